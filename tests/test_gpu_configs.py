"""Bit-exact parity on the BASELINE.json configs at their stated sizes, against
the reference itself (oracle/_ref: the unmodified headers compiled in place).

* every per-class lcom (raw bits), lcom_ck and cbo against the reference's
  parallel_class_metrics + parallel_lcom_ck (parallel.hpp:149,164) on all host
  threads, and both threshold means against its compute_thresholds
  (suggest.hpp:46-61);
* the ordered cohesion+coupling suggestion list (device mean thresholds,
  union, best-only: the bench step) against suggest_all (suggest.hpp:303-350)
  — in full for C4, and for C3 / C5 (hours of reference what-ifs in full) on
  SURVEY.md §8c's deterministic sample: every 97th method in class-segment
  order plus methods of the 8 largest classes. The reference side is
  ref_sweep (oracle/ref_shim.cpp): the reference's own per-method body of
  suggest_by_cohesion / suggest_by_coupling (detail::used_classes,
  detail::emit_for_method, what_if_move) on host threads, then suggest_all's
  merge; per-method decisions are independent given the report and the
  thresholds, so the sample's list is suggest_all's list restricted to the
  sampled methods (checked against suggest_all itself in
  tests/test_oracle.py::test_ref_sweep_equals_suggest_all). C3's class 0
  has 10,218 members, so this is also the giant / 1024-thread CTA path's
  sweep against the reference.
"""
import os

import numpy as np
import pytest

import oracle
from conftest import first_diff, records_equal
from paper_1308_4011_b200 import Engine, System, abi

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]

COH_COUP = abi.MM_CRIT_COHESION | abi.MM_CRIT_COUPLING
THREADS = os.cpu_count() or 1

C3 = dict(seed=1, n_classes=10000, n_methods=100000, n_attributes=200000, k_max_calls=4, k_max_accesses=4,
          intra_class_bias=0.5, zipf_s=1.0)
C4 = dict(seed=1, n_classes=100000, n_methods=1000000, n_attributes=2000000, k_max_calls=4, k_max_accesses=4,
          intra_class_bias=0.5)
C5 = dict(seed=3, n_classes=5000, n_methods=2500000, n_attributes=320000, k_max_calls=4, k_max_accesses=32,
          intra_class_bias=0.9)


def metrics_and_thresholds(e: Engine, s: System, R: "oracle.RefModel"):
    e.upload(s)
    gl, gk, gc = e.class_metrics_all()
    wl, wk, wc = R.class_metrics(THREADS)  # parallel_class_metrics + parallel_lcom_ck
    assert gl.tobytes() == wl.tobytes(), "lcom bits"
    assert np.array_equal(gk, wk), "lcom_ck"
    assert np.array_equal(gc, wc), "cbo"
    t = e.compute_thresholds()                # device means
    wt = oracle.ref_thresholds(wl, wc)        # the reference's compute_thresholds
    assert (t.lcom, t.cbo) == (wt.lcom, wt.cbo)
    return wl, wc, t


def sample_methods(s: System, every: int = 97, per_big: int = 16, n_big: int = 8) -> np.ndarray:
    """every `every`-th method in class-segment order, plus
    `per_big` evenly spaced members of each of the n_big largest classes."""
    pos = np.arange(0, s.n_methods, every)
    picks = [s.class_methods[pos]]
    msz = np.diff(s.class_method_off.astype(np.int64))
    for c in np.argsort(-msz, kind="stable")[:n_big]:
        mem = s.members(int(c))
        picks.append(mem[np.linspace(0, len(mem) - 1, min(per_big, len(mem))).astype(np.int64)])
    return np.unique(np.concatenate(picks)).astype(np.uint32)


def gpu_list(e: Engine):
    e.run(thresholds=None)  # the bench step: one graph replay (metric pass + device means + sweep)
    return e.suggestions()


def test_config_c4_full_ordered_list(gpu_engine):
    s = System.generate(**C4)
    R = oracle.RefModel(s)
    wl, wc, t = metrics_and_thresholds(gpu_engine, s, R)
    got = gpu_list(gpu_engine)
    want, cand = R.sweep(wl, wc, COH_COUP, t.lcom, t.cbo, n_workers=THREADS, dynamic=True)
    assert cand == 1998056 and len(want) == 86684  # SURVEY.md §8a / BASELINE.md §3
    assert records_equal(got, want), first_diff(got, want)


def test_config_c3_zipf(gpu_engine):
    s = System.generate(**C3)
    assert int(np.diff(s.class_method_off).max()) > 2048  # class 0 (10,218 members): the giant / 1024-thread CTA path
    R = oracle.RefModel(s)
    wl, wc, t = metrics_and_thresholds(gpu_engine, s, R)
    got = gpu_list(gpu_engine)
    sample = sample_methods(s)
    want, _ = R.sweep(wl, wc, COH_COUP, t.lcom, t.cbo, methods=sample, n_workers=THREADS, dynamic=True)
    sel = got[np.isin(got["method"], sample)]
    assert len(want) > 0 and records_equal(sel, want), first_diff(sel, want)
    # every record on the device list is a method/destination the reference also scores
    assert np.all(got["origin"] == s.method_owner[got["method"]])


def test_config_c5_dense(gpu_engine):
    s = System.generate(**C5)
    R = oracle.RefModel(s)
    wl, wc, t = metrics_and_thresholds(gpu_engine, s, R)
    got = gpu_list(gpu_engine)
    sample = sample_methods(s)
    want, _ = R.sweep(wl, wc, COH_COUP, t.lcom, t.cbo, methods=sample, n_workers=THREADS, dynamic=True)
    sel = got[np.isin(got["method"], sample)]
    assert len(want) > 0 and records_equal(sel, want), first_diff(sel, want)


def test_config_c3_all_candidates_and_intersection(gpu_engine):
    # the other modes on the skewed shape, on a smaller sample
    s = System.generate(**C3)
    R = oracle.RefModel(s)
    gpu_engine.upload(s)
    wl, _, wc = gpu_engine.class_metrics_all()
    t = gpu_engine.compute_thresholds()
    sample = sample_methods(s, every=389, per_big=4)
    for comb, allc in ((0, True), (1, False)):
        got = gpu_engine.suggest_all(t, all_candidates=allc, combine=comb)
        want, _ = R.sweep(wl, wc, COH_COUP, t.lcom, t.cbo, comb, allc, methods=sample, n_workers=THREADS)
        sel = got[np.isin(got["method"], sample)]
        assert records_equal(sel, want), (comb, allc, first_diff(sel, want))
