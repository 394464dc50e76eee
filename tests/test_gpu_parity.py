"""GPU parity: libmmgpu.so (sm_100a) against the reference's golden outputs and the oracle.

Bar: bit-exact — lcom doubles compared as raw bits, every integer equal, the
ordered suggestion list equal record by record (all 64 bytes but padding).
All calls go through the C ABI (paper_1308_4011_b200.Engine is a ctypes shim).
"""
import os

import numpy as np
import pytest

import oracle
from conftest import first_diff, golden_names, golden_records, golden_system, load_golden, records_equal, unhex
from paper_1308_4011_b200 import (Combine, Criterion, Engine, MMArgError, MMError, MMRangeError, System, ThresholdOverrides,
                                  Thresholds, abi)
from paper_1308_4011_b200.engine import criteria_mask

pytestmark = pytest.mark.gpu

COH, COUP = abi.MM_CRIT_COHESION, abi.MM_CRIT_COUPLING
CRIT = {COH: [Criterion.Cohesion], COUP: [Criterion.Coupling], COH | COUP: [Criterion.Cohesion, Criterion.Coupling]}


def gpu_metrics(e: Engine, s: System):
    e.upload(s)
    return e.class_metrics_all()


def assert_metrics_equal(got, want, ctx=""):
    gl, gk, gc = got
    wl, wk, wc = want
    assert gl.tobytes() == np.ascontiguousarray(wl, np.float64).tobytes(), f"lcom differs {ctx}"
    assert np.array_equal(gk, np.asarray(wk, np.uint64)), f"lcom_ck differs {ctx}"
    assert np.array_equal(gc, np.asarray(wc, np.uint32)), f"cbo differs {ctx}"


@pytest.mark.parametrize("name", golden_names())
def test_gpu_matches_reference_golden(gpu_engine, name):
    case = load_golden(name)
    s = golden_system(case)
    got = gpu_metrics(gpu_engine, s)
    assert_metrics_equal(got, ([unhex(h) for h in case["lcom"]], case["lcom_ck"], case["cbo"]), name)
    t = gpu_engine.compute_thresholds()
    assert t.lcom == unhex(case["thresholds_mean"]["lcom"]) and t.cbo == unhex(case["thresholds_mean"]["cbo"])
    for run in case["suggest"]:
        thr = Thresholds(0.0, unhex(run["thr_lcom"]), unhex(run["thr_cbo"]), run["thresholds"] == "explicit")
        out = gpu_engine.suggest_all(thr, CRIT[run["criteria"]], Combine(run["combine"]), run["all_candidates"])
        want = golden_records(run["suggestions"])
        assert records_equal(out, want), (name, run["criteria"], run["combine"], first_diff(out, want))
    for w in case.get("what_if", []):
        if w["status"]:
            exc = MMRangeError if w["status"] == abi.MM_E_RANGE else MMArgError
            with pytest.raises(exc):
                gpu_engine.what_if_move(w["u"], w["o"], w["d"])
            continue
        wm = gpu_engine.what_if_move(w["u"], w["o"], w["d"])
        for f, v in w["w"].items():
            assert (wm[f] == unhex(v)) if f.startswith("lcom") else (int(wm[f]) == v), (name, w, f)


def test_device_threshold_source_equals_explicit(gpu_engine):
    s = System.generate(seed=1, n_classes=1000, n_methods=10000, n_attributes=20000)
    gpu_engine.upload(s)
    t = gpu_engine.compute_thresholds()
    a = gpu_engine.suggest_all(t)
    gpu_engine.sweep(thresholds=None)
    b = gpu_engine.suggestions()
    assert records_equal(a, b) and len(a) == 955  # C2 -> 955 suggestions


def random_cfg(rng, seed, big=False):
    if big:  # acceptance.cpp:139-153 ranges (m 10-2000, c 2-200)
        m = int(10 + rng.integers(0, 1991))
        c = int(2 + rng.integers(0, 199))
        a = int(1 + rng.integers(0, max(1, m // 2)))
    else:
        m, c, a = int(rng.integers(4, 120)), int(rng.integers(2, 30)), int(rng.integers(1, 60))
    return dict(seed=seed, n_classes=c, n_methods=m, n_attributes=a, k_max_calls=int(rng.integers(0, 5)),
                k_max_accesses=int(rng.integers(0, 5)), intra_class_bias=float(rng.random()))


def check_against_oracle(e, s, ctx, modes=None, top_ks=(1,), cache=None):
    """Engine e against the oracle on system s. `cache` (a dict) keeps the
    oracle's answers when several engines check the same system."""
    got = gpu_metrics(e, s)
    key = s.digest() if cache is not None else None
    if cache is not None and ("metrics", key) in cache:
        want = cache[("metrics", key)]
    else:
        want = oracle.class_metrics(s)
        if cache is not None:
            cache[("metrics", key)] = want
    assert_metrics_equal(got, want, ctx)
    lcom, ck, cbo = want
    t_or = oracle.thresholds(lcom, cbo)
    t = e.compute_thresholds()
    assert (t.lcom, t.cbo) == (t_or.lcom, t_or.cbo), ctx
    for mask, comb, allc in modes or ((COH | COUP, 0, False), (COH | COUP, 1, False), (COH, 0, False),
                                     (COUP, 0, False), (COH | COUP, 0, True), (COH | COUP, 1, True)):
        for k in top_ks:
            g = e.suggest_all(t, CRIT[mask], Combine(comb), allc, top_k=k)
            ck_ = ("suggest", key, mask, comb, allc, k)
            if cache is not None and ck_ in cache:
                o = cache[ck_]
            else:
                o = oracle.suggest(s, lcom, cbo, mask, comb, allc, k, t.lcom, t.cbo)
                if cache is not None:
                    cache[ck_] = o
            assert records_equal(g, o), (ctx, mask, comb, allc, k, first_diff(g, o))


def test_gpu_random_small_systems(gpu_engine):
    for seed in range(40):
        s = System.generate(**random_cfg(np.random.default_rng(seed), seed))
        check_against_oracle(gpu_engine, s, f"seed {seed}", top_ks=(1, 3))


def test_gpu_random_acceptance_sized(gpu_engine):
    # acceptance criterion 2/3 sizes: 50 systems, m in [10, 2000], c in [2, 200]
    for seed in range(50):
        s = System.generate(**random_cfg(np.random.default_rng(7000 + seed), seed, big=True))
        check_against_oracle(gpu_engine, s, f"acc seed {seed}", modes=((COH | COUP, 0, False), (COH | COUP, 1, True)))


def test_gpu_what_if_every_pair_random(gpu_engine):
    # what_if_move for every (method, destination), including non-candidate destinations
    for seed in range(8):
        s = System.generate(**random_cfg(np.random.default_rng(300 + seed), seed))
        gpu_engine.upload(s)
        for u in range(s.n_methods):
            o = int(s.method_owner[u])
            for d in range(s.n_classes):
                st, w = oracle.what_if(s, u, o, d)
                if st:
                    with pytest.raises(MMError):
                        gpu_engine.what_if_move(u, o, d)
                    continue
                g = gpu_engine.what_if_move(u, o, d)
                for f in abi.WHATIF_FIELDS:
                    assert g[f] == getattr(w, f), (seed, u, o, d, f)


def test_gpu_large_class_paths(gpu_engine, monkeypatch):
    # classes with > 32 members, > 64 attributes and methods of degree > 16
    # exercise the CTA path of the metric pass and the streaming sweep path
    cfgs = [
        dict(seed=3, n_classes=20, n_methods=10000, n_attributes=1280, k_max_calls=4, k_max_accesses=32,
             intra_class_bias=0.9),   # C5-like: 500 methods and 64 attributes per class
        dict(seed=5, n_classes=7, n_methods=700, n_attributes=2000, k_max_calls=12, k_max_accesses=12,
             intra_class_bias=0.3),
        dict(seed=11, n_classes=300, n_methods=3000, n_attributes=6000, k_max_calls=4, k_max_accesses=4,
             intra_class_bias=0.5, zipf_s=1.0),  # C3-like Zipf skew
        dict(seed=12, n_classes=1, n_methods=300, n_attributes=40, k_max_calls=20, k_max_accesses=20,
             intra_class_bias=0.7),   # single class
        dict(seed=13, n_classes=150, n_methods=9000, n_attributes=3000, k_max_calls=6, k_max_accesses=6,
             intra_class_bias=0.1),   # dense coupling: U rows > 64 -> exact class bitmaps
        dict(seed=14, n_classes=40, n_methods=4000, n_attributes=30000, k_max_calls=3, k_max_accesses=24,
             intra_class_bias=0.6),   # A > 256 per class: attribute-bitmap LCOM-CK, degree > 16
    ]
    # CTA-path U rows come from an smem class histogram (4·C ≤ 64 KB, as here)
    # or from sorted keys (many classes); MMGPU_HIST_MAX_BYTES=0 forces the latter
    # MMGPU_GIANT_MIN=64 sends every histogram class of ≥ 64 members with
    # global attribute bitmaps through the multi-CTA giant phase 1
    from paper_1308_4011_b200 import Engine
    monkeypatch.setenv("MMGPU_GIANT_MIN", "64")
    giant_engine = Engine(0)
    monkeypatch.delenv("MMGPU_GIANT_MIN")
    # dense classes (A ≤ 64, ≥ 128 members) count LCOM-CK pairs with tcgen05
    # MMA by default; MMGPU_CK_MMA_MIN past every class keeps the popc path
    monkeypatch.setenv("MMGPU_CK_MMA_MIN", str(1 << 30))
    popc_engine = Engine(0)
    monkeypatch.delenv("MMGPU_CK_MMA_MIN")
    monkeypatch.setenv("MMGPU_HIST_MAX_BYTES", "0")
    cache = {}  # the oracle's (recompute-based) answers, shared by the four engines
    systems = [System.generate(**cfg) for cfg in cfgs]
    with Engine(0) as keys_engine, giant_engine, popc_engine:
        for e, tag in ((gpu_engine, "hist"), (keys_engine, "keys"), (giant_engine, "giant"), (popc_engine, "popc")):
            for cfg, s in zip(cfgs, systems):
                check_against_oracle(e, s, f"{tag} {cfg}", modes=((COH | COUP, 0, False), (COH | COUP, 0, True),
                                                                   (COH | COUP, 1, False)), top_ks=(1, 4),
                                     cache=cache)


def test_gpu_explicit_thresholds_and_degenerate(gpu_engine):
    # empty classes, classes without attributes, isolated methods
    s = System.build([([], [0, 1]), ([0, 1], []), ([2], [2, 3, 4]), ([], [])],
                     [[2], [], [0, 1], [], [3]], [[0, 2], [1], [2], [], [0]])
    check_against_oracle(gpu_engine, s, "degenerate")
    gpu_engine.upload(s)
    for thr in (Thresholds(0, -1.0, -1.0), Thresholds(0, 2.0, 99.0), Thresholds(0, 0.0, 0.0)):
        lcom, ck, cbo = oracle.class_metrics(s)
        g = gpu_engine.suggest_all(thr)
        o = oracle.suggest(s, lcom, cbo, COH | COUP, 0, False, 1, thr.lcom, thr.cbo)
        assert records_equal(g, o)


def test_gpu_empty_system(gpu_engine):
    s = System.build([([], [])], [], [])
    gpu_engine.upload(s)
    lcom, ck, cbo = gpu_engine.class_metrics_all()
    assert lcom.tolist() == [0.0] and ck.tolist() == [0] and cbo.tolist() == [0]
    assert len(gpu_engine.suggest_all(gpu_engine.compute_thresholds())) == 0


def test_gpu_errors(gpu_engine):
    s = System.build([([0, 1], [0, 1]), ([2, 3], [2])], [[2], [], []], [[2, 3], [0, 1], [2]])
    gpu_engine.upload(s)
    with pytest.raises(MMArgError):
        gpu_engine.what_if_move(0, 0, 0)
    with pytest.raises(MMArgError):
        gpu_engine.what_if_move(2, 0, 1)
    with pytest.raises(MMRangeError):
        gpu_engine.what_if_move(0, 0, 9)
    with pytest.raises(MMRangeError):
        gpu_engine.what_if_move(0, 7, 1)
    with pytest.raises(MMRangeError):
        gpu_engine.lcom_normalized(5)
    with pytest.raises(MMArgError):
        gpu_engine.suggest_all(Thresholds(), [])
    with pytest.raises(MMError) as ei:  # the similarity criterion has no top-k extension
        gpu_engine.suggest_all(Thresholds(), [Criterion.Similarity], top_k=3)
    assert ei.value.status == abi.MM_E_UNSUPPORTED
    with pytest.raises(MMRangeError):
        gpu_engine.suggest_all(Thresholds(), class_range=(0, 9))
    # malformed input is rejected on upload instead of faulting
    bad = System.build([([0, 1], [0, 1]), ([2, 3], [2])], [[2], [], []], [[2, 3], [0, 1], [2]])
    bad.acc_tgt[0] = 99
    with pytest.raises(MMArgError):
        gpu_engine.upload(bad)


def test_gpu_shards_concatenate_to_full_list(gpu_engine):
    from paper_1308_4011_b200 import plan_shards
    s = System.generate(seed=2, n_classes=500, n_methods=6000, n_attributes=9000, k_max_calls=5, k_max_accesses=5,
                        intra_class_bias=0.4)
    gpu_engine.upload(s)
    t = gpu_engine.compute_thresholds()
    full = gpu_engine.suggest_all(t)
    for n in (2, 3, 8):
        b = plan_shards(s, n)
        parts = [gpu_engine.suggest_all(t, class_range=(int(b[i]), int(b[i + 1]))) for i in range(n)]
        assert records_equal(np.concatenate(parts), full)


@pytest.mark.slow
def test_gpu_config_c4_metrics_and_sampled_sweep(gpu_engine):
    """C4 (100k classes / 1M methods): every class value vs the oracle; the sweep
    vs the oracle on class ranges; size-independent properties on the full list."""
    s = System.generate(seed=1, n_classes=100000, n_methods=1000000, n_attributes=2000000)
    got = gpu_metrics(gpu_engine, s)
    want = oracle.class_metrics(s)
    assert_metrics_equal(got, want, "C4")
    t = gpu_engine.compute_thresholds()
    t_or = oracle.thresholds(want[0], want[2])
    assert (t.lcom, t.cbo) == (t_or.lcom, t_or.cbo)
    full = gpu_engine.suggest_all(t)
    stats = gpu_engine.sweep_stats()
    assert stats["candidates"] == s.n_candidates() == 1998056
    assert len(full) == 86684                                     # BASELINE.md §3 (reference, C4)
    assert stats["gated_whatifs"] == 960003 + 1236116
    key = (full["origin"].astype(np.uint64) << np.uint64(40)) | (full["method"].astype(np.uint64) << np.uint64(20)) \
        | full["destination"].astype(np.uint64)
    assert np.all(np.diff(key.astype(np.int64)) > 0)  # strictly (origin, method, destination) ordered
    for lo, hi in ((0, 1000), (50000, 50500), (99000, 100000)):
        o = oracle.suggest(s, want[0], want[2], COH | COUP, 0, False, 1, t.lcom, t.cbo, class_range=(lo, hi))
        sel = (full["origin"] >= lo) & (full["origin"] < hi)
        assert records_equal(full[sel], o), (lo, hi)


def _seq_mean(vals):
    s = 0.0
    for v in vals:
        s += float(v)  # IEEE double round-to-nearest, left to right (suggest.hpp:48-53)
    return s / len(vals) if len(vals) else 0.0


def test_gpu_sequential_mean_adversarial(gpu_engine):
    rng = np.random.default_rng(0)
    u = 2.0 ** -53
    cases = []
    for n in (1, 2, 3, 31, 1000, 1024, 1025, 4097, 100000, 333333):
        cases.append(rng.integers(0, 2 ** 53 + 1, n).astype(np.float64) * u)            # uniform grid values
        cases.append(np.round(rng.random(n) * 8) / 8)                                    # dyadic -> exact ties
        cases.append(0.5 + rng.integers(0, 4, n) * 2.0 ** -53)                           # ties at every binade
        cases.append(np.where(rng.random(n) < 0.5, 1.0, 0.0))                            # exact binade hits
        cases.append(1.0 - rng.integers(1, 1 << 20, n) * u)                              # near-1 values
    cases.append(np.zeros(5000))
    for vals in cases:
        got, fast = gpu_engine.sequential_mean(vals)
        assert got == _seq_mean(vals), (len(vals), vals[:4])
        assert fast, "fast path should accept grid values"
    # outside the fast path's precondition: still exact (device serial fallback)
    for vals in (rng.random(3000) * 0.3, -rng.random(100), rng.random(2000) * 3):
        got, fast = gpu_engine.sequential_mean(vals)
        assert got == _seq_mean(vals) and not fast


def test_gpu_threshold_fast_path_on_systems(gpu_engine):
    for cfg in (dict(seed=1, n_classes=100000, n_methods=300000, n_attributes=200000),
                dict(seed=4, n_classes=77777, n_methods=500000, n_attributes=100000, k_max_accesses=9)):
        s = System.generate(**cfg)
        gpu_engine.upload(s)
        lcom, ck, cbo = gpu_engine.class_metrics_all()
        t = gpu_engine.compute_thresholds()
        assert t.lcom == _seq_mean(lcom) and t.cbo == _seq_mean(cbo.astype(np.float64))
        assert gpu_engine.sequential_mean(lcom) == (t.lcom, True)


def test_gpu_graph_step_equals_eager(gpu_engine):
    # mm_run replays a captured CUDA graph of metric pass + sweep: same bits as the eager calls
    s = System.generate(seed=21, n_classes=2000, n_methods=30000, n_attributes=40000, k_max_calls=5,
                        k_max_accesses=5, intra_class_bias=0.45)
    gpu_engine.upload(s)
    t = gpu_engine.compute_thresholds()
    eager = gpu_engine.suggest_all(t)
    for _ in range(3):
        gpu_engine.run(thresholds=None)  # capture, then replays
        assert records_equal(gpu_engine.suggestions(), eager)
    lcom, ck, cbo = gpu_engine.class_metrics_all()
    want = oracle.class_metrics(s)
    assert_metrics_equal((lcom, ck, cbo), want, "graph")
    # a new model invalidates the graph
    s2 = System.generate(seed=22, n_classes=2000, n_methods=30000, n_attributes=40000)
    gpu_engine.upload(s2)
    gpu_engine.run(thresholds=None)
    l2, k2, c2 = oracle.class_metrics(s2)
    t2 = oracle.thresholds(l2, c2)
    o2 = oracle.suggest(s2, l2, c2, COH | COUP, 0, False, 1, t2.lcom, t2.cbo)
    assert records_equal(gpu_engine.suggestions(), o2)


def test_gpu_upload_without_owner_tables(gpu_engine):
    # mm_system with NULL owner tables: the device derives them from the
    # membership lists; every result equals the full upload's
    for cfg in (dict(seed=31, n_classes=300, n_methods=4000, n_attributes=6000, k_max_calls=5, k_max_accesses=5,
                     intra_class_bias=0.5),
                dict(seed=32, n_classes=40, n_methods=6000, n_attributes=3000, k_max_calls=4, k_max_accesses=12,
                     intra_class_bias=0.6, zipf_s=1.0)):
        s = System.generate(**cfg)
        gpu_engine.upload(s)
        want_m = gpu_metrics(gpu_engine, s)
        t = gpu_engine.compute_thresholds()
        want = gpu_engine.suggest_all(t, all_candidates=True)
        gpu_engine.upload(s, owner_tables=False)
        got_m = gpu_metrics(gpu_engine, s)
        assert_metrics_equal(got_m, want_m, str(cfg))
        assert records_equal(gpu_engine.suggest_all(t, all_candidates=True), want)
        for u in range(0, s.n_methods, 97):
            o = int(s.method_owner[u])
            d = int((o + 1 + u % (s.n_classes - 1)) % s.n_classes)
            g = gpu_engine.what_if_move(u, o, d)
            w = oracle.what_if(s, u, o, d)[1]
            assert all(g[f] == getattr(w, f) for f in abi.WHATIF_FIELDS)
    # a method no class lists has no derivable owner: rejected like a bad id
    bad = System.build([([0, 1], [0, 1]), ([2, 3], [2])], [[2], [], []], [[2, 3], [0, 1], [2]])
    bad.class_methods = bad.class_methods.copy()
    bad.class_methods[-1] = 0  # method 2 unlisted, method 0 listed twice
    with pytest.raises(MMArgError):
        gpu_engine.upload(bad, owner_tables=False)


def test_gpu_class_metrics_async(gpu_engine):
    # enqueued D2H under the sweep: same values once synchronized; the next
    # metric pass waits for the copies
    s = System.generate(seed=41, n_classes=2000, n_methods=25000, n_attributes=30000)
    gpu_engine.upload(s, owner_tables=False)
    gpu_engine.compute_metrics()
    lcom, ck, cbo = gpu_engine.class_metrics_async()
    gpu_engine.sweep(thresholds=None, want_count=False)
    gpu_engine.compute_metrics()
    gpu_engine.synchronize()
    got = (lcom.copy(), ck.copy(), cbo.copy())
    assert_metrics_equal(got, oracle.class_metrics(s), "async")


def test_gpu_fan_metrics(gpu_engine):
    # MetricsReport::fan_in / fan_out (metrics.hpp:79-93) against the oracle,
    # the golden systems through C4
    systems = [golden_system(load_golden(n)) for n in golden_names()[:4]]
    systems += [System.generate(**random_cfg(np.random.default_rng(900 + k), k)) for k in range(10)]
    systems.append(System.generate(seed=1, n_classes=100000, n_methods=1000000, n_attributes=2000000))
    for s in systems:
        gpu_engine.upload(s)
        fi, fo = gpu_engine.fan_metrics()
        wi, wo = oracle.fan_metrics(s)
        assert (fi == wi).all() and (fo == wo).all()


def test_gpu_estimate_workload(gpu_engine):
    # WorkloadEstimate (metrics.hpp:195-233): device max-reduce + closed forms
    for s in (System.generate(seed=51, n_classes=300, n_methods=5000, n_attributes=7000, k_max_calls=7,
                              k_max_accesses=3),
              System.build([([], [])], [], []),
              System.generate(seed=1, n_classes=100000, n_methods=1000000, n_attributes=2000000)):
        gpu_engine.upload(s)
        w = gpu_engine.estimate_workload()
        m, c = s.n_methods, s.n_classes
        k_m = int(np.diff(s.call_off).max()) if m else 0
        k_a = int(np.diff(s.acc_off).max()) if m else 0
        n_sim = m * (m - 1) // 2 if m else 0
        want = dict(m=m, c=c, k_m=k_m, k_a=k_a, n_fan=2 * m, n_sim=n_sim, n_lcom=c * (m + 1), n_cbo=c * (m + 1),
                    n_total=2 * m + n_sim + 2 * c * (m + 1))
        assert w == want


def test_gpu_giant_phase1_equals_single_cta(gpu_engine, monkeypatch):
    # a Zipf system whose largest class (> 2048 members) takes the multi-CTA
    # giant path by default: metrics against the oracle, every sweep mode
    # against the single-CTA path (the oracle's recompute-based sweep needs
    # minutes per mode on a 2k-member class)
    from paper_1308_4011_b200 import Engine
    s = System.generate(seed=16, n_classes=150, n_methods=12000, n_attributes=20000, k_max_calls=4,
                        k_max_accesses=4, intra_class_bias=0.5, zipf_s=1.0)
    assert np.diff(s.class_method_off).max() > 2048
    monkeypatch.setenv("MMGPU_GIANT_MIN", str(1 << 30))
    with Engine(0) as single:
        single.upload(s)
        gpu_engine.upload(s)
        assert_metrics_equal(gpu_metrics(gpu_engine, s), oracle.class_metrics(s), "giant")
        assert_metrics_equal(gpu_metrics(single, s), oracle.class_metrics(s), "single")
        t = gpu_engine.compute_thresholds()
        for crit in ([Criterion.Cohesion, Criterion.Coupling], [Criterion.Coupling]):
            for comb in (Combine.Union, Combine.Intersection):
                for allc in (False, True):
                    a = gpu_engine.suggest_all(t, crit, comb, allc)
                    b = single.suggest_all(t, crit, comb, allc)
                    assert records_equal(a, b), (crit, comb, allc, first_diff(a, b))
        for k in (2, 5):
            assert records_equal(gpu_engine.suggest_all(t, top_k=k), single.suggest_all(t, top_k=k))


def boundary_system(rng, sizes, attrs, max_calls, max_accs, intra=0.7, shuffle=True):
    """Classes of the given member / attribute counts (ids shuffled across
    classes), dependencies drawn like the reference generator: each edge stays
    in the own class with probability `intra`."""
    n_m, n_a = int(sum(sizes)), int(sum(attrs))
    mids = rng.permutation(n_m) if shuffle else np.arange(n_m)
    aids = rng.permutation(n_a) if shuffle else np.arange(n_a)
    classes, mo, ao = [], np.zeros(n_m, np.int64), np.zeros(n_a, np.int64)
    mo_off = ao_off = 0
    for c, (m, a) in enumerate(zip(sizes, attrs)):
        ms, as_ = mids[mo_off:mo_off + m], aids[ao_off:ao_off + a]
        mo[ms], ao[as_] = c, c
        classes.append((as_.tolist(), ms.tolist()))
        mo_off += m
        ao_off += a
    members = [np.array(cl[1]) for cl in classes]
    owned = [np.array(cl[0]) for cl in classes]
    calls, accs = [], []
    for p in range(n_m):
        c = mo[p]
        cl, al = set(), set()
        for _ in range(int(rng.integers(0, max_calls + 1))):
            pool = members[c] if rng.random() < intra else members[int(rng.integers(0, len(sizes)))]
            t = int(pool[rng.integers(0, len(pool))])
            if t != p:
                cl.add(t)
        for _ in range(int(rng.integers(0, max_accs + 1))):
            pool = owned[c] if (rng.random() < intra and len(owned[c])) else owned[int(rng.integers(0, len(sizes)))]
            if len(pool):
                al.add(int(pool[rng.integers(0, len(pool))]))
        calls.append(sorted(cl))
        accs.append(sorted(al))
    return System.build(classes, calls, accs)


def test_gpu_path_boundaries(gpu_engine):
    # classes on both sides of every planning threshold: warp path limits
    # (32 members, 64 attributes, degree 16, 32 foreign edges), the popc /
    # tensor-core LCOM-CK cut (128 members), the giant cut (512), mask width
    # (64 / 65 / 256 / 257 attributes) — metrics and the sweep against the oracle
    rng = np.random.default_rng(2024)
    cases = [
        ([31, 32, 33, 1, 2, 40], [63, 64, 65, 1, 0, 10], 4, 12),
        ([127, 128, 129, 5, 6], [64, 64, 64, 3, 3], 3, 16),
        ([20, 20, 20, 20], [257, 256, 255, 8], 2, 18),
        ([511, 512, 513, 3], [40, 300, 70, 2], 3, 6),
        ([32] * 12, [64] * 12, 6, 10),
    ]
    for sizes, attrs, mc, ma in cases:
        s = boundary_system(rng, sizes, attrs, mc, ma)
        check_against_oracle(gpu_engine, s, f"sizes {sizes} attrs {attrs}",
                             modes=((COH | COUP, 0, False), (COH | COUP, 0, True), (COH | COUP, 1, False)),
                             top_ks=(1, 3))
        for u in range(0, s.n_methods, 53):
            o = int(s.method_owner[u])
            for d in range(s.n_classes):
                if d == o:
                    continue
                g = gpu_engine.what_if_move(u, o, d)
                w = oracle.what_if(s, u, o, d)[1]
                assert all(g[f] == getattr(w, f) for f in abi.WHATIF_FIELDS), (sizes, u, o, d)


def test_gpu_c4x8_metrics_and_sampled_sweep(gpu_engine):
    # 800k classes / 8M methods: every class metric and both threshold means
    # (the cooperative sequential-sum emulation over 391 tiles) against the
    # oracle, the sweep on a 20k-class range of the full-system pass
    s = System.generate(seed=1, n_classes=800000, n_methods=8000000, n_attributes=16000000)
    gpu_engine.upload(s, owner_tables=False)
    got = gpu_metrics(gpu_engine, s)
    want = oracle.class_metrics(s)
    assert_metrics_equal(got, want, "c4x8")
    t_or = oracle.thresholds(want[0], want[2])
    t = gpu_engine.compute_thresholds()
    assert (t.lcom, t.cbo) == (t_or.lcom, t_or.cbo)
    g = gpu_engine.suggest_all(t, class_range=(0, 20000))
    o = oracle.suggest(s, want[0], want[2], COH | COUP, 0, False, 1, t.lcom, t.cbo, class_range=(0, 20000))
    assert records_equal(g, o), first_diff(g, o)


def test_gpu_similarities(gpu_engine):
    # all_similarities (metrics.hpp:39-77): pairs, order and every double
    # against the oracle; the golden systems, random ones, a dense one whose
    # rows take the wide kernel, and an empty system
    systems = [golden_system(load_golden(n)) for n in golden_names()[:4]]
    systems += [System.generate(**random_cfg(np.random.default_rng(500 + k), k)) for k in range(12)]
    systems.append(System.generate(seed=9, n_classes=8, n_methods=1200, n_attributes=90, k_max_calls=6,
                                   k_max_accesses=20, intra_class_bias=0.9))
    systems.append(System.build([([], [])], [], []))
    for s in systems:
        gpu_engine.upload(s)
        g = gpu_engine.similarities()
        o = oracle.similarities(s)
        assert g.tobytes() == o.tobytes(), (len(g), len(o))
    # a 20k-method system against the compiled reference's parallel engine
    s = System.generate(seed=1, n_classes=2000, n_methods=20000, n_attributes=40000)
    gpu_engine.upload(s, owner_tables=False)
    g = gpu_engine.similarities()
    if oracle.ref_available():
        o = oracle.RefModel(s).similarities(8)
    else:
        o = oracle.similarities(s)
    assert g.tobytes() == o.tobytes()


def test_gpu_similarity_limits_and_full_report(gpu_engine):
    # rows whose candidate lists pass 4096 entries take the huge-row path (a
    # table equal to the oracle's, no error); the full report's fields agree
    # with their own calls
    n = 5000
    s = System.build([(list(range(2)), list(range(n)))], [], [[0, 1]] * n)
    gpu_engine.upload(s)
    g = gpu_engine.similarities()
    assert len(g) == n * (n - 1) // 2 and g.tobytes() == oracle.similarities(s).tobytes()
    s = System.generate(seed=61, n_classes=50, n_methods=800, n_attributes=600, k_max_calls=5, k_max_accesses=5)
    gpu_engine.upload(s)
    r = gpu_engine.full_report()
    assert r["similarity"].tobytes() == oracle.similarities(s).tobytes()
    fi, fo = oracle.fan_metrics(s)
    assert (r["fan_in"] == fi).all() and (r["fan_out"] == fo).all()
    assert_metrics_equal((r["lcom"], r["lcom_ck"], r["cbo"]), oracle.class_metrics(s), "full_report")


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_gpu_similarity_criterion_vs_reference(gpu_engine):
    # suggest_all with every criterion combination that includes Similarity,
    # union / intersection, best / all candidates, mean and explicit
    # thresholds — against the compiled reference (report.similarity =
    # all_similarities)
    combos = [[Criterion.Similarity], [Criterion.Similarity, Criterion.Cohesion],
              [Criterion.Similarity, Criterion.Coupling],
              [Criterion.Similarity, Criterion.Cohesion, Criterion.Coupling]]
    systems = [golden_system(load_golden(n)) for n in golden_names()[:3]]
    systems += [System.generate(**random_cfg(np.random.default_rng(700 + k), k)) for k in range(10)]
    for s in systems:
        gpu_engine.upload(s)
        lcom, ck, cbo = gpu_metrics(gpu_engine, s)
        table = gpu_engine.similarities()
        R = oracle.RefModel(s)
        sim_mean = float(np.sum(table["value"]) / len(table)) if len(table) else 0.0
        t_mean = oracle.thresholds(lcom, cbo, table["value"])
        for thr in (Thresholds(t_mean.similarity, t_mean.lcom, t_mean.cbo), Thresholds(0.3, 0.2, 1.0),
                    Thresholds(0.0, -1.0, -1.0)):
            for crit in combos:
                for comb in (Combine.Union, Combine.Intersection):
                    for allc in (False, True):
                        g = gpu_engine.suggest_all(thr, crit, comb, allc)
                        o = R.suggest_full(lcom, cbo, criteria_mask(crit), int(comb), allc, thr.similarity,
                                           thr.lcom, thr.cbo)
                        assert records_equal(g, o), (crit, comb, allc, thr, first_diff(g, o))
        del sim_mean


def hub_system(rng, n_classes=220, per=5, hubs=((0, 150, 120), (7, 40, 31), (13, 31, 0), (21, 33, 2))):
    """Classes of `per` methods / attributes; hub methods (method id, classes
    called into, classes accessed) use 31..270 classes; the rest draw a few
    dependencies. Ids are class-major (method p of class p // per)."""
    n_m = n_a = n_classes * per
    classes = [(list(range(c * per, (c + 1) * per)), list(range(c * per, (c + 1) * per))) for c in range(n_classes)]
    calls = [[] for _ in range(n_m)]
    accs = [[] for _ in range(n_m)]
    for p in range(n_m):
        for _ in range(int(rng.integers(0, 4))):
            t = int(rng.integers(0, n_m))
            if t != p:
                calls[p].append(t)
        for _ in range(int(rng.integers(0, 3))):
            accs[p].append(int(rng.integers(0, n_a)) if rng.random() < 0.8 else (p // per) * per + int(rng.integers(0, per)))
    for p, n_call, n_acc in hubs:
        own = p // per
        for q in range(own * per, (own + 1) * per):  # a cohesive home class: moving the hub out lowers its lcom
            if q != p:
                accs[q].extend(range(own * per, (own + 1) * per))
        others = [c for c in range(n_classes) if c != own]
        for c in rng.choice(others, size=n_call, replace=False):
            calls[p].append(int(c) * per + int(rng.integers(0, per)))
        for c in rng.choice(others, size=n_acc, replace=False):  # two attributes in each: lcom(dest) can drop
            accs[p].extend([int(c) * per, int(c) * per + 1])
        accs[p].append(own * per)  # and one own attribute
    return System.build(classes, calls, accs)


def test_gpu_hub_methods_all_candidates_and_topk(gpu_engine):
    # top-k / all-candidates modes for methods using 32..271 classes (the
    # reference's emit_for_method has no bound on |used(u)|, suggest.hpp:165-187)
    for seed in range(3):
        s = hub_system(np.random.default_rng(77 + seed))
        used = s.used_classes()
        assert used.max() >= 150 and (used >= 32).sum() >= 4
        check_against_oracle(gpu_engine, s, f"hub {seed}",
                             modes=((COH | COUP, 0, True), (COH | COUP, 1, True), (COH, 0, True), (COUP, 0, True),
                                    (COH | COUP, 0, False), (COH | COUP, 1, False)), top_ks=(1, 3, 8))
        for thr in (Thresholds(0, -1.0, -1.0), Thresholds(0, 0.0, 0.0)):
            lcom, ck, cbo = oracle.class_metrics(s)
            for mask, comb, allc, k in ((COH | COUP, 0, True, 1), (COH | COUP, 1, True, 1), (COH | COUP, 0, False, 5)):
                g = gpu_engine.suggest_all(thr, CRIT[mask], Combine(comb), allc, top_k=k)
                o = oracle.suggest(s, lcom, cbo, mask, comb, allc, k, thr.lcom, thr.cbo)
                assert records_equal(g, o), (seed, thr, mask, comb, allc, k, first_diff(g, o))
        if oracle.ref_available():  # and the reference itself, all-candidates
            R = oracle.RefModel(s)
            lcom, ck, cbo = R.class_metrics()
            gpu_engine.upload(s)
            for comb in (0, 1):  # every class gated in: the hubs emit up to ~120 records each
                want, _ = R.sweep(lcom, cbo, COH | COUP, -1.0, -1.0, comb, True, n_workers=4)
                g = gpu_engine.suggest_all(Thresholds(0, -1.0, -1.0), all_candidates=True, combine=Combine(comb))
                if comb == 0:
                    assert (want["method"] == 0).sum() > 100
                assert records_equal(g, want), (seed, comb, first_diff(g, want))


def test_gpu_similarity_huge_rows_and_mean(gpu_engine):
    # all_similarities has no row bound (metrics.hpp:67-77): an attribute with
    # 10,200 users (every user's candidate list is > 4096 entries) and a
    # method with 1,500 properties take the huge-row path (global scratch +
    # segmented sort); against the oracle and the compiled reference. The
    # similarity mean of compute_thresholds (suggest.hpp:55-56) on the device
    # table bit-equals the reference's sequential mean.
    rng = np.random.default_rng(5)
    n_cls, per = 60, 200
    n_m = n_a = n_cls * per
    classes = [(list(range(c * per, (c + 1) * per)), list(range(c * per, (c + 1) * per))) for c in range(n_cls)]
    calls = [[int(t) for t in rng.integers(0, n_m, size=int(rng.integers(0, 3))) if t != p] for p in range(n_m)]
    accs = [[int(a) for a in rng.integers(0, n_a, size=int(rng.integers(0, 3)))] for p in range(n_m)]
    for p in range(10200):
        accs[p].append(7)  # attribute 7: 10,200 users
    calls[11000] = [t for t in range(1500) if t != 11000]  # 1,499 call properties
    s = System.build(classes, calls, accs)
    gpu_engine.upload(s)
    g = gpu_engine.similarities()
    assert len(g) > 10200 * 10199 // 2
    o = oracle.similarities(s)
    assert g.tobytes() == o.tobytes(), (len(g), len(o))
    del o
    lcom, ck, cbo = gpu_engine.class_metrics_all()
    t = gpu_engine.compute_thresholds()
    want = oracle.thresholds(lcom, cbo, g["value"])
    assert (t.similarity, t.lcom, t.cbo) == (want.similarity, want.lcom, want.cbo)
    if oracle.ref_available():
        r = oracle.RefModel(s).similarities(os.cpu_count() or 1)
        assert g.tobytes() == r.tobytes()
        del r
        wr = oracle.ref_thresholds(lcom, cbo, g["value"])
        assert (t.similarity, t.lcom, t.cbo) == (wr.similarity, wr.lcom, wr.cbo)
        # compute_thresholds on a caller's report, every override combination
        for ov in (None, ThresholdOverrides(lcom=0.25), ThresholdOverrides(0.1, None, 3.0)):
            a = gpu_engine.report_thresholds(lcom, cbo, g, ov)
            b = oracle.ref_thresholds(lcom, cbo, g["value"], None if ov is None else
                                      {k: getattr(ov, k) for k in ("similarity", "lcom", "cbo")})
            assert (a.similarity, a.lcom, a.cbo, a.explicit_mode) == (b.similarity, b.lcom, b.cbo,
                                                                      bool(b.explicit_mode)), ov


def test_gpu_report_thresholds_random(gpu_engine):
    # the device means of arbitrary report vectors (the drop-in's
    # gpu::compute_thresholds) against the reference's compute_thresholds
    rng = np.random.default_rng(11)
    for n in (0, 1, 5, 2047, 2048, 2049, 100000, 333333):
        lcom = rng.integers(0, 2 ** 53 + 1, n).astype(np.float64) * 2.0 ** -53
        cbo = rng.integers(0, 200, n).astype(np.uint32)
        sim = rng.random(n // 3 + 1)
        a = gpu_engine.report_thresholds(lcom, cbo, sim)
        b = oracle.thresholds(lcom, cbo, sim)
        assert (a.similarity, a.lcom, a.cbo) == (b.similarity, b.lcom, b.cbo), n
    a = gpu_engine.report_thresholds(rng.random(10), rng.integers(0, 9, 7).astype(np.uint32), None)
    assert a.similarity == 0.0


@pytest.mark.parametrize("env", [{}, {"MMGPU_GROUP": "0"}, {"MMGPU_LEAN": "0"}, {"MMGPU_SCORE_FAST": "0"}],
                         ids=["default", "warp-per-class", "method+class-small", "general-scorer"])
def test_gpu_metric_pass_and_scorer_variants(monkeypatch, env):
    """Every route a small class can take through the metric pass — groups of
    whole classes per warp (k_class_group), one warp per class (k_class_lean:
    the solo list of members with degree 9..16, and everything under
    MMGPU_GROUP=0), the round-1 k_method + k_class_small chain (MMGPU_LEAN=0)
    — and both best-only scorers, against the oracle on systems whose member
    degrees reach 16 (so solo classes, record overflow and listed warp-path
    classes all occur)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    with Engine(0) as e:
        for seed in range(10):
            rng = np.random.default_rng(4100 + seed)
            cfg = dict(seed=seed, n_classes=int(rng.integers(20, 300)), n_methods=int(rng.integers(200, 4000)),
                       n_attributes=int(rng.integers(100, 6000)), k_max_calls=int(rng.integers(0, 9)),
                       k_max_accesses=int(rng.integers(0, 9)), intra_class_bias=float(rng.random()))
            s = System.generate(**cfg)
            check_against_oracle(e, s, f"{env} seed {seed}",
                                 modes=((COH | COUP, 0, False), (COH | COUP, 1, False), (COH | COUP, 0, True)))
