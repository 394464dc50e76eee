"""Several engines driven from several host threads (the e2e request pipeline
bench.py measures): every request's results equal one engine's serial run,
bit for bit. Exercises the library's shared state across contexts (kernel
attributes raised by one engine while another launches, per-device
co-residency limits) and the upload path's pinned staging."""
import threading

import numpy as np
import pytest

from conftest import first_diff, records_equal
from paper_1308_4011_b200 import Engine, System

pytestmark = pytest.mark.gpu

SHAPES = [
    # uniform lean classes (group / lean kernels)
    dict(seed=5, n_classes=2000, n_methods=20000, n_attributes=40000, k_max_calls=4, k_max_accesses=4,
         intra_class_bias=0.5),
    # Zipf sizes: CTA-path classes, giants split over CTAs
    dict(seed=6, n_classes=1000, n_methods=20000, n_attributes=40000, k_max_calls=4, k_max_accesses=4,
         intra_class_bias=0.5, zipf_s=1.0),
    # dense classes: 100 members x 60 attributes (tensor-core LCOM-CK, per-thread scoring)
    dict(seed=7, n_classes=50, n_methods=5000, n_attributes=3000, k_max_calls=4, k_max_accesses=32,
         intra_class_bias=0.9),
]


def request(e: Engine, s: System):
    e.upload(s, owner_tables=False)
    e.compute_metrics()
    lcom, ck, cbo = e.class_metrics_all()
    e.sweep(thresholds=None, want_count=False)
    return lcom, ck, cbo, e.suggestions()


def test_engines_on_threads_match_serial():
    systems = [System.generate(**kw) for kw in SHAPES]
    with Engine(0) as ref:
        want = [request(ref, s) for s in systems]
    engines = [Engine(0) for _ in range(3)]
    got, errors = {}, []

    def worker(i):
        try:
            for rep in range(3):
                for j in range((i + rep) % 3, (i + rep) % 3 + 3):  # engines on different shapes at once
                    got[(i, rep, j % 3)] = request(engines[i], systems[j % 3])
        except Exception as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(engines))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in engines:
        e.close()
    assert not errors, errors
    assert len(got) == 27
    for (i, rep, j), (lcom, ck, cbo, recs) in got.items():
        wl, wk, wc, wr = want[j]
        ctx = f"engine {i} round {rep} shape {j}"
        assert lcom.tobytes() == wl.tobytes(), ctx
        assert np.array_equal(ck, wk) and np.array_equal(cbo, wc), ctx
        assert records_equal(recs, wr), f"{ctx}: {first_diff(recs, wr)}"
