"""A small end-to-end workload for compute-sanitizer (tests/test_sanitizer.py).

Runs every kernel family of libmmgpu.so once on small systems — upload
(validation, expansion, plan), the metric pass (warp path, CTA path incl.
giant phase 1 / split LCOM-CK / tensor-core LCOM-CK), the threshold means
(one-CTA and cooperative), the sweep in every mode (screen + fallback, top-k,
all-candidates incl. wide methods, the decoupled look-back offsets, the
record writer), what-if, fan metrics, the similarity table incl. the huge-row
path and its criterion, and a one-GPU group with the NCCL exchange — and exits
0. No oracle: this checks memory / race / sync hygiene, not values."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1308_4011_b200 import Combine, Criterion, Engine, Group, System, Thresholds  # noqa: E402


def main():
    os.environ.setdefault("MMGPU_GIANT_MIN", "64")
    systems = [
        System.generate(seed=1, n_classes=300, n_methods=3000, n_attributes=6000),
        System.generate(seed=3, n_classes=8, n_methods=4000, n_attributes=512, k_max_calls=4, k_max_accesses=32,
                        intra_class_bias=0.9),   # dense: CTA path, tensor-core LCOM-CK
        System.generate(seed=11, n_classes=200, n_methods=6000, n_attributes=9000, k_max_calls=6, k_max_accesses=6,
                        intra_class_bias=0.5, zipf_s=1.0),  # giants
        System.generate(seed=14, n_classes=40, n_methods=2000, n_attributes=20000, k_max_calls=3,
                        k_max_accesses=24, intra_class_bias=0.6),  # A > 256, degree > 16
    ]
    n = 600  # a hub-ish system: one attribute with 600 users (similarity huge rows need > 4096: see below)
    systems.append(System.build([(list(range(4)), list(range(n)))], [[(p + 1) % n] for p in range(n)],
                                [[0, 1]] * n))
    with Engine(0) as e:
        for s in systems:
            e.upload(s)
            e.compute_metrics()
            t = e.compute_thresholds()
            for allc, k in ((False, 1), (False, 3), (True, 1)):
                for comb in (Combine.Union, Combine.Intersection):
                    e.suggest_all(t, all_candidates=allc, top_k=k, combine=comb)
            e.run(thresholds=None)
            e.run(thresholds=None)
            e.suggestions()
            e.fan_metrics()
            e.estimate_workload()
            for u in range(0, s.n_methods, max(1, s.n_methods // 7)):
                o = int(s.method_owner[u])
                e.what_if_move(u, o, (o + 1) % s.n_classes) if s.n_classes > 1 else None
            if s.n_methods <= 6000:
                e.suggest_all(t, [Criterion.Similarity, Criterion.Cohesion], Combine.Union)
        big = 4200  # > 4096 candidates per row: the similarity huge-row path
        s = System.build([(list(range(2)), list(range(big)))], [], [[0, 1]] * big)
        e.upload(s)
        e.similarities()
        e.sequential_mean(np.random.default_rng(0).random(5000))
        e.sequential_mean(np.arange(300000, dtype=np.float64) * 2.0 ** -53)
    with Group(n=1) as g:
        g.upload(systems[0])
        g.run(thresholds=None)
        g.suggestions()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
