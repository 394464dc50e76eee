"""Generate tests/golden/*.json by running the REFERENCE itself.

The reference headers (/root/reference/proj/include) are compiled in place by
oracle/Makefile into oracle/_ref/libmmref.so; this script drives that library
on the bundled samples, the reference's own test fixtures, small generated
systems and config C2, and records raw results (doubles as IEEE-754 hex) so
tests can check the oracle and the GPU bit for bit without the reference
present. Re-run: `python tests/golden/make_golden.py` (needs /root/reference).
"""
from __future__ import annotations

import json
import struct
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_1308_4011_b200 import System, abi  # noqa: E402

OUT = Path(__file__).resolve().parent
REF_SAMPLES = Path("/root/reference/proj/samples")


def hexd(x: float) -> str:
    return struct.pack("<d", float(x)).hex()


def rec_to_json(r) -> dict:
    d = {k: int(r[k]) for k in ("method", "origin", "destination", "cbo_origin_before", "cbo_origin_after",
                                "cbo_dest_before", "cbo_dest_after", "criteria", "origin_degenerate_after",
                                "dest_degenerate_after")}
    for k in ("lcom_origin_before", "lcom_origin_after", "lcom_dest_before", "lcom_dest_after"):
        d[k] = hexd(r[k])
    return d


def system_json(s: System) -> dict:
    return {"classes": [[s.attrs(c).tolist(), s.members(c).tolist()] for c in range(s.n_classes)],
            "calls": [s.calls(p).tolist() for p in range(s.n_methods)],
            "accesses": [s.accesses(p).tolist() for p in range(s.n_methods)]}


def run_case(name: str, s: System, spec: dict, explicit=None, sugg=True, whatifs=True) -> None:
    R = oracle.RefModel(s)
    assert R.validate() == 0, name
    lcom, ck, cbo = R.class_metrics()
    case = {"name": name, "system": spec, "digest": s.digest(),
            "lcom": [hexd(v) for v in lcom], "lcom_ck": [int(v) for v in ck], "cbo": [int(v) for v in cbo]}
    t_mean = oracle.ref_thresholds(lcom, cbo)
    case["thresholds_mean"] = {"lcom": hexd(t_mean.lcom), "cbo": hexd(t_mean.cbo)}
    runs = []
    thr_sets = [("mean", t_mean.lcom, t_mean.cbo)]
    if explicit:
        thr_sets.append(("explicit", explicit[0], explicit[1]))
    if sugg:
        for tname, tl, tc in thr_sets:
            for mask in (abi.MM_CRIT_COHESION, abi.MM_CRIT_COUPLING, abi.MM_CRIT_COHESION | abi.MM_CRIT_COUPLING):
                for comb in (0, 1):
                    for allc in (False, True):
                        if mask != 6 and comb == 1:
                            continue
                        st, out = R.suggest(lcom, cbo, mask, comb, allc, tl, tc)
                        assert st == 0, (name, st)
                        runs.append({"thresholds": tname, "thr_lcom": hexd(tl), "thr_cbo": hexd(tc),
                                     "criteria": mask, "combine": comb, "all_candidates": allc,
                                     "suggestions": [rec_to_json(r) for r in out]})
    case["suggest"] = runs
    if whatifs:
        w = []
        for u in range(s.n_methods):
            o = int(s.method_owner[u])
            for d in range(s.n_classes):
                st, wm = R.what_if(u, o, d)
                w.append({"u": u, "o": o, "d": d, "status": st,
                          "w": None if st else {f: (hexd(getattr(wm, f)) if f.startswith("lcom") else
                                                    int(getattr(wm, f))) for f in abi.WHATIF_FIELDS}})
        case["what_if"] = w
    (OUT / f"{name}.json").write_text(json.dumps(case, separators=(",", ":")))
    print(name, "classes", s.n_classes, "methods", s.n_methods, "runs", len(runs))


def main() -> None:
    for sample in ("billing", "generated"):
        s = System.from_facts(REF_SAMPLES / f"{sample}.json")
        run_case(f"sample_{sample}", s, {"build": system_json(s)}, explicit=(0.4, 0.5))
    # the reference's named fixtures, tests/test_suggest.cpp:17-40 and :284-309
    fixtures = {
        "fixture_envy": ([([0, 1], [0, 1]), ([2, 3], [2])], [[2], [], []], [[2, 3], [0, 1], [2]], (0.4, 0.5)),
        "fixture_cohesion": ([([0, 1], [0, 1]), ([2, 3], [2])], [[], [2], []], [[0, 1], [2, 3], [2]], (0.3, 0.5)),
        "fixture_coupling": ([([], [0]), ([], [1]), ([], [2])], [[1, 2], [2], []], [], (2.0, 1.5)),
        "fixture_tie": ([([0], [0, 1]), ([1], [2]), ([2], [3])], [[], [], [], []], [[1, 2], [0], [], []],
                        (0.4, 99.0)),
    }
    for name, (classes, calls, accs, expl) in fixtures.items():
        s = System.build(classes, calls, accs)
        run_case(name, s, {"build": system_json(s)}, explicit=expl)
    # generated systems: test_suggest.cpp:402-430 style draws
    for seed in range(10):
        rng = np.random.default_rng(seed * 13 + 5)
        cfg = dict(seed=seed, n_classes=int(2 + rng.integers(0, 7)), n_methods=int(4 + rng.integers(0, 22)),
                   n_attributes=int(2 + rng.integers(0, 14)), k_max_calls=int(rng.integers(0, 5)),
                   k_max_accesses=int(rng.integers(0, 5)), intra_class_bias=float(rng.random()))
        s = System.generate(**cfg)
        run_case(f"gen_small_{seed}", s, {"generate": cfg}, explicit=(0.3, 1.0))
    # config C2: metrics + mean-threshold suggestions, no what-if table
    cfg = dict(seed=1, n_classes=1000, n_methods=10000, n_attributes=20000, k_max_calls=4, k_max_accesses=4,
               intra_class_bias=0.5)
    run_case("config_c2", System.generate(**cfg), {"generate": cfg}, whatifs=False)


if __name__ == "__main__":
    main()
