"""The CPU oracle (oracle/mmoracle.c) pinned against the reference.

(a) Known answers from the reference's own tests and README, cited inline.
(b) tests/golden/*.json — outputs of the reference itself (make_golden.py).
(c) When oracle/_ref/libmmref.so is present (built here from the reference
    headers), oracle == reference on randomly generated systems.
"""
import math

import numpy as np
import pytest

import oracle
from conftest import golden_names, golden_records, golden_system, load_golden, records_equal, unhex, first_diff
from paper_1308_4011_b200 import System, abi

COH, COUP = abi.MM_CRIT_COHESION, abi.MM_CRIT_COUPLING


def test_lcom_worked_example():
    # test_metrics.cpp:102-109 — two attributes, two methods, 3 of 4 accesses -> 0.25
    s = System.build([([0, 1], [0, 1])], [[], []], [[0, 1], [0]])
    assert oracle.class_metrics(s)[0][0] == 0.25


@pytest.mark.parametrize("classes,calls,accs,want", [
    ([([0, 1], [0, 1])], [[], []], [[0, 1], [0, 1]], 0.0),                 # perfect cohesion, :112-115
    ([([0], [0, 1]), ([1], [2])], [[], [], []], [[1], [], []], 1.0),       # no own access, :116-120
    ([([], [0, 1]), ([0], [])], [[], []], [[0], [0]], 0.0),                # no attributes, :121-124
    ([([0], []), ([], [0])], [[]], [[0]], 0.0),                            # no methods, :125-128
])
def test_lcom_degenerate(classes, calls, accs, want):
    assert oracle.class_metrics(System.build(classes, calls, accs))[0][0] == want


@pytest.mark.parametrize("classes,accs,want", [
    ([([0, 1, 2], [0, 1, 2])], [[0], [1], [2]], 3),    # test_metrics.cpp:138-145
    ([([0, 1], [0, 1, 2])], [[0], [0], [1]], 1),       # :146-152
    ([([0, 1], [0, 1, 2])], [[0], [0], [0]], 0),       # :154-159 clamp
    ([([0], [0])], [[0]], 0),                          # :161-164 fewer than two
    ([([0], [0, 1]), ([1], [])], [[1], [1]], 1),       # :165-171 foreign attrs don't count
])
def test_lcom_ck_known(classes, accs, want):
    s = System.build(classes, [[] for _ in accs], accs)
    assert int(oracle.class_metrics(s)[1][0]) == want


def test_cbo_known():
    # test_metrics.cpp:173-192
    s = System.build([([], [0]), ([], [1]), ([0], [2])], [[1, 2], [], []], [[0], [], []])
    assert oracle.class_metrics(s)[2].tolist() == [2, 0, 0]
    s = System.build([([0], [0, 1])], [[1], []], [[0], [0]])
    assert oracle.class_metrics(s)[2].tolist() == [0]


def test_thresholds_known():
    # test_suggest.cpp:52-86
    t = oracle.thresholds([0.25, 0.75], [1, 2], similarity=[0.5, 1.0])
    assert (t.similarity, t.lcom, t.cbo, t.explicit_mode) == (0.75, 0.5, 1.5, 0)
    t = oracle.thresholds([], [])
    assert (t.similarity, t.lcom, t.cbo) == (0.0, 0.0, 0.0)
    t = oracle.thresholds([0.4], [3], similarity=[0.5], overrides={"lcom": 0.9})
    assert (t.similarity, t.lcom, t.cbo, t.explicit_mode) == (0.5, 0.9, 3.0, 1)


def test_what_if_envy_and_errors():
    # test_suggest.cpp:88-109
    s = System.build([([0, 1], [0, 1]), ([2, 3], [2])], [[2], [], []], [[2, 3], [0, 1], [2]])
    st, w = oracle.what_if(s, 0, 0, 1)
    assert st == 0
    assert (w.lcom_origin_before, w.lcom_origin_after, w.lcom_dest_before, w.lcom_dest_after) == (0.5, 0.0, 0.5, 0.25)
    assert (w.cbo_origin_before, w.cbo_origin_after, w.cbo_dest_before, w.cbo_dest_after) == (1, 0, 0, 0)
    assert oracle.what_if(s, 0, 0, 0)[0] == abi.MM_E_ARG
    assert oracle.what_if(s, 2, 0, 1)[0] == abi.MM_E_ARG
    assert oracle.what_if(s, 0, 0, 9)[0] == abi.MM_E_RANGE
    assert oracle.what_if(s, 0, 7, 1)[0] == abi.MM_E_RANGE


def test_billing_readme_known_answers():
    # SURVEY.md §8c (README.md:69-94 reproduced): lcom [0.5,0.5], ck [1,0], cbo [1,0];
    # mean thresholds lcom 0.5 cbo 0.5; one coupling move m1 0->1
    case = load_golden("sample_billing")
    s = golden_system(case)
    lcom, ck, cbo = oracle.class_metrics(s)
    assert lcom.tolist() == [0.5, 0.5] and ck.tolist() == [1, 0] and cbo.tolist() == [1, 0]
    t = oracle.thresholds(lcom, cbo)
    assert (t.lcom, t.cbo) == (0.5, 0.5)
    out = oracle.suggest(s, lcom, cbo, COH | COUP, 0, False, 1, t.lcom, t.cbo)
    assert len(out) == 1 and (out[0]["method"], out[0]["origin"], out[0]["destination"]) == (1, 0, 1)
    assert out[0]["criteria"] == COUP
    assert (out[0]["lcom_origin_after"], out[0]["lcom_dest_after"]) == (0.0, 0.25)


def test_generated_sample_known_answers():
    # samples/generated.json == generate(seed 42, 5c/30m/12a, k 3/3, bias .6)
    s = System.generate(seed=42, n_classes=5, n_methods=30, n_attributes=12, k_max_calls=3, k_max_accesses=3,
                        intra_class_bias=0.6)
    assert s.digest() == load_golden("sample_generated")["digest"]
    lcom, ck, cbo = oracle.class_metrics(s)
    assert lcom.tolist() == [0.72222222222222221, 0.72222222222222221, 0.66666666666666674,
                             0.66666666666666674, 0.66666666666666674]
    assert ck.tolist() == [11, 9, 9, 3, 11] and cbo.tolist() == [3, 4, 4, 3, 4]
    t = oracle.thresholds(lcom, cbo)
    assert t.lcom == 0.68888888888888888 and t.cbo == 3.6000000000000001
    out = oracle.suggest(s, lcom, cbo, COH | COUP, 0, False, 1, t.lcom, t.cbo)
    moves = [(int(r["method"]), int(r["origin"]), int(r["destination"]), int(r["criteria"])) for r in out]
    # m1 1->0 [coupling]; m11 1->2 [cohesion, coupling]; m12 2->1; m19 4->1; m29 4->2 [coupling]
    assert moves == [(1, 1, 0, COUP), (11, 1, 2, COH | COUP), (12, 2, 1, COUP), (19, 4, 1, COUP), (29, 4, 2, COUP)]
    assert len(oracle.suggest(s, lcom, cbo, COH | COUP, 0, True, 1, t.lcom, t.cbo)) == 7


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_golden(name):
    case = load_golden(name)
    s = golden_system(case)
    lcom, ck, cbo = oracle.class_metrics(s)
    assert [unhex(h) for h in case["lcom"]] == lcom.tolist()
    assert lcom.tobytes() == np.array([unhex(h) for h in case["lcom"]]).tobytes()
    assert ck.tolist() == case["lcom_ck"] and cbo.tolist() == case["cbo"]
    t = oracle.thresholds(lcom, cbo)
    assert t.lcom == unhex(case["thresholds_mean"]["lcom"]) and t.cbo == unhex(case["thresholds_mean"]["cbo"])
    for run in case["suggest"]:
        got = oracle.suggest(s, lcom, cbo, run["criteria"], run["combine"], run["all_candidates"], 1,
                             unhex(run["thr_lcom"]), unhex(run["thr_cbo"]))
        want = golden_records(run["suggestions"])
        assert records_equal(got, want), (run["criteria"], run["combine"], first_diff(got, want))
    for w in case.get("what_if", []):
        st, wm = oracle.what_if(s, w["u"], w["o"], w["d"])
        assert st == w["status"]
        if not st:
            for f, v in w["w"].items():
                got = getattr(wm, f)
                assert (got == unhex(v)) if f.startswith("lcom") else (got == v), (w, f)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_matches_compiled_reference_random():
    for seed in range(60):
        rng = np.random.default_rng(1000 + seed)
        cfg = dict(seed=seed, n_classes=int(rng.integers(2, 40)), n_methods=int(rng.integers(4, 400)),
                   n_attributes=int(rng.integers(1, 200)), k_max_calls=int(rng.integers(0, 6)),
                   k_max_accesses=int(rng.integers(0, 6)), intra_class_bias=float(rng.random()))
        s = System.generate(**cfg)
        R = oracle.RefModel(s)
        l, k, c = oracle.class_metrics(s)
        l2, k2, c2 = R.class_metrics()
        assert l.tobytes() == l2.tobytes() and (k == k2).all() and (c == c2).all()
        fi, fo = oracle.fan_metrics(s)
        for w in (0, 3):  # fan_in/fan_out and parallel_fan_metrics
            fi2, fo2 = R.fan_metrics(w)
            assert (fi == fi2).all() and (fo == fo2).all()
        t = oracle.thresholds(l, c)
        for mask, comb, allc in ((COH | COUP, 0, False), (COH | COUP, 1, True), (COH, 0, False), (COUP, 0, True)):
            a = oracle.suggest(s, l, c, mask, comb, allc, 1, t.lcom, t.cbo)
            st, b = R.suggest(l, c, mask, comb, allc, t.lcom, t.cbo)
            assert st == 0 and records_equal(a, b), (seed, mask, first_diff(a, b))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_ref_sweep_equals_suggest_all():
    # ref_sweep (the reference's per-method code on threads + suggest_all's
    # merge) is suggest_all itself over all methods, and suggest_all
    # restricted to the methods given otherwise — the basis of the sampled
    # parity tests at the BASELINE sizes
    for seed in range(25):
        rng = np.random.default_rng(4000 + seed)
        cfg = dict(seed=seed, n_classes=int(rng.integers(2, 60)), n_methods=int(rng.integers(4, 600)),
                   n_attributes=int(rng.integers(1, 300)), k_max_calls=int(rng.integers(0, 7)),
                   k_max_accesses=int(rng.integers(0, 7)), intra_class_bias=float(rng.random()),
                   zipf_s=float(rng.choice([0.0, 1.0])))
        s = System.generate(**cfg)
        R = oracle.RefModel(s)
        l, k, c = R.class_metrics()
        t = oracle.ref_thresholds(l, c)
        for mask, comb, allc in ((COH | COUP, 0, False), (COH | COUP, 1, False), (COH | COUP, 0, True),
                                 (COH | COUP, 1, True), (COH, 0, False), (COUP, 0, True)):
            st, want = R.suggest(l, c, mask, comb, allc, t.lcom, t.cbo)
            assert st == 0
            for workers, dyn in ((1, False), (3, True), (4, False)):
                got, cand = R.sweep(l, c, mask, t.lcom, t.cbo, comb, allc, n_workers=workers, dynamic=dyn)
                assert records_equal(got, want), (seed, mask, comb, allc, workers, first_diff(got, want))
                assert cand == s.n_candidates()
            sub = np.sort(rng.choice(s.n_methods, size=max(1, s.n_methods // 5), replace=False)).astype(np.uint32)
            got, _ = R.sweep(l, c, mask, t.lcom, t.cbo, comb, allc, methods=sub[::-1].copy(), n_workers=2)
            assert records_equal(got, want[np.isin(want["method"], sub)])


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_reference_generate_without_product():
    # bench.py's reference arm builds its input with the reference's own
    # generate() (no product library); it equals the product generator, Zipf
    # variant (config C3) included
    for cfg in (dict(seed=1, n_classes=1000, n_methods=10000, n_attributes=20000, k_max_calls=4, k_max_accesses=4,
                     intra_class_bias=0.5),
                dict(seed=1, n_classes=2000, n_methods=20000, n_attributes=40000, k_max_calls=4, k_max_accesses=4,
                     intra_class_bias=0.5, zipf_s=1.0),
                dict(seed=7, n_classes=37, n_methods=900, n_attributes=50, k_max_calls=6, k_max_accesses=2,
                     intra_class_bias=0.2, zipf_s=0.7)):
        r = oracle.ref_generate(**cfg)
        assert System.generate(**cfg).equals(r), cfg
        R = oracle.ref_generate_model(**cfg)
        assert R.validate() == 0
        assert R.candidates() == System.generate(**cfg).n_candidates()
