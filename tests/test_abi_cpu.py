"""CPU-side checks of the C ABI library: it loads, exports every symbol the
header declares, host-only entry points work, and compute entry points fail
cleanly (never fall back to the CPU) when no CUDA device is present."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_1308_4011_b200 import Engine, MMError, System, abi, lib, plan_shards
from paper_1308_4011_b200._lib import EXPORTED

HEADER = Path(__file__).resolve().parents[1] / "include" / "mmgpu.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(mm_[a-z_]+)\s*\(", text)))


def test_header_symbols_exported():
    l = lib()
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(l, n), f"libmmgpu.so does not export {n}"
    assert set(names) == set(EXPORTED), "ctypes binding table out of sync with include/mmgpu.h"
    assert l.mm_abi_version() == 1


def test_struct_sizes_match_header():
    assert C.sizeof(abi.mm_suggestion) == 64
    assert C.sizeof(abi.mm_whatif) == 56
    assert C.sizeof(abi.mm_sweep_params) == 48
    assert C.sizeof(abi.mm_system) == 16 + 10 * 8


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(MMError) as ei:
        Engine(0)
    assert ei.value.status == abi.MM_E_CUDA


def test_generator_matches_reference_golden_digests():
    # digests of the reference generate() output, recorded by make_golden.py
    from conftest import load_golden
    for name in ("sample_generated", "config_c2"):
        case = load_golden(name)
        spec = case["system"]
        s = System.generate(**spec["generate"]) if "generate" in spec else System.generate(
            seed=42, n_classes=5, n_methods=30, n_attributes=12, k_max_calls=3, k_max_accesses=3,
            intra_class_bias=0.6)
        assert s.digest() == case["digest"], name


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_generator_matches_compiled_reference():
    rng = np.random.default_rng(5)
    for seed in range(40):
        cfg = dict(seed=seed, n_classes=int(rng.integers(1, 50)), n_methods=int(rng.integers(0, 500)),
                   n_attributes=int(rng.integers(0, 300)), k_max_calls=int(rng.integers(0, 6)),
                   k_max_accesses=int(rng.integers(0, 6)), intra_class_bias=float(rng.random()))
        assert System.generate(**cfg).equals(oracle.ref_generate(**cfg)), cfg
    cfg = dict(seed=1, n_classes=10000, n_methods=100000, n_attributes=200000, k_max_calls=4, k_max_accesses=4,
               intra_class_bias=0.5)
    assert System.generate(**cfg).equals(oracle.ref_generate(**cfg))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_zipf_generator_validates():
    s = System.generate(seed=1, n_classes=500, n_methods=5000, n_attributes=10000, zipf_s=1.0)
    assert oracle.RefModel(s).validate() == 0
    sizes = np.diff(s.class_method_off)
    assert sizes.min() >= 1 and sizes.sum() == 5000 and sizes.max() > 20 * np.median(sizes)


def test_generator_rejects_bad_config():
    with pytest.raises(MMError):
        System.generate(seed=0, n_classes=0, n_methods=1, n_attributes=0)
    with pytest.raises(MMError):
        System.generate(seed=0, n_classes=1, n_methods=1, n_attributes=0, intra_class_bias=1.5)


def test_plan_shards_contiguous_balanced():
    s = System.generate(seed=3, n_classes=1000, n_methods=20000, n_attributes=5000, zipf_s=1.0)
    for n in (1, 2, 4, 8, 3000):
        b = plan_shards(s, n)
        assert b[0] == 0 and b[-1] == s.n_classes and np.all(np.diff(b.astype(np.int64)) >= 0)
    with pytest.raises(MMError):
        plan_shards(s, 0)


def test_system_build_matches_fixture_semantics():
    # fixtures.hpp:22-69 sorts memberships and dedupes dependency lists
    s = System.build([([1, 0], [1, 0]), ([2], [2])], [[2, 2], [], []], [[1, 0, 1], [], [2]])
    assert s.members(0).tolist() == [0, 1] and s.attrs(0).tolist() == [0, 1]
    assert s.calls(0).tolist() == [2] and s.accesses(0).tolist() == [0, 1]
    assert s.method_owner.tolist() == [0, 0, 1]


def test_candidate_count_matches_survey_c2():
    s = System.generate(seed=1, n_classes=1000, n_methods=10000, n_attributes=20000)
    assert s.n_candidates() == 19933
