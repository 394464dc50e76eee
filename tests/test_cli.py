"""tools/_build/mmgpu — the reference CLI's subcommands with `--engine gpu`
(tools/mmgpu_cli.cpp), after the reference's tests/test_cli.cpp.

Host-only cases run the reference engines (sequential / parallel) and the
shared paths (generate, validate, exit codes). The GPU cases require the gpu
engine's output to equal the reference engine's BYTE FOR BYTE for analyze and
suggest (json and text, criteria subsets, intersection, all-candidates,
explicit thresholds) — the renderers are the reference's own, so this is the
full_report / suggest_all parity seen through the CLI."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parents[1] / "tools" / "_build" / "mmgpu"
pytestmark = pytest.mark.skipif(not BIN.exists(), reason="tools/_build/mmgpu not built (needs the reference headers)")


def cli(*args, check=True):
    r = subprocess.run([str(BIN), *map(str, args)], capture_output=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stderr.decode()
    return r


def gen(tmp_path, name, classes, methods, attributes, seed=1, kc=4, ka=4, bias=0.5):
    p = tmp_path / f"{name}.json"
    cli("generate", "--classes", classes, "--methods", methods, "--attributes", attributes, "--kmax-calls", kc,
        "--kmax-accesses", ka, "--intra-bias", bias, "--seed", seed, "--out", p)
    return p


def test_generate_then_validate(tmp_path):
    p = gen(tmp_path, "g", 6, 40, 20, seed=5)
    r = cli("validate", "--facts", p)
    assert r.stdout.decode().startswith("ok:") and "40 methods" in r.stdout.decode()


def test_generate_is_deterministic(tmp_path):
    a, b = gen(tmp_path, "a", 5, 30, 12, seed=9), gen(tmp_path, "b", 5, 30, 12, seed=9)
    c = gen(tmp_path, "c", 5, 30, 12, seed=10)
    assert a.read_bytes() == b.read_bytes() != c.read_bytes()


def test_reference_engines_agree(tmp_path):
    p = gen(tmp_path, "g", 30, 300, 200)
    seq = cli("analyze", "--facts", p, "--engine", "sequential").stdout
    par = cli("analyze", "--facts", p, "--engine", "parallel", "--workers", 3).stdout
    assert seq and seq == par
    txt = cli("analyze", "--facts", p, "--engine", "sequential", "--format", "text").stdout.decode()
    assert "300 methods" in txt and "n_total=" in txt


def test_exit_codes(tmp_path):
    assert cli("analyze", "--facts", tmp_path / "none.json", check=False).returncode == 4
    bad = tmp_path / "bad.json"
    bad.write_text('{"schema_version": "1", "classes": [')
    r = cli("validate", "--facts", bad, check=False)
    assert r.returncode == 2 and b"JSON parse error at line 1" in r.stderr
    inv = tmp_path / "inv.json"
    inv.write_text('{"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [],'
                   ' "methods": [{"id": 0, "name": "f", "calls": [12], "accesses": []}]}]}')
    r = cli("validate", "--facts", inv, check=False)
    assert r.returncode == 3 and b"  - method 0 calls unknown method 12" in r.stderr
    assert cli("analyze", "--engine", "x", "--facts", inv, check=False).returncode == 64
    assert cli("suggest", "--facts", inv, "--criteria", "speed", check=False).returncode == 64
    assert cli(check=False).returncode == 64


def test_gpu_engine_never_falls_back(tmp_path):
    # no device here: the gpu engine (the default) must fail loudly, not compute on the CPU
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    p = gen(tmp_path, "g", 4, 20, 10)
    r = cli("analyze", "--facts", p, check=False)
    assert r.returncode == 1 and b"no usable CUDA device" in r.stderr and not r.stdout


SUGGEST_VARIANTS = [
    (),
    ("--format", "text"),
    ("--criteria", "cohesion,coupling"),
    ("--criteria", "similarity", "--combine", "intersection"),
    ("--criteria", "coupling,similarity", "--combine", "intersection"),
    ("--all-candidates",),
    ("--threshold-similarity", "0.2", "--threshold-lcom", "0.4", "--threshold-cbo", "0.5"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(5, 30, 12, 42, 3, 3, 0.6), (60, 600, 900, 1, 4, 4, 0.5),
                                   (12, 400, 64, 3, 4, 16, 0.9), (1000, 10000, 20000, 1, 4, 4, 0.5)])
def test_gpu_engine_bytes_equal_reference(tmp_path, shape):
    c, m, a, seed, kc, ka, bias = shape
    p = gen(tmp_path, "s", c, m, a, seed=seed, kc=kc, ka=ka, bias=bias)
    for fmt in ("json", "text"):
        ref = cli("analyze", "--facts", p, "--engine", "sequential", "--format", fmt).stdout
        got = cli("analyze", "--facts", p, "--engine", "gpu", "--format", fmt).stdout
        assert got == ref, f"analyze {fmt}"
    variants = SUGGEST_VARIANTS if m <= 1000 else SUGGEST_VARIANTS[:3]
    for v in variants:
        ref = cli("suggest", "--facts", p, "--engine", "sequential", *v).stdout
        got = cli("suggest", "--facts", p, *v).stdout  # gpu is the default engine
        assert got == ref, f"suggest {v}"
