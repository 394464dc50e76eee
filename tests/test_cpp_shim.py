"""The C++ drop-in (include/modmetrics/gpu.hpp) against the reference itself.

oracle/_ref/shim_parity is built here from the unmodified reference headers and
links libmmgpu.so; on a GPU box it compares, with the reference's own types and
operator==, parallel_class_metrics / parallel_lcom_ck / lcom_normalized / cbo /
lcom_ck / what_if_move / suggest_by_cohesion / suggest_by_coupling /
suggest_all (vector ORDER included, exception types included)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "shim_parity"


@pytest.mark.gpu
@pytest.mark.skipif(not BIN.exists(), reason="oracle/_ref/shim_parity not built (needs /root/reference at build time)")
def test_cpp_dropin_equals_reference():
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900)
    tail = res.stdout[-4000:]
    assert res.returncode == 0, tail
    assert "PASS" in tail
