"""compute-sanitizer over the whole kernel set (tools/sanitize_case.py).

memcheck runs in the GPU suite (out-of-bounds / misaligned accesses, leaks of
device allocations, API errors). racecheck and synccheck (shared-memory races,
barrier misuse) are run one tool per GPU call — several sanitizer tools in one
process have left a B200 unusable on this pool — and their logs are kept
under profiles/ (r2_sanitizer_*.log); set MMGPU_SANITIZE_ALL=1 to run them
here too."""
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CASE = ROOT / "tools" / "sanitize_case.py"
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not Path(SAN).exists(), reason="compute-sanitizer not found")]


def run_tool(tool: str):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9"]
    if tool == "memcheck":
        cmd += ["--leak-check", "full"]
    r = subprocess.run(cmd + [sys.executable, str(CASE)], capture_output=True, text=True, timeout=1200,
                       env=dict(os.environ, PYTHONUNBUFFERED="1"))
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "sanitize case ok" in out, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]


def test_memcheck():
    run_tool("memcheck")


@pytest.mark.skipif(os.environ.get("MMGPU_SANITIZE_ALL") != "1", reason="one sanitizer tool per GPU call")
@pytest.mark.parametrize("tool", ["racecheck", "synccheck", "initcheck"])
def test_other_tools(tool):
    run_tool(tool)
