"""Build the in-tree native libraries.

    libmmgpu.so  (paper_1308_4011_b200/)  the product: CUDA kernels for sm_100a + the C ABI
    oracle/liboracle.so, oracle/_ref/libmmref.so  test/baseline infrastructure (oracle/Makefile)

Everything is compiled explicitly with nvcc / gcc into the source tree so the
built .so files travel with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libmmgpu.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",          # IEEE mul/add everywhere; the fp64 metric paths also use _rn intrinsics
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False) -> Path:
    deps = _sources() + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "mmgpu.h", ROOT / "include" / "mmfacts.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    # one nvcc per translation unit, in parallel (no device code crosses
    # units), then one link
    from concurrent.futures import ThreadPoolExecutor
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    srcs = _sources()
    objs = [objdir / (s.name + ".o") for s in srcs]
    cmds = [[NVCC, *NVCC_FLAGS, "-c", "-o", str(o), str(s)] for s, o in zip(srcs, objs)]
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds))
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(LIB), *map(str, objs)]
    if all(r.returncode == 0 for r in results):
        results.append(subprocess.run(link, capture_output=True, text=True))
    log = PKG / "build.log"
    log.write_text("\n\n".join(" ".join(c) + "\n" + r.stdout + r.stderr for c, r in zip(cmds + [link], results)))
    if any(r.returncode != 0 for r in results):
        sys.stderr.write("".join(r.stdout + r.stderr for r in results if r.returncode != 0))
        raise RuntimeError(f"nvcc failed building {LIB.name} (see {log})")
    if verbose:
        sys.stderr.write("".join(r.stderr for r in results))
    return LIB


def build_variant(name: str, defines) -> Path:
    """A/B build of the same sources with extra -D flags (development only):
    paper_1308_4011_b200/_variants/libmmgpu_<name>.so, selected at run time by
    MMGPU_LIB=<path> (the product is always libmmgpu.so)."""
    out = PKG / "_variants" / f"libmmgpu_{name}.so"
    out.parent.mkdir(exist_ok=True)
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-shared", "-o", str(out), *map(str, _sources())]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(res.stdout + res.stderr)
    return out


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)


def build_tools() -> None:
    """tools/_build/mmgpu (the CLI with --engine gpu; needs the reference headers)."""
    subprocess.run(["make", "-s", "-C", str(ROOT / "tools")], check=True)


def build_all(force: bool = False) -> None:
    build_lib(force=force)
    build_oracle()
    build_tools()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built", LIB)
