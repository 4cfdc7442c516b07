"""Build the in-tree CUDA library ``_lib/libwindvox_b200.so`` for sm_100a.

Plain nvcc (no torch headers): every .cu under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into one
shared object that exports the C ABI of ``include/windvox_b200.h``.  The
f64 staging/parity files are compiled with ``-fmad=false`` so their
expressions are the same IEEE sequence as the numpy/numba reference.

    python -m paper_2407_11272_b200._build [--verbose]
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUTDIR = PKG / "_lib"
OBJDIR = OUTDIR / "obj"
LIB = OUTDIR / "libwindvox_b200.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", str(CSRC), "-I", str(INCLUDE)]
# files whose f64 arithmetic must not be FMA-contracted
# host code that runs on all cores (parallel sorts of the strip builder)
OPENMP = {"wv_strip.cu", "wv_trail.cu"}
NO_FMAD = {"wv_pack.cu", "wv_f64.cu", "wv_mc.cu", "wv_metrics.cu", "wv_strip.cu", "wv_trail.cu"}


def _nvcc() -> str:
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        raise RuntimeError("nvcc not found; the windvox_b200 CUDA library cannot be built")
    return nvcc


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, objdir: Path | None = None,
          lib: Path | None = None) -> Path:
    """Compile every csrc/*.cu (stale ones only) and link the library.
    ``objdir`` / ``lib``: another object directory and output (A/B variant
    builds, tools/build_variant.py)."""
    nvcc = _nvcc()
    OBJDIR_ = objdir or OBJDIR
    LIB_ = lib or LIB
    OBJDIR_.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    objs = []
    for src in sources():
        obj = OBJDIR_ / (src.stem + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [src, *headers]):
            continue
        # WV_NVCC_DEFINES: extra -D flags for A/B builds of kernel variants
        extra = os.environ.get("WV_NVCC_DEFINES", "").split()
        cmd = [nvcc, *ARCH, *COMMON, *extra, "-c", str(src), "-o", str(obj)]
        if src.name in NO_FMAD:
            cmd.insert(-4, "-fmad=false")
        if src.name in OPENMP:
            cmd[-4:-4] = ["-Xcompiler", "-fopenmp"]
        if verbose:
            cmd.insert(-4, "-Xptxas=-v")
        print("[windvox_b200] nvcc", src.name, flush=True)
        subprocess.run(cmd, check=True)
    if force or _stale(LIB_, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", str(LIB_), *map(str, objs), "-lcudart_static",
               "-lrt", "-lpthread", "-ldl", "-lgomp"]
        subprocess.run(cmd, check=True)
    return LIB_


def build_probe() -> Path:
    """tools/ffma2_probe: the FP32 peak microbenchmark bench.py reports."""
    src = PKG.parent / "tools" / "ffma2_probe.cu"
    exe = src.with_suffix("")
    if _stale(exe, [src]):
        subprocess.run([_nvcc(), *ARCH, "-O3", "-o", str(exe), str(src)], check=True)
    return exe


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force="--force" in sys.argv)
    build_probe()
    print(LIB)
