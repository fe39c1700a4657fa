"""Build the CUDA engine in-tree: ``libzks_b200.so`` next to this file (sm_100a only)."""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = [os.path.join(HERE, "csrc", "zks_capi.cu")]
HEADERS = [
    os.path.join(HERE, "csrc", f)
    for f in ("zks_stream.cuh", "zks_series.cuh", "zks_replicate.cuh", "zks_select.cuh", "zks_probe.cuh", "zks_fit.cuh", "zks_batch.cuh", "zks_ks.cuh", "zks_samples.cuh", "zks_rows.cuh", "zks_lanes.cuh")
] + [os.path.join(os.path.dirname(HERE), "include", "zipfks_b200.h")]
LIB = os.environ.get("ZKS_LIB") or os.path.join(HERE, "libzks_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found; the engine is CUDA-only (sm_100a)")
    return path


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    built = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > built for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the engine if any source is newer than the library; return its path."""
    if not force and not stale():
        return LIB
    tmp = LIB + ".tmp"
    extra = os.environ.get("ZKS_NVCC_EXTRA", "").split()  # tuning experiments, e.g. -DZKS_DRAW_MINB=3
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", tmp, *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


DEBUG_LIB = os.path.join(HERE, "libzks_b200_debug.so")


def build_debug_bounds() -> str:
    """The bounds-checked variant (-DZKS_DEBUG_BOUNDS: violated indices trap), loaded instead of the
    product library with ZKS_LIB=<path>; for tests only."""
    tmp = DEBUG_LIB + ".tmp"
    subprocess.run([nvcc(), *NVCC_FLAGS, "-DZKS_DEBUG_BOUNDS", "-o", tmp, *SOURCES], check=True)
    os.replace(tmp, DEBUG_LIB)
    return DEBUG_LIB


if __name__ == "__main__":
    import sys

    print(build_debug_bounds() if "--debug-bounds" in sys.argv else build(force=True, verbose=True))
