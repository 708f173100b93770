"""Build libs5gpu.so in-tree for sm_100a (nvcc; no JIT cache)."""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB_PATH = LIB_DIR / "libs5gpu.so"
GEN_PATH = LIB_DIR / "libs5gen.so"  # corpus generator (bench / test infrastructure)
GEN_SOURCES = [CSRC / "s5g_gen.cu"]
GEN_DEPS = GEN_SOURCES + [ROOT / "include" / "s5g_gen.h"]
SOURCES = [CSRC / "s5g.cu"]
DEPS = SOURCES + [CSRC / "s5g_device.cuh", CSRC / "s5g_kernels.cuh", CSRC / "s5g_warpsort.cuh", CSRC / "s5g_merge.cuh", ROOT / "include" / "s5g.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-I", str(ROOT / "include"),
]


def nvcc() -> str:
    cand = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda")) / "bin" / "nvcc"
    return str(cand) if cand.exists() else "nvcc"


def up_to_date(path: Path = LIB_PATH, deps=DEPS) -> bool:
    if not path.exists():
        return False
    t = path.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in deps)


def _compile(path: Path, sources, extra_flags=()) -> subprocess.Popen:
    tmp = path.with_suffix(".so.tmp")
    extra = os.environ.get("S5G_NVCC_EXTRA", "").split()  # tuning experiments only
    cmd = [nvcc(), *NVCC_FLAGS, *extra_flags, *extra, "-o", str(tmp), *map(str, sources)]
    return cmd, tmp


def build_library(force: bool = False, verbose: bool = False) -> Path:
    """Build libs5gpu.so (the sorter) and libs5gen.so (corpus generator),
    the two nvcc runs side by side."""
    LIB_DIR.mkdir(exist_ok=True)
    jobs = []
    if force or not up_to_date():
        jobs.append((LIB_PATH, *_compile(LIB_PATH, SOURCES, ["-Xcompiler", "-fopenmp", "-lgomp"])))
    if force or not up_to_date(GEN_PATH, GEN_DEPS):
        jobs.append((GEN_PATH, *_compile(GEN_PATH, GEN_SOURCES, ["-Xcompiler", "-fopenmp", "-lgomp"])))
    procs = []
    for path, cmd, tmp in jobs:
        if verbose:
            print(" ".join(cmd))
        procs.append((path, tmp, subprocess.Popen(cmd)))
    for path, tmp, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, str(path))
        os.replace(tmp, path)
    return LIB_PATH


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))
