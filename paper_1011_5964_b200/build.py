"""Build the native library ``libtvdeblur_b200.so`` in-tree with nvcc (sm_100a).

    python -m paper_1011_5964_b200.build [--force]

Each translation unit compiles to an object in parallel (no cross-unit device
code), then nvcc links the shared library.  ``TVD_EXTRA_NVCC_FLAGS`` appends
flags (profiling builds, e.g. ``-DTVD_PIPE_TIMING``).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import shlex
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libtvdeblur_b200.so"
OBJ = PKG / "_obj"
SOURCES = ["tvd_lines.cu", "tvd_pfa.cu", "tvd_rader.cu", "tvd_stencil.cu", "tvd_band_mma.cu", "tvd_cg.cu",
           "tvd_capi.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not LIB.exists():
        return True
    newest = max(p.stat().st_mtime for p in list(CSRC.glob("*")) + [PKG.parent / "include" / "tvdeblur_b200.h"])
    return newest > LIB.stat().st_mtime


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    if not force and not _stale():
        return LIB
    OBJ.mkdir(exist_ok=True)
    extra = shlex.split(os.environ.get("TVD_EXTRA_NVCC_FLAGS", ""))
    nvcc = _nvcc()

    def compile_one(src: str) -> pathlib.Path:
        obj = OBJ / (pathlib.Path(src).stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", "-o", str(obj), str(CSRC / src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(LIB),
           *[str(o) for o in objs]]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
