"""In-tree build of the sm_100a C-ABI library ``libspmoe.so``.

``nvcc`` cross-compiles for ``sm_100a`` without a GPU, so this runs in the
CPU container (``__graft_entry__.build``) and the resulting ``.so`` travels
to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
REPO = PKG_DIR.parent
LIB_PATH = PKG_DIR / "libspmoe.so"

SOURCES = [CSRC / "spmoe_kernels.cu", CSRC / "spmoe_tc.cu", CSRC / "spmoe_codec.cu", CSRC / "spmoe_attn.cu",
           CSRC / "spmoe_runtime.cpp"]
HEADERS = [CSRC / "spmoe_common.cuh", REPO / "include" / "spmoe.h"]

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; the spmoe CUDA library cannot be built")
    return cand


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    return any(p.exists() and p.stat().st_mtime > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile ``libspmoe.so`` for sm_100a if any source is newer than it."""
    if not force and not _stale():
        return LIB_PATH
    srcs = [str(s) for s in SOURCES if s.exists()]
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [
        nvcc_path(),
        *ARCH_FLAGS,
        "-O3",
        "-lineinfo",
        "-std=c++17",
        "-Xcompiler",
        "-fPIC,-O3",
        "-Xptxas",
        "-v" if verbose else "-O3",
        "-shared",
        "-o",
        str(tmp),
        *srcs,
        "-lpthread",
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    import sys

    build(force="-f" in sys.argv, verbose="-v" in sys.argv)
    print(LIB_PATH)
