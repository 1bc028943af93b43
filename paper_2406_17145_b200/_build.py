"""In-tree nvcc build of ``libgpp_b200.so`` (sm_100a only).

The built library lives next to this file so it travels with the repo snapshot
to the GPU box (see ``.gitignore``: ``*.so`` stays out of history).
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
INCLUDE = PKG_DIR.parent / "include"
LIB_PATH = PKG_DIR / "libgpp_b200.so"
STAMP_PATH = PKG_DIR / ".libgpp_b200.stamp"

SOURCES = ["gemm_sm100.cu", "gemm_simt.cu", "ops.cu", "comm.cu", "mmt_ops.cu", "dlrm_ops.cu", "attn_sm100.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC",
    "-shared",
]


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _source_digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile the CUDA sources into ``libgpp_b200.so`` unless it is up to date."""
    digest = _source_digest()
    if not force and LIB_PATH.exists() and STAMP_PATH.exists() and STAMP_PATH.read_text() == digest:
        return LIB_PATH
    srcs = [str(CSRC / s) for s in SOURCES if (CSRC / s).exists()]
    out_tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [_nvcc(), *NVCC_FLAGS, "-I", str(INCLUDE), *srcs, "-o", str(out_tmp)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out_tmp, LIB_PATH)
    STAMP_PATH.write_text(digest)
    return LIB_PATH


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB_PATH)
