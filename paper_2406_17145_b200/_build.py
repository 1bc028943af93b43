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

SOURCES = ["gemm_sm100.cu", "gemm_simt.cu", "ops.cu", "comm.cu", "mmt_ops.cu", "dlrm_ops.cu", "attn_sm100.cu", "attn_flash_sm100.cu"]
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


def binary_is_current(path: Path = LIB_PATH, digest: str | None = None) -> bool:
    """True iff the binary at ``path`` was built from the current sources: the digest is
    compiled INTO the library (``gpp_source_digest()``), so a stale untracked .so left
    behind by a checkout can never pass for a fresh one."""
    if not path.exists():
        return False
    tag = ("gpp-digest:" + (digest or _source_digest())).encode()
    return tag in path.read_bytes()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile the CUDA sources into ``libgpp_b200.so`` unless it is up to date.

    Each translation unit is compiled to an object in parallel (``build/``), an unchanged
    unit (same source digest + flags) is reused, then one nvcc link makes the library."""
    from concurrent.futures import ThreadPoolExecutor

    digest = _source_digest()
    if not force and binary_is_current(LIB_PATH, digest):
        return LIB_PATH
    objdir = PKG_DIR.parent / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    hdr = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))):
        hdr.update(p.read_bytes())
    hdr.update(" ".join(compile_flags).encode())

    def compile_one(name: str) -> str:
        src = CSRC / name
        # ops.cu carries the library digest; the others only depend on their own text + headers
        unit = hashlib.sha256(hdr.digest() + src.read_bytes() + (digest.encode() if name == "ops.cu" else b""))
        obj = objdir / f"{src.stem}-{unit.hexdigest()[:16]}.o"
        if force or not obj.exists():
            cmd = [_nvcc(), *compile_flags, "-c", f"-DGPP_SOURCE_DIGEST=\"{digest}\"", "-I", str(INCLUDE),
                   str(src), "-o", str(obj) + ".tmp"]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
            os.replace(str(obj) + ".tmp", obj)
        return str(obj)

    names = [s for s in SOURCES if (CSRC / s).exists()]
    with ThreadPoolExecutor(max_workers=min(len(names), os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, names))
    out_tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", *objs,
           "-o", str(out_tmp)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out_tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB_PATH)
