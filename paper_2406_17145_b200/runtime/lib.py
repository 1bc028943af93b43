"""ctypes binding of the C-ABI library ``libgpp_b200.so`` (include/gpp_b200.h).

PyTorch supplies device memory and streams only; every compute call below goes
through the sm_100a library.  There is no CPU or eager-PyTorch fallback: if the
library is missing or a call fails, a ``RuntimeError`` is raised.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent.parent
LIB_PATH = _PKG / "libgpp_b200.so"

F32, BF16 = 0, 1
ACT = {"none": 0, "relu": 1, "gelu": 2}

_lib = None

_vp, _i64, _i32, _f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float

_SIGS = {
    "gpp_version": ([], _i32),
    "gpp_source_digest": ([], ctypes.c_char_p),
    "gpp_last_error": ([], ctypes.c_char_p),
    "gpp_launch_count": ([], ctypes.c_uint64),
    "gpp_linear_fwd": ([_vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp], _i32),
    "gpp_linear_dgrad": ([_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp], _i32),
    "gpp_linear_wgrad": ([_vp, _i64, _vp, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp], _i32),
    "gpp_linear_wgrad_sgd": ([_vp, _i64, _vp, _i64, _vp, _i64, _f32, _i32, _i32, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _vp, _i32, _vp], _i32),
    "gpp_gemm_prefetch_hint": ([_vp, _i64], _i32),
    "gpp_gemm": ([_vp, _i64, _vp, _i64, _i32, _vp, _i64, _i32, _i64, _i64, _i64, _f32, _f32, _i32, _i32, _vp], _i32),
    "gpp_rowdot_fwd": ([_vp, _vp, _i64, _vp, _vp, _i64, _i64, _i32, _vp], _i32),
    "gpp_rowdot_bwd": ([_vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i32, _i64, _i64, _i32, _i32, _vp], _i32),
    "gpp_rowdot_loss": ([_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _i32, _f32, _i32, _vp], _i32),
    "gpp_mse_loss": ([_vp, _vp, _vp, _vp, _i64, _f32, _vp], _i32),
    "gpp_bce_loss": ([_vp, _vp, _vp, _vp, _i64, _f32, _vp], _i32),
    "gpp_ce_loss": ([_vp, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _f32, _i32, _vp], _i32),
    "gpp_colsum_multi": ([_i32, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp], _i32),
    "gpp_colsum": ([_vp, _vp, _i64, _i64, _i64, _i32, _i32, _vp], _i32),
    "gpp_sgd_step": ([_vp, _vp, _vp, _i64, _f32, _vp], _i32),
    "gpp_copy_rows": ([_vp, _i64, _vp, _i64, _i64, _i64, _i32, _vp], _i32),
    "gpp_copy_rows_multi": ([_i32, _vp, _vp, _vp, _vp, _i64, _vp, _i32, _vp], _i32),
    "gpp_cast": ([_vp, _i32, _vp, _i32, _i64, _vp], _i32),
    "gpp_nccl_available": ([], _i32),
    "gpp_nccl_unique_id": ([_vp], _i32),
    "gpp_comm_init_group": ([_i32, _vp, _vp, _vp, _vp], _i32),
    "gpp_comm_destroy": ([_vp], _i32),
    "gpp_send": ([_vp, _vp, _i64, _i32, _vp], _i32),
    "gpp_recv": ([_vp, _vp, _i64, _i32, _vp], _i32),
    "gpp_allreduce_f32": ([_vp, _vp, _i64, _vp], _i32),
    "gpp_allgather": ([_vp, _vp, _vp, _i64, _vp], _i32),
    "gpp_group_start": ([], _i32),
    "gpp_group_end": ([], _i32),
    "gpp_layernorm_fwd": ([_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _f32, _vp], _i32),
    "gpp_layernorm_bwd": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i32, _vp], _i32),
    "gpp_softmax_fwd": ([_vp, _vp, _i64, _i64, _vp], _i32),
    "gpp_softmax_bwd": ([_vp, _vp, _vp, _i64, _i64, _f32, _vp], _i32),
    "gpp_meanpool_fwd": ([_vp, _i64, _vp, _i64, _i64, _i64, _vp], _i32),
    "gpp_meanpool_bwd": ([_vp, _vp, _i64, _i64, _i64, _i64, _vp], _i32),
    "gpp_gemm_batched": ([_vp, _i64, _vp, _i64, _i64, _i32, _vp, _i64, _i64, _i32, _i64, _i64, _i64, _f32, _f32, _i32, _vp, _vp], _i32),
    "gpp_flash_attn_fwd": ([_vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _f32, _vp], _i32),
    "gpp_flash_attn_bwd": ([_vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _i64, _i64, _i64, _f32, _vp], _i32),
    "gpp_attn_fwd": ([_vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _f32, _vp], _i32),
    "gpp_attn_bwd": ([_vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _i64, _i64, _i64, _f32, _vp], _i32),
    "gpp_attn_softmax": ([_vp, _i64, _vp, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _f32, _vp, _vp], _i32),
    "gpp_attn_softmax_bwd": ([_vp, _i64, _vp, _i64, _vp, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _f32, _vp, _vp], _i32),
    "gpp_embbag_bad_indices": ([ctypes.POINTER(ctypes.c_uint64), _i32], _i32),
    "gpp_embbag_fwd": ([_vp, _i64, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp], _i32),
    "gpp_embbag_sgd_multi": ([_i32, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _f32, _vp], _i32),
    "gpp_embbag_sgd": ([_vp, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _f32, _vp], _i32),
    "gpp_interaction_fwd": ([_vp, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _vp], _i32),
    "gpp_interaction_bwd": ([_vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _vp], _i32),
}


def declared_symbols() -> list[str]:
    """Every entry point the binding expects the C-ABI library to export."""
    return sorted(_SIGS)


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes handle; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"libgpp_b200.so not found at {p}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
        )
    if path is None and os.environ.get("GPP_ALLOW_STALE_LIB") != "1":
        from .. import _build

        if _build.CSRC.exists() and not _build.binary_is_current(p):
            raise RuntimeError(
                f"{p} was not built from the current csrc/ sources (digest mismatch); rebuild with "
                "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue  # optional entry points are checked by tests against the header
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(rc: int, name: str) -> None:
    if rc != 0:
        msg = _lib.gpp_last_error().decode(errors="replace") if _lib is not None else "?"
        raise RuntimeError(f"{name} failed (status {rc}): {msg}")


def call(name: str, *args) -> None:
    lib = load()
    fn = getattr(lib, name, None)
    if fn is None:
        raise RuntimeError(f"{name} is not exported by {LIB_PATH}")
    _check(fn(*args), name)


def launch_count() -> int:
    return int(load().gpp_launch_count())


# ---------------------------------------------------------------------------
# Tensor-level helpers (device tensors; row-major 2-D with unit inner stride).
# ---------------------------------------------------------------------------


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _ld(t: torch.Tensor | None) -> int:
    if t is None:
        return 0
    if t.dim() == 1:
        return t.shape[0]
    assert t.stride(-1) == 1, "inner dimension must be contiguous"
    return t.stride(0)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def linear_fwd(y, x, w, bias=None, act="none", residual=None, pre=None, stream=None):
    M, K = x.shape
    N = w.shape[0]
    call("gpp_linear_fwd", _ptr(y), _ld(y), _ptr(x), _ld(x), _ptr(w), _ld(w), _ptr(bias),
         _ptr(residual), _ld(residual), _ptr(pre), _ld(pre), M, N, K, ACT[act], _dt(x), _stream(stream))


def linear_dgrad(dx, dy, w, saved=None, act="none", stream=None):
    M, N = dy.shape
    K = w.shape[1]
    call("gpp_linear_dgrad", _ptr(dx), _ld(dx), _ptr(dy), _ld(dy), _ptr(w), _ld(w), _ptr(saved),
         _ld(saved), M, N, K, ACT[act], _dt(dy), _stream(stream))


def linear_wgrad(dw, dbias, dy, x, accumulate=False, stream=None):
    M, N = dy.shape
    K = x.shape[1]
    call("gpp_linear_wgrad", _ptr(dw), _ld(dw), _ptr(dbias), _ptr(dy), _ld(dy), _ptr(x), _ld(x),
         M, N, K, int(bool(accumulate)), _dt(dy), _stream(stream))


def linear_wgrad_sgd(master, shadow, grad, dy, x, lr, accumulate=False, store_grad=False, dbias=None,
                     stream=None):
    """Last-micro-batch wgrad with the SGD update fused into the epilogue; ``dbias`` (optional)
    receives the bias GRADIENT (+= with ``accumulate``), summed inside the same kernel."""
    M, N = dy.shape
    K = x.shape[1]
    call("gpp_linear_wgrad_sgd", _ptr(master), _ld(master), _ptr(shadow), _ld(shadow), _ptr(grad), _ld(grad),
         float(lr), int(bool(accumulate)), int(bool(store_grad)), _ptr(dy), _ld(dy), _ptr(x), _ld(x),
         M, N, K, _ptr(dbias), _dt(dy), _stream(stream))


def gemm(c, a, b, a_mn=False, b_mn=False, alpha=1.0, beta=0.0, stream=None):
    """c[M,N] = alpha * A·Bᵀ + beta*c with A(m,k)/B(n,k) in K- or MN-major storage."""
    M = a.shape[1] if a_mn else a.shape[0]
    K = a.shape[0] if a_mn else a.shape[1]
    N = b.shape[1] if b_mn else b.shape[0]
    call("gpp_gemm", _ptr(c), _ld(c), _ptr(a), _ld(a), int(a_mn), _ptr(b), _ld(b), int(b_mn),
         M, N, K, float(alpha), float(beta), int(c.dtype == torch.float32), _dt(a), _stream(stream))


def rowdot_fwd(out, x, w, bias=None, stream=None):
    M, K = x.shape
    call("gpp_rowdot_fwd", _ptr(out), _ptr(x), _ld(x), _ptr(w), _ptr(bias), M, K, _dt(x), _stream(stream))


def rowdot_bwd(dx, dw, dbias, dout, x, w, saved=None, act="none", accumulate=False, stream=None):
    M, K = x.shape
    call("gpp_rowdot_bwd", _ptr(dx), _ld(dx), _ptr(dw), _ptr(dbias), _ptr(dout), _ptr(x), _ld(x),
         _ptr(w), _ptr(saved), _ld(saved), ACT[act], M, K, int(bool(accumulate)), _dt(x), _stream(stream))


def mse_loss(loss_acc, dpred, pred, y, scale: float, stream=None):
    call("gpp_mse_loss", _ptr(loss_acc), _ptr(dpred), _ptr(pred), _ptr(y), pred.numel(), float(scale), _stream(stream))


def bce_loss(loss_acc, dlogit, logit, y, scale: float, stream=None):
    call("gpp_bce_loss", _ptr(loss_acc), _ptr(dlogit), _ptr(logit), _ptr(y), logit.numel(), float(scale), _stream(stream))


def ce_loss(loss_acc, dlogits, logits, labels, scale: float, stream=None):
    M, C = logits.shape
    call("gpp_ce_loss", _ptr(loss_acc), _ptr(dlogits), _ld(dlogits), _ptr(logits), _ld(logits),
         _ptr(labels), M, C, float(scale), _dt(logits), _stream(stream))


def rowdot_loss(z, dz, loss_acc, x, w, bias, y, kind: str, scale: float, stream=None):
    """Fused N=1 head + loss (kind "mse" | "bce"): z = x.w + b, the loss into loss_acc, dz."""
    M, K = x.shape
    call("gpp_rowdot_loss", _ptr(z), _ptr(dz), _ptr(loss_acc), _ptr(x), _ld(x), _ptr(w), _ptr(bias), _ptr(y), M, K,
         {"mse": 0, "bce": 1}[kind], float(scale), _dt(x), _stream(stream))


def colsum_multi(outs, xs, accumulate=False, stream=None):
    """out_i (+)= column sums of x_i (2-D, one dtype) for every pair, in as few launches as possible."""
    n = len(xs)
    if n == 0:
        return
    P = ctypes.c_void_p * n
    I = ctypes.c_int64 * n
    call("gpp_colsum_multi", n, P(*[_ptr(x) for x in xs]), I(*[_ld(x) for x in xs]), I(*[x.shape[0] for x in xs]),
         I(*[x.shape[1] for x in xs]), P(*[_ptr(o) for o in outs]), int(bool(accumulate)), _dt(xs[0]),
         _stream(stream))


def colsum(out, x, accumulate=False, stream=None):
    M, N = x.shape
    call("gpp_colsum", _ptr(out), _ptr(x), _ld(x), M, N, int(bool(accumulate)), _dt(x), _stream(stream))


def sgd_step(master, shadow, grad, lr: float, stream=None):
    call("gpp_sgd_step", _ptr(master), _ptr(shadow), _ptr(grad), master.numel(), float(lr), _stream(stream))


def copy_rows(dst, src, stream=None):
    rows, cols = src.shape
    call("gpp_copy_rows", _ptr(dst), _ld(dst), _ptr(src), _ld(src), rows, cols, src.element_size(), _stream(stream))


def copy_rows_multi(dsts, srcs, stream=None):
    """All slices of one concat / split (same row count, same dtype) in one launch."""
    n = len(dsts)
    if n == 0:
        return
    rows = srcs[0].shape[0]
    if any(s.shape[0] != rows or d.shape != s.shape or d.dtype != s.dtype for d, s in zip(dsts, srcs)):
        raise ValueError("copy_rows_multi: slices must share rows and dtype and match shapes")
    P, L = ctypes.c_void_p * n, ctypes.c_int64 * n
    call("gpp_copy_rows_multi", n, P(*[_ptr(d) for d in dsts]), L(*[_ld(d) for d in dsts]),
         P(*[_ptr(s) for s in srcs]), L(*[_ld(s) for s in srcs]), rows, L(*[s.shape[1] for s in srcs]),
         srcs[0].element_size(), _stream(stream))


def embbag_fwd(out, table, idx, stream=None):
    M, bag = idx.shape
    call("gpp_embbag_fwd", _ptr(out), _ld(out), _ptr(table), _ptr(idx), _ld(idx), M, bag, table.shape[1],
         table.shape[0], _stream(stream))


def embbag_sgd_multi(tables, dpooled, idxs, lr, stream=None):
    """Deterministic sparse SGD of several tables in one call (same M x bag index shape and
    dpooled row pitch for every table)."""
    n = len(tables)
    M, bag = idxs[0].shape
    P = ctypes.c_void_p * n
    call("gpp_embbag_sgd_multi", n, P(*[_ptr(t) for t in tables]), (ctypes.c_int64 * n)(*[t.shape[0] for t in tables]),
         P(*[_ptr(d) for d in dpooled]), _ld(dpooled[0]), P(*[_ptr(i) for i in idxs]), _ld(idxs[0]), M, bag,
         tables[0].shape[1], float(lr), _stream(stream))


def embbag_sgd(table, dpooled, idx, lr, stream=None):
    M, bag = idx.shape
    call("gpp_embbag_sgd", _ptr(table), _ptr(dpooled), _ld(dpooled), _ptr(idx), _ld(idx), M, bag,
         table.shape[1], table.shape[0], float(lr), _stream(stream))


def embbag_check_indices(reset: bool = True) -> None:
    """Raise IndexError if any gather / scatter since the last check saw an index outside
    its table (those bag elements were skipped, never redirected; synchronising read)."""
    n = ctypes.c_uint64(0)
    call("gpp_embbag_bad_indices", ctypes.byref(n), 1 if reset else 0)
    if n.value:
        raise IndexError(f"embedding bag: {n.value} indices out of range of their table")


def interaction_fwd(out, z, F, out_cols, stream=None):
    M = z.shape[0]
    call("gpp_interaction_fwd", _ptr(out), _ld(out), out_cols, _ptr(z), _ld(z), M, F, 64, _stream(stream))


def interaction_bwd(dz, dout, z, F, mask_first, stream=None):
    M = z.shape[0]
    call("gpp_interaction_bwd", _ptr(dz), _ld(dz), _ptr(dout), _ld(dout), _ptr(z), _ld(z), M, F, 64,
         int(bool(mask_first)), _stream(stream))


def layernorm_fwd(y, mean, rstd, x, gamma, beta, eps=1e-5, stream=None):
    T, D = x.shape
    call("gpp_layernorm_fwd", _ptr(y), _ptr(mean), _ptr(rstd), _ptr(x), _ptr(gamma), _ptr(beta), T, D,
         float(eps), _stream(stream))


def layernorm_bwd(dx, dgamma, dbeta, dy, x, mean, rstd, gamma, dres=None, accumulate=False, stream=None):
    T, D = x.shape
    call("gpp_layernorm_bwd", _ptr(dx), _ptr(dgamma), _ptr(dbeta), _ptr(dy), _ptr(x), _ptr(mean), _ptr(rstd),
         _ptr(gamma), _ptr(dres), T, D, int(bool(accumulate)), _stream(stream))


def softmax_fwd(p, scores, stream=None):
    R, L = scores.shape
    call("gpp_softmax_fwd", _ptr(p), _ptr(scores), R, L, _stream(stream))


def softmax_bwd(ds, p, dp, scale, stream=None):
    R, L = dp.shape
    call("gpp_softmax_bwd", _ptr(ds), _ptr(p), _ptr(dp), R, L, float(scale), _stream(stream))


def meanpool_fwd(out, x, M, S, D, stream=None):
    call("gpp_meanpool_fwd", _ptr(out), _ld(out), _ptr(x), M, S, D, _stream(stream))


def meanpool_bwd(dx, dout, M, S, D, stream=None):
    call("gpp_meanpool_bwd", _ptr(dx), _ptr(dout), _ld(dout), M, S, D, _stream(stream))


def gemm_batched(c, ldc, a, lda, a_rows, a_mn, b, ldb, b_rows, b_mn, M, N, K, spec, alpha=1.0, beta=0.0,
                 out_f32=False, stream=None):
    """Batched GEMM on flat buffers; ``spec`` = 17 ints (see include/gpp_b200.h)."""
    assert len(spec) == 17
    arr = (ctypes.c_int64 * 17)(*[int(v) for v in spec])
    call("gpp_gemm_batched", _ptr(c), ldc, _ptr(a), lda, a_rows, int(a_mn), _ptr(b), ldb, b_rows, int(b_mn),
         M, N, K, float(alpha), float(beta), int(bool(out_f32)), ctypes.cast(arr, ctypes.c_void_p), _stream(stream))


def attn_softmax(p, ldp, q, ldq, q_rows, k, ldk, k_rows, M, N, K, scale, spec, stream=None):
    """p[z] = softmax(scale * q[z] k[z]^T) per batch (fused tcgen05 epilogue, keys <= 512)."""
    arr = (ctypes.c_int64 * 17)(*[int(v) for v in spec])
    call("gpp_attn_softmax", _ptr(p), ldp, _ptr(q), ldq, q_rows, _ptr(k), ldk, k_rows, M, N, K, float(scale),
         ctypes.cast(arr, ctypes.c_void_p), _stream(stream))


def attn_softmax_bwd(ds, ldc, p, ldp, dout, ldo, o_rows, v, ldv, v_rows, M, N, K, scale, spec, stream=None):
    """ds[z] = scale * p o (dout v^T - rowsum(p o dout v^T)) per batch (fused epilogue)."""
    arr = (ctypes.c_int64 * 17)(*[int(x) for x in spec])
    call("gpp_attn_softmax_bwd", _ptr(ds), ldc, _ptr(p), ldp, _ptr(dout), ldo, o_rows, _ptr(v), ldv, v_rows, M, N,
         K, float(scale), ctypes.cast(arr, ctypes.c_void_p), _stream(stream))


def attn_fwd(qkv, p, o, m, S, d, H, scale, stream=None):
    """Fused MMT attention forward: p = softmax(scale q k^T) (kept for the backward),
    o[:, h*64..] = p v (one tcgen05 kernel; packed qkv [m*S, 3d], p [m*H*S, S])."""
    call("gpp_attn_fwd", _ptr(qkv), _ptr(p), _ptr(o), _ld(o), m, S, d, H, float(scale), _stream(stream))


def attn_bwd(qkv, p, o, dout, ds, dqkv, m, S, d, H, scale, stream=None):
    """Fused MMT attention backward: ds = scale p o (dout v^T - rowsum(dout o o)) and the
    Q block of dqkv = ds k (one tcgen05 kernel)."""
    call("gpp_attn_bwd", _ptr(qkv), _ptr(p), _ptr(o), _ld(o), _ptr(dout), _ld(dout), _ptr(ds), _ptr(dqkv), m, S, d,
         H, float(scale), _stream(stream))


def flash_attn_fwd(qkv, lse2, o, m, S, d, H, scale, stream=None):
    """MMT attention forward, P never stored: o[:, h*64..] = softmax(scale q k^T) v and the
    base-2 row log-sum-exp lse2 [m*H, S] fp32 (packed qkv [m*S, 3d])."""
    call("gpp_flash_attn_fwd", _ptr(qkv), _ptr(lse2), _ptr(o), _ld(o), m, S, d, H, float(scale), _stream(stream))


def flash_attn_bwd(qkv, lse2, o, dout, dvec, dqkv, m, S, d, H, scale, stream=None):
    """MMT attention backward with P recomputed from q, k and lse2: the Q, K and V blocks
    of dqkv (dvec: [m*H, S] fp32 scratch for scale * rowsum(dout o o))."""
    call("gpp_flash_attn_bwd", _ptr(qkv), _ptr(lse2), _ptr(o), _ld(o), _ptr(dout), _ld(dout), _ptr(dvec),
         _ptr(dqkv), m, S, d, H, float(scale), _stream(stream))


def prefetch_hint(t):
    """Next GEMM launched from this thread prefetches tensor ``t`` into L2."""
    call("gpp_gemm_prefetch_hint", _ptr(t), 0 if t is None else t.numel() * t.element_size())
