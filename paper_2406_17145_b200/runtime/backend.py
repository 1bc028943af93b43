"""Kernel backend of the stage executor: every compute op goes to libgpp_b200.so.

The executor (``runtime.executor``) is written against this small tensor-level
interface.  ``CudaBackend`` is the only product implementation; the torch-CPU
restatement with identical signatures lives in ``oracle/torch_backend.py`` and
is used by tests only (multi-rank gloo tests of the executor's host logic).
"""

from __future__ import annotations

import torch

from . import lib


class CudaBackend:
    name = "cuda"

    def __init__(self, device: torch.device | int | str):
        if not torch.cuda.is_available():
            raise RuntimeError("CudaBackend needs a CUDA device (there is no CPU fallback)")
        self.device = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
        lib.load()

    # stream plumbing -------------------------------------------------------
    def current_stream(self):
        return torch.cuda.current_stream(self.device)

    def prefetch_hint(self, t):
        lib.prefetch_hint(t)

    # dense operator --------------------------------------------------------
    def linear_fwd(self, y, x, w, bias, act, residual=None, pre=None):
        lib.linear_fwd(y, x, w, bias=bias, act=act, residual=residual, pre=pre)

    def linear_dgrad(self, dx, dy, w, saved, act):
        lib.linear_dgrad(dx, dy, w, saved=saved, act=act)

    def linear_wgrad(self, dw, db, dy, x, accumulate):
        lib.linear_wgrad(dw, db, dy, x, accumulate=accumulate)

    def linear_wgrad_sgd(self, master, shadow, grad, dy, x, lr, accumulate, store_grad, dbias=None):
        lib.linear_wgrad_sgd(master, shadow, grad, dy, x, lr, accumulate=accumulate, store_grad=store_grad,
                             dbias=dbias)

    def rowdot_loss(self, z, dz, loss_acc, x, w, bias, y, kind, scale):
        lib.rowdot_loss(z, dz, loss_acc, x, w, bias, y, kind, scale)

    def colsum_multi(self, outs, xs, accumulate):
        lib.colsum_multi(outs, xs, accumulate=accumulate)

    def colsum(self, out, x, accumulate):
        lib.colsum(out, x, accumulate=accumulate)

    # heads / losses --------------------------------------------------------
    def rowdot_fwd(self, out, x, w, bias):
        lib.rowdot_fwd(out, x, w, bias)

    def rowdot_bwd(self, dx, dw, db, dout, x, w, saved, act, accumulate):
        lib.rowdot_bwd(dx, dw, db, dout, x, w, saved=saved, act=act, accumulate=accumulate)

    def mse_loss(self, loss_acc, dpred, pred, y, scale):
        lib.mse_loss(loss_acc, dpred, pred, y, scale)

    def bce_loss(self, loss_acc, dz, z, y, scale):
        lib.bce_loss(loss_acc, dz, z, y, scale)

    def ce_loss(self, loss_acc, dlogits, logits, labels, scale):
        lib.ce_loss(loss_acc, dlogits, logits, labels, scale)

    # data movement / optimizer --------------------------------------------
    def copy_rows(self, dst, src):
        lib.copy_rows(dst, src)

    def copy_rows_multi(self, dsts, srcs):
        lib.copy_rows_multi(dsts, srcs)

    def sgd_step(self, master, shadow, grad, lr):
        lib.sgd_step(master, shadow, grad, lr)

    # DLRM ------------------------------------------------------------------
    def embbag_fwd(self, out, table, idx):
        lib.embbag_fwd(out, table, idx)

    def embbag_sgd_multi(self, tables, dpooled, idxs, lr):
        lib.embbag_sgd_multi(tables, dpooled, idxs, lr)

    def embbag_sgd(self, table, dpooled, idx, lr):
        lib.embbag_sgd(table, dpooled, idx, lr)

    def interaction_fwd(self, out, z, F, out_cols):
        lib.interaction_fwd(out, z, F, out_cols)

    def interaction_bwd(self, dz, dout, z, F, mask_first):
        lib.interaction_bwd(dz, dout, z, F, mask_first)

    # MMT -------------------------------------------------------------------
    def layernorm_fwd(self, y, mean, rstd, x, g, b, eps=1e-5):
        lib.layernorm_fwd(y, mean, rstd, x, g, b, eps)

    def layernorm_bwd(self, dx, dg, db, dy, x, mean, rstd, g, dres=None, accumulate=False):
        lib.layernorm_bwd(dx, dg, db, dy, x, mean, rstd, g, dres=dres, accumulate=accumulate)

    def softmax_fwd(self, p, scores):
        lib.softmax_fwd(p, scores)

    def softmax_bwd(self, ds, p, dp, scale):
        lib.softmax_bwd(ds, p, dp, scale)

    def meanpool_fwd(self, out, x, M, S, D):
        lib.meanpool_fwd(out, x, M, S, D)

    def meanpool_bwd(self, dx, dout, M, S, D):
        lib.meanpool_bwd(dx, dout, M, S, D)

    def attn_softmax(self, p, ldp, q, ldq, q_rows, k, ldk, k_rows, M, N, K, scale, spec):
        lib.attn_softmax(p, ldp, q, ldq, q_rows, k, ldk, k_rows, M, N, K, scale, spec)

    def attn_softmax_bwd(self, ds, ldc, p, ldp, dout, ldo, o_rows, v, ldv, v_rows, M, N, K, scale, spec):
        lib.attn_softmax_bwd(ds, ldc, p, ldp, dout, ldo, o_rows, v, ldv, v_rows, M, N, K, scale, spec)

    def flash_attn_fwd(self, qkv, lse2, o, m, S, d, H, scale):
        lib.flash_attn_fwd(qkv, lse2, o, m, S, d, H, scale)

    def flash_attn_bwd(self, qkv, lse2, o, dout, dvec, dqkv, m, S, d, H, scale):
        lib.flash_attn_bwd(qkv, lse2, o, dout, dvec, dqkv, m, S, d, H, scale)

    def attn_fwd(self, qkv, p, o, m, S, d, H, scale):
        lib.attn_fwd(qkv, p, o, m, S, d, H, scale)

    def attn_bwd(self, qkv, p, o, dout, ds, dqkv, m, S, d, H, scale):
        lib.attn_bwd(qkv, p, o, dout, ds, dqkv, m, S, d, H, scale)

    def gemm_batched(self, c, ldc, a, lda, a_rows, a_mn, b, ldb, b_rows, b_mn, M, N, K, spec, alpha=1.0,
                     out_f32=False):
        lib.gemm_batched(c, ldc, a, lda, a_rows, a_mn, b, ldb, b_rows, b_mn, M, N, K, spec, alpha=alpha,
                         out_f32=out_f32)
