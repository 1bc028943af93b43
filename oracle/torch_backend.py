"""TEST INFRASTRUCTURE ONLY.  torch-CPU restatement of the executor kernel interface.

Same method signatures and numeric contract as ``runtime.backend.CudaBackend``
(include/gpp_b200.h): fp32 math, results rounded to the destination dtype.
"""

from __future__ import annotations

import math

import torch


def _act(z, act):
    if act == "relu":
        return torch.relu(z)
    if act == "gelu":
        return torch.nn.functional.gelu(z, approximate="tanh")
    return z


def _dact(saved, act):
    s = saved.float()
    if act == "relu":
        return (s > 0).float()
    if act == "gelu":  # d/dx of x * sigmoid(2u), u = sqrt(2/pi) (x + 0.044715 x^3)
        c = math.sqrt(2.0 / math.pi)
        sg = torch.sigmoid(2.0 * c * (s + 0.044715 * s ** 3))
        return sg + s * sg * (1.0 - sg) * 2.0 * c * (1.0 + 3.0 * 0.044715 * s * s)
    return torch.ones_like(s)


class TorchBackend:
    name = "torch-cpu"

    def __init__(self, device="cpu"):
        self.device = torch.device(device)

    def prefetch_hint(self, t):
        pass

    def linear_fwd(self, y, x, w, bias, act, residual=None, pre=None):
        z = x.float() @ w.float().t()
        if bias is not None:
            z = z + bias
        if pre is not None:
            pre.copy_(z)
        out = _act(z, act)
        if residual is not None:
            out = out + residual.float()
        y.copy_(out)

    def linear_dgrad(self, dx, dy, w, saved, act):
        v = dy.float() @ w.float()
        if act != "none":
            v = v * _dact(saved, act)
        dx.copy_(v)

    def linear_wgrad(self, dw, db, dy, x, accumulate):
        v = dy.float().t() @ x.float()
        if accumulate:
            dw.add_(v)
        else:
            dw.copy_(v)
        if db is not None:
            s = dy.float().sum(0)
            if accumulate:
                db.add_(s)
            else:
                db.copy_(s)

    def linear_wgrad_sgd(self, master, shadow, grad, dy, x, lr, accumulate, store_grad, dbias=None):
        if dbias is not None:
            self.colsum(dbias, dy, accumulate)
        g = dy.float().t() @ x.float()
        if accumulate:
            g = g + grad
        if store_grad:
            grad.copy_(g)
        master.sub_(lr * g)
        if shadow is not None:
            shadow.copy_(master)

    def rowdot_loss(self, z, dz, loss_acc, x, w, bias, y, kind, scale):
        self.rowdot_fwd(z, x, w, bias)
        (self.mse_loss if kind == "mse" else self.bce_loss)(loss_acc, dz, z, y, scale)

    def colsum_multi(self, outs, xs, accumulate):
        for o, x in zip(outs, xs):
            self.colsum(o, x, accumulate)

    def colsum(self, out, x, accumulate):
        s = x.float().sum(0)
        out.add_(s) if accumulate else out.copy_(s)

    def rowdot_fwd(self, out, x, w, bias):
        v = x.float() @ w
        if bias is not None:
            v = v + bias[0]
        out.copy_(v)

    def rowdot_bwd(self, dx, dw, db, dout, x, w, saved, act, accumulate):
        if dx is not None:
            v = dout[:, None] * w[None, :]
            if act != "none":
                v = v * _dact(saved, act)
            dx.copy_(v)
        if dw is not None:
            v = dout @ x.float()
            dw.add_(v) if accumulate else dw.copy_(v)
        if db is not None:
            v = dout.sum().reshape(1)
            db.add_(v) if accumulate else db.copy_(v)

    def mse_loss(self, loss_acc, dpred, pred, y, scale):
        d = pred - y
        loss_acc.add_(scale * (d * d).sum())
        dpred.copy_(2.0 * scale * d)

    def bce_loss(self, loss_acc, dz, z, y, scale):
        l = torch.clamp(z, min=0) - z * y + torch.log1p(torch.exp(-z.abs()))
        loss_acc.add_(scale * l.sum())
        dz.copy_(scale * (torch.sigmoid(z) - y))

    def ce_loss(self, loss_acc, dlogits, logits, labels, scale):
        lf = logits.float()
        lse = torch.logsumexp(lf, dim=1)
        loss_acc.add_(scale * (lse - lf.gather(1, labels[:, None]).squeeze(1)).sum())
        p = torch.softmax(lf, dim=1)
        p[torch.arange(lf.shape[0]), labels] -= 1.0
        dlogits.copy_(scale * p)

    def copy_rows(self, dst, src):
        dst.copy_(src)

    def copy_rows_multi(self, dsts, srcs):
        for d, s in zip(dsts, srcs):
            d.copy_(s)

    def sgd_step(self, master, shadow, grad, lr):
        master.sub_(lr * grad)
        if shadow is not None:
            shadow.copy_(master)

    # DLRM ------------------------------------------------------------------
    def embbag_fwd(self, out, table, idx):
        out.copy_(table[idx].sum(1))

    def embbag_sgd_multi(self, tables, dpooled, idxs, lr):
        for t, d, i in zip(tables, dpooled, idxs):
            self.embbag_sgd(t, d, i, lr)

    def embbag_sgd(self, table, dpooled, idx, lr):
        M, bag = idx.shape
        upd = (-lr * dpooled.float())[:, None, :].expand(M, bag, table.shape[1]).reshape(-1, table.shape[1])
        table.index_add_(0, idx.reshape(-1), upd)

    @staticmethod
    def _pairs(F):
        return [(i, j) for i in range(F) for j in range(i)]

    def interaction_fwd(self, out, z, F, out_cols):
        zz = z.float().reshape(z.shape[0], F, 64)
        dots = torch.bmm(zz, zz.transpose(1, 2))
        ii = torch.tensor([p[0] for p in self._pairs(F)])
        jj = torch.tensor([p[1] for p in self._pairs(F)])
        res = torch.zeros(z.shape[0], out_cols)
        res[:, :64] = zz[:, 0]
        res[:, 64:64 + len(ii)] = dots[:, ii, jj]
        out.copy_(res)

    def interaction_bwd(self, dz, dout, z, F, mask_first):
        zz = z.float().reshape(z.shape[0], F, 64)
        P = len(self._pairs(F))
        g = torch.zeros(z.shape[0], F, F)
        for p, (i, j) in enumerate(self._pairs(F)):
            g[:, i, j] = dout[:, 64 + p].float()
            g[:, j, i] = dout[:, 64 + p].float()
        d = torch.bmm(g, zz)
        d[:, 0] += dout[:, :64].float()
        if mask_first:
            d[:, 0] *= (zz[:, 0] > 0).float()
        dz.copy_(d.reshape(z.shape[0], F * 64))

    # MMT -------------------------------------------------------------------
    def layernorm_fwd(self, y, mean, rstd, x, g, b, eps=1e-5):
        xf = x.float()
        mu = xf.mean(1)
        var = ((xf - mu[:, None]) ** 2).mean(1)
        rs = torch.rsqrt(var + eps)
        y.copy_((xf - mu[:, None]) * rs[:, None] * g + b)
        mean.copy_(mu)
        rstd.copy_(rs)

    def layernorm_bwd(self, dx, dg, db, dy, x, mean, rstd, g, dres=None, accumulate=False):
        xf, dyf = x.float(), dy.float()
        xh = (xf - mean[:, None]) * rstd[:, None]
        gy = dyf * g
        m1 = gy.mean(1, keepdim=True)
        m2 = (gy * xh).mean(1, keepdim=True)
        v = rstd[:, None] * (gy - m1 - xh * m2)
        if dres is not None:
            v = v + dres.float()
        dx.copy_(v)
        a, c = (dyf * xh).sum(0), dyf.sum(0)
        if accumulate:
            dg.add_(a)
            db.add_(c)
        else:
            dg.copy_(a)
            db.copy_(c)

    def softmax_fwd(self, p, scores):
        p.copy_(torch.softmax(scores, dim=1))

    def softmax_bwd(self, ds, p, dp, scale):
        pf = p.float()
        ds.copy_(scale * pf * (dp - (dp * pf).sum(1, keepdim=True)))

    def meanpool_fwd(self, out, x, M, S, D):
        out.copy_(x.float().reshape(M, S, D).mean(1))

    def meanpool_bwd(self, dx, dout, M, S, D):
        dx.copy_((dout.float()[:, None, :] / S).expand(M, S, D).reshape(M * S, D))

    @staticmethod
    def _heads(t, m, S, H, col0, dh):
        """[m*S, >=col0+H*dh] head-interleaved columns -> [m*H, S, dh] fp32."""
        return t[:, col0:col0 + H * dh].float().reshape(m, S, H, dh).permute(0, 2, 1, 3).reshape(m * H, S, dh)

    def flash_attn_fwd(self, qkv, lse2, o, m, S, d, H, scale):
        """Emulates gpp_flash_attn_fwd: O = softmax(scale Q K^T) V (P rounded to bf16 as the
        A operand of the P.V MMA), lse2 = base-2 log-sum-exp of the scaled scores."""
        dh = d // H
        q, k, v = (self._heads(qkv, m, S, H, c, dh) for c in (0, d, 2 * d))
        s2 = scale * (q @ k.transpose(1, 2)) * 1.4426950408889634
        l2 = torch.logsumexp(s2 * 0.6931471805599453, dim=2) * 1.4426950408889634
        lse2.copy_(l2.reshape(-1))
        pr = torch.exp2(s2 - l2[..., None]).to(o.dtype).float()
        oz = pr @ v
        o[:, :d].copy_(oz.reshape(m, H, S, dh).permute(0, 2, 1, 3).reshape(m * S, d))

    def flash_attn_bwd(self, qkv, lse2, o, dout, dvec, dqkv, m, S, d, H, scale):
        """Emulates gpp_flash_attn_bwd: P recomputed from lse2, D = rowsum(dO o O),
        dS = scale P (dO V^T - D); dQ = dS K, dK = dS^T Q, dV = P^T dO (bf16 operands).
        dvec receives scale * D (the device kernels' pre-scaled form)."""
        dh = d // H
        q, k, v = (self._heads(qkv, m, S, H, c, dh) for c in (0, d, 2 * d))
        g, oz = self._heads(dout, m, S, H, 0, dh), self._heads(o, m, S, H, 0, dh)
        D = (g * oz).sum(2, keepdim=True)
        dvec.copy_(scale * D.reshape(-1))
        s2 = scale * (q @ k.transpose(1, 2)) * 1.4426950408889634
        pz = torch.exp2(s2 - lse2.reshape(m * H, S, 1))
        dsz = scale * pz * (g @ v.transpose(1, 2) - D)
        pb, dsb = pz.to(dqkv.dtype).float(), dsz.to(dqkv.dtype).float()
        for col0, t in ((0, dsb @ k), (d, dsb.transpose(1, 2) @ q), (2 * d, pb.transpose(1, 2) @ g)):
            dqkv[:, col0:col0 + d].copy_(t.reshape(m, H, S, dh).permute(0, 2, 1, 3).reshape(m * S, d))

    def attn_fwd(self, qkv, p, o, m, S, d, H, scale):
        """Emulates gpp_attn_fwd: P = softmax(scale Q K^T) (bf16, kept), O = bf16(P) V."""
        dh = d // H
        q, k, v = (self._heads(qkv, m, S, H, c, dh) for c in (0, d, 2 * d))
        pr = torch.softmax(scale * (q @ k.transpose(1, 2)), dim=2).to(p.dtype)
        p.copy_(pr.reshape(m * H * S, S))
        oz = pr.float() @ v
        o[:, :d].copy_(oz.reshape(m, H, S, dh).permute(0, 2, 1, 3).reshape(m * S, d))

    def attn_bwd(self, qkv, p, o, dout, ds, dqkv, m, S, d, H, scale):
        """Emulates gpp_attn_bwd: dP = dO V^T, D = rowsum(dO o O), dS = scale P (dP - D),
        dQ = bf16(dS) K into the Q block of dqkv."""
        dh = d // H
        k, v = self._heads(qkv, m, S, H, d, dh), self._heads(qkv, m, S, H, 2 * d, dh)
        g, oz = self._heads(dout, m, S, H, 0, dh), self._heads(o, m, S, H, 0, dh)
        pz = p.float().reshape(m * H, S, S)
        D = (g * oz).sum(2, keepdim=True)
        dsz = (scale * pz * (g @ v.transpose(1, 2) - D)).to(ds.dtype)
        ds.copy_(dsz.reshape(m * H * S, S))
        dq = dsz.float() @ k
        dqkv[:, :d].copy_(dq.reshape(m, H, S, dh).permute(0, 2, 1, 3).reshape(m * S, d))

    def attn_softmax(self, p, ldp, q, ldq, q_rows, k, ldk, k_rows, M, N, K, scale, spec):
        """Emulates gpp_attn_softmax: scores GEMM (fp32) then row softmax, per batch."""
        nb = spec[0]
        sc = torch.zeros(nb * M * N, dtype=torch.float32)
        self.gemm_batched(sc, N, q, ldq, q_rows, False, k, ldk, k_rows, False, M, N, K,
                          tuple(spec[:14]) + (0, _hi_stride(spec, M, N), M * N), alpha=scale,
                          out_f32=True)
        self._scatter_rows(p, ldp, spec, M, N, torch.softmax(sc.reshape(nb * M, N), dim=1))

    def attn_softmax_bwd(self, ds, ldc, p, ldp, dout, ldo, o_rows, v, ldv, v_rows, M, N, K, scale, spec):
        """Emulates gpp_attn_softmax_bwd: dP = dout v^T (fp32), ds = scale p (dP - rowsum(p dP))."""
        nb = spec[0]
        dp = torch.zeros(nb * M * N, dtype=torch.float32)
        self.gemm_batched(dp, N, dout, ldo, o_rows, False, v, ldv, v_rows, False, M, N, K,
                          tuple(spec[:14]) + (0, _hi_stride(spec, M, N), M * N), out_f32=True)
        dp = dp.reshape(nb * M, N)
        pf = self._gather_rows(p, ldp, spec, M, N)
        self._scatter_rows(ds, ldc, spec, M, N, scale * pf * (dp - (dp * pf).sum(1, keepdim=True)))

    @staticmethod
    def _row_index(ld, spec, M, N):
        nb, nlo, c0, chi, clo = spec[0], spec[1], spec[14], spec[15], spec[16]
        idx = []
        for z in range(nb):
            hi, lo = divmod(z, nlo)
            off = c0 + hi * chi + lo * clo
            idx.append(off + torch.arange(M)[:, None] * ld + torch.arange(N)[None, :])
        return torch.cat(idx).reshape(-1)

    def _scatter_rows(self, out, ld, spec, M, N, vals):
        out.reshape(-1)[self._row_index(ld, spec, M, N)] = vals.reshape(-1).to(out.dtype)

    def _gather_rows(self, t, ld, spec, M, N):
        return t.reshape(-1)[self._row_index(ld, spec, M, N)].float().reshape(-1, N)

    def gemm_batched(self, c, ldc, a, lda, a_rows, a_mn, b, ldb, b_rows, b_mn, M, N, K, spec, alpha=1.0,
                     out_f32=False):
        (nb, nlo, am0, amh, aml, ak0, akh, akl, bn0, bnh, bnl, bk0, bkh, bkl, c0, chi, clo) = spec
        A2 = a.reshape(a_rows, lda).float()
        B2 = b.reshape(b_rows, ldb).float()
        cf = c.reshape(-1)
        for z in range(nb):
            hi, lo = divmod(z, nlo)
            am, ak = am0 + hi * amh + lo * aml, ak0 + hi * akh + lo * akl
            bn, bk = bn0 + hi * bnh + lo * bnl, bk0 + hi * bkh + lo * bkl
            Am = A2[ak:ak + K, am:am + M].t() if a_mn else A2[am:am + M, ak:ak + K]
            Bm = B2[bk:bk + K, bn:bn + N].t() if b_mn else B2[bn:bn + N, bk:bk + K]
            Cz = alpha * (Am @ Bm.t())
            off = c0 + hi * chi + lo * clo
            idx = off + torch.arange(M)[:, None] * ldc + torch.arange(N)[None, :]
            cf[idx.reshape(-1)] = Cz.reshape(-1).to(cf.dtype)


def _hi_stride(spec, M, N):
    """Contiguous per-batch [M, N] scratch: batch z = hi*nlo + lo sits at z*M*N."""
    return spec[1] * M * N
