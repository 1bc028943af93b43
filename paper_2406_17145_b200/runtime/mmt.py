"""One pre-LN transformer encoder layer of the Multi-Modal Transformer.

    h1 = LN1(x);  qkv = h1 Wqkv^T + bqkv;  P = softmax(Q K^T / sqrt(dh));  o = P V
    y1 = o Wo^T + bo + x;  h2 = LN2(y1);  f = GELU(h2 W1^T + b1);  y2 = f W2^T + b2 + y1
    [pool: out = mean over the S tokens of y2 — the branch output fed to the concat]

Every matrix product is a libgpp_b200 tcgen05 GEMM: the four projections with fused
bias / GELU (+ pre-activation) / residual epilogues.  Attention with 64-wide heads and
S in {128, ..., 512} recomputes P (csrc/attn_flash_sm100.cu): the forward keeps only O
and the row log-sum-exp; ONE backward kernel rebuilds P from Q, K and the LSE and
produces dQ, dK and dV (dK/dV accumulated in TMEM, dQ partials summed across a CTA
cluster) -- no [S x S] matrix of any kind reaches HBM.  (GPP_ATTN_IMPL=p selects the
P-storing kernels of csrc/attn_sm100.cu plus dV / dK batched GEMMs.)  Other shapes use
the scores GEMM with the softmax in its epilogue plus batched GEMMs.
LayerNorm and mean-pool are warp-per-row kernels.  Rows of the executor's [m, S*d] buffers are viewed as [m*S, d] token matrices.
"""

from __future__ import annotations

import math
import os

import torch

WEIGHTS = ("wqkv", "wo", "w1", "w2")  # dense weights (fused-SGD region)


def mmt_params(spec, op_id: int, seed: int):
    S, d, H, ffn, pool = spec.extra
    g = torch.Generator().manual_seed(seed * 1_000_003 + op_id * 7919 + 17)
    r = lambda *s: torch.randn(*s, generator=g)
    return [
        ("ln1_g", 1.0 + 0.1 * r(d)), ("ln1_b", 0.1 * r(d)),
        ("wqkv", r(3 * d, d) / d**0.5), ("bqkv", 0.01 * r(3 * d)),
        ("wo", r(d, d) / d**0.5), ("bo", 0.01 * r(d)),
        ("ln2_g", 1.0 + 0.1 * r(d)), ("ln2_b", 0.1 * r(d)),
        ("w1", r(ffn, d) / d**0.5), ("b1", 0.01 * r(ffn)),
        ("w2", r(d, ffn) / ffn**0.5), ("b2", 0.01 * r(d)),
    ]


def _spec(nb, nlo, a_m0=0, a_m_hi=0, a_m_lo=0, a_k0=0, a_k_hi=0, a_k_lo=0,
          b_n0=0, b_n_hi=0, b_n_lo=0, b_k0=0, b_k_hi=0, b_k_lo=0, c0=0, c_hi=0, c_lo=0):
    return (nb, nlo, a_m0, a_m_hi, a_m_lo, a_k0, a_k_hi, a_k_lo, b_n0, b_n_hi, b_n_lo,
            b_k0, b_k_hi, b_k_lo, c0, c_hi, c_lo)


class MMTLayer:
    def __init__(self, ex, o: int, spec):
        self.ex, self.o, self.spec = ex, o, spec
        self.S, self.d, self.H, self.ffn, self.pool = spec.extra
        self.dh = self.d // self.H
        m, S, d, H, f = ex.m, self.S, self.d, self.H, self.ffn
        self.T = m * S
        self.Z = m * H
        T, Z = self.T, self.Z
        dt, dev = ex.dtype, ex.dev
        ring = ex._ring
        self.h1, self.h2, self.o_, self.y1 = ring((T, d)), ring((T, d)), ring((T, d)), ring((T, d))
        self.qkv = ring((T, 3 * d))
        self.pre1, self.f = ring((T, f)), ring((T, f))
        self.y2 = ring((T, d)) if self.pool else None
        st = lambda: [torch.zeros(T, dtype=torch.float32, device=dev) for _ in range(ex.ell)]
        self.mean1, self.rstd1, self.mean2, self.rstd2 = st(), st(), st(), st()
        z = lambda shape, t=dt: torch.zeros(shape, dtype=t, device=dev)
        # one-kernel attention (softmax + P.V / softmax-bwd + dS.K) for 64-wide heads and
        # S in {128..512}; else the scores kernel with the softmax in its epilogue when the
        # key row fits TMEM; else unfused GEMM + softmax kernels
        self.flash = S % 128 == 0 and S <= 512 and self.dh == 64 and dt == torch.bfloat16
        self.fused = S <= 512 and S % 32 == 0 and self.dh % 64 == 0 and dt == torch.bfloat16
        # default for 64-wide heads: recompute attention (O + base-2 LSE forward, P rebuilt in
        # the backward; csrc/attn_flash_sm100.cu) -- GPP_ATTN_IMPL=p keeps the P-storing kernels
        self.recompute = self.flash and os.environ.get("GPP_ATTN_IMPL", "flash") != "p"
        if self.recompute:
            self.lse = [torch.zeros(Z * S, dtype=torch.float32, device=dev) for _ in range(ex.ell)]
            self.dvec = torch.zeros(Z * S, dtype=torch.float32, device=dev)
            self.P = None
        else:
            self.P = ring((Z * S, S))
        self.scores = None if self.fused else z((Z * S, S), torch.float32)
        self.dP = None if self.fused else z((Z * S, S), torch.float32)
        self.dS = None if self.recompute else z((Z * S, S))
        self.dy2 = z((T, d)) if self.pool else None
        self.df, self.dh2, self.dy1, self.do = z((T, f)), z((T, d)), z((T, d)), z((T, d))
        self.dqkv, self.dh1 = z((T, 3 * d)), z((T, d))
        self.dx_scratch = z((T, d))
        self.scale = 1.0 / math.sqrt(self.dh)

    def _w(self, name):
        return self.ex.W[(self.o, name)]

    def _p(self, name):
        return self.ex.P[(self.o, name)]

    def forward(self, x2d: torch.Tensor, out: torch.Tensor, slot: int):
        be, S, d, H, dh, T, Z = self.ex.be, self.S, self.d, self.H, self.dh, self.T, self.Z
        h1, qkv, o_ = self.h1[slot], self.qkv[slot], self.o_[slot]
        P = self.P[slot] if self.P is not None else None
        be.layernorm_fwd(h1, self.mean1[slot], self.rstd1[slot], x2d, self._p("ln1_g"), self._p("ln1_b"))
        be.linear_fwd(qkv, h1, self._w("wqkv"), self._p("bqkv"), "none")
        if self.recompute:
            be.flash_attn_fwd(qkv, self.lse[slot], o_, self.ex.m, S, d, H, self.scale)
        elif self.flash:
            be.attn_fwd(qkv, P, o_, self.ex.m, S, d, H, self.scale)
        else:
            self._attention_fwd(qkv, P, o_)
        y1 = self.y1[slot]
        be.linear_fwd(y1, o_, self._w("wo"), self._p("bo"), "none", residual=x2d)
        h2 = self.h2[slot]
        be.layernorm_fwd(h2, self.mean2[slot], self.rstd2[slot], y1, self._p("ln2_g"), self._p("ln2_b"))
        be.linear_fwd(self.f[slot], h2, self._w("w1"), self._p("b1"), "gelu", pre=self.pre1[slot])
        y2 = self.y2[slot] if self.pool else out.view(T, d)
        be.linear_fwd(y2, self.f[slot], self._w("w2"), self._p("b2"), "none", residual=y1)
        if self.pool:
            be.meanpool_fwd(out, y2, self.ex.m, S, d)

    def _attention_fwd(self, qkv, P, o_):
        be, S, d, H, dh, T, Z = self.ex.be, self.S, self.d, self.H, self.dh, self.T, self.Z
        # P[z] = softmax(Q_z K_z^T * scale)  (z = sample * H + head)
        spec = _spec(Z, H, a_m_hi=S, a_k_lo=dh, b_n_hi=S, b_k0=d, b_k_lo=dh, c_hi=H * S * S, c_lo=S * S)
        if self.fused:
            be.attn_softmax(P, S, qkv, 3 * d, T, qkv, 3 * d, T, S, S, dh, self.scale, spec)
        else:
            be.gemm_batched(self.scores, S, qkv, 3 * d, T, False, qkv, 3 * d, T, False, S, S, dh, spec,
                            alpha=self.scale, out_f32=True)
            be.softmax_fwd(P, self.scores)
        # o[z] = P_z V_z  -> head-interleaved columns of o
        be.gemm_batched(o_, d, P, S, Z * S, False, qkv, 3 * d, T, True, S, dh, S,
                        _spec(Z, H, a_m_hi=H * S, a_m_lo=S, b_n0=2 * d, b_n_lo=dh, b_k_hi=S, c_hi=S * d, c_lo=dh))

    def _wgrad(self, name, bname, dz, xin, accumulate, last):
        ex, be = self.ex, self.ex.be
        o = self.o
        ex.bias_queue.append((ex.G[(o, bname)], dz))  # summed with the task's other biases, one launch
        if ex.fuse and last:
            be.linear_wgrad_sgd(ex.P[(o, name)], ex.W[(o, name)] if ex.shadow is not None else None,
                                ex.G[(o, name)], dz, xin, ex.lr, accumulate, ex.keep_grads)
        else:
            be.linear_wgrad(ex.G[(o, name)], None, dz, xin, accumulate)
            if ex.d > 1 and last:
                ex._ar_handles.append(ex.tp.allreduce_async(ex.G[(o, name)]))

    def backward(self, dz_out: torch.Tensor, x2d: torch.Tensor, dx2d, slot: int, accumulate: bool, last: bool):
        ex, be = self.ex, self.ex.be
        o, S, d, H, dh, T, Z = self.o, self.S, self.d, self.H, self.dh, self.T, self.Z
        G = ex.G
        if self.pool:
            be.meanpool_bwd(self.dy2, dz_out, ex.m, S, d)
            dy2 = self.dy2
        else:
            dy2 = dz_out.view(T, d)
        # FFN: dgrad before the (possibly fused) weight update
        be.linear_dgrad(self.df, dy2, self._w("w2"), self.pre1[slot], "gelu")
        self._wgrad("w2", "b2", dy2, self.f[slot], accumulate, last)
        be.linear_dgrad(self.dh2, self.df, self._w("w1"), None, "none")
        self._wgrad("w1", "b1", self.df, self.h2[slot], accumulate, last)
        be.layernorm_bwd(self.dy1, G[(o, "ln2_g")], G[(o, "ln2_b")], self.dh2, self.y1[slot],
                         self.mean2[slot], self.rstd2[slot], self._p("ln2_g"), dres=dy2, accumulate=accumulate)
        be.linear_dgrad(self.do, self.dy1, self._w("wo"), None, "none")
        self._wgrad("wo", "bo", self.dy1, self.o_[slot], accumulate, last)
        qkv = self.qkv[slot]
        if self.recompute:
            # dQ, dK, dV in one kernel, P recomputed from Q, K and the forward's LSE
            be.flash_attn_bwd(qkv, self.lse[slot], self.o_[slot], self.do, self.dvec, self.dqkv, ex.m, S, d, H,
                              self.scale)
        else:
            self._attention_bwd_stored_p(qkv, self.P[slot], slot)
        be.linear_dgrad(self.dh1, self.dqkv, self._w("wqkv"), None, "none")
        self._wgrad("wqkv", "bqkv", self.dqkv, self.h1[slot], accumulate, last)
        target = dx2d if dx2d is not None else self.dx_scratch
        be.layernorm_bwd(target, G[(o, "ln1_g")], G[(o, "ln1_b")], self.dh1, x2d, self.mean1[slot],
                         self.rstd1[slot], self._p("ln1_g"), dres=self.dy1, accumulate=accumulate)

    def _attention_bwd_stored_p(self, qkv, P, slot):
        ex, be = self.ex, self.ex.be
        S, d, H, dh, T, Z = self.S, self.d, self.H, self.dh, self.T, self.Z
        # dV[z] = P_z^T dO_z
        be.gemm_batched(self.dqkv, 3 * d, P, S, Z * S, True, self.do, d, T, True, S, dh, S,
                        _spec(Z, H, a_k_hi=H * S, a_k_lo=S, b_n_lo=dh, b_k_hi=S, c0=2 * d, c_hi=S * 3 * d, c_lo=dh))
        if self.flash:
            # dS = scale * P o (dO V^T - rowsum(dO o O)) and dQ = dS K in one kernel
            be.attn_bwd(qkv, P, self.o_[slot], self.do, self.dS, self.dqkv, ex.m, S, d, H, self.scale)
        else:
            # dP[z] = dO_z V_z^T ;  dS = scale * P o (dP - rowsum(P o dP))
            spec = _spec(Z, H, a_m_hi=S, a_k_lo=dh, b_n_hi=S, b_k0=2 * d, b_k_lo=dh, c_hi=H * S * S, c_lo=S * S)
            if self.fused:
                be.attn_softmax_bwd(self.dS, S, P, S, self.do, d, T, qkv, 3 * d, T, S, S, dh, self.scale, spec)
            else:
                be.gemm_batched(self.dP, S, self.do, d, T, False, qkv, 3 * d, T, False, S, S, dh, spec, out_f32=True)
                be.softmax_bwd(self.dS, P, self.dP, self.scale)
            # dQ[z] = dS_z K_z
            be.gemm_batched(self.dqkv, 3 * d, self.dS, S, Z * S, False, qkv, 3 * d, T, True, S, dh, S,
                            _spec(Z, H, a_m_hi=H * S, a_m_lo=S, b_n0=d, b_n_lo=dh, b_k_hi=S, c_hi=S * 3 * d,
                                  c_lo=dh))
        # dK[z] = dS_z^T Q_z
        be.gemm_batched(self.dqkv, 3 * d, self.dS, S, Z * S, True, qkv, 3 * d, T, True, S, dh, S,
                        _spec(Z, H, a_k_hi=H * S, a_k_lo=S, b_n_lo=dh, b_k_hi=S, c0=d, c_hi=S * 3 * d, c_lo=dh))
