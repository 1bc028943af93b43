"""Kernel-level numerics of libgpp_b200.so against a plain PyTorch fp32 reference.

bf16 kernels: inputs are bf16, the reference is fp32 math on the same bf16 values,
so only accumulation order / final rounding differ.  fp32 kernels: rtol 1e-5.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(128, 256, 64), (256, 512, 128), (1000, 520, 200), (384, 128, 4096), (1024, 4096, 1024),
          (16, 4096, 4096), (1024, 1024, 28672), (96, 136, 2000),  # split-K paths
          (512, 1024, 4096), (256, 512, 3136)]  # split counts that do not divide the k-blocks


def _gelu(t):  # the model's GELU: tanh form (csrc/common.cuh act_fwd)
    return torch.nn.functional.gelu(t, approximate="tanh")


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / (b.float().abs().max() + 1e-6)).item()


def _op(x_rows_k, mn):
    """Return storage for an operand with logical (rows, k): MN-major stores its transpose."""
    return x_rows_k.t().contiguous() if mn else x_rows_k.contiguous()


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_bf16_layouts(cuda_lib, a_mn, b_mn, shape):
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K + a_mn * 2 + b_mn)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.float32)
    cuda_lib.gemm(C, _op(A, a_mn), _op(B, b_mn), a_mn=a_mn, b_mn=b_mn)
    ref = A.float() @ B.float().t()
    torch.cuda.synchronize()
    assert _rel(C, ref) < 1e-4


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
def test_gemm_f32_layouts(cuda_lib, a_mn, b_mn):
    M, N, K = 200, 136, 72
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g)
    C = torch.full((M, N), 2.0, device="cuda")
    cuda_lib.gemm(C, _op(A, a_mn), _op(B, b_mn), a_mn=a_mn, b_mn=b_mn, alpha=0.5, beta=1.0)
    ref = 0.5 * (A.double() @ B.double().t()) + 2.0
    torch.cuda.synchronize()
    assert _rel(C, ref) < 1e-5


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("act", ["none", "relu", "gelu"])
def test_linear_fwd_bwd(cuda_lib, dtype, act):
    M, N, K = 512, 768, 384
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(M, K, device="cuda", generator=g).to(dtype)
    w = (torch.randn(N, K, device="cuda", generator=g) / K**0.5).to(dtype)
    b = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g).to(dtype)
    y = torch.empty(M, N, device="cuda", dtype=dtype)
    pre = torch.empty(M, N, device="cuda", dtype=dtype)
    cuda_lib.linear_fwd(y, x, w, bias=b, act=act, residual=res, pre=pre)
    z = x.float() @ w.float().t() + b
    fa = {"none": lambda t: t, "relu": torch.relu, "gelu": _gelu}[act]
    ref = fa(z) + res.float()
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-5
    torch.cuda.synchronize()
    assert _rel(y, ref) < tol
    assert _rel(pre, z) < tol

    # dgrad with the act' of the predecessor: saved = output (relu) or pre-activation (gelu)
    dy = torch.randn(M, N, device="cuda", generator=g).to(dtype)
    saved = torch.randn(M, K, device="cuda", generator=g).to(dtype)
    dx = torch.empty(M, K, device="cuda", dtype=dtype)
    cuda_lib.linear_dgrad(dx, dy, w, saved=saved, act=act)
    dxr = dy.float() @ w.float()
    s = saved.float()
    if act == "relu":
        dxr = dxr * (s > 0)
    elif act == "gelu":
        s = s.clone().requires_grad_(True)
        _gelu(s).backward(torch.ones_like(s))
        dxr = dxr * s.grad
    torch.cuda.synchronize()
    assert _rel(dx, dxr) < tol

    dw = torch.full((N, K), 1.0, device="cuda")
    db = torch.full((N,), 1.0, device="cuda")
    cuda_lib.linear_wgrad(dw, db, dy, x, accumulate=True)
    torch.cuda.synchronize()
    assert _rel(dw, dy.float().t() @ x.float() + 1.0) < (1e-4 if dtype == torch.bfloat16 else 1e-5)
    assert _rel(db, dy.float().sum(0) + 1.0) < 1e-4


def test_big_tile_shapes(cuda_lib):
    # CANDLE tower layer at b=1024: fw / dgrad / wgrad
    M, N, K = 1024, 4096, 4096
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = (torch.randn(N, K, device="cuda", generator=g) / 64).bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cuda_lib.linear_fwd(y, x, w, act="relu")
    torch.cuda.synchronize()
    assert _rel(y, torch.relu(x.float() @ w.float().t())) < 1e-2
    dw = torch.empty(N, K, device="cuda")
    cuda_lib.linear_wgrad(dw, None, y, x)
    torch.cuda.synchronize()
    assert _rel(dw, y.float().t() @ x.float()) < 1e-4


def test_heads_and_losses(cuda_lib):
    M, K = 1000, 300
    g = torch.Generator(device="cuda").manual_seed(9)
    for dtype in (torch.float32, torch.bfloat16):
        x = torch.randn(M, K, device="cuda", generator=g).to(dtype)
        w = torch.randn(K, device="cuda", generator=g)
        out = torch.empty(M, device="cuda")
        cuda_lib.rowdot_fwd(out, x, w, torch.full((1,), 0.25, device="cuda"))
        torch.cuda.synchronize()
        assert _rel(out, x.float() @ w + 0.25) < 1e-4
        y = torch.randn(M, device="cuda", generator=g)
        loss = torch.zeros(1, device="cuda")
        dpred = torch.empty(M, device="cuda")
        cuda_lib.mse_loss(loss, dpred, out, y, 1.0 / M)
        torch.cuda.synchronize()
        ref = ((out - y) ** 2).mean()
        assert abs(loss.item() - ref.item()) / ref.item() < 1e-5
        assert _rel(dpred, 2 * (out - y) / M) < 1e-5
        dx = torch.empty(M, K, device="cuda", dtype=dtype)
        dw = torch.empty(K, device="cuda")
        db = torch.empty(1, device="cuda")
        cuda_lib.rowdot_bwd(dx, dw, db, dpred, x, w, saved=x, act="relu")
        torch.cuda.synchronize()
        assert _rel(dx, dpred[:, None] * w[None, :] * (x.float() > 0)) < 1e-2
        assert _rel(dw, dpred @ x.float()) < 1e-4
        assert abs(db.item() - dpred.sum().item()) < 1e-5
    # CE
    C = 1000
    logits = torch.randn(64, C, device="cuda", generator=g)
    labels = torch.randint(0, C, (64,), device="cuda", generator=g)
    dl = torch.empty_like(logits)
    loss = torch.zeros(1, device="cuda")
    cuda_lib.ce_loss(loss, dl, logits, labels, 1.0 / 64)
    lt = logits.clone().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(lt, labels)
    ref.backward()
    torch.cuda.synchronize()
    assert abs(loss.item() - ref.item()) < 1e-4
    assert _rel(dl, lt.grad) < 1e-4
    # BCE
    z = torch.randn(500, device="cuda", generator=g)
    yb = (torch.rand(500, device="cuda", generator=g) > 0.5).float()
    dz = torch.empty_like(z)
    loss.zero_()
    cuda_lib.bce_loss(loss, dz, z, yb, 1.0 / 500)
    zt = z.clone().requires_grad_(True)
    ref = torch.nn.functional.binary_cross_entropy_with_logits(zt, yb)
    ref.backward()
    torch.cuda.synchronize()
    assert abs(loss.item() - ref.item()) < 1e-5
    assert _rel(dz, zt.grad) < 1e-5


def test_sgd_and_colsum(cuda_lib):
    g = torch.Generator(device="cuda").manual_seed(1)
    n = 1000003
    m = torch.randn(n, device="cuda", generator=g)
    gr = torch.randn(n, device="cuda", generator=g)
    sh = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    ref = m - 0.1 * gr
    cuda_lib.sgd_step(m, sh, gr, 0.1)
    torch.cuda.synchronize()
    assert torch.allclose(m, ref, rtol=1e-6, atol=1e-7)  # FMA vs two roundings
    assert torch.equal(sh, m.bfloat16())
    x = torch.randn(777, 333, device="cuda", generator=g)
    out = torch.empty(333, device="cuda")
    cuda_lib.colsum(out, x)
    torch.cuda.synchronize()
    assert _rel(out, x.sum(0)) < 1e-5


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("M,N,ld", [(1024, 4096, 4096), (1, 8, 8), (3000, 1000, 1000),
                                    (513, 264, 272), (64, 65536, 65536), (100, 333, 333)])
def test_colsum_paths(cuda_lib, dtype, M, N, ld):
    """Vectorised single-launch path (aligned) and the generic two-pass path (ragged);
    repeated calls must give bit-identical results (arrival counters re-armed)."""
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    x = torch.randn(M, ld, device="cuda", generator=g).to(dtype)[:, :N]
    ref = x.float().sum(0, dtype=torch.float64).float()
    out = torch.empty(N, device="cuda")
    cuda_lib.colsum(out, x)
    first = out.clone()
    for _ in range(3):
        cuda_lib.colsum(out, x)
    assert torch.equal(out, first)
    assert _rel(out, ref) < 1e-5
    base = torch.randn(N, device="cuda", generator=g)
    acc = base.clone()
    cuda_lib.colsum(acc, x, accumulate=True)
    torch.cuda.synchronize()
    assert _rel(acc, base + ref) < 1e-5


@pytest.mark.parametrize("M", [64, 1024])
@pytest.mark.parametrize("accumulate", [False, True])
def test_wgrad_sgd_fused(cuda_lib, M, accumulate):
    N, K = 1024, 512
    g = torch.Generator(device="cuda").manual_seed(M + accumulate)
    dy = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    master = torch.randn(N, K, device="cuda", generator=g)
    shadow = torch.empty(N, K, device="cuda", dtype=torch.bfloat16)
    grad = torch.randn(N, K, device="cuda", generator=g)
    grad0, master0 = grad.clone(), master.clone()
    db = torch.randn(N, device="cuda", generator=g)
    db0 = db.clone()
    cuda_lib.linear_wgrad_sgd(master, shadow, grad, dy, x, 0.01, accumulate=accumulate, store_grad=True, dbias=db)
    torch.cuda.synchronize()
    gref = dy.float().t() @ x.float() + (grad0 if accumulate else 0)
    assert _rel(grad, gref) < 1e-4
    # bias gradient summed inside the GEMM (pair kernel at M = 1024, fallback kernel at 64)
    assert torch.allclose(db, dy.float().sum(0) + (db0 if accumulate else 0), rtol=1e-4, atol=1e-3)
    assert torch.allclose(master, master0 - 0.01 * gref, rtol=1e-5, atol=1e-5)
    assert torch.equal(shadow, master.bfloat16())


@pytest.mark.parametrize("N,K,M", [(4096, 4096, 1024), (1000, 520, 300), (264, 4104, 64), (1024, 28672, 1024)])
def test_wgrad_sgd_fast_path(cuda_lib, N, K, M):
    """Production fused update (no grad store, beta = 0): cp.async-staged master chunks."""
    g = torch.Generator(device="cuda").manual_seed(N + K)
    dy = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    master = torch.randn(N, K, device="cuda", generator=g)
    shadow = torch.empty(N, K, device="cuda", dtype=torch.bfloat16)
    grad = torch.zeros(N, K, device="cuda")  # not touched (store_grad off)
    master0 = master.clone()
    db = torch.full((N,), float("nan"), device="cuda")
    cuda_lib.linear_wgrad_sgd(master, shadow, grad, dy, x, 0.01, dbias=db)
    torch.cuda.synchronize()
    gref = dy.float().t() @ x.float()
    assert torch.allclose(master, master0 - 0.01 * gref, rtol=1e-5, atol=2e-5)
    assert torch.equal(shadow, master.bfloat16())
    assert torch.allclose(db, dy.float().sum(0), rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("M,N,K", [(8192, 1024, 1024), (8192, 3072, 1024), (1024, 4096, 4096), (300, 520, 264)])
@pytest.mark.parametrize("accumulate", [False, True])
def test_wgrad_fused_bias_colsum(cuda_lib, M, N, K, accumulate):
    """linear_wgrad's dbias: summed by the CTA-pair kernel's column-sum warp from the staged
    dy tiles (unsplit launches) or by the column-sum kernel (split-K / small shapes)."""
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    dy = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    dw = torch.randn(N, K, device="cuda", generator=g)
    db = torch.randn(N, device="cuda", generator=g)
    dw0, db0 = dw.clone(), db.clone()
    cuda_lib.linear_wgrad(dw, db, dy, x, accumulate=accumulate)
    torch.cuda.synchronize()
    assert _rel(dw, dy.float().t() @ x.float() + (dw0 if accumulate else 0)) < 1e-4
    assert torch.allclose(db, dy.float().sum(0) + (db0 if accumulate else 0), rtol=1e-4, atol=2e-3)


@pytest.mark.parametrize("F", [7, 26, 27])
def test_embbag_and_interaction_kernels(cuda_lib, F, monkeypatch):
    g = torch.Generator(device="cuda").manual_seed(21)
    rows, M, bag = 5000, 300, 100
    table = torch.randn(rows, 64, device="cuda", generator=g)
    idx = torch.randint(0, rows, (M, bag), device="cuda", generator=g)
    out = torch.empty(M, 64, device="cuda", dtype=torch.bfloat16)
    cuda_lib.embbag_fwd(out, table, idx)
    torch.cuda.synchronize()
    ref = torch.nn.functional.embedding_bag(idx, table, mode="sum")
    assert _rel(out, ref) < 1e-2
    dp = torch.randn(M, 64, device="cuda", generator=g).bfloat16()
    t2 = table.clone()
    cuda_lib.embbag_sgd(t2, dp, idx, 0.1)
    exp = table.clone().index_add_(0, idx.reshape(-1), (-0.1 * dp.float())[:, None, :].expand(M, bag, 64).reshape(-1, 64))
    torch.cuda.synchronize()
    assert torch.allclose(t2, exp, rtol=1e-5, atol=1e-5)
    z = torch.randn(M, F * 64, device="cuda", generator=g).bfloat16()
    cols = 64 + F * (F - 1) // 2 + 1
    o = torch.empty(M, cols, device="cuda", dtype=torch.bfloat16)
    cuda_lib.interaction_fwd(o, z, F, cols)
    zz = z.float().reshape(M, F, 64)
    d = torch.bmm(zz, zz.transpose(1, 2))
    ii = torch.tensor([i for i in range(F) for j in range(i)], device="cuda")
    jj = torch.tensor([j for i in range(F) for j in range(i)], device="cuda")
    ref = torch.cat([zz[:, 0], d[:, ii, jj], torch.zeros(M, cols - 64 - len(ii), device="cuda")], 1)
    torch.cuda.synchronize()
    assert _rel(o, ref) < 1e-2
    dout = torch.randn(M, cols, device="cuda", generator=g).bfloat16()
    dz = torch.empty_like(z)
    cuda_lib.interaction_bwd(dz, dout, z, F, True)
    zt = zz.clone().requires_grad_(True)
    dd = torch.bmm(zt, zt.transpose(1, 2))
    y = torch.cat([zt[:, 0], dd[:, ii, jj]], 1)
    y.backward(dout.float()[:, :64 + len(ii)])
    gref = zt.grad.clone()
    gref[:, 0] *= (zz[:, 0] > 0).float()
    torch.cuda.synchronize()
    assert _rel(dz.float().reshape(M, F, 64), gref) < 1e-2
    # the register-tiled F=27 kernel and the generic smem kernel: bit-identical
    monkeypatch.setenv("GPP_INTERACTION_GENERIC", "1")
    dz_gen = torch.empty_like(z)
    cuda_lib.interaction_bwd(dz_gen, dout, z, F, True)
    torch.cuda.synchronize()
    assert torch.equal(dz_gen, dz)


def test_embbag_bad_indices_skipped_and_reported(cuda_lib):
    """Out-of-range indices are skipped (never redirected to row 0) and reported."""
    rows = 100
    table = torch.randn(rows, 64, device="cuda")
    idx = torch.tensor([[1, 2, rows], [-1, 3, 4]], device="cuda")
    cuda_lib.embbag_check_indices()  # clear
    out = torch.empty(2, 64, device="cuda", dtype=torch.bfloat16)
    cuda_lib.embbag_fwd(out, table, idx)
    with pytest.raises(IndexError):
        cuda_lib.embbag_check_indices()
    exp = torch.stack([table[1] + table[2], table[3] + table[4]])
    assert torch.allclose(out.float(), exp, rtol=1e-2, atol=1e-2)
    t2 = table.clone()
    cuda_lib.embbag_sgd(t2, torch.ones(2, 64, device="cuda", dtype=torch.bfloat16), idx, 1.0)
    with pytest.raises(IndexError):
        cuda_lib.embbag_check_indices()
    assert torch.equal(t2[0], table[0]) and torch.equal(t2[rows - 1], table[rows - 1])
    assert torch.allclose(t2[1], table[1] - 1)
    cuda_lib.embbag_check_indices()  # reset by the previous read: no error


@pytest.mark.parametrize("D", [96, 1024])
def test_meanpool_kernels(cuda_lib, D):
    """Token mean-pool fw (into a strided concat slice) and bw against fp32 torch; D = 1024
    takes the 16-byte vector kernels, D = 96 the scalar ones."""
    M, S = 3, 128
    x = torch.randn(M * S, D, device="cuda").bfloat16()
    cat = torch.zeros(M, 3 * D, device="cuda", dtype=torch.bfloat16)
    out = cat[:, D:2 * D]
    cuda_lib.meanpool_fwd(out, x, M, S, D)
    ref = x.float().reshape(M, S, D).mean(1)
    torch.testing.assert_close(out.float(), ref, rtol=1e-2, atol=1e-2)
    assert torch.count_nonzero(cat[:, :D]) == 0 and torch.count_nonzero(cat[:, 2 * D:]) == 0
    dcat = torch.randn(M, 3 * D, device="cuda").bfloat16()
    dx = torch.empty(M * S, D, device="cuda", dtype=torch.bfloat16)
    cuda_lib.meanpool_bwd(dx, dcat[:, D:2 * D], M, S, D)
    refd = (dcat[:, D:2 * D].float() / S).repeat_interleave(S, 0)
    torch.testing.assert_close(dx.float(), refd, rtol=1e-2, atol=1e-4)


@pytest.mark.parametrize("D", [128, 512, 1024])
def test_layernorm_kernels(cuda_lib, D):
    g = torch.Generator(device="cuda").manual_seed(D)
    T = 777
    x = torch.randn(T, D, device="cuda", generator=g).bfloat16()
    gam = 1 + 0.1 * torch.randn(D, device="cuda", generator=g)
    bet = 0.1 * torch.randn(D, device="cuda", generator=g)
    y = torch.empty_like(x)
    mean = torch.empty(T, device="cuda")
    rstd = torch.empty(T, device="cuda")
    cuda_lib.layernorm_fwd(y, mean, rstd, x, gam, bet)
    xt = x.float().clone().requires_grad_(True)
    gt = gam.clone().requires_grad_(True)
    bt = bet.clone().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xt, (D,), gt, bt, eps=1e-5)
    torch.cuda.synchronize()
    assert _rel(y, ref) < 1e-2
    dy = torch.randn(T, D, device="cuda", generator=g).bfloat16()
    dres = torch.randn(T, D, device="cuda", generator=g).bfloat16()
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    dg = torch.empty(D, device="cuda")
    db = torch.empty(D, device="cuda")
    cuda_lib.layernorm_bwd(dx, dg, db, dy, x, mean, rstd, gam, dres=dres)
    torch.cuda.synchronize()
    assert _rel(dx, xt.grad + dres.float()) < 1e-2
    assert _rel(dg, gt.grad) < 1e-3
    assert _rel(db, bt.grad) < 1e-3


def test_softmax_kernels(cuda_lib):
    g = torch.Generator(device="cuda").manual_seed(4)
    R, L = 1000, 512
    s = 3 * torch.randn(R, L, device="cuda", generator=g)
    p = torch.empty(R, L, device="cuda", dtype=torch.bfloat16)
    cuda_lib.softmax_fwd(p, s)
    torch.cuda.synchronize()
    assert _rel(p, torch.softmax(s, 1)) < 1e-2
    dp = torch.randn(R, L, device="cuda", generator=g)
    ds = torch.empty_like(p)
    cuda_lib.softmax_bwd(ds, p, dp, 0.125)
    pf = p.float()
    torch.cuda.synchronize()
    assert _rel(ds, 0.125 * pf * (dp - (dp * pf).sum(1, keepdim=True))) < 1e-2


@pytest.mark.parametrize("m,S,d,H", [(3, 256, 256, 4), (4, 512, 1024, 16)])
def test_batched_attention_gemms_match_emulation(cuda_lib, m, S, d, H):
    """The seven attention GEMM specs of runtime/mmt.py, GPU vs the torch emulation
    (the second shape is the MMT layer: many tiles, two CTAs per SM)."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.torch_backend import TorchBackend
    from paper_2406_17145_b200.runtime.mmt import _spec
    g = torch.Generator(device="cuda").manual_seed(8)
    dh, T, Z = d // H, m * S, m * H
    qkv = torch.randn(T, 3 * d, device="cuda", generator=g).bfloat16()
    P = torch.softmax(torch.randn(Z * S, S, device="cuda", generator=g), 1).bfloat16()
    do = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    cases = [
        ("scores", (Z * S, S), torch.float32, S, qkv, 3 * d, T, False, qkv, 3 * d, T, False, S, S, dh,
         _spec(Z, H, a_m_hi=S, a_k_lo=dh, b_n_hi=S, b_k0=d, b_k_lo=dh, c_hi=H * S * S, c_lo=S * S)),
        ("pv", (T, d), torch.bfloat16, d, P, S, Z * S, False, qkv, 3 * d, T, True, S, dh, S,
         _spec(Z, H, a_m_hi=H * S, a_m_lo=S, b_n0=2 * d, b_n_lo=dh, b_k_hi=S, c_hi=S * d, c_lo=dh)),
        ("dv", (T, 3 * d), torch.bfloat16, 3 * d, P, S, Z * S, True, do, d, T, True, S, dh, S,
         _spec(Z, H, a_k_hi=H * S, a_k_lo=S, b_n_lo=dh, b_k_hi=S, c0=2 * d, c_hi=S * 3 * d, c_lo=dh)),
        ("dp", (Z * S, S), torch.float32, S, do, d, T, False, qkv, 3 * d, T, False, S, S, dh,
         _spec(Z, H, a_m_hi=S, a_k_lo=dh, b_n_hi=S, b_k0=2 * d, b_k_lo=dh, c_hi=H * S * S, c_lo=S * S)),
        ("dq", (T, 3 * d), torch.bfloat16, 3 * d, P, S, Z * S, False, qkv, 3 * d, T, True, S, dh, S,
         _spec(Z, H, a_m_hi=H * S, a_m_lo=S, b_n0=d, b_n_lo=dh, b_k_hi=S, c_hi=S * 3 * d, c_lo=dh)),
        ("dk", (T, 3 * d), torch.bfloat16, 3 * d, P, S, Z * S, True, qkv, 3 * d, T, True, S, dh, S,
         _spec(Z, H, a_k_hi=H * S, a_k_lo=S, b_n_lo=dh, b_k_hi=S, c0=d, c_hi=S * 3 * d, c_lo=dh)),
    ]
    tb = TorchBackend("cpu")
    for name, shape, dt, ldc, a, lda, ar, amn, b, ldb, br, bmn, M, N, K, spec in cases:
        c = torch.zeros(shape, device="cuda", dtype=dt)
        cuda_lib.gemm_batched(c, ldc, a, lda, ar, amn, b, ldb, br, bmn, M, N, K, spec, alpha=0.5,
                              out_f32=dt == torch.float32)
        ref = torch.zeros(shape, dtype=dt)
        tb.gemm_batched(ref, ldc, a.cpu(), lda, ar, amn, b.cpu(), ldb, br, bmn, M, N, K, spec, alpha=0.5,
                        out_f32=dt == torch.float32)
        torch.cuda.synchronize()
        assert _rel(c.cpu(), ref) < 1e-2, name


@pytest.mark.parametrize("M,N,K", [(1024, 4096, 4096), (1024, 2560, 4096), (768, 4096, 1024)])
@pytest.mark.parametrize("act", ["relu", "gelu"])
def test_pair_epilogues_partial_wave(cuda_lib, M, N, K, act):
    """Pair GEMMs whose tiles do not fill the 74 pairs (64 / 40 / 48 tiles): fw with bias /
    act / pre-activation / residual and dgrad with the act' mask, twice in a row, against
    fp32 torch."""
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = (torch.randn(N, K, device="cuda", generator=g) / K**0.5).bfloat16()
    b = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    fa = {"relu": torch.relu, "gelu": _gelu}[act]
    z = x.float() @ w.float().t() + b
    for _ in range(2):
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        pre = torch.empty_like(y)
        cuda_lib.linear_fwd(y, x, w, bias=b, act=act, residual=res, pre=pre)
        torch.cuda.synchronize()
        assert _rel(pre, z) < 1e-2
        assert _rel(y, fa(z) + res.float()) < 2e-2
    dy = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    saved = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    s = saved.float().clone().requires_grad_(True)
    fa(s).backward(torch.ones_like(s))
    ref = (dy.float() @ w.float()) * s.grad
    for _ in range(2):
        dx = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
        cuda_lib.linear_dgrad(dx, dy, w, saved=saved, act=act)
        torch.cuda.synchronize()
        assert _rel(dx, ref) < 2e-2


@pytest.mark.parametrize("m,S,d,H", [(3, 256, 256, 4), (2, 512, 1024, 16), (2, 96, 256, 4)])
def test_fused_attention_softmax(cuda_lib, m, S, d, H):
    """Scores GEMM with the softmax (and its backward) in the tcgen05 epilogue vs the
    unfused emulation (fp32 scores, row softmax) on the MMT packed-QKV layout."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.torch_backend import TorchBackend
    from paper_2406_17145_b200.runtime.mmt import _spec
    g = torch.Generator(device="cuda").manual_seed(S + d)
    dh, T, Z = d // H, m * S, m * H
    scale = dh ** -0.5
    qkv = torch.randn(T, 3 * d, device="cuda", generator=g).bfloat16()
    do = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    spec_f = _spec(Z, H, a_m_hi=S, a_k_lo=dh, b_n_hi=S, b_k0=d, b_k_lo=dh, c_hi=H * S * S, c_lo=S * S)
    spec_b = _spec(Z, H, a_m_hi=S, a_k_lo=dh, b_n_hi=S, b_k0=2 * d, b_k_lo=dh, c_hi=H * S * S, c_lo=S * S)
    P = torch.empty(Z * S, S, device="cuda", dtype=torch.bfloat16)
    cuda_lib.attn_softmax(P, S, qkv, 3 * d, T, qkv, 3 * d, T, S, S, dh, scale, spec_f)
    tb = TorchBackend("cpu")
    Pr = torch.zeros(Z * S, S, dtype=torch.bfloat16)
    tb.attn_softmax(Pr, S, qkv.cpu(), 3 * d, T, qkv.cpu(), 3 * d, T, S, S, dh, scale, spec_f)
    torch.cuda.synchronize()
    assert _rel(P.cpu(), Pr) < 1e-2
    assert torch.allclose(P.float().sum(1).cpu(), torch.ones(Z * S), atol=2e-2)
    dS = torch.empty_like(P)
    cuda_lib.attn_softmax_bwd(dS, S, P, S, do, d, T, qkv, 3 * d, T, S, S, dh, scale, spec_b)
    dSr = torch.zeros(Z * S, S, dtype=torch.bfloat16)
    tb.attn_softmax_bwd(dSr, S, P.cpu(), S, do.cpu(), d, T, qkv.cpu(), 3 * d, T, S, S, dh, scale, spec_b)
    torch.cuda.synchronize()
    assert _rel(dS.cpu(), dSr) < 2e-2


@pytest.mark.parametrize("m,S,d,H", [(2, 128, 128, 2), (3, 256, 256, 4), (2, 384, 256, 4), (2, 512, 1024, 16)])
def test_fused_attention_fwd_bwd(cuda_lib, m, S, d, H):
    """One-kernel attention (csrc/attn_sm100.cu) vs the torch restatement in
    oracle/torch_backend.py on the MMT packed-QKV layout: P and O forward, dS and the Q
    block of dQKV backward (bf16 operands / outputs, fp32 accumulation)."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.torch_backend import TorchBackend
    g = torch.Generator(device="cuda").manual_seed(7 * S + d)
    T, Z = m * S, m * H
    scale = 64 ** -0.5
    qkv = torch.randn(T, 3 * d, device="cuda", generator=g).bfloat16()
    do = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    P = torch.empty(Z * S, S, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    cuda_lib.attn_fwd(qkv, P, o, m, S, d, H, scale)
    tb = TorchBackend("cpu")
    Pr, orf = torch.zeros(Z * S, S, dtype=torch.bfloat16), torch.zeros(T, d, dtype=torch.bfloat16)
    tb.attn_fwd(qkv.cpu(), Pr, orf, m, S, d, H, scale)
    torch.cuda.synchronize()
    assert _rel(P.cpu(), Pr) < 1e-2
    assert _rel(o.cpu(), orf) < 1e-2
    dS = torch.empty_like(P)
    dqkv = torch.full((T, 3 * d), 7.0, device="cuda", dtype=torch.bfloat16)
    cuda_lib.attn_bwd(qkv, P, o, do, dS, dqkv, m, S, d, H, scale)
    dSr, dqr = torch.zeros(Z * S, S, dtype=torch.bfloat16), torch.zeros(T, 3 * d, dtype=torch.bfloat16)
    tb.attn_bwd(qkv.cpu(), P.cpu(), o.cpu(), do.cpu(), dSr, dqr, m, S, d, H, scale)
    torch.cuda.synchronize()
    assert _rel(dS.cpu(), dSr) < 2e-2
    assert _rel(dqkv[:, :d].cpu(), dqr[:, :d]) < 2e-2
    assert (dqkv[:, d:] == 7.0).all(), "attn_bwd wrote outside the Q block of dqkv"


def test_fused_attention_fwd_smem_p_variant(cuda_lib):
    """The smem-P forward kernel (GPP_ATTN_FWD2=0) in a fresh process, vs the oracle."""
    import os, subprocess, sys
    env = dict(os.environ, GPP_ATTN_FWD2="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", os.path.abspath(__file__),
                        "-k", "test_fused_attention_fwd_bwd"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.uint8])
@pytest.mark.parametrize("rows,cols,ld_src,ld_dst,off", [
    (1024, 4096, 4096, 28672, 8192),   # CANDLE concat: tower output -> column slice (16 B vectors)
    (1024, 4096, 28672, 4096, 0),      # and the backward split
    (8192, 64, 64, 1728, 64 * 5),      # DLRM interaction slices
    (37, 13, 13, 45, 3),               # odd widths / offsets: narrow vector paths
    (5, 1, 1, 7, 6),
    (0, 16, 16, 16, 0),
])
def test_copy_rows(cuda_lib, dtype, rows, cols, ld_src, ld_dst, off):
    g = torch.Generator(device="cuda").manual_seed(rows + cols + off)
    src_full = (torch.rand(max(rows, 1), ld_src, device="cuda", generator=g) * 200).to(dtype)
    dst_full = torch.zeros(max(rows, 1), ld_dst, device="cuda", dtype=dtype)
    src = src_full[:rows, (ld_src - cols) if ld_src > cols else 0:][:, :cols]
    dst = dst_full[:rows, off:off + cols] if ld_dst > cols else dst_full[:rows]
    cuda_lib.copy_rows(dst, src)
    torch.cuda.synchronize()
    assert torch.equal(dst, src)
    mask = torch.ones_like(dst_full, dtype=torch.bool)
    mask[:rows, off:off + cols] = False  # nothing outside the slice is touched
    assert torch.equal(dst_full[mask], torch.zeros_like(dst_full[mask]))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("widths,rows", [([4096] * 7, 1024), ([64] * 27, 8192), ([13, 64, 8], 37),
                                          ([64] * 40, 16)])  # > 32 slices: two launches
def test_copy_rows_multi(cuda_lib, dtype, widths, rows):
    g = torch.Generator(device="cuda").manual_seed(rows + len(widths))
    parts = [(torch.rand(rows, w, device="cuda", generator=g) * 100).to(dtype) for w in widths]
    cat = torch.empty(rows, sum(widths), device="cuda", dtype=dtype)
    offs = [sum(widths[:i]) for i in range(len(widths))]
    cuda_lib.copy_rows_multi([cat[:, o:o + w] for o, w in zip(offs, widths)], parts)  # concat
    back = [torch.empty_like(p) for p in parts]
    cuda_lib.copy_rows_multi(back, [cat[:, o:o + w] for o, w in zip(offs, widths)])  # split
    torch.cuda.synchronize()
    assert torch.equal(cat, torch.cat(parts, dim=1))
    assert all(torch.equal(a, b) for a, b in zip(back, parts))


@pytest.mark.parametrize("act", ["none", "relu", "gelu"])
def test_rowdot_bwd_vector_path(cuda_lib, act):
    """K % 8 == 0 bf16 head (the DLRM top-MLP output layer shape, scaled down): 16 B vector dx
    kernel and the one-block dbias sum (with accumulate)."""
    M, K = 4096, 1024
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = torch.randn(K + 1, device="cuda", generator=g)[1:]  # 4 B-offset weights are fine
    dpred = torch.randn(M, device="cuda", generator=g)
    dx = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
    dw = torch.zeros(K, device="cuda")
    db = torch.full((1,), 0.5, device="cuda")
    cuda_lib.rowdot_bwd(dx, dw, db, dpred, x, w, saved=x if act != "none" else None, act=act, accumulate=True)
    torch.cuda.synchronize()
    ref = dpred[:, None] * w[None, :]
    if act == "relu":
        ref = ref * (x.float() > 0)
    elif act == "gelu":
        xf = x.float().requires_grad_()
        _gelu(xf).backward(torch.ones_like(xf))
        ref = ref * xf.grad
    assert _rel(dx, ref) < 1e-2
    assert abs(db.item() - (0.5 + dpred.sum().item())) < 1e-3


def _attn_ref(qkv, dout, m, S, H, scale):
    """fp32 torch reference of MMT attention on packed qkv [m*S, 3d] (head-interleaved)."""
    d = H * 64
    x = qkv.float().clone().requires_grad_(True)
    q, k, v = (x[:, c:c + d].reshape(m, S, H, 64).transpose(1, 2) for c in (0, d, 2 * d))
    p = torch.softmax(scale * (q @ k.transpose(-1, -2)), dim=-1)
    o = (p @ v).transpose(1, 2).reshape(m * S, d)
    o.backward(dout.float())
    lse2 = torch.logsumexp(scale * (q @ k.transpose(-1, -2)), dim=-1) * 1.4426950408889634
    return o.detach(), x.grad, lse2.detach().reshape(-1)


@pytest.mark.parametrize("m,S,H", [(2, 128, 2), (1, 256, 4), (2, 384, 2), (2, 512, 16)])
def test_flash_attention_fwd_bwd(cuda_lib, m, S, H):
    """Recompute attention (csrc/attn_flash_sm100.cu) vs fp32 torch: O, the base-2 LSE and
    dQ / dK / dV; the cluster's fixed-order dQ reduction is bit-reproducible."""
    g = torch.Generator(device="cuda").manual_seed(S + H)
    d = 64 * H
    qkv = torch.randn(m * S, 3 * d, device="cuda", generator=g).bfloat16()
    dout = torch.randn(m * S, d, device="cuda", generator=g).bfloat16()
    scale = 0.125
    o = torch.empty(m * S, d, device="cuda", dtype=torch.bfloat16)
    lse2 = torch.empty(m * H * S, device="cuda")
    cuda_lib.flash_attn_fwd(qkv, lse2, o, m, S, d, H, scale)
    dqkv = torch.zeros(m * S, 3 * d, device="cuda", dtype=torch.bfloat16)
    dvec = torch.empty(m * H * S, device="cuda")
    cuda_lib.flash_attn_bwd(qkv, lse2, o, dout, dvec, dqkv, m, S, d, H, scale)
    torch.cuda.synchronize()
    o_ref, dqkv_ref, lse_ref = _attn_ref(qkv, dout, m, S, H, scale)
    assert _rel(o, o_ref) < 1e-2
    assert torch.allclose(lse2, lse_ref, atol=2e-2, rtol=1e-3)
    for c, name in ((0, "dQ"), (d, "dK"), (2 * d, "dV")):
        assert _rel(dqkv[:, c:c + d], dqkv_ref[:, c:c + d]) < 2e-2, name
    again = torch.zeros_like(dqkv)
    cuda_lib.flash_attn_bwd(qkv, lse2, o, dout, dvec, again, m, S, d, H, scale)
    torch.cuda.synchronize()
    assert torch.equal(again, dqkv)


def test_flash_attention_fwd_growing_scores(cuda_lib):
    """Keys of later 64-key blocks scaled up so every row's running max grows block after
    block: the online forward must rescale its O accumulators (csrc/attn_flash_sm100.cu,
    attn_fwd_online_kernel) and still match fp32 torch in O and the base-2 LSE."""
    m, S, H = 2, 512, 2
    g = torch.Generator(device="cuda").manual_seed(11)
    d = 64 * H
    qkv = torch.randn(m * S, 3 * d, device="cuda", generator=g)
    growth = (1 + torch.arange(S, device="cuda") // 64).float().repeat(m)  # key block kb -> x (kb + 1)
    qkv[:, d:2 * d] *= growth[:, None]
    qkv = qkv.bfloat16()
    dout = torch.randn(m * S, d, device="cuda", generator=g).bfloat16()
    scale = 0.125
    o = torch.empty(m * S, d, device="cuda", dtype=torch.bfloat16)
    lse2 = torch.empty(m * H * S, device="cuda")
    cuda_lib.flash_attn_fwd(qkv, lse2, o, m, S, d, H, scale)
    torch.cuda.synchronize()
    o_ref, _, lse_ref = _attn_ref(qkv, dout, m, S, H, scale)
    assert _rel(o, o_ref) < 1e-2
    assert torch.allclose(lse2, lse_ref, atol=2e-2, rtol=1e-3)


@pytest.mark.parametrize("kind", ["mse", "bce"])
@pytest.mark.parametrize("K,dt", [(1024, torch.bfloat16), (4096, torch.bfloat16), (300, torch.float32)])
def test_rowdot_loss_fused(cuda_lib, kind, K, dt):
    """Head GEMV + loss + dLoss in one kernel vs torch; deterministic across runs."""
    g = torch.Generator(device="cuda").manual_seed(K)
    M = 5000
    x = torch.randn(M, K, device="cuda", generator=g).to(dt)
    w = torch.randn(K, device="cuda", generator=g) / K ** 0.5
    b = torch.randn(1, device="cuda", generator=g)
    y = (torch.rand(M, device="cuda", generator=g) > 0.5).float() if kind == "bce" else torch.randn(M, device="cuda", generator=g)
    z, dz, acc = torch.empty(M, device="cuda"), torch.empty(M, device="cuda"), torch.zeros(1, device="cuda")
    scale = 1.0 / M
    cuda_lib.rowdot_loss(z, dz, acc, x, w, b, y, kind, scale)
    torch.cuda.synchronize()
    zr = (x.float() @ w + b).requires_grad_(True)
    lr = ((zr - y) ** 2).sum() * scale if kind == "mse" else \
        torch.nn.functional.binary_cross_entropy_with_logits(zr, y, reduction="sum") * scale
    lr.backward()
    assert torch.allclose(z, zr.detach(), rtol=1e-4, atol=1e-4)
    assert torch.allclose(dz, zr.grad, rtol=1e-4, atol=1e-7)
    assert abs(acc.item() - lr.item()) <= 1e-4 * abs(lr.item())
    acc2 = torch.zeros(1, device="cuda")
    cuda_lib.rowdot_loss(z, dz, acc2, x, w, b, y, kind, scale)
    torch.cuda.synchronize()
    assert torch.equal(acc, acc2)


def test_colsum_multi_matches_per_tensor(cuda_lib):
    """Several bias-gradient column sums in one launch (shapes of an MMT layer + ragged /
    unaligned ones that fall back), accumulate on and off, deterministic."""
    g = torch.Generator(device="cuda").manual_seed(5)
    shapes = [(8192, 1024), (8192, 4096), (8192, 3072), (300, 520), (777, 100), (64, 8)]
    xs = [torch.randn(m, n, device="cuda", generator=g).bfloat16() for m, n in shapes]
    for acc in (False, True):
        outs = [torch.randn(n, device="cuda", generator=g) for _, n in shapes]
        base = [o.clone() for o in outs]
        cuda_lib.colsum_multi(outs, xs, accumulate=acc)
        torch.cuda.synchronize()
        for o, b, x in zip(outs, base, xs):
            ref = x.float().sum(0) + (b if acc else 0)
            assert torch.allclose(o, ref, rtol=1e-4, atol=2e-3)
        again = [b.clone() for b in base]
        cuda_lib.colsum_multi(again, xs, accumulate=acc)
        torch.cuda.synchronize()
        assert all(torch.equal(a, o) for a, o in zip(again, outs))


@pytest.mark.parametrize("rows,M,bag,hot", [(5000, 300, 100, False), (200, 256, 20, True), (1000, 64, 3, False)])
def test_embbag_sgd_multi_deterministic(cuda_lib, rows, M, bag, hot):
    """Multi-table deterministic sparse SGD vs index_add_ (fp32): equal within fp32
    reassociation, bit-identical across runs; hot rows (> 32 hits) take the min-extraction path."""
    g = torch.Generator(device="cuda").manual_seed(rows + M)
    T = 3
    tables = [torch.randn(rows, 64, device="cuda", generator=g) for _ in range(T)]
    idxs = [torch.randint(0, 8 if hot else rows, (M, bag), device="cuda", generator=g) for _ in range(T)]
    dps = [torch.randn(M, 64, device="cuda", generator=g).bfloat16() for _ in range(T)]
    outs = []
    for _ in range(2):
        t2 = [t.clone() for t in tables]
        cuda_lib.embbag_sgd_multi(t2, dps, idxs, 0.1)
        torch.cuda.synchronize()
        outs.append(t2)
    for t, t2, idx, dp in zip(tables, outs[0], idxs, dps):
        exp = t.clone().index_add_(0, idx.reshape(-1), (-0.1 * dp.float())[:, None, :].expand(M, bag, 64).reshape(-1, 64))
        assert torch.allclose(t2, exp, rtol=1e-5, atol=1e-4)
    assert all(torch.equal(a, b) for a, b in zip(outs[0], outs[1]))
