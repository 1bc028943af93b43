"""End-to-end numerics: the GPU executor (libgpp_b200.so) vs the CPU oracle.

Per-step loss and every parameter gradient, plus the updated weights after the
SGD step, for the fp32 toy (rtol 1e-4) and the bf16 workloads (rtol 2e-2) —
BASELINE.json north_star's tolerances, on every gradient, Frobenius AND max-abs
(tests/_parity.py).  ReLU nets: the oracle takes the device's ReLU masks.
Includes the benchmarked configurations: CANDLE-Uno at B=1024 with b=256 (four
micro-batches) and DLRM with 26 x 1M-row tables, bag 100, hidden 4096.
"""

import pytest
import torch

from oracle.reference_model import ReferenceModel
from paper_2406_17145_b200 import model as M
from paper_2406_17145_b200 import sched as S
from paper_2406_17145_b200 import workloads as W
from paper_2406_17145_b200.runtime.backend import CudaBackend
from paper_2406_17145_b200.runtime.data import make_batch, to_device_rows
from paper_2406_17145_b200.runtime.executor import Executor

from _parity import assert_close, masks_from_taps, relerr_max

pytestmark = pytest.mark.gpu


def _single_stage(wl, b):
    return S.schedule_stage_graph(M.StageGraph([M.Stage(0, wl.graph.op_ids, b, frozenset({0}))], [], wl.mini_batch))


def _check(wl, b, tol, steps=2, lr=1e-2):
    fp32 = wl.dtype == "fp32"
    dev = torch.device("cuda", 0)
    sg = _single_stage(wl, b)
    ex = Executor(wl, sg, 0, 1, CudaBackend(dev), lr=lr, keep_grads=True)
    ref = ReferenceModel(wl)
    for step in range(steps):
        full = make_batch(wl, step)
        # per-step parity: the oracle evaluates loss/gradients at the executor's current
        # weights, so rounding drift of earlier steps is not compounded into later ones
        ref.load_params(ex.P)
        before = {k: v.detach().clone().cpu() for k, v in ex.P.items()}
        ex.tap = {}
        loss = ex.run_iteration(to_device_rows(ex, full, ex.dtype, dev))
        torch.cuda.synchronize()
        rl, rg = ref.step(full, lr, masks_from_taps([(0, ex.tap)], sg, wl))
        ex.tap = None
        assert abs(loss.item() - rl.item()) <= tol * abs(rl.item()), (step, loss.item(), rl.item())
        for k, g in rg.items():
            if fp32:
                assert relerr_max(ex.G[k].cpu(), g) < tol, (step, k)
            else:
                assert_close(ex.G[k].cpu(), g, tol, (step, k))
        for k in ref.params:
            # the SGD update itself: p' = p - lr * g (exact up to fp32 rounding)
            expect = before[k] - lr * ex.G[k].cpu()
            assert torch.allclose(ex.P[k].cpu(), expect, rtol=1e-6, atol=1e-7), ("sgd", step, k)
    return ex


def test_toy_fp32_matches_oracle(cuda_lib):
    _check(W.toy(B=64), 16, 1e-4)


def test_small_towers_gelu_bf16_matches_oracle(cuda_lib):
    _check(W.multi_tower("mini-gelu", 3, 3, 256, 256, 128, 128, act="gelu"), 32, 2e-2, steps=3)


def test_small_towers_relu_bf16_matches_oracle(cuda_lib):
    _check(W.multi_tower("mini", 3, 2, 256, 256, 128, 128), 32, 2e-2, steps=3)


def test_candle_full_width_bf16(cuda_lib):
    # full CANDLE-Uno layer widths (4096 / 28672 / 1024), small batch, two micro-batches
    _check(W.candle(B=64), 32, 2e-2, steps=2)


def test_candle_benchmarked_config_bf16(cuda_lib):
    """The benchmarked CANDLE-Uno config: 7 towers x 4 x 4096, B = 1024, here as four
    micro-batches of 256 (the bench's N=1 plan runs one of 1024; kFkB interleaving and
    the cross-micro-batch gradient accumulation are exercised this way)."""
    _check(W.candle(B=1024), 256, 2e-2, steps=1)


def test_candle_full_width_gelu_bf16(cuda_lib):
    _check(W.multi_tower("candle-gelu", 2, 4, 4096, 4096, 1024, 64, act="gelu"), 32, 2e-2, steps=2)


@pytest.mark.parametrize("act", ["gelu", "relu"])
def test_fused_optimizer_fast_path(cuda_lib, act):
    """Production path (keep_grads=False): the SGD update fused into the last wgrad
    epilogue.  The gradient is recovered from the update, (p_before - p_after) / lr,
    and checked against the oracle; the same run with the fusion disabled must give
    the same weights."""
    wl = W.multi_tower("fused", 2, 3, 512, 256, 256, 128, act=act)
    dev = torch.device("cuda", 0)
    lr = 1e-2
    sg = _single_stage(wl, 64)
    fast = Executor(wl, sg, 0, 1, CudaBackend(dev), lr=lr)
    slow = Executor(wl, sg, 0, 1, CudaBackend(dev), lr=lr, fuse_optimizer=False)
    assert fast.fuse and not slow.fuse
    ref = ReferenceModel(wl)
    full = make_batch(wl, 0)
    before = {k: v.detach().clone().cpu() for k, v in fast.P.items()}
    fast.tap = {}
    fast.run_iteration(to_device_rows(fast, full, fast.dtype, dev))
    slow.run_iteration(to_device_rows(slow, full, slow.dtype, dev))
    torch.cuda.synchronize()
    _, rg = ref.step(full, lr, masks_from_taps([(0, fast.tap)], sg, wl))
    for k, g in rg.items():
        rec = (before[k] - fast.P[k].cpu()) / lr
        # the recovered gradient carries the fp32 rounding of p - lr*g: scale-relative 1e-4
        assert_close(rec, g, 2e-2, k)
        assert torch.allclose(fast.P[k], slow.P[k], rtol=1e-6, atol=1e-7), k


def _dlrm_check(wl, b, steps, lr=1e-2):
    """DLRM (embedding bags + interaction + MLPs + BCE) on the GPU executor vs the oracle.
    Table gradients are recovered from the sparse SGD update on the rows the batch
    touches; every other row must be bit-unchanged."""
    dev = torch.device("cuda", 0)
    sg = _single_stage(wl, b)
    ex = Executor(wl, sg, 0, 1, CudaBackend(dev), lr=lr, keep_grads=True)
    ref = ReferenceModel(wl)
    tables = [k for k in ex.P if k[1] == "table"]
    for step in range(steps):
        full = make_batch(wl, step)
        ref.load_params(ex.P)
        before = {k: v.detach().clone() for k, v in ex.P.items()}  # on the device
        ex.tap = {}
        loss = ex.run_iteration(to_device_rows(ex, full, ex.dtype, dev))
        torch.cuda.synchronize()
        rl, rg = ref.step(full, lr, masks_from_taps([(0, ex.tap)], sg, wl))
        ex.tap = None
        assert abs(loss.item() - rl.item()) <= 2e-2 * abs(rl.item()), (step, loss.item(), rl.item())
        for k, g in rg.items():
            if k in tables:
                rows = full[wl.layers[k[0]].data_key].reshape(-1).unique().to(dev)
                got = ((before[k][rows] - ex.P[k][rows]) / lr).cpu()
                assert_close(got, g[rows.cpu()], 2e-2, (step, k))
                changed = (before[k] != ex.P[k]).any(1)
                changed[rows] = False
                assert not bool(changed.any()), ("untouched table rows changed", step, k)
            else:
                assert_close(ex.G[k].cpu(), g, 2e-2, (step, k))
    from paper_2406_17145_b200.runtime import lib
    lib.embbag_check_indices()


def test_dlrm_small_bf16_matches_oracle(cuda_lib):
    _dlrm_check(W.dlrm(B=128, tables=6, rows=2000, bag=20, hidden=512), 32, steps=2)


def test_dlrm_benchmarked_tables_bf16(cuda_lib):
    """The benchmarked DLRM model: 26 tables x 1M rows x 64, bag 100, MLP hidden 4096;
    small mini-batch (B = 256, b = 64) for the CPU oracle."""
    _dlrm_check(W.dlrm(B=256), 64, steps=1)


def test_mmt_small_bf16_matches_oracle(cuda_lib):
    """Multi-Modal Transformer (pre-LN layers, one-kernel attention, mean-pool, concat,
    CE head) on the GPU executor vs the oracle."""
    wl = W.mmt(B=8, branches=2, layers=2, S=128, d=128, H=2, ffn=256, classes=64)
    _check(wl, 4, 2e-2, steps=2)


def test_mmt_full_width_layer(cuda_lib):
    """One full-size MMT layer (S=512, d=1024, 16 heads, FFN 4096) per branch, B=2."""
    wl = W.mmt(B=2, branches=2, layers=1, S=512, d=1024, H=16, ffn=4096, classes=1000)
    _check(wl, 1, 2e-2, steps=1)


def test_dlrm_deterministic_sparse_sgd_bit_reproducible(cuda_lib, monkeypatch):
    """GPP_EMB_SGD=deterministic: the same DLRM step twice from the same state gives bit-identical
    tables (the default fp32-atomic scatter does not promise that), and matches the oracle."""
    monkeypatch.setenv("GPP_EMB_SGD", "deterministic")
    wl = W.dlrm(B=128, tables=6, rows=2000, bag=20, hidden=512)
    dev = torch.device("cuda", 0)
    outs = []
    for _ in range(2):
        ex = Executor(wl, _single_stage(wl, 32), 0, 1, CudaBackend(dev), lr=1e-2)
        assert not ex._emb_atomic
        ex.run_iteration(to_device_rows(ex, make_batch(wl, 0), ex.dtype, dev))
        torch.cuda.synchronize()
        outs.append({k: v.clone() for k, v in ex.P.items() if k[1] == "table"})
    assert outs[0].keys() and all(torch.equal(outs[0][k], outs[1][k]) for k in outs[0])
    _dlrm_check(wl, 32, steps=1)


def test_pdl_is_bit_identical(cuda_lib):
    """Programmatic dependent launch only moves kernel prologues ahead of the previous
    kernel's tail: the trained weights are bit-identical with it on (all families) and off."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    digests = []
    for mask in ("0", "-1"):
        env = dict(os.environ, GPP_PDL=mask, PYTHONPATH=os.pathsep.join([root, here]))
        r = subprocess.run([sys.executable, os.path.join(here, "_pdl_step.py")], env=env, cwd=root,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        digests.append(r.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1]
