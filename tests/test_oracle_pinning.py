"""Pinning the numerics oracle (oracle/reference_model.py), CPU only.

The reference has no numerics to compare against, so the torch oracle the GPU
executor is checked against is itself pinned three ways:
  1. its forward loss equals an independent float64 numpy restatement (oracle/numpy_ref.py)
     on every workload kind (dense + ReLU/GELU towers, concat, MSE / BCE / CE heads,
     embedding bags, the dot interaction, the pre-LN MMT encoder layer with attention);
  2. its autograd gradients equal central finite differences of that numpy forward at
     random coordinates of every parameter tensor (float64);
  3. its bf16 rounding points round-to-nearest-even exactly like the device's
     __float2bfloat16_rn, and the ReLU-mask hook reproduces the unmasked loss when fed the
     model's own ReLU pattern.
"""

import numpy as np
import pytest
import torch

from oracle import numpy_ref
from oracle.reference_model import ReferenceModel, _round
from paper_2406_17145_b200 import workloads as W
from paper_2406_17145_b200.runtime.data import make_batch

CASES = {
    "toy": lambda: W.toy(B=8),
    "towers-gelu": lambda: W.multi_tower("g", 2, 2, 16, 12, 8, B=6, act="gelu"),
    "dlrm": lambda: W.dlrm(B=6, tables=3, rows=20, bag=4, hidden=16, dense_in=5),
    "mmt": lambda: W.mmt(B=2, branches=2, layers=1, S=8, d=16, H=2, ffn=32, classes=5),
}


def _fp64_oracle(wl):
    ref = ReferenceModel(wl)
    ref.bf16, ref.native, ref.cd = False, False, torch.float64
    with torch.no_grad():
        for k, p in ref.params.items():
            ref.params[k] = p.detach().double().requires_grad_(True)
    return ref


def _np(batch):
    return {k: (v.numpy().astype(np.float64) if v.is_floating_point() else v.numpy()) for k, v in batch.items()}


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_forward_equals_independent_numpy(name):
    wl = CASES[name]()
    ref = _fp64_oracle(wl)
    batch = make_batch(wl, 3)
    lt = ref.loss({k: v.double() if v.is_floating_point() else v for k, v in batch.items()}).item()
    ln = numpy_ref.loss(wl, {k: p.detach().numpy() for k, p in ref.params.items()}, _np(batch))
    assert ln == pytest.approx(lt, rel=1e-11, abs=1e-12)


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_gradients_equal_finite_differences(name):
    wl = CASES[name]()
    ref = _fp64_oracle(wl)
    batch = make_batch(wl, 4)
    tb = {k: v.double() if v.is_floating_point() else v for k, v in batch.items()}
    for p in ref.params.values():
        p.grad = None
    ref.loss(tb).backward()
    P = {k: p.detach().numpy().copy() for k, p in ref.params.items()}
    nb = _np(batch)
    rng = np.random.default_rng(7)
    eps = 1e-6
    checked = 0
    for k, p in ref.params.items():
        g = p.grad.numpy()
        flat = P[k].reshape(-1)
        if k[1] == "table":  # only rows the batch touches carry gradient
            rows = np.unique(nb[wl.layers[k[0]].data_key])
            coords = [int(r) * P[k].shape[1] + int(c) for r in rng.choice(rows, 3) for c in rng.integers(0, P[k].shape[1], 1)]
        else:
            coords = rng.integers(0, flat.size, size=min(4, flat.size)).tolist()
        for i in coords:
            old = flat[i]
            flat[i] = old + eps
            up = numpy_ref.loss(wl, P, nb)
            flat[i] = old - eps
            dn = numpy_ref.loss(wl, P, nb)
            flat[i] = old
            fd = (up - dn) / (2 * eps)
            assert fd == pytest.approx(g.reshape(-1)[i], rel=1e-5, abs=1e-8), (k, i)
            checked += 1
    assert checked >= 2 * len(ref.params)


def test_bf16_rounding_is_round_to_nearest_even():
    x = torch.randn(100000) * torch.exp2(torch.randint(-20, 20, (100000,)).float())
    got = _round(x, True)
    bits = x.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    rne = ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16) << 16
    exp = (rne & 0xFFFFFFFF).to(torch.int64)
    exp = torch.where(exp >= 2**31, exp - 2**32, exp).to(torch.int32).view(torch.float32)
    assert torch.equal(got, exp)
    assert torch.equal(got, x.bfloat16().float())


def test_relu_mask_hook_reproduces_the_model():
    """Feeding the oracle its OWN ReLU pattern leaves loss and gradients unchanged."""
    wl = W.multi_tower("m", 2, 3, 16, 12, 8, B=6)
    ref = ReferenceModel(wl)
    batch = make_batch(wl, 0)
    masks = {}
    with torch.no_grad():  # the model's own ReLU pattern, op by op
        g, P = wl.graph, ref.params
        out = {}
        for o in g.topo_order:
            s = wl.layers[o]
            if s.kind == "dense":
                x = _round(batch[s.data_key].float(), True) if s.data_key else out[g.predecessors(o)[0]]
                z = x @ _round(P[(o, "w")], True).t() + P[(o, "b")]
                masks[o] = z > 0
                out[o] = _round(torch.relu(z), True)
            elif s.kind == "concat":
                out[o] = torch.cat([out[u] for u in g.predecessors(o)], dim=1)
    l0, g0 = ref.step(batch, 0.0)
    l1, g1 = ref.step(batch, 0.0, masks)
    assert torch.equal(l0, l1)
    assert all(torch.equal(g0[k], g1[k]) for k in g0)
