"""TEST INFRASTRUCTURE ONLY.  An independent float64 numpy restatement of the workloads'
training loss -- the check ON the torch oracle (oracle/reference_model.py).

The reference ships no numerics, so the torch-CPU model cannot be pinned
against reference outputs.  It is pinned instead against (1) this second, separately
written implementation of the same forward pass (plain numpy, no autograd, no torch
layer functions: LayerNorm, softmax attention, tanh-GELU, embedding-bag, the dot
interaction, MSE / BCE-with-logits / CE written out) and (2) central finite differences
of this forward, which check the oracle's autograd gradients coordinate by coordinate
(tests/test_oracle_pinning.py).  The model definitions follow PAPER.md:1089-1093
(Appendix B) as restated in workloads.py.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = ["loss"]

_SQ = math.sqrt(2.0 / math.pi)


def _gelu(z):
    return 0.5 * z * (1.0 + np.tanh(_SQ * (z + 0.044715 * z ** 3)))


def _layer_norm(x, g, b, eps=1e-5):
    mu = x.mean(axis=1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def _softmax_rows(s):
    m = s.max(axis=-1, keepdims=True)
    e = np.exp(s - m)
    return e / e.sum(axis=-1, keepdims=True)


def _mmt_layer(P, o, spec, xflat):
    S, d, H, ffn, pool = spec.extra
    B = xflat.shape[0]
    x = xflat.reshape(B * S, d)
    h1 = _layer_norm(x, P[(o, "ln1_g")], P[(o, "ln1_b")])
    qkv = h1 @ P[(o, "wqkv")].T + P[(o, "bqkv")]
    dh = d // H
    att = np.empty((B * S, d))
    for bi in range(B):
        rows = slice(bi * S, (bi + 1) * S)
        for h in range(H):
            cols = slice(h * dh, (h + 1) * dh)
            q = qkv[rows, cols]
            k = qkv[rows, d + h * dh:d + (h + 1) * dh]
            v = qkv[rows, 2 * d + h * dh:2 * d + (h + 1) * dh]
            att[rows, cols] = _softmax_rows(q @ k.T / math.sqrt(dh)) @ v
    y1 = att @ P[(o, "wo")].T + P[(o, "bo")] + x
    h2 = _layer_norm(y1, P[(o, "ln2_g")], P[(o, "ln2_b")])
    f = _gelu(h2 @ P[(o, "w1")].T + P[(o, "b1")])
    y2 = f @ P[(o, "w2")].T + P[(o, "b2")] + y1
    if pool:
        return y2.reshape(B, S, d).mean(axis=1)
    return y2.reshape(B, S * d)


def loss(wl, P: dict, batch: dict) -> float:
    """Mini-batch loss of workload ``wl`` (every op in topological order) in float64.
    ``P``: {(op, name): ndarray}; ``batch``: {data key: ndarray} (full mini-batch)."""
    g = wl.graph
    B = wl.mini_batch
    out: dict[int, np.ndarray] = {}
    total = 0.0
    for o in g.topo_order:
        spec = wl.layers[o]
        preds = g.predecessors(o)
        x = batch[spec.data_key].astype(np.float64) if spec.data_key is not None else (
            out[preds[0]] if len(preds) == 1 else None)
        if spec.kind == "dense":
            z = x @ P[(o, "w")].T + P[(o, "b")]
            out[o] = np.maximum(z, 0.0) if spec.act == "relu" else (_gelu(z) if spec.act == "gelu" else z)
        elif spec.kind == "concat":
            out[o] = np.concatenate([out[u] for u in preds], axis=1)
        elif spec.kind == "embbag":
            out[o] = P[(o, "table")][batch[spec.data_key]].sum(axis=1)
        elif spec.kind == "interaction":
            zz = np.stack([out[u] for u in preds], axis=1)  # [B, F, D]
            F = zz.shape[1]
            pairs = [np.einsum("bd,bd->b", zz[:, i], zz[:, j]) for i in range(F) for j in range(i)]
            pad = spec.out_dim - zz.shape[2] - len(pairs)
            out[o] = np.concatenate([zz[:, 0], np.stack(pairs, axis=1), np.zeros((zz.shape[0], pad))], axis=1)
        elif spec.kind == "mmt_layer":
            out[o] = _mmt_layer(P, o, spec, x)
        elif spec.kind == "mse_head":
            pred = x @ P[(o, "w")] + P[(o, "b")][0]
            total += float(((pred - batch[spec.label_key]) ** 2).sum() / B)
        elif spec.kind == "bce_head":
            z = x @ P[(o, "w")] + P[(o, "b")][0]
            y = batch[spec.label_key]
            total += float((np.maximum(z, 0.0) - z * y + np.log1p(np.exp(-np.abs(z)))).sum() / B)
        elif spec.kind == "ce_head":
            logits = x @ P[(o, "w")].T + P[(o, "b")]
            m = logits.max(axis=1, keepdims=True)
            lse = (m[:, 0] + np.log(np.exp(logits - m).sum(axis=1)))
            lab = batch[spec.label_key]
            total += float((lse - logits[np.arange(logits.shape[0]), lab]).sum() / B)
        else:
            raise NotImplementedError(spec.kind)
    return total
