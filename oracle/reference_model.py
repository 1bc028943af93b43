"""TEST INFRASTRUCTURE ONLY.  Monolithic torch-CPU model of a workload.

The numerics oracle for the pipelined executor (BASELINE.json north_star:
"per-step loss and parameter gradients must match within rtol 2e-2 in bf16
(1e-4 in fp32)").  No pipeline, no micro-batches, no stages: the whole
mini-batch through the computation graph in op order, autograd for the
gradients.  For bf16 workloads it rounds exactly where the device path stores
bf16 (weights used by GEMMs, every layer output); gradients flow straight-
through the roundings, and all math is fp32.

Also the CPU baseline of bench.py (``--impl reference`` / ``cpu_baseline``):
the training step the reference would run on host cores.
"""

from __future__ import annotations

import torch

from paper_2406_17145_b200.runtime.executor import init_params


def _round(t, bf16: bool):
    if not bf16:
        return t
    return t + (t.to(torch.bfloat16).float() - t).detach()


class ReferenceModel:
    """``native_bf16``: the CPU BASELINE variant (bench.py cpu_baseline / --impl reference):
    parameters, activations and GEMMs in bf16 directly (oneDNN / AMX on the host), no
    rounding emulation — the fastest honest CPU training step of the workload, not the
    parity oracle (which computes in fp32 and rounds where the device stores bf16)."""

    def __init__(self, wl, seed: int = 0, native_bf16: bool = False):
        self.wl = wl
        self.bf16 = wl.dtype != "fp32"
        self.native = native_bf16 and self.bf16
        self.cd = torch.bfloat16 if self.native else torch.float32
        self.params: dict[tuple[int, str], torch.Tensor] = {}
        for o in wl.graph.topo_order:
            for name, t in init_params(wl.layers[o], o, seed):
                self.params[(o, name)] = t.to(self.cd).clone().requires_grad_(True)

    def _r(self, t):
        return t if self.native else _round(t, self.bf16)

    def loss(self, batch: dict[str, torch.Tensor], relu_masks: dict | None = None) -> torch.Tensor:
        """``relu_masks`` (op -> bool [B, width], global sample order): take the ReLU
        pattern of those ops from the device run instead of recomputing it.  A ReLU's
        gradient is discontinuous at 0, so a pre-activation within bf16 rounding of zero
        may land on either side under a different (equally valid) summation order and
        move a whole gradient row; with the device's own masks the comparison measures
        the arithmetic, not those coin flips."""
        wl, g, P = self.wl, self.wl.graph, self.params
        B = wl.mini_batch
        out: dict[int, torch.Tensor] = {}
        total = None
        for o in g.topo_order:
            spec = wl.layers[o]
            if spec.data_key is not None:
                x = self._r(batch[spec.data_key].to(self.cd))
            else:
                preds = g.predecessors(o)
                x = out[preds[0]] if len(preds) == 1 else None
            if spec.kind == "dense":
                w = self._r(P[(o, "w")])
                z = x @ w.t() + P[(o, "b")]
                if spec.act == "relu" and relu_masks is not None and o in relu_masks:
                    y = z * relu_masks[o].to(z.dtype)
                else:
                    y = torch.relu(z) if spec.act == "relu" else (torch.nn.functional.gelu(z, approximate="tanh") if spec.act == "gelu" else z)
                out[o] = self._r(y)
            elif spec.kind == "concat":
                out[o] = torch.cat([out[u] for u in g.predecessors(o)], dim=1)
            elif spec.kind == "mmt_layer":
                out[o] = self._mmt_layer(o, spec, x)
            elif spec.kind == "embbag":
                pooled = torch.nn.functional.embedding_bag(batch[spec.data_key], P[(o, "table")], mode="sum")
                out[o] = self._r(pooled)
            elif spec.kind == "interaction":
                zz = torch.stack([out[u] for u in g.predecessors(o)], dim=1)  # [B, F, D]
                F = zz.shape[1]
                dots = torch.bmm(zz, zz.transpose(1, 2))
                ii = torch.tensor([i for i in range(F) for j in range(i)])
                jj = torch.tensor([j for i in range(F) for j in range(i)])
                pad = spec.out_dim - zz.shape[2] - len(ii)
                y = torch.cat([zz[:, 0], dots[:, ii, jj], torch.zeros(zz.shape[0], pad, dtype=zz.dtype)], dim=1)
                out[o] = self._r(y)
            elif spec.kind == "mse_head":
                pred = x @ P[(o, "w")] + P[(o, "b")][0]
                l = ((pred - batch[spec.label_key].to(self.cd)) ** 2).sum() / B
                total = l if total is None else total + l
            elif spec.kind == "bce_head":
                z = x @ P[(o, "w")] + P[(o, "b")][0]
                l = torch.nn.functional.binary_cross_entropy_with_logits(z, batch[spec.label_key].to(self.cd), reduction="sum") / B
                total = l if total is None else total + l
            elif spec.kind == "ce_head":
                w = self._r(P[(o, "w")])
                logits = self._r(x @ w.t() + P[(o, "b")])
                l = torch.nn.functional.cross_entropy(logits, batch[spec.label_key], reduction="sum") / B
                total = l if total is None else total + l
            else:
                raise NotImplementedError(spec.kind)
        return total

    def _mmt_layer(self, o, spec, xflat):
        """Pre-LN encoder layer with the device path's bf16 rounding points."""
        S, d, H, ffn, pool = spec.extra
        P = self.params
        R = self._r
        W = lambda n: self._r(P[(o, n)])
        B = xflat.shape[0]
        x = xflat.reshape(B * S, d)
        h1 = R(torch.nn.functional.layer_norm(x, (d,), P[(o, "ln1_g")], P[(o, "ln1_b")], eps=1e-5))
        qkv = R(h1 @ W("wqkv").t() + P[(o, "bqkv")])
        dh = d // H
        q, k, v = (qkv[:, i * d:(i + 1) * d].reshape(B, S, H, dh).transpose(1, 2) for i in range(3))
        scores = (q @ k.transpose(-1, -2)) / dh**0.5
        pr = R(torch.softmax(scores, dim=-1))
        att = R((pr @ v).transpose(1, 2).reshape(B * S, d))
        y1 = R(att @ W("wo").t() + P[(o, "bo")] + x)
        h2 = R(torch.nn.functional.layer_norm(y1, (d,), P[(o, "ln2_g")], P[(o, "ln2_b")], eps=1e-5))
        f = R(torch.nn.functional.gelu(h2 @ W("w1").t() + P[(o, "b1")], approximate="tanh"))
        y2 = R(f @ W("w2").t() + P[(o, "b2")] + y1)
        if pool:
            return R(y2.reshape(B, S, d).mean(1))
        return y2.reshape(B, S * d)

    def load_params(self, params: dict):
        """Re-synchronise to another run's master weights (per-step parity without drift)."""
        with torch.no_grad():
            for k, p in self.params.items():
                p.copy_(params[k].detach().to(self.cd).cpu().reshape(p.shape))

    def step(self, batch, lr: float, relu_masks: dict | None = None):
        """loss, grads (dict) and the SGD update applied in place."""
        for p in self.params.values():
            p.grad = None
        loss = self.loss(batch, relu_masks)
        loss.backward()
        grads = {k: p.grad.detach().clone() for k, p in self.params.items()}
        with torch.no_grad():
            for p in self.params.values():
                p.sub_(lr * p.grad)
        return loss.detach(), grads
