"""Shared parity checks: GPU executor vs the CPU oracle (oracle/reference_model.py).

Tolerances are BASELINE.json north_star's: bf16 rtol 2e-2, fp32 rtol 1e-4.  A
gradient tensor passes when BOTH its Frobenius-relative error and its max-abs
error relative to the tensor's max-abs value are below the tolerance (the
element-wise criterion: no element is off by more than tol x the tensor's
scale).  For ReLU networks the oracle takes the device's own ReLU masks
(``masks_from_taps``), so near-zero pre-activations cannot flip sides between
the two runs (the ReLU gradient is discontinuous there).
"""

from __future__ import annotations

import torch


def relerr_fro(a, b) -> float:
    a, b = a.double(), b.double()
    return ((a - b).norm() / (b.norm() + 1e-30)).item()


def relerr_max(a, b) -> float:
    a, b = a.double(), b.double()
    return ((a - b).abs().max() / (b.abs().max() + 1e-30)).item()


def assert_close(got, ref, tol: float, what) -> None:
    fro, mx = relerr_fro(got, ref), relerr_max(got, ref)
    assert fro < tol and mx < tol, (what, f"frobenius {fro:.3e}", f"max-abs {mx:.3e}", f"tol {tol}")


def masks_from_taps(taps_by_rank, sg, wl) -> dict[int, torch.Tensor]:
    """Assemble every tapped ReLU op's output sign into a full [B, width] mask in global
    sample order.  ``taps_by_rank``: list of (rank, {(op, task): output tensor}) from
    executors with ``ex.tap = {}``; rank r of stage S with DP degree d holds rows
    [j*b + q*b/d, j*b + (q+1)*b/d) of task j (cost.py:61)."""
    B = sg.mini_batch
    owner = {op: st for st in sg.stages for op in st.op_ids}
    out: dict[int, torch.Tensor] = {}
    for rank, taps in taps_by_rank:
        for (o, j), t in taps.items():
            spec = wl.layers[o]
            if spec.kind != "dense" or spec.act != "relu":
                continue
            st = owner[o]
            devs = sorted(st.devices)
            m = st.micro_batch // len(devs)
            r0 = j * st.micro_batch + devs.index(rank) * m
            full = out.setdefault(o, torch.zeros(B, t.shape[1], dtype=torch.bool))
            full[r0:r0 + m] = t.float().cpu() > 0
    return out
