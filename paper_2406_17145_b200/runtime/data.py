"""Synthetic mini-batches (no datasets offline): seeded, identical on CPU and GPU runs.

SURVEY.md §8(d) "Common inputs": data for step s is drawn from a CPU generator
seeded with seed + 1 + s; each data key gets its own stream so a rank can draw
only the keys its stage reads.
"""

from __future__ import annotations

import torch

from ..workloads import Workload


def make_batch(wl: Workload, step: int, seed: int = 0, keys=None) -> dict[str, torch.Tensor]:
    """Full [B, ...] CPU tensors for every data key (or only ``keys``)."""
    out = {}
    for n, key in enumerate(sorted(wl.data)):
        if keys is not None and key not in keys:
            continue
        shape, kind = wl.data[key]
        g = torch.Generator().manual_seed((seed + 1 + step) * 1_000_003 + n * 7_919)
        B = wl.mini_batch
        if kind == "normal":
            t = torch.randn((B, *shape), generator=g)
        elif kind.startswith("normal_pad:"):  # n real features, zero-padded to shape (TMA: ld % 8)
            real = int(kind.split(":")[1])
            t = torch.zeros((B, *shape))
            t[..., :real] = torch.randn((B, *shape[:-1], real), generator=g)
        elif kind == "binary":
            t = (torch.rand((B, *shape), generator=g) > 0.5).float()
        elif kind.startswith("label:"):
            t = torch.randint(0, int(kind.split(":")[1]), (B, *shape), generator=g)
        elif kind.startswith("index:"):
            t = torch.randint(0, int(kind.split(":")[1]), (B, *shape), generator=g)
        else:
            raise ValueError(f"unknown data kind {kind}")
        out[key] = t
    return out


def to_device_rows(ex, full: dict[str, torch.Tensor], dtype: torch.dtype, device, pin: bool = False):
    """This rank's rows of each key, cast for the compute dtype, on ``device``."""
    out = {}
    for key in ex.data_keys():
        t = ex.local_rows(full[key])
        if t.is_floating_point():
            t = t.to(dtype) if t.dim() > 1 else t.float()
        if pin:
            t = t.pin_memory()
        out[key] = t.to(device, non_blocking=pin)
    return out
