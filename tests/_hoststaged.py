"""TEST INFRASTRUCTURE: a host-staged gloo transport for several executor ranks that
share ONE GPU (the driver's GPU test box has one B200).

Same interface as runtime/transport.py's transports.  Every piece is copied
device -> pinned host -> gloo -> host -> device, synchronously with the compute
stream, so the multi-stage executor logic (pieces, DP re-shard, tokens, DP
all-reduce) runs with the real CUDA kernels (CudaBackend) on a single device.
Only the transport is staged through the host; there is no compute on the CPU.
Never selected by the product: tests pass it as ``Executor(transport=...)``.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def _wire(t: torch.Tensor) -> torch.Tensor:
    """Bytes-equivalent view gloo can move (bf16 travels as raw bytes)."""
    return t.view(torch.uint8) if t.dtype == torch.bfloat16 else t


class _Recv:
    def __init__(self, work, host, dst):
        self.work, self.host, self.dst = work, host, dst

    def wait(self):
        if self.work is not None:
            self.work.wait()
            self.dst.copy_(self.host)
            self.work = None


class _Send:
    def __init__(self, work, host):
        self.work, self.host = work, host

    def wait(self):
        if self.work is not None:
            self.work.wait()
            self.work = None


class HostStagedTransport:
    name = "host-staged gloo (tests: ranks sharing one GPU)"

    def __init__(self, rank: int, pairs, dp_groups, device):
        self.rank = rank
        self.p2p = {}
        for (a, b) in sorted(pairs):
            self.p2p[(a, b)] = dist.new_group(ranks=sorted({a, b}), backend="gloo")
        self.dp = None
        for devs in dp_groups:
            g = dist.new_group(ranks=sorted(devs), backend="gloo")
            if rank in devs:
                self.dp = g

    def irecv_many(self, items):
        out = []
        for buf, src in items:
            host = torch.empty(buf.shape, dtype=buf.dtype)
            w = dist.irecv(_wire(host), src=src, group=self.p2p[(src, self.rank)])
            out.append(_Recv(w, host, buf))
        return out

    def isend_many(self, items):
        out = []
        for buf, dst in items:
            host = buf.detach().cpu()  # waits for the producing kernels on this stream
            w = dist.isend(_wire(host), dst=dst, group=self.p2p[(self.rank, dst)])
            out.append(_Send(w, host))
        return out

    def allreduce(self, t):
        h = t.cpu()
        dist.all_reduce(h, group=self.dp)
        t.copy_(h)

    def allreduce_async(self, t):
        self.allreduce(t)
        return None

    def allgather(self, out, t):
        src = t.detach().cpu().contiguous()
        parts = [torch.empty_like(src) for _ in range(dist.get_world_size(self.dp))]
        dist.all_gather([_wire(p) for p in parts], _wire(src), group=self.dp)
        out.copy_(torch.cat(parts, 0).reshape(out.shape))

    def join(self, handles):
        pass
