"""NCCL all-reduce bus bandwidth through libgpp_b200 (the DP-stage gradient sync).

    torchrun --nproc-per-node N tools/bench_allreduce.py      (on a B200 box, via gpurun)

Prints one JSON line per size: bytes, ms, busbw GB/s = 2(N-1)/N * bytes / t (the same
formula cost.dp_sync_time prices, cost.py:44-48), so the result is the B200 value of
DeviceCluster.intra_bw for the DP sync.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import torch.distributed as dist

from paper_2406_17145_b200.runtime.transport import NcclTransport


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    tp = NcclTransport(rank, set(), [tuple(range(world))], dev)
    for mb in (25, 100, 400, 1200, 2400):
        t = torch.ones(mb * (1 << 20) // 4, device=dev)
        for _ in range(3):
            tp.allreduce(t)
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        s.record()
        for _ in range(reps):
            tp.allreduce(t)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        mt = torch.tensor([ms], device=dev)
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        ms = float(mt.item())
        nbytes = t.numel() * 4
        if rank == 0:
            print(json.dumps({"n": world, "bytes": nbytes, "ms": round(ms, 4),
                              "busbw_gbs": round(2 * (world - 1) / world * nbytes / ms / 1e6, 1)}), flush=True)
        del t
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
