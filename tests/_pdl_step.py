"""Helper for test_parity_gpu.test_pdl_is_bit_identical: two training steps of a small MMT
and a GELU tower workload on cuda:0 in THIS process (GPP_PDL is read once per process),
printing a digest of every parameter afterwards."""

import hashlib
import sys

import torch

from paper_2406_17145_b200 import model as M
from paper_2406_17145_b200 import sched as S
from paper_2406_17145_b200 import workloads as W
from paper_2406_17145_b200.runtime.backend import CudaBackend
from paper_2406_17145_b200.runtime.data import make_batch, to_device_rows
from paper_2406_17145_b200.runtime.executor import Executor


def main():
    dev = torch.device("cuda", 0)
    h = hashlib.sha256()
    for wl, b in ((W.mmt(B=4, branches=2, layers=2, S=128, d=128, H=2, ffn=256, classes=64), 2),
                  (W.multi_tower("pdl", 2, 3, 512, 256, 256, 128, act="gelu"), 64)):
        sg = S.schedule_stage_graph(M.StageGraph([M.Stage(0, wl.graph.op_ids, b, frozenset({0}))], [], wl.mini_batch))
        ex = Executor(wl, sg, 0, 1, CudaBackend(dev), lr=1e-2)
        for step in range(2):
            ex.run_iteration(to_device_rows(ex, make_batch(wl, step), ex.dtype, dev))
        torch.cuda.synchronize()
        for k in sorted(ex.P, key=str):
            h.update(ex.P[k].detach().cpu().contiguous().view(torch.uint8).numpy().tobytes())
    sys.stdout.write(h.hexdigest() + "\n")


if __name__ == "__main__":
    main()
