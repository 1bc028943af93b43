"""Measure B200 table cost curves for the workload operators -> profiles/cost_curves_b200.json.

    python tools/profile_costs.py            (on a B200, via gpurun)

The JSON is committed so the partitioner uses the same frozen B200 curves on CPU
and GPU runs ("profile B200 curves and freeze them").
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2406_17145_b200.runtime.profiler import profile_dense, profile_mmt_layer


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    only = sys.argv[1] if len(sys.argv) > 1 else "all"
    bs = [2 ** k for k in range(4, 15)]  # 16 .. 16384 samples per task (per device)
    # every bf16 dense shape of the CANDLE / DLRM presets (workloads.dense_profile_key)
    shapes = [(4096, 4096, "relu", True), (4096, 4096, "relu", False), (28672, 1024, "relu", True),
              (16, 4096, "relu", False), (416, 4096, "relu", True), (4096, 64, "relu", True),
              (1024, 4096, "gelu", True), (4096, 1024, "none", True), (1024, 3072, "none", True),
              (1024, 1024, "none", True)]
    base = os.path.join(ROOT, "profiles", "cost_curves_b200.json")
    if only != "all" and os.path.exists(base):
        with open(base) as f:
            res = json.load(f)  # re-profile a subset, keep the other frozen curves
    else:
        res = {"device": torch.cuda.get_device_name(dev), "unit": "ms per task", "curves": {}}
    if only in ("all", "dense"):
        for din, dout, act, dg in shapes:
            bl = [b for b in bs if b * max(din, dout) <= (1 << 27)]
            key = f"dense:{din}x{dout}:{act}:{'dgrad' if dg else 'nodgrad'}"
            res["curves"][key] = profile_dense(din, dout, act, bl, dev, has_dgrad=dg)
            print(key, [round(1e3 * t, 1) for t in res["curves"][key]["fwd_ms"]], flush=True)
    if only in ("all", "mmt"):
        # MMT encoder layer (workloads.mmt): 1 .. 32 samples of 512 tokens per device and task
        for pool in (False, True):
            key = f"mmt:512x1024x16x4096:{'pool' if pool else 'seq'}"
            res["curves"][key] = profile_mmt_layer(512, 1024, 16, 4096, pool, [1, 2, 4, 8, 16, 32], dev)
            print(key, [round(t, 3) for t in res["curves"][key]["fwd_ms"]],
                  [round(t, 3) for t in res["curves"][key]["bwd_ms"]], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", "cost_curves_b200.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)
    print(path)


if __name__ == "__main__":
    main()
