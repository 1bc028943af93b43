"""One MMT training iteration (B = 16, one branch of two pre-LN layers: the MMT step's
per-layer shapes, T = 8192 tokens, d = 1024, FFN 4096, 16 heads, S = 512) inside a
cudaProfilerStart/Stop range, for

    ncu --profile-from-start off --set full ... python tools/ncu_mmt_layer.py

(every kernel of the iteration captured once; `--full`: the bench's 4 x 12-layer model, for a
`--metrics gpu__time_duration.sum` launch list of one step).  `--summarise REPORT.csv` turns the
`ncu -i X --page raw --csv` export of that capture into the per-kernel summary committed
under profiles/ (time, tensor / issue / XU utilisation, DRAM bytes) plus the GEMM-family
DRAM bytes per layer and per logical GEMM launch that bench.py's MMT roofline reports.
"""
import argparse
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# algorithmic bytes of one layer's 12 logical GEMMs (T = 8192, d = 1024, FFN 4096, bf16
# operands / outputs, fp32 master read + write and bf16 shadow for wgrad + SGD), in MB
_T, _D, _F = 8192, 1024, 4096
_MB = 1e-6


def _alg_layer_mb():
    a = lambda r, c: 2.0 * r * c * _MB  # bf16 matrix
    sgd = lambda r, c: 10.0 * r * c * _MB  # fp32 master r + w + bf16 shadow
    fw = [a(_T, _D) + a(3 * _D, _D) + a(_T, 3 * _D),                     # QKV + bias
          a(_T, _D) + a(_D, _D) + 2 * a(_T, _D),                         # out-proj + residual
          a(_T, _D) + a(_F, _D) + 2 * a(_T, _F),                         # FFN1 + GELU (+ pre-activation)
          a(_T, _F) + a(_D, _F) + 2 * a(_T, _D)]                         # FFN2 + residual
    dg = [a(_T, _D) + a(_D, _F) + 2 * a(_T, _F),                         # FFN2 dgrad x GELU'(pre)
          a(_T, _F) + a(_F, _D) + a(_T, _D),                             # FFN1 dgrad
          2 * a(_T, _D) + a(_D, _D),                                     # out-proj dgrad
          a(_T, 3 * _D) + a(3 * _D, _D) + a(_T, _D)]                     # QKV dgrad
    wg = [a(_T, 3 * _D) + a(_T, _D) + sgd(3 * _D, _D),
          2 * a(_T, _D) + sgd(_D, _D),
          a(_T, _F) + a(_T, _D) + sgd(_F, _D),
          a(_T, _D) + a(_T, _F) + sgd(_D, _F)]
    return sum(fw) + sum(dg) + sum(wg)


def run(branches=1, layers=2):
    import torch

    from paper_2406_17145_b200 import model as M
    from paper_2406_17145_b200 import sched as S
    from paper_2406_17145_b200 import workloads as W
    from paper_2406_17145_b200.runtime.backend import CudaBackend
    from paper_2406_17145_b200.runtime.data import make_batch, to_device_rows
    from paper_2406_17145_b200.runtime.executor import Executor

    dev = torch.device("cuda", 0)
    wl = W.mmt(B=16, branches=branches, layers=layers)
    sg = S.schedule_stage_graph(M.StageGraph([M.Stage(0, wl.graph.op_ids, 16, frozenset({0}))], [], wl.mini_batch))
    ex = Executor(wl, sg, 0, 1, CudaBackend(dev), lr=1e-3)
    batch = to_device_rows(ex, make_batch(wl, 0), ex.dtype, dev)
    for _ in range(2):
        ex.run_iteration(batch)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ex.run_iteration(batch)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


_COLS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
         "smsp__issue_active.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
         "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size", "launch__registers_per_thread"]


def summarise(raw_csv, out_csv, out_json):
    rows = list(csv.reader(open(raw_csv)))
    h, units, data = rows[0], rows[1], rows[2:]
    idx = {c: h.index(c) for c in _COLS if c in h}
    ki = h.index("Kernel Name")
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}

    def mb(r, c):
        return float(r[idx[c]].replace(",", "")) * scale.get(units[idx[c]], 1.0)

    out = []
    gemm_mb = gemm_us = 0.0
    n_gemm = 0
    for r in data:
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
        rec = {"kernel": name}
        for c in _COLS:
            if c in idx:
                rec[c] = r[idx[c]]
        out.append(rec)
        if re.search(r"gemm_tc|splitk_reduce", name):
            gemm_mb += mb(r, "dram__bytes_read.sum") + mb(r, "dram__bytes_write.sum")
            gemm_us += float(r[idx["gpu__time_duration.sum"]].replace(",", "")) * (
                1e-3 if units[idx["gpu__time_duration.sum"]] in ("nsecond", "ns") else 1.0)
            n_gemm += 1
    with open(out_csv, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["kernel"] + [c for c in _COLS if c in idx])
        w.writeheader()
        w.writerow({"kernel": "(units)", **{c: units[idx[c]] for c in idx}})
        w.writerows(out)
    # two layers + the CE head; head GEMMs are small (16 x 1000 / 1024), counted with the layers
    layers = 2
    res = {"what": "one MMT iteration (B=16, 1 branch x 2 layers) under ncu --set full; GEMM family = gemm_tc* + splitk_reduce",
           "gemm_launches": n_gemm, "gemm_dram_MB": round(gemm_mb, 1), "gemm_us_cold": round(gemm_us, 1),
           "logical_gemms_per_layer": 12, "traffic_MB_per_logical_gemm": round(gemm_mb / (12 * layers), 1),
           "algorithmic_MB_per_logical_gemm": round(_alg_layer_mb() / 12, 1)}
    json.dump(res, open(out_json, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--summarise", nargs=3, metavar=("RAW_CSV", "OUT_CSV", "OUT_JSON"))
    ap.add_argument("--full", action="store_true", help="the bench's whole MMT model (4 x 12 layers), e.g. for a launch list")
    a = ap.parse_args()
    if a.summarise:
        summarise(*a.summarise)
    else:
        run(*((4, 12) if a.full else (1, 2)))
