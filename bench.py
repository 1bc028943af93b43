#!/usr/bin/env python
"""Benchmark: GPP training throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--workload candle|toy] [--mode gpp|spp]

One process per GPU (torchrun for N > 1).  A "step" is one synchronous training
iteration of the workload's configured StageGraph: every stage's kFkB task
list, the P2P activation/gradient transfers, the DP all-reduce and the SGD
update.  Workload at N GPUs: CANDLE-Uno (BASELINE configs[1]) with mini-batch
1024*N (PAPER.md:1100 scales B with the device count; 4096 at 4 GPUs), random
init, synthetic N(0,1) features.

value : samples/s with the inputs already resident in HBM (CUDA events, max
        over ranks; per-iteration working set = 0.94 GB bf16 weights + 1.9 GB
        fp32 master/grad >> 126 MB L2, so every timed step starts L2-cold).
e2e   : same metric through the public API with pinned HOST buffers: every
        step's H2D input copy (double-buffered on a copy stream) and the D2H
        loss read are inside the timed region.
--impl reference : the CPU path (oracle/reference_model.py: the monolithic
        torch-CPU training step) on a bounded sample, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled DURING the timed region.

    NVML polled every 5 ms from a thread (a 20-step region is ~70 ms: one nvidia-smi
    process per sample caught at most one reading), the device matched by PCI bus id;
    falls back to polling nvidia-smi if NVML is unavailable."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows: list[list[str]] = []
        self.sm: list[float] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        self._h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            h = None
            try:
                pr = torch.cuda.get_device_properties(gpu_index)
                for fmt in ("{:08x}:{:02x}:{:02x}.0", "{:04x}:{:02x}:{:02x}.0"):
                    try:
                        h = pynvml.nvmlDeviceGetHandleByPciBusId(
                            fmt.format(pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id).encode())
                        break
                    except Exception:  # noqa: BLE001
                        continue
            except Exception:  # noqa: BLE001
                h = None
            self._h = h or pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self._nv = pynvml
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:  # noqa: BLE001
            self._nv = None

    def _run_nvml(self):
        nv, h = self._nv, self._h
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, b in bits.items():
                    if r & b:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.005)

    def _run_smi(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def start(self):
        self._t = threading.Thread(target=self._run_nvml if self._nv else self._run_smi, daemon=True)
        self._t.start()

    def stop(self) -> dict:
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if self._nv:
            return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 5 ms"}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows), "source": "nvidia-smi"}


def _workload(name: str, world: int, per_gpu: int | None, branches: int | None = None):
    from paper_2406_17145_b200 import workloads as W

    if name == "candle":
        return W.candle(B=(per_gpu or 1024) * world)
    if name == "toy":
        return W.toy(B=(per_gpu or 64) * world)
    if name == "dlrm":
        return W.dlrm(B=(per_gpu or 8192) * world)
    if name == "mmt":  # --branches: the BASELINE configs[4] branch sweep (2 / 4 / 8 branches)
        return W.mmt(B=(per_gpu or 16) * world, branches=branches or 4)
    raise SystemExit(f"unknown workload {name}")


def cpu_reference_run(wl_name: str, sample_B: int, steps: int, min_seconds: float = 0.0, warmup: int = 1):
    """Time the reference's CPU path (monolithic torch-CPU step) on a bounded sample:
    ``steps`` steps, continued until at least ``min_seconds`` of CPU work are timed.
    Returns (samples/s, seconds, steps run)."""
    from oracle.reference_model import ReferenceModel
    from paper_2406_17145_b200.runtime.data import make_batch

    torch.set_num_threads(os.cpu_count() or 1)
    wl = _workload(wl_name, 1, sample_B)
    ref = ReferenceModel(wl)
    for w in range(max(1, warmup)):  # warm-up (allocations, thread pools)
        ref.step(make_batch(wl, 10_000 + w), 1e-3)
    t0 = time.perf_counter()
    n = 0
    while n < steps or (time.perf_counter() - t0 < min_seconds and n < 1000):
        ref.step(make_batch(wl, n + 1), 1e-3)
        n += 1
    dt = time.perf_counter() - t0
    return sample_B * n / dt, dt, n


def run_reference(args, rank, world):
    if rank != 0:
        return
    sample = {"candle": 32, "toy": 64, "dlrm": 16, "mmt": 1}[args.workload]
    # every step is one bounded CPU sample of the workload (B = sample); K steps
    val, dt, n_run = cpu_reference_run(args.workload, sample, max(1, min(args.steps, 50)),
                                       warmup=min(args.warmup, 5))
    cores = torch.get_num_threads()
    line = {
        "metric": "train samples/sec", "value": round(val, 3), "unit": "samples/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": n_run, "warmup": min(args.warmup, 5),
        "ms_per_step": round(1e3 * dt / n_run, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16-emulated fp32 (CPU)", "data": "synthetic",
        "config": {"workload": f"{args.workload} (CPU sample B={sample} per step)", "device": "host CPU"},
        "cpu_baseline": {"value": round(val, 3), "unit": "samples/s", "cores": cores, "kind": "port",
                         "sample": f"{args.workload} mini-batch of {sample} samples, monolithic torch-CPU step"},
        "e2e": {"value": round(val, 3), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _gemm_traffic(workload: str) -> dict:
    """DRAM bytes per GEMM launch from the committed ncu --set full capture of one CANDLE
    step (profiles/ncu_step_gemms_r1d_summary.csv), averaged over the step's launch mix
    (28 tower fw, 21 tower dgrad, 28 tower wgrad+SGD, one of each tail GEMM), beside the
    algorithmic bytes of the same mix (operands + outputs + fp32 master read/write + bf16
    shadow).  Only the CANDLE step was captured; other workloads report null."""
    if workload != "candle":
        return {"traffic": None}
    import csv

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_step_gemms_r1d_summary.csv")
    try:
        rows = list(csv.reader(open(path)))
    except OSError:
        return {"traffic": None}
    h = rows[0]
    mb = {r[0]: float(r[h.index("dram__bytes_read.sum")]) + float(r[h.index("dram__bytes_write.sum")]) for r in rows[2:]}
    mix = {"fw tower": (28, 48.0), "fw tail": (1, 119.4), "dgrad tail": (1, 178.2), "wgrad+SGD tail": (1, 353.3),
           "dgrad tower": (21, 56.0), "wgrad+SGD tower": (28, 176.0)}
    tot = alg = n = 0.0
    for role, v in mb.items():
        key = next((k for k in mix if role.startswith(k + " ")), None)
        if key is None:
            continue
        c, a = mix[key]
        tot, alg, n = tot + c * v, alg + c * a, n + c
    if not n:
        return {"traffic": None}
    return {"traffic": round(tot / n, 1), "traffic_unit": "MB per GEMM launch (ncu dram read+write, step mix)",
            "algorithmic_MB_per_launch": round(alg / n, 1),
            "traffic_source": "profiles/ncu_step_gemms_r1d_summary.csv"}


def _time_arm(wl, world, rank, dev, mode, args, clocks=True):
    """Plan ``mode`` (gpp | spp) for ``world`` GPUs, build this rank's executor, capture its
    iteration in a CUDA graph and time ``args.steps`` replays (max over ranks)."""
    from paper_2406_17145_b200.runtime import lib
    from paper_2406_17145_b200.runtime.api import plan
    from paper_2406_17145_b200.runtime.data import make_batch, to_device_rows
    from paper_2406_17145_b200.runtime.executor import Executor
    from paper_2406_17145_b200.runtime.profiler import TimedBackend

    t_plan = time.perf_counter()
    strategy = plan(wl, world, mode, costs=args.costs)
    t_plan = time.perf_counter() - t_plan
    sg = strategy.stage_graph
    be = TimedBackend(dev)
    be.enabled = False
    ex = Executor(wl, sg, rank, world, be, lr=1e-4)
    keys = set(ex.data_keys()) if ex.stage else set()
    full = make_batch(wl, 0, keys=keys)
    dev_batch = to_device_rows(ex, full, ex.dtype, dev) if ex.stage else {}
    graphed = None
    graphed_launches = 0
    if not args.no_graph and (ex.stage is not None or world > 1):
        from paper_2406_17145_b200.runtime.graph import GraphedIteration

        n_before = lib.launch_count()
        ex.run_iteration(dev_batch)
        graphed_launches = lib.launch_count() - n_before  # libgpp kernels per iteration
        graphed = GraphedIteration(ex, dev_batch)
        for b in graphed.bufs:
            for k in b:
                b[k].copy_(dev_batch[k])

    def step(i=0):
        return graphed.replay(i) if graphed is not None else ex.run_iteration(dev_batch)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(dev.index) if clocks else None
    if sampler:
        sampler.start()
    launches0 = lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nvtx = os.environ.get("GPP_NVTX") == "1"  # ncu --nvtx --nvtx-include "timed/": steady-state launch lists
    torch.cuda.synchronize()
    if nvtx:
        torch.cuda.nvtx.range_push("timed")
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if nvtx:
        torch.cuda.nvtx.range_pop()
    launches = lib.launch_count() - launches0
    if graphed is not None:  # replays launch the captured kernels without host calls
        launches = graphed_launches * args.steps
    ms = e0.elapsed_time(e1)
    clk = sampler.stop() if sampler else None
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        lt = torch.tensor([float(launches)], device=dev)
        dist.all_reduce(lt)
        launches = int(lt.item())
    return {"ex": ex, "sg": sg, "graphed": graphed, "dev_batch": dev_batch, "ms": ms, "launches": launches,
            "clocks": clk, "plan_s": t_plan, "be": be}


def _ncu_cross_check(workload: str, peak: float) -> dict | None:
    """The committed ncu --set full capture of the CANDLE step's forward tower GEMMs
    (profiles/ncu_candle_fw_gemm_r1g_summary.csv): per-launch duration without the event
    nodes the live timing needs (which add ~2-4 us per launch), for comparison."""
    if workload != "candle":
        return None
    import csv

    path = os.path.join(ROOT, "profiles", "ncu_candle_fw_gemm_r1g_summary.csv")
    try:
        rows = list(csv.reader(open(path)))
    except OSError:
        return None
    h = rows[0]
    us = [float(r[h.index("gpu__time_duration.sum")].split()[0]) for r in rows[1:]]
    tens = [float(r[h.index("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")].split()[0]) for r in rows[1:]]
    avg = sum(us) / len(us)
    tf = 2.0 * 1024 * 4096 * 4096 / (avg * 1e-6) / 1e12
    return {"kernel": "fw tower GEMM 1024x4096x4096 (+bias+ReLU)", "us": round(avg, 2), "tflops": round(tf, 1),
            "frac": round(tf / peak, 4), "tensor_pipe_active_pct": round(sum(tens) / len(tens), 1),
            "source": "profiles/ncu_candle_fw_gemm_r1g_summary.csv"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="candle", choices=["candle", "toy", "dlrm", "mmt"])
    ap.add_argument("--mode", default="gpp", choices=["gpp", "spp"])
    ap.add_argument("--costs", default="measured", choices=["measured", "analytic"],
                    help="partitioner cost curves: frozen B200 tables (profiles/) or analytic FLOP curves")
    ap.add_argument("--per-gpu-batch", type=int, default=None)
    ap.add_argument("--branches", type=int, default=None, help="MMT branch count (default 4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels eagerly (no CUDA graph)")
    ap.add_argument("--no-spp", action="store_true", help="skip the SPP comparison arm (N > 1)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    from paper_2406_17145_b200.runtime.api import dist_env

    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2406_17145_b200.runtime.data import make_batch
    from paper_2406_17145_b200.runtime.api import twin
    from paper_2406_17145_b200.workloads import b200_cluster, with_measured_curves

    wl = _workload(args.workload, world, args.per_gpu_batch, args.branches)
    dev = torch.device("cuda", local)
    arm = _time_arm(wl, world, rank, dev, args.mode, args)
    ex, sg, graphed, dev_batch, ms, launches, clk, t_plan, be = (
        arm["ex"], arm["sg"], arm["graphed"], arm["dev_batch"], arm["ms"], arm["launches"], arm["clocks"],
        arm["plan_s"], arm["be"])
    keys = set(ex.data_keys()) if ex.stage else set()
    value = wl.mini_batch * args.steps / (ms / 1e3)

    # ---------------- e2e: host buffers through the public API ----------------
    host = []
    h2d_bytes = 0
    for s in range(2):
        fb = make_batch(wl, s + 1, keys=keys)
        hb = {}
        for k in ex.data_keys() if ex.stage else []:
            t = ex.local_rows(fb[k])
            if t.is_floating_point():
                t = t.to(ex.dtype) if t.dim() > 1 else t.float()
            hb[k] = t.pin_memory()
        host.append(hb)
    h2d_bytes = sum(t.numel() * t.element_size() for t in host[0].values())
    dbufs = graphed.bufs if graphed is not None else [{k: torch.empty_like(v, device=dev) for k, v in hb.items()} for hb in host]
    loss_host = torch.zeros(args.steps, dtype=torch.float32).pin_memory()
    copy_stream = torch.cuda.Stream(dev)
    ready = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()

    def h2d(i):
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[i % 2])
            for k, v in host[i % 2].items():
                dbufs[i % 2][k].copy_(v, non_blocking=True)
            ready[i % 2].record(copy_stream)

    for i in range(2):
        consumed[i].record()
    h2d(0)
    for i in range(args.steps):
        if i + 1 < args.steps:
            h2d(i + 1)
        torch.cuda.current_stream().wait_event(ready[i % 2])
        loss = graphed.replay(i % 2) if graphed is not None else ex.run_iteration(dbufs[i % 2])
        consumed[i % 2].record()
        if loss is not None:
            loss_host[i:i + 1].copy_(loss, non_blocking=True)
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = wl.mini_batch * args.steps / (e2e_ms / 1e3)

    # ---------------- roofline + busy time: events around every kernel call ----------------
    # One iteration captured in a CUDA graph with an event-record node on each side of every
    # kernel call (external events keep their timestamps across replays) and replayed: the
    # durations are those of the graph-replayed step.  Fallback: eager iterations with the
    # GPU queue kept ahead of the host (a sleep longer than the host's enqueue time).
    prof_iters = 1
    timing = "cuda-graph event nodes"
    torch.cuda.synchronize()
    be.enabled = True
    be.external = True
    be.reset()
    try:
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        pg = torch.cuda.CUDAGraph()
        if world > 1:
            dist.barrier()
        with torch.cuda.graph(pg):
            ex.run_iteration(dev_batch)
        be.enabled = False
        for _ in range(3):
            pg.replay()
        torch.cuda.synchronize()
    except Exception as exc:  # noqa: BLE001 - report and fall back to eager timing
        timing = f"eager events, queue preloaded (graph capture failed: {type(exc).__name__})"
        be.external = False
        be.enabled = False
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        h0 = time.perf_counter()
        ex.run_iteration(dev_batch)
        host_s = time.perf_counter() - h0
        torch.cuda.synchronize()
        be.enabled = True
        be.reset()
        if world > 1:
            dist.barrier()
        be.preload(host_s)
        ex.run_iteration(dev_batch)
        torch.cuda.synchronize()
    summ = be.summary() if ex.stage else {"flops": 0.0, "ms": 0.0, "busy_ms": 0.0, "tflops": 0.0, "launches": 0}
    be.enabled = False
    # the same iteration's GEMMs replayed back to back from one graph, two events around
    # it: per-launch durations free of the event nodes above (timed on this rank; the
    # GEMMs do no communication)
    alone = None
    if ex.stage is not None:
        try:
            alone = be.time_gemms_alone(lambda: ex.run_iteration(dev_batch))
        except Exception as exc:  # noqa: BLE001 - report, keep the event-node figure
            alone = {"error": f"{type(exc).__name__}: {exc}"[:200]}
    peaks, peak_src = _peaks()
    t_iter = ms / args.steps
    cuda_graph = graphed is not None
    gemm_share = (summ["ms"] / prof_iters) / t_iter if ms > 0 else 0.0
    busy = summ["busy_ms"] / prof_iters  # this rank's kernel time per iteration
    busy_sum = busy
    if world > 1:
        bt = torch.tensor([busy], device=dev, dtype=torch.float64)
        dist.all_reduce(bt)
        busy_sum = float(bt.item())
    bubble = max(0.0, 1.0 - busy_sum / (world * t_iter))
    # summed stage-compute roofline: every sample's algorithmic FLOPs at the
    # sustained tensor peak plus its HBM-bound bytes at the measured copy bandwidth, over N GPUs
    t_roof = wl.mini_batch * (wl.flops_per_sample / (peaks["bf16_tflops_sustained"] * 1e12)
                              + wl.bytes_per_sample / (peaks["hbm_gbs"] * 1e9)) / world * 1e3

    # ---------------- GPP vs the sequential pipeline (SPP) on the same runtime ----------------
    spp = None
    if world > 1 and args.mode == "gpp" and not args.no_spp:
        spp_sg_gpp = [(len(s.op_ids), s.micro_batch, s.dp_degree) for s in sg.stages]
        del graphed, ex, dev_batch, arm
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        sp = _time_arm(wl, world, rank, dev, "spp", args, clocks=False)
        spp_value = wl.mini_batch * args.steps / (sp["ms"] / 1e3)
        spp = {"value": round(spp_value, 3), "ms_per_step": round(sp["ms"] / args.steps, 4),
               "gpp_vs_spp_speedup": round(value / spp_value, 4), "plan_s": round(sp["plan_s"], 3),
               "stages": [{"ops": len(s.op_ids), "b": s.micro_batch, "d": s.dp_degree} for s in sp["sg"].stages],
               "gpp_stages": [{"ops": a, "b": b, "d": d} for a, b, d in spp_sg_gpp],
               # the GPP sweep keeps a sequential candidate when the twin rates it faster
               "gpp_picked_sequential": ([(s.op_ids, s.micro_batch) for s in sg.stages], sg.edges)
                                        == ([(s.op_ids, s.micro_batch) for s in sp["sg"].stages], sp["sg"].edges),
               "note": "SPP = spp_optimize (SPEC.md:384-392) strategy on this same runtime, CUDA-graph replay"}

    # ---------------- simulated twin + bubble estimate ----------------
    cluster = b200_cluster(world)
    sim_graph = with_measured_curves(wl)[0].graph if args.costs == "measured" else wl.graph
    sim = twin(sg, cluster, sim_graph)

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only (the contract)
            sample = {"candle": 32, "toy": 64, "dlrm": 16, "mmt": 1}[args.workload]
            cv, cdt, cn = cpu_reference_run(args.workload, sample, 2, min_seconds=10.0)
            cpu = {"value": round(cv, 3), "unit": "samples/s", "cores": torch.get_num_threads(), "kind": "port",
                   "sample": f"{args.workload}, {cn} steps x B={sample}, monolithic torch-CPU training step "
                             f"(oracle/reference_model.py), {cdt:.1f}s"}
        peak = peaks["bf16_tflops_sustained"]
        achieved = alone["tflops"] if alone and alone.get("tflops") else summ["tflops"]
        line = {
            "metric": "train samples/sec", "value": round(value, 3), "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16" if wl.dtype != "fp32" else "fp32", "data": "synthetic",
            "config": {
                "workload": f"{wl.name}: 7 towers x 4 x Linear(4096,4096)+ReLU -> concat -> Linear(28672,1024)+ReLU -> Linear(1024,1) MSE"
                if wl.name == "candle" else (f"mmt: {args.branches or 4} branches x 12 pre-LN layers, d=1024, S=512"
                                            if wl.name == "mmt" else wl.name),
                "global_batch": wl.mini_batch, "mode": args.mode,
                "parallelism": f"{args.mode} stages={len(sg.stages)} depth={sim.depth}",
                "stages": [{"ops": len(s.op_ids), "b": s.micro_batch, "d": s.dp_degree,
                            "inflight": s.sched_cfg.inflight_samples} for s in sg.stages],
                "l2": {"candle": "per-step working set (weights+master+grads ~2.9 GB) >> 126 MB L2",
                       "dlrm": "per-step working set (26 x 256 MB fp32 tables + MLP master/grads) >> 126 MB L2",
                       "mmt": "per-step working set (48 layers x ~150 MB master/grad/shadow + activations) >> 126 MB L2",
                       "toy": "toy model fits in L2 (launch-bound; no roofline claim)"}.get(args.workload),
                "optimizer": "SGD fp32 master + bf16 shadow (fused into last wgrad epilogue when DP=1)",
                "plan_s": round(t_plan, 3), "cuda_graph": cuda_graph, "costs": args.costs,
            },
            "e2e": {"value": round(e2e, 3), "unit": "samples/s", "h2d_bytes_per_step": int(h2d_bytes),
                    "d2h_bytes_per_step": 4},
            "gpu_launches": int(launches),
            "roofline": {"bound": "tensor", "kernel": "gemm_tc_pair_kernel (tcgen05 cta_group::2 bf16 GEMM, all dense fw/dgrad/wgrad+SGD)",
                         "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                         "frac": round(achieved / peak, 4) if peak else None,
                         **_gemm_traffic(args.workload),
                         "peak_source": f"{peak_src} bf16_tflops_sustained",
                         "timing": "one iteration's GEMM launches replayed back to back from a CUDA graph, "
                                   "CUDA events around the replay (gemms_alone); the event-node figures below time "
                                   "each launch inside the full iteration graph",
                         "gemms_alone": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in (alone or {}).items()},
                         "achieved_event_nodes": round(summ["tflops"], 2),
                         "share_of_step": round(gemm_share, 4), "event_node_timing": timing,
                         "ncu_cross_check": _ncu_cross_check(args.workload, peak),
                         "by_kind": summ.get("by_kind", {}),
                         "other_kernels_ms": summ.get("other_ms", {})},
            "clocks": clk,
            "step_roofline": {"t_roof_ms": round(t_roof, 4), "frac": round(t_roof / t_iter, 4),
                              "flops_per_sample": wl.flops_per_sample, "bytes_per_sample": wl.bytes_per_sample,
                              "note": "summed stage-compute roofline: B*(F/P_sustained + bytes/BW_hbm)/N vs measured step"},
            "bubble": {"measured": round(bubble, 4), "busy_ms_per_gpu": round(busy_sum / world, 4),
                       "model": round(sim.bubble_fraction, 4),
                       "note": "1 - sum over ranks of kernel busy time / (N * step time); busy from events around "
                               "every kernel call in eager iterations"},
            "sim": {"iteration_ms_model": round(sim.iteration_ms, 4), "bubble_fraction_model": round(sim.bubble_fraction, 4)},
            "spp": spp,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
        if os.environ.get("GPP_BENCH_DETAIL"):
            print(json.dumps({"gemm_by_shape": summ.get("by_shape", {})}), file=sys.stderr)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
