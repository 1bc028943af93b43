#!/usr/bin/env python
"""Benchmark: GPP training throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--workload all|mmt|candle|dlrm|toy] [--mode gpp|spp]

One process per GPU.  ``--gpus N`` with N > 1 outside torchrun re-launches this
script under ``torch.distributed.run`` (127.0.0.1) with N ranks; every rank
checks WORLD_SIZE == N.  A "step" is one synchronous training iteration of the
workload's configured StageGraph: every stage's kFkB task list, the P2P
activation/gradient transfers, the DP all-reduce and the SGD update.

Headline: the Multi-Modal Transformer (BASELINE configs[2], the north-star
target: 4 branches x 12 pre-LN layers, d=1024, S=512), mini-batch 16 per GPU
(weak scaling; PAPER.md:1099-1101 doubles B per doubling of devices).  With the
default ``--workload all`` the line carries ``sub_results`` for CANDLE-Uno
(configs[1], B = 1024 N) and DLRM (configs[3], B = 8192 N), each with its own
value / e2e / roofline / cpu_baseline / GPP-vs-SPP fields.  Strategies come from
the frozen StrategyFiles in profiles/strategies/ (planned afresh if stale).

value : samples/s with the inputs already resident in HBM, the iteration replayed
        from a CUDA graph, CUDA events, max over ranks (the per-step working set —
        weights + fp32 master/grad — is GBs >> the 126 MB L2: every step is L2-cold).
e2e   : the same metric through the public API ``runtime.api.execute``: pinned host
        batches, each step's H2D copy (double-buffered) and the loss D2H inside the
        timed region.
--impl reference : the CPU path (the monolithic torch-CPU training step of the
        workload, native bf16 on the host cores) on a bounded sample, rank 0 only.
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
CPU_SAMPLE = {"mmt": 2, "candle": 256, "dlrm": 1024, "toy": 64}  # per CPU step (bounded sample)


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


def _describe(wl, branches=None) -> str:
    if wl.name == "candle":
        return "candle: 7 towers x 4 x Linear(4096,4096)+ReLU -> concat -> Linear(28672,1024)+ReLU -> Linear(1024,1) MSE"
    if wl.name == "mmt":
        return (f"mmt: {branches or 4} branches x 12 pre-LN encoder layers (d=1024, 16 heads, FFN 4096 GELU, S=512) "
                "-> mean-pool -> concat -> Linear(., 1000) CE")
    if wl.name == "dlrm":
        return "dlrm: bottom 13->4096x3->64, 26 x 1M x 64 fp32 tables bag 100 (sum), dot interaction 415, top 416->4096x3->1 BCE"
    return wl.name


def cpu_reference_run(wl_name: str, sample_B: int, steps: int, min_seconds: float = 0.0, warmup: int = 1,
                      branches: int | None = None):
    """Time the reference's CPU path (the monolithic torch-CPU training step of the same
    model, parameters and activations in native bf16 on the host cores, all threads) on
    a bounded sample: ``steps`` steps of ``sample_B`` samples, continued until at least
    ``min_seconds`` are timed.  Returns (samples/s, seconds, steps run, threads)."""
    from oracle.reference_model import ReferenceModel
    from paper_2406_17145_b200.runtime.data import make_batch

    torch.set_num_threads(os.cpu_count() or 1)
    wl = _workload(wl_name, 1, sample_B, branches)
    ref = ReferenceModel(wl, native_bf16=True)
    batches = [make_batch(wl, i) for i in range(2)]
    for w in range(max(1, warmup)):  # warm-up (allocations, thread pools, oneDNN kernels)
        ref.step(batches[w % 2], 1e-4)
    t0 = time.perf_counter()
    n = 0
    while n < steps or (time.perf_counter() - t0 < min_seconds and n < 1000):
        ref.step(batches[n % 2], 1e-4)
        n += 1
    dt = time.perf_counter() - t0
    return sample_B * n / dt, dt, n, torch.get_num_threads()


def run_reference(args, rank, world):
    """--impl reference: rank 0 times the CPU path of the headline workload; others exit."""
    if rank != 0:
        return
    name = "mmt" if args.workload == "all" else args.workload
    sample = CPU_SAMPLE[name]
    # warm-up honours the contract's W >= 3 (capped at 3: each warm-up step is a full CPU step)
    val, dt, n_run, cores = cpu_reference_run(name, sample, max(1, min(args.steps, 20)),
                                              warmup=min(args.warmup, 3), branches=args.branches)
    wl = _workload(name, world, args.per_gpu_batch, args.branches)
    line = {
        "metric": "train samples/sec", "value": round(val, 4), "unit": "samples/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": n_run, "warmup": min(args.warmup, 3),
        "ms_per_step": round(1e3 * dt / n_run, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": _describe(wl, args.branches), "global_batch": wl.mini_batch,
                   "cpu_sample_per_step": sample, "device": "host CPU"},
        "cpu_baseline": {"value": round(val, 4), "unit": "samples/s", "cores": cores, "kind": "port",
                         "sample": f"{name}: {n_run} steps x B={sample}, monolithic torch-CPU training step in "
                                   f"native bf16 (oracle/reference_model.py, native_bf16=True), {dt:.1f}s"},
        "e2e": {"value": round(val, 4), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _gemm_traffic(workload: str) -> dict:
    """DRAM bytes per GEMM launch from the committed ncu --set full capture of one CANDLE
    step (profiles/ncu_step_gemms_r1d_summary.csv), averaged over the step's launch mix
    (28 tower fw, 21 tower dgrad, 28 tower wgrad+SGD, one of each tail GEMM), beside the
    algorithmic bytes of the same mix (operands + outputs + fp32 master read/write + bf16
    shadow).  MMT: the GEMM-family DRAM bytes of one captured iteration (1 branch x 2 layers,
    the bench's per-layer shapes; tools/ncu_mmt_layer.py) per logical GEMM (12 per layer),
    beside the same mix's algorithmic bytes.  DLRM reports null."""
    if workload == "mmt":
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_mmt_layer_r2_gemm.json")
        try:
            d = json.load(open(path))
        except (OSError, ValueError):
            return {"traffic": None}
        return {"traffic": d["traffic_MB_per_logical_gemm"], "traffic_unit": "MB per GEMM launch (ncu dram read+write, layer mix)",
                "algorithmic_MB_per_launch": d["algorithmic_MB_per_logical_gemm"],
                "traffic_source": "profiles/ncu_mmt_layer_r2_gemm.json"}
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


def _time_arm(wl, sg, world, rank, dev, args, clocks=True):
    """Build this rank's executor for ``sg``, capture its iteration in a CUDA graph and time
    ``args.steps`` replays on device-resident inputs (max over ranks)."""
    from paper_2406_17145_b200.runtime import lib
    from paper_2406_17145_b200.runtime.data import make_batch, to_device_rows
    from paper_2406_17145_b200.runtime.executor import Executor
    from paper_2406_17145_b200.runtime.graph import GraphedIteration
    from paper_2406_17145_b200.runtime.profiler import TimedBackend

    be = TimedBackend(dev)
    be.enabled = False
    ex = Executor(wl, sg, rank, world, be, lr=1e-4)
    keys = set(ex.data_keys()) if ex.stage else set()
    dev_batch = to_device_rows(ex, make_batch(wl, 0, keys=keys), ex.dtype, dev) if ex.stage else {}
    n0 = lib.launch_count()
    ex.run_iteration(dev_batch)
    per_iter = lib.launch_count() - n0  # this rank's libgpp kernels per iteration
    graphed = None if args.no_graph else GraphedIteration(ex, dev_batch)

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
    ms = e0.elapsed_time(e1)
    clk = sampler.stop() if sampler else None
    launches = per_iter * args.steps
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        lt = torch.tensor([float(launches)], device=dev)
        dist.all_reduce(lt)
        launches = int(lt.item())
    return {"ex": ex, "graphed": graphed, "dev_batch": dev_batch, "ms": ms, "launches": launches, "clocks": clk,
            "be": be}


def _dlrm_bf16_roof(wl, peaks, world, t_iter) -> dict:
    """DLRM's tables are fp32 here (exact sparse SGD); SURVEY section
    8(d) config 4 names bf16 tables.  The same roofline with the bf16 config's table bytes
    (gather 2 B, read-modify-write 2 x 2 B per element) -- the stricter denominator."""
    spec = next(s for s in wl.layers.values() if s.kind == "embbag")
    tables = sum(1 for s in wl.layers.values() if s.kind == "embbag")
    bag, emb = spec.extra[0], spec.out_dim
    byts = tables * (3 * bag * emb * 2 + 2 * bag * 8 + 2 * emb * 2)
    t = wl.mini_batch * (wl.flops_per_sample / (peaks["bf16_tflops_sustained"] * 1e12)
                         + byts / (peaks["hbm_gbs"] * 1e9)) / world * 1e3
    return {"bf16_table_config": {"bytes_per_sample": byts, "t_roof_ms": round(t, 4), "frac": round(t / t_iter, 4)}}


def _attn_flops_per_launch(wl, ex) -> dict:
    """Algorithmic FLOPs of one attention launch on this rank (all heads of a micro-batch):
    fw = 2 GEMMs (QK^T, PV) = 4 S^2 dh per head; bw = 5 GEMM-equivalents with the
    recompute of S = QK^T (dV, dP, dQ, dK, S) = 10 S^2 dh per head, 2 without it."""
    for o in (ex.ops if ex.stage else []):
        spec = wl.layers[o]
        if spec.kind == "mmt_layer":
            S, d, H, _, _ = spec.extra
            z = ex.m * H
            fw, bw = 4.0 * S * S * (d // H) * z, 10.0 * S * S * (d // H) * z
            return {"attn_fwd": fw, "attn_bwd": bw, "flash_attn_fwd": fw, "flash_attn_bwd": bw}
    return {}


def _plan(wl, world, rank, mode, costs):
    """Rank 0 loads (or plans) the strategy and broadcasts it as a StrategyFile document, so
    N ranks never plan N times (and all run the identical StageGraph)."""
    from paper_2406_17145_b200.cli import strategy_from_json, strategy_to_json
    from paper_2406_17145_b200.runtime.api import plan_cached

    if world == 1:
        return plan_cached(wl, world, mode, costs=costs)
    box = [None]
    if rank == 0:
        sg, meta = plan_cached(wl, world, mode, costs=costs)
        box = [(strategy_to_json(sg, wl.graph), meta)]
    dist.broadcast_object_list(box, src=0)
    doc, meta = box[0]
    return strategy_from_json(doc)[0], meta


def bench_workload(name, args, rank, world, dev, peaks, peak_src, cpu_ok: bool) -> dict | None:
    from paper_2406_17145_b200.runtime.api import execute, twin
    from paper_2406_17145_b200.runtime.data import make_batch
    from paper_2406_17145_b200.runtime.trace import trace_diff
    from paper_2406_17145_b200.workloads import b200_cluster, with_measured_curves

    wl = _workload(name, world, args.per_gpu_batch, args.branches if name == "mmt" else None)
    cluster = b200_cluster(world)
    sg, meta = _plan(wl, world, rank, args.mode, args.costs)
    arm = _time_arm(wl, sg, world, rank, dev, args)
    ex, be, ms = arm["ex"], arm["be"], arm["ms"]
    launches, clk, graphed_flag = arm["launches"], arm["clocks"], arm["graphed"] is not None
    value = wl.mini_batch * args.steps / (ms / 1e3)

    # e2e through the public API: pinned host batches, H2D + loss D2H every step
    fulls = [make_batch(wl, s + 1, keys=set(ex.data_keys()) if ex.stage else set()) for s in range(2)]
    rep = execute(sg, cluster, wl, batch_source=lambda i: fulls[i % 2], iters=args.steps, graph=not args.no_graph,
                  ex=ex)
    e2e = rep.samples_per_s
    # one traced iteration: CUDA-event nodes around every kernel (graph-replayed) -> measured
    # Chrome trace, busy / idle per stage, kernel-family times; diffed against the twin
    be.reset()
    trep = execute(sg, cluster, wl, batch_source=lambda i: fulls[i % 2], iters=2, graph=not args.no_graph,
                   trace=True, ex=ex)
    summ = be.summary() if ex.stage else {"flops": 0.0, "ms": 0.0, "busy_ms": 0.0, "tflops": 0.0, "launches": 0}
    sim_graph = with_measured_curves(wl)[0].graph if args.costs == "measured" else wl.graph
    sim = twin(sg, cluster, sim_graph)
    tdiff = trace_diff(trep.task_times, sim)
    if args.trace_out and rank == 0:
        with open(f"{args.trace_out}.{name}.n{world}.measured.json", "w") as f:
            f.write(trep.trace)
        from paper_2406_17145_b200.sim import emit_trace

        with open(f"{args.trace_out}.{name}.n{world}.sim.json", "w") as f:
            f.write(emit_trace(sim))
    # the same iteration's dense GEMMs replayed back to back from one graph (no event nodes)
    alone = None
    if ex.stage is not None:
        try:
            alone = be.time_gemms_alone(lambda: ex.run_iteration(arm["dev_batch"]))
        except Exception as exc:  # noqa: BLE001 - report, keep the event-node figure
            alone = {"error": f"{type(exc).__name__}: {exc}"[:200]}
    # attention kernels (MMT): algorithmic FLOPs / event-node durations of the traced iteration
    attn = {}
    fl = _attn_flops_per_launch(wl, ex)
    for k, f in fl.items():
        o = summ.get("other_ms", {}).get(k)
        if o and o["launches"]:
            us = 1e3 * o["ms"] / o["launches"]
            attn[k] = {"launches_per_step": o["launches"], "avg_us": round(us, 2),
                       "tflops": round(f / (us * 1e-6) / 1e12, 1), "frac_burst": round(f / (us * 1e-6) / 1e12 / peaks["bf16_tflops"], 4),
                       "ms_per_step": round(o["ms"], 3)}
    t_iter = ms / args.steps
    busy = summ["busy_ms"]
    bt = torch.tensor([busy], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(bt)
    bubble = max(0.0, 1.0 - float(bt.item()) / (world * t_iter))
    t_roof = wl.mini_batch * (wl.flops_per_sample / (peaks["bf16_tflops_sustained"] * 1e12)
                              + wl.bytes_per_sample / (peaks["hbm_gbs"] * 1e9)) / world * 1e3

    spp = None
    if world > 1 and args.mode == "gpp" and not args.no_spp:
        gpp_sg = [(sorted(s.op_ids), s.micro_batch, s.sched_cfg.k if s.sched_cfg else None) for s in sg.stages]
        del arm, ex, be
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        ssg, smeta = _plan(wl, world, rank, "spp", args.costs)
        sp = _time_arm(wl, ssg, world, rank, dev, args, clocks=False)
        spp_value = wl.mini_batch * args.steps / (sp["ms"] / 1e3)
        sp_sg = [(sorted(s.op_ids), s.micro_batch, s.sched_cfg.k if s.sched_cfg else None) for s in ssg.stages]
        spp = {"value": round(spp_value, 3), "ms_per_step": round(sp["ms"] / args.steps, 4),
               "gpp_vs_spp_speedup": round(value / spp_value, 4), "plan": smeta.get("source"),
               "stages": [{"ops": len(s.op_ids), "b": s.micro_batch, "d": s.dp_degree} for s in ssg.stages],
               # the runtime sweep keeps a sequential candidate when the twin rates it faster;
               # equal (op sets, micro-batch, k) per stage and equal edges = the same pipeline
               "gpp_picked_sequential": (gpp_sg, sorted(sg.edges)) == (sp_sg, sorted(ssg.edges)),
               "note": "SPP = spp_optimize (SPEC.md:384-392) strategy on this same runtime, CUDA-graph replay"}
        del sp
        gc.collect()
        torch.cuda.empty_cache()
    if rank != 0:
        return None
    cpu = None
    if cpu_ok and world == 1 and not args.no_cpu_baseline:
        sample = CPU_SAMPLE[name]
        cv, cdt, cn, cores = cpu_reference_run(name, sample, 2, min_seconds=args.cpu_seconds,
                                               branches=args.branches if name == "mmt" else None)
        cpu = {"value": round(cv, 4), "unit": "samples/s", "cores": cores, "kind": "port",
               "sample": f"{name}: {cn} steps x B={sample}, monolithic torch-CPU training step in native bf16 "
                         f"(oracle/reference_model.py, native_bf16=True), {cdt:.1f}s"}
    peak = peaks["bf16_tflops"]  # the GEMMs are timed ALONE (back to back): the burst figure
    achieved = alone["tflops"] if alone and alone.get("tflops") else summ["tflops"]
    gp = meta.get("gpp_partitioner")
    line = {
        "metric": "train samples/sec", "value": round(value, 3), "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_iter, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16" if wl.dtype != "fp32" else "fp32", "data": "synthetic",
        "config": {
            "workload": _describe(wl, args.branches), "global_batch": wl.mini_batch, "mode": args.mode,
            "parallelism": f"{args.mode} stages={len(sg.stages)} depth={sim.depth}",
            "stages": [{"ops": len(s.op_ids), "b": s.micro_batch, "d": s.dp_degree,
                        "inflight": s.sched_cfg.inflight_samples} for s in sg.stages],
            "plan": {k: v for k, v in meta.items() if k != "gpp_partitioner"},
            "gpp_partitioner": None if gp is None else {"twin_ms": gp["twin_ms"],
                                                        "stages": [{"ops": len(s["ops"]), "b": s["b"], "d": len(s["devices"])}
                                                                   for s in gp["stages"]]},
            "l2": {"candle": "per-step working set (weights+master+grads ~2.9 GB) >> 126 MB L2",
                   "dlrm": "per-step working set (26 x 256 MB fp32 tables + MLP master/grads) >> 126 MB L2",
                   "mmt": "per-step working set (48 layers x ~150 MB master/grad/shadow + activations) >> 126 MB L2",
                   "toy": "toy model fits in L2 (launch-bound; no roofline claim)"}.get(name),
            "optimizer": "SGD fp32 master + bf16 shadow (fused into the last wgrad epilogue when DP=1)",
            "cuda_graph": graphed_flag, "costs": args.costs,
        },
        "e2e": {"value": round(e2e, 3), "unit": "samples/s", "h2d_bytes_per_step": rep.h2d_bytes_per_step,
                "d2h_bytes_per_step": rep.d2h_bytes_per_step, "api": "paper_2406_17145_b200.runtime.api.execute"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "tensor", "kernel": "gemm_tc_pair_kernel / gemm_tc_kernel (tcgen05 bf16 GEMM family: every dense "
                                                  "fw / dgrad / wgrad(+SGD) launch of the iteration)",
                     "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4) if peak else None,
                     **(_gemm_traffic(name)),
                     "peak_source": f"{peak_src} bf16_tflops (burst: the GEMMs are replayed alone)",
                     "timing": "one iteration's GEMM launches replayed back to back from a CUDA graph, CUDA events "
                               "around the replay (gemms_alone)",
                     "gemms_alone": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in (alone or {}).items()},
                     "achieved_event_nodes": round(summ["tflops"], 2),
                     "share_of_step": round(summ["ms"] / t_iter, 4) if t_iter > 0 else None,
                     "attention": attn or None,
                     "by_kind": summ.get("by_kind", {}), "other_kernels_ms": summ.get("other_ms", {})},
        "clocks": clk,
        "step_roofline": {"t_roof_ms": round(t_roof, 4), "frac": round(t_roof / t_iter, 4),
                          "flops_per_sample": wl.flops_per_sample, "bytes_per_sample": wl.bytes_per_sample,
                          **(_dlrm_bf16_roof(wl, peaks, world, t_iter) if name == "dlrm" else {}),
                          "note": "summed stage-compute roofline: B*(F/P_sustained + bytes/BW_hbm)/N vs measured step"},
        "bubble": {"measured": round(bubble, 4), "model": round(sim.bubble_fraction, 4),
                   "note": "1 - sum over ranks of kernel busy time / (N * step time); kernel time from CUDA-event "
                           "nodes around every kernel of a graph-replayed iteration"},
        "report": {"iteration_ms": round(trep.iteration_ms, 4), "peak_inflight_samples": trep.peak_inflight_samples,
                   "busy_ms": {k: round(v, 4) for k, v in trep.busy_ms.items()},
                   "idle_ms": {k: round(v, 4) for k, v in trep.idle_ms.items()},
                   "peak_mem_gb": {k: round(v / 1e9, 2) for k, v in trep.peak_mem_bytes.items()},
                   "warm_up_microbatches": trep.warm_up_microbatches, "depth": trep.depth,
                   "note": "runtime.api.execute(trace=True) RunReport (SimReport fields, measured)"},
        "trace_vs_sim": tdiff,
        "sim": {"iteration_ms_model": round(sim.iteration_ms, 4), "bubble_fraction_model": round(sim.bubble_fraction, 4)},
        "spp": spp,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    return line


def _spawn_ranks(args) -> int:
    """``--gpus N`` (N > 1) outside torchrun: re-launch this script with N ranks under
    torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def _init_ranks(args, rank, world, local):
    """One process per GPU: NCCL (or gloo for --dry-run) process group; every rank prints
    its init line so the rank/world check is observable."""
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with torchrun --nproc-per-node "
                         f"{args.gpus} (or without torchrun and let bench.py spawn the ranks)")
    if args.dry_run:
        if world > 1:
            dist.init_process_group("gloo")
        print(f"[bench] rank {rank}/{world} backend={'gloo' if world > 1 else 'none'} dry-run pid={os.getpid()}",
              file=sys.stderr, flush=True)
        return None
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        nccl = ".".join(str(x) for x in torch.cuda.nccl.version())
    print(f"[bench] rank {rank}/{world} on cuda:{local} ({torch.cuda.get_device_name(dev)}) "
          f"backend={'nccl ' + nccl if nccl else 'none'} pid={os.getpid()}", file=sys.stderr, flush=True)
    return dev


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="all", choices=["all", "mmt", "candle", "dlrm", "toy"],
                    help="all = MMT headline + CANDLE-Uno and DLRM sub-results")
    ap.add_argument("--mode", default="gpp", choices=["gpp", "spp"])
    ap.add_argument("--costs", default="measured", choices=["measured", "analytic"],
                    help="partitioner cost curves: frozen B200 tables (profiles/) or analytic FLOP curves")
    ap.add_argument("--per-gpu-batch", type=int, default=None)
    ap.add_argument("--branches", type=int, default=None, help="MMT branch count (default 4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="minimum timed CPU work per cpu_baseline")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels eagerly (no CUDA graph)")
    ap.add_argument("--no-spp", action="store_true", help="skip the SPP comparison arm (N > 1)")
    ap.add_argument("--trace-out", default=None, help="write measured + simulated Chrome traces to PREFIX.*.json")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch / rendezvous only (gloo, no GPU): print one line per rank and exit")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    from paper_2406_17145_b200.runtime.api import dist_env

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args))
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    dev = _init_ranks(args, rank, world, local)
    if args.dry_run:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world}), flush=True)
        return
    peaks, peak_src = _peaks()
    names = ["mmt", "candle", "dlrm"] if args.workload == "all" else [args.workload]
    results = {}
    for i, name in enumerate(names):
        results[name] = bench_workload(name, args, rank, world, dev, peaks, peak_src, cpu_ok=True)
        import gc

        gc.collect()
        torch.cuda.empty_cache()
    if rank == 0:
        head = results[names[0]]
        if len(names) > 1:
            head["sub_results"] = {n: results[n] for n in names[1:]}
        print(json.dumps(head), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
