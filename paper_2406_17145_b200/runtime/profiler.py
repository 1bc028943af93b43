"""Live kernel timing for the roofline report and measured cost curves.

``TimedBackend`` wraps the CUDA backend and brackets every dense-operator GEMM
(``linear_fwd``/``linear_dgrad``/``linear_wgrad``) with CUDA events on the
launching stream, recording algorithmic FLOPs per launch.  ``profile_ops``
measures fw/bw task times per operator over micro-batch sizes and returns
table ``CostCurve``s (model.py:18-97) — B200 profiles for the partitioner
(SURVEY.md §8(f) row 1).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .backend import CudaBackend


@dataclass
class _Rec:
    kind: str
    flops: float
    m: int
    n: int
    k: int
    start: torch.cuda.Event
    end: torch.cuda.Event
    task: tuple | None = None  # (stage id, "fw" | "bw", micro-batch index) being executed


GEMM_KINDS = ("fwd", "dgrad", "wgrad")
# every other kernel-launching backend call, timed for the per-rank busy time
_OTHER_CALLS = ("colsum", "colsum_multi", "rowdot_loss", "rowdot_fwd", "rowdot_bwd", "mse_loss", "bce_loss", "ce_loss", "copy_rows", "copy_rows_multi",
                "sgd_step", "embbag_fwd", "embbag_sgd", "embbag_sgd_multi", "interaction_fwd", "interaction_bwd",
                "layernorm_fwd", "layernorm_bwd", "softmax_fwd", "softmax_bwd", "meanpool_fwd",
                "meanpool_bwd", "attn_softmax", "attn_softmax_bwd", "gemm_batched", "attn_fwd", "attn_bwd",
                "flash_attn_fwd", "flash_attn_bwd")


class TimedBackend(CudaBackend):
    """CudaBackend with CUDA events around every kernel-launching call (when enabled).

    Dense-operator GEMMs are recorded with their algorithmic FLOPs (the roofline's
    tensor-bound kernel family); every other call is recorded with 0 FLOPs so that
    ``summary()['busy_ms']`` is the rank's total kernel time (the pipeline-bubble
    measure).  Events are recorded on the launching (current) stream.  Callers that
    want undistorted durations keep the GPU queue ahead of the host (``preload``)."""

    def __init__(self, device):
        super().__init__(device)
        self.records: list[_Rec] = []
        self.enabled = True
        self.external = False  # graph capture: event-record nodes that keep their timestamps
        self.gemm_calls = None  # list -> record every dense GEMM call (replayable closure)
        self.task = None  # set by the executor around each task (measured task trace)
        self.t_origin = None  # event recorded at the start of the last iteration
        for name in _OTHER_CALLS:
            base = getattr(CudaBackend, name, None)
            if base is not None:
                setattr(self, name, self._wrap(name, base))

    def _wrap(self, name, base):
        def call(*a, **kw):
            return self._timed(name, 0, 0, 0, lambda: base(self, *a, **kw))
        return call

    def _timed(self, kind, m, n, k, fn):
        if self.gemm_calls is not None and kind in GEMM_KINDS:
            self.gemm_calls.append((kind, 2.0 * m * n * k, fn))
        if not self.enabled:
            return fn()
        s = torch.cuda.Event(enable_timing=True, external=self.external)
        e = torch.cuda.Event(enable_timing=True, external=self.external)
        s.record()
        r = fn()
        e.record()
        self.records.append(_Rec(kind, 2.0 * m * n * k, m, n, k, s, e, self.task))
        return r

    def set_task(self, task) -> None:
        """Executor hook: the kernels that follow belong to ``task`` = (stage, dir, index);
        ``("iteration", ...)`` marks the start of an iteration (the trace's time origin)."""
        if task is not None and task[0] == "iteration":
            self.task = None
            if self.enabled:
                ev = torch.cuda.Event(enable_timing=True, external=self.external)
                ev.record()
                self.t_origin = ev
            return
        self.task = task

    def task_times(self) -> dict:
        """Measured {(stage, dir, index): (start_ms, end_ms, busy_ms)} of the recorded
        iteration: first kernel start / last kernel end relative to the iteration's start
        event, and the summed kernel time (waits for peers excluded).  Synchronises."""
        torch.cuda.synchronize()
        out: dict = {}
        for r in self.records:
            if r.task is None or self.t_origin is None:
                continue
            t0 = self.t_origin.elapsed_time(r.start)
            t1 = self.t_origin.elapsed_time(r.end)
            a = out.get(r.task)
            d = r.start.elapsed_time(r.end)
            out[r.task] = (t0, t1, d) if a is None else (min(a[0], t0), max(a[1], t1), a[2] + d)
        return out

    def linear_fwd(self, y, x, w, bias, act, residual=None, pre=None):
        self._timed("fwd", x.shape[0], w.shape[0], x.shape[1],
                    lambda: super(TimedBackend, self).linear_fwd(y, x, w, bias, act, residual, pre))

    def linear_dgrad(self, dx, dy, w, saved, act):
        self._timed("dgrad", dy.shape[0], w.shape[1], dy.shape[1],
                    lambda: super(TimedBackend, self).linear_dgrad(dx, dy, w, saved, act))

    def linear_wgrad(self, dw, db, dy, x, accumulate):
        self._timed("wgrad", dy.shape[1], x.shape[1], dy.shape[0],
                    lambda: super(TimedBackend, self).linear_wgrad(dw, None, dy, x, accumulate))
        if db is not None:
            self.colsum(db, dy, accumulate)

    def linear_wgrad_sgd(self, master, shadow, grad, dy, x, lr, accumulate, store_grad, dbias=None):
        # the bias column sum is its own kernel (the GEMM-fused variant is off by default):
        # timed apart so the GEMM family's roofline sees only the GEMM
        self._timed("wgrad", dy.shape[1], x.shape[1], dy.shape[0],
                    lambda: super(TimedBackend, self).linear_wgrad_sgd(master, shadow, grad, dy, x, lr,
                                                                       accumulate, store_grad, None))
        if dbias is not None:
            self.colsum(dbias, dy, accumulate)

    def time_gemms_alone(self, run_iteration, reps: int = 3) -> dict:
        """Record one iteration's dense GEMM launches (kind, FLOPs, closure), capture them
        back to back in one CUDA graph and time its replay with two events: the average
        GEMM launch duration without any per-launch event node (those add ~2-4 us each).
        The replays repeat the fused-SGD updates (benchmark-only side effect)."""
        self.gemm_calls = []
        try:
            run_iteration()
        finally:
            calls, self.gemm_calls = self.gemm_calls, None
        torch.cuda.synchronize()
        if not calls:
            return {"launches": 0, "flops": 0.0, "ms": 0.0, "tflops": 0.0}
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                for _, _, fn in calls:
                    fn()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            g.replay()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        fl = sum(f for _, f, _ in calls)
        by_kind = {}
        for kd, f, _ in calls:
            a = by_kind.setdefault(kd, [0, 0.0])
            a[0] += 1
            a[1] += f
        return {"launches": len(calls), "flops": fl, "ms": ms, "tflops": fl / (ms * 1e-3) / 1e12 if ms > 0 else 0.0,
                "by_kind_launches": {k: v[0] for k, v in by_kind.items()}}

    @staticmethod
    def preload(host_seconds: float, sm_hz: float = 1.965e9) -> None:
        """Queue a GPU sleep longer than the host's enqueue time of what follows, so the
        following launches run back to back and each event pair brackets only its kernel
        (otherwise a host slower than the GPU stretches every measured duration)."""
        torch.cuda._sleep(int(max(host_seconds, 1e-3) * 1.5 * sm_hz))

    def summary(self) -> dict:
        """GEMM FLOPs / device time (dense-operator GEMMs) and the total kernel time of
        every recorded call (``busy_ms``); synchronises first."""
        torch.cuda.synchronize()
        tot_f = tot_ms = busy = 0.0
        by_kind: dict[str, list[float]] = {}
        by_shape: dict[tuple, list[float]] = {}
        other: dict[str, list[float]] = {}
        for r in self.records:
            ms = r.start.elapsed_time(r.end)
            busy += ms
            if r.kind not in GEMM_KINDS:
                o = other.setdefault(r.kind, [0.0, 0])
                o[0] += ms
                o[1] += 1
                continue
            tot_f += r.flops
            tot_ms += ms
            agg = by_kind.setdefault(r.kind, [0.0, 0.0, 0])
            agg[0] += r.flops
            agg[1] += ms
            agg[2] += 1
            sh = by_shape.setdefault((r.kind, r.m, r.n, r.k), [0.0, 0.0, 0])
            sh[0] += r.flops
            sh[1] += ms
            sh[2] += 1
        return {
            "launches": sum(v[2] for v in by_kind.values()),
            "flops": tot_f,
            "ms": tot_ms,
            "busy_ms": busy,
            "tflops": (tot_f / (tot_ms * 1e-3) / 1e12) if tot_ms > 0 else 0.0,
            "by_kind": {k: {"launches": v[2], "tflops": v[0] / (v[1] * 1e-3) / 1e12 if v[1] else 0.0,
                            "ms": v[1]} for k, v in by_kind.items()},
            "other_ms": {k: {"launches": v[1], "ms": v[0]} for k, v in sorted(other.items())},
            "by_shape": {f"{k[0]}:{k[1]}x{k[2]}x{k[3]}": {"launches": v[2], "avg_us": 1e3 * v[1] / v[2],
                                                           "tflops": v[0] / (v[1] * 1e-3) / 1e12 if v[1] else 0.0}
                         for k, v in sorted(by_shape.items())},
        }

    def reset(self):
        self.records.clear()


# ---------------------------------------------------------------------------
# Measured cost curves: table CostCurves from B200 timings.
# ---------------------------------------------------------------------------


def _time_us(fn, reps: int) -> float:
    """Device time per call of ``fn``, replayed from a CUDA graph of ``reps`` calls: the
    executor replays captured iterations, so host launch overhead is not a task cost."""
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps


def profile_dense(din: int, dout: int, act: str, batches, device, dtype=torch.bfloat16, reps: int = 10,
                  has_dgrad: bool = True) -> dict:
    """fw and bw (dgrad + fused wgrad/SGD + bias colsum) milliseconds of Linear(din, dout)
    at each micro-batch size in ``batches``, through the production kernels."""
    be = CudaBackend(device)
    w = (torch.randn(dout, din, device=device) / din**0.5).to(dtype)
    master = torch.randn(dout, din, device=device) / din**0.5
    grad = torch.zeros(dout, din, device=device)
    bias = torch.zeros(dout, device=device)
    gb = torch.zeros(dout, device=device)
    out = {"b": [], "fwd_ms": [], "bwd_ms": []}
    for b in batches:
        x = torch.randn(b, din, device=device).to(dtype)
        y = torch.empty(b, dout, device=device, dtype=dtype)
        dz = torch.randn(b, dout, device=device).to(dtype)
        dx = torch.empty(b, din, device=device, dtype=dtype)
        f = _time_us(lambda: be.linear_fwd(y, x, w, bias, act), reps)

        def bw():
            if has_dgrad:
                be.linear_dgrad(dx, dz, w, x, act)
            if dtype == torch.bfloat16:
                be.linear_wgrad_sgd(master, w, grad, dz, x, 0.0, False, False, dbias=gb)
            else:
                be.linear_wgrad(grad, gb, dz, x, False)

        bwt = _time_us(bw, reps)
        out["b"].append(int(b))
        out["fwd_ms"].append(f / 1e3)
        out["bwd_ms"].append(bwt / 1e3)
    return out


class _LayerHost:
    """The Executor attributes an ``MMTLayer`` reads, for profiling one layer alone
    (single stage, no DP: the fused wgrad+SGD production path, one ring slot)."""

    def __init__(self, be, m: int, spec, device):
        from .mmt import mmt_params

        self.be, self.m, self.dev = be, m, device
        self.dtype, self.ell = torch.bfloat16, 1
        self.fuse, self.lr, self.keep_grads, self.d, self.tp = True, 0.0, False, 1, None
        self._ar_handles = []
        params = mmt_params(spec, 0, 0)
        self.P = {(0, n): t.to(device) for n, t in params}
        self.G = {(0, n): torch.zeros_like(t, device=device) for n, t in params}
        self.W = {(0, n): t.to(device, torch.bfloat16) for n, t in params}
        self.shadow = True

    def _ring(self, shape, dtype=None):
        return [torch.zeros(shape, dtype=dtype or self.dtype, device=self.dev)]


def profile_mmt_layer(S: int, d: int, H: int, ffn: int, pool: bool, batches, device, reps: int = 5) -> dict:
    """fw and bw milliseconds of one MMT encoder layer (runtime.mmt.MMTLayer, the production
    kernels) at each per-device micro-batch size in ``batches`` (samples of S tokens)."""
    from ..workloads import LayerSpec
    from .mmt import MMTLayer

    be = CudaBackend(device)
    spec = LayerSpec("mmt_layer", S * d, d if pool else S * d, extra=(S, d, H, ffn, pool))
    out = {"b": [], "fwd_ms": [], "bwd_ms": []}
    for b in batches:
        host = _LayerHost(be, b, spec, device)
        layer = MMTLayer(host, 0, spec)
        x = torch.randn(b * S, d, device=device).to(torch.bfloat16)
        y = torch.empty(b, spec.out_dim, device=device, dtype=torch.bfloat16)
        dz = (0.01 * torch.randn(b, spec.out_dim, device=device)).to(torch.bfloat16)
        dx = torch.empty(b * S, d, device=device, dtype=torch.bfloat16)
        f = _time_us(lambda: layer.forward(x, y, 0), reps)
        layer.forward(x, y, 0)
        bwt = _time_us(lambda: layer.backward(dz, x, dx, 0, False, True), reps)
        out["b"].append(int(b))
        out["fwd_ms"].append(f / 1e3)
        out["bwd_ms"].append(bwt / 1e3)
        del layer, host
        torch.cuda.empty_cache()
    return out
