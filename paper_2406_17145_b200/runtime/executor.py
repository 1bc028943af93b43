"""GPP stage executor: runs a configured StageGraph for real, one process per GPU.

This is the hot path the reference delegates to FlexFlow (
out of scope in SPEC.md:8).  Its contract is the simulator's semantics
(``sim.simulate``):

* rank r runs the stage S with r in S.devices; inside a DP stage of degree d,
  DP index q owns rows [q*b/d, (q+1)*b/d) of every micro-batch (cost.py:61);
* the stage executes its task list Pi strictly in order;
* fw(y, j) consumes every predecessor's outputs covering samples
  [j*b_y, (j+1)*b_y); bw(x, j) every successor's gradients covering x's range
  — realised as *pieces*: intersections of producer (task, rank) row ranges
  with consumer (task, rank) row ranges, each moved by one P2P message;
* activations live in rings of l = peak-in-flight slots indexed j mod l
  (kFkB never holds more than l micro-batches);
* after the last task, DP stages all-reduce their flat gradient buffer once
  (NCCL), then one fused SGD kernel updates master weights + bf16 shadows.

Transport: ``torch.distributed`` P2P (NCCL over NVLink on B200) with one
process group per ordered rank pair and direction, so forward and backward
streams never serialise against each other; pieces on a pair are posted in
global sample order on both sides, which is what makes NCCL's in-order
matching correct.  Compute: every kernel goes through the ``backend`` (the
sm_100a C-ABI library in production).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from ..model import Stage, StageGraph
from ..workloads import LayerSpec, Workload

__all__ = ["Piece", "build_pieces", "Executor", "init_params"]

_ALIGN = 64  # elements; keeps every parameter view 128-byte aligned (TMA needs 16 B)


@dataclass(frozen=True)
class Piece:
    tensor: int          # producer op id
    producer: int        # rank
    consumer: int        # rank
    p_task: int
    c_task: int
    p_row0: int          # row offset inside the producer's rank-local micro-batch block
    c_row0: int          # row offset inside the consumer's rank-local micro-batch block
    rows: int
    start: int           # global sample index of the first row (ordering key)


class _OrderedSends:
    """Posts a task's outgoing pieces as soon as their tensors are final, keeping each
    peer's posting order equal to the list order the peer posts its receives in."""

    def __init__(self, pieces, peer_of):
        self.pieces = list(pieces)
        self.posted = [False] * len(self.pieces)
        self.ready: set[int] = set()
        self.peer_of = peer_of

    def mark(self, tensor: int) -> None:
        self.ready.add(tensor)

    def flush(self, post_many, everything: bool = False) -> list:
        """Post every piece that is ready and not held back by an earlier piece to the same
        peer, as ONE grouped transfer (``post_many(pieces) -> works``)."""
        todo, blocked = [], set()
        for i, pc in enumerate(self.pieces):
            if self.posted[i]:
                continue
            peer = self.peer_of(pc)
            if peer in blocked:
                continue
            if everything or pc.tensor in self.ready:
                todo.append(pc)
                self.posted[i] = True
            else:
                blocked.add(peer)
        return post_many(todo) if todo else []


def _rank_rows(st: Stage, rank: int) -> tuple[int, int]:
    devs = sorted(st.devices)
    q = devs.index(rank)
    m = st.micro_batch // len(devs)
    return q * m, m


def build_pieces(prod: Stage, cons: Stage, tensors: list[int], B: int) -> list[Piece]:
    """All (producer task, rank) x (consumer task, rank) row-range intersections."""
    out: list[Piece] = []
    bp, bc = prod.micro_batch, cons.micro_batch
    for p in sorted(prod.devices):
        p_off, mp = _rank_rows(prod, p)
        for c in sorted(cons.devices):
            c_off, mc = _rank_rows(cons, c)
            for i in range(B // bp):
                lo_p = i * bp + p_off
                hi_p = lo_p + mp
                for j in range(lo_p // bc, (hi_p - 1) // bc + 1):
                    lo_c = j * bc + c_off
                    hi_c = lo_c + mc
                    s, e = max(lo_p, lo_c), min(hi_p, hi_c)
                    if s >= e:
                        continue
                    for t in tensors:
                        out.append(Piece(t, p, c, i, j, s - lo_p, s - lo_c, e - s, s))
    return out


def _order(pieces):
    return sorted(pieces, key=lambda pc: (pc.start, pc.tensor))


def init_params(spec: LayerSpec, op_id: int, seed: int) -> list[tuple[str, torch.Tensor]]:
    """Deterministic fp32 parameters of one op (CPU generator per (seed, op))."""
    g = torch.Generator().manual_seed(seed * 1_000_003 + op_id * 7919 + 17)
    if spec.kind == "dense" or spec.kind == "ce_head":
        w = torch.randn(spec.out_dim, spec.in_dim, generator=g) / spec.in_dim**0.5
        b = torch.randn(spec.out_dim, generator=g) * 0.01
        return [("w", w), ("b", b)]
    if spec.kind in ("mse_head", "bce_head"):
        w = torch.randn(spec.in_dim, generator=g) / spec.in_dim**0.5
        b = torch.randn(1, generator=g) * 0.01
        return [("w", w), ("b", b)]
    if spec.kind == "embbag":
        return [("table", torch.randn(spec.in_dim, spec.out_dim, generator=g) * 0.05)]
    if spec.kind == "mmt_layer":
        from .mmt import mmt_params
        return mmt_params(spec, op_id, seed)
    return []


def init_table(spec: LayerSpec, op_id: int, seed: int, device) -> torch.Tensor:
    """Embedding table: CPU-identical init when small (oracle-checkable), device RNG when big."""
    if spec.in_dim * spec.out_dim <= (1 << 22):
        return init_params(spec, op_id, seed)[0][1].to(device)
    g = torch.Generator(device=device).manual_seed(seed * 1_000_003 + op_id * 7919 + 17)
    return torch.randn(spec.in_dim, spec.out_dim, generator=g, device=device) * 0.05


def _width(spec: LayerSpec) -> int:
    return spec.out_dim


class Executor:
    """One rank's share of a GPP strategy."""

    def __init__(self, wl: Workload, sg: StageGraph, rank: int, world: int, backend,
                 lr: float = 1e-3, seed: int = 0, use_dist: bool | None = None,
                 fuse_optimizer: bool = True, keep_grads: bool = False, transport: str = "auto"):
        self.wl, self.sg, self.rank, self.world, self.be = wl, sg, rank, world, backend
        self.lr = float(lr)
        self.seed = seed
        self.B = sg.mini_batch
        self.dev = backend.device
        self.dtype = torch.float32 if wl.dtype == "fp32" else torch.bfloat16
        self.use_dist = (world > 1) if use_dist is None else use_dist
        self.keep_grads = keep_grads
        self._fuse_req = fuse_optimizer
        self._transport_kind = transport
        self.bias_queue: list = []  # (bias-gradient view, output gradient) of the running task
        import os

        # sparse table SGD: fp32-atomic scatter (default: at the HBM roofline, 1.9 ms per DLRM
        # step) or GPP_EMB_SGD=deterministic (bit-reproducible counting-sort kernel, 5.3 ms)
        self._emb_atomic = os.environ.get("GPP_EMB_SGD", "atomic") != "deterministic"
        # test hook: when a dict, every dense op's forward output is copied into it under
        # (op, task) -- the oracle takes the device's ReLU masks from these (tests only)
        self.tap: dict | None = None
        g = wl.graph
        self.owner = {op: st.id for st in sg.stages for op in st.op_ids}
        mine = [st for st in sg.stages if rank in st.devices]
        self.stage: Stage | None = mine[0] if mine else None
        self._make_groups()
        if self.stage is None:
            return
        st = self.stage
        self.d = st.dp_degree
        self.row_off, self.m = _rank_rows(st, rank)
        self.n = self.B // st.micro_batch
        # ring depth = peak in-flight micro-batches along Pi
        live = hi = 0
        for t in st.schedule:
            live += 1 if t.direction == "fw" else -1
            hi = max(hi, live)
        self.ell = max(1, hi)
        self.ops = [o for o in g.topo_order if o in st.op_ids]
        self.layers = {o: wl.layers[o] for o in self.ops}
        for o in self.ops:
            succ = g.successors(o)
            if len(succ) > 1:
                raise NotImplementedError(f"op {o} fans out to {len(succ)} consumers (unsupported)")
        # SGD fused into the last micro-batch's wgrad epilogue: only without data
        # parallelism (a DP stage must all-reduce its gradients first).
        self.fuse = self._fuse_req and self.d == 1 and hasattr(backend, "linear_wgrad_sgd")
        self._build_plan()
        self._alloc_params()
        self._alloc_buffers()

    # ------------------------------------------------------------------ plan
    def _make_groups(self):
        """Transport: one channel per ordered (src, dst) rank pair with traffic, one DP group per
        DP stage.  Every rank builds every channel in the same order (collective setup)."""
        self.tp = None
        self.dp_group = None
        if not self.use_dist:
            return
        pairs = set()
        for (a, b) in sorted(self.sg.edges):
            sa, sb = self.sg.by_id[a], self.sg.by_id[b]
            for p in sa.devices:
                for c in sb.devices:
                    pairs.add((p, c))
                    pairs.add((c, p))
        dp_groups = [tuple(sorted(st.devices)) for st in self.sg.stages if st.dp_degree > 1]
        kind = self._transport_kind
        if callable(kind):  # an injected transport (tests: host-staged gloo, ranks sharing a GPU)
            self.tp = kind(self.rank, pairs, dp_groups, self.dev)
            self.dp_group = getattr(self.tp, "dp", None)
            return
        if kind == "auto":
            kind = "nccl" if self.dev.type == "cuda" else "torch"
        if kind == "nccl":
            from .transport import NcclTransport
            self.tp = NcclTransport(self.rank, pairs, dp_groups, self.dev)
        else:
            from .transport import TorchTransport
            self.tp = TorchTransport(self.rank, pairs, dp_groups)
            self.dp_group = self.tp.dp

    def _build_plan(self):
        g = self.wl.graph
        st = self.stage
        mine = set(self.ops)
        # remote producers of local consumers / local producers with remote consumers
        self.in_remote: dict[int, int] = {}     # producer op -> producer stage id
        self.out_remote: dict[int, int] = {}    # local op -> consumer stage id
        for o in self.ops:
            for u in g.predecessors(o):
                if u not in mine:
                    self.in_remote[u] = self.owner[u]
            for v in g.successors(o):
                if v not in mine:
                    self.out_remote[o] = self.owner[v]
        self.recv_fw = {j: [] for j in range(self.n)}
        self.send_fw = {j: [] for j in range(self.n)}
        by_stage_in: dict[int, list[int]] = {}
        for u, sid in self.in_remote.items():
            by_stage_in.setdefault(sid, []).append(u)
        for sid, tensors in by_stage_in.items():
            for pc in build_pieces(self.sg.by_id[sid], st, sorted(tensors), self.B):
                if pc.consumer == self.rank:
                    self.recv_fw[pc.c_task].append(pc)
        by_stage_out: dict[int, list[int]] = {}
        for u, sid in self.out_remote.items():
            by_stage_out.setdefault(sid, []).append(u)
        for sid, tensors in by_stage_out.items():
            for pc in build_pieces(st, self.sg.by_id[sid], sorted(tensors), self.B):
                if pc.producer == self.rank:
                    self.send_fw[pc.p_task].append(pc)
        for j in range(self.n):
            self.recv_fw[j] = _order(self.recv_fw[j])
            self.send_fw[j] = _order(self.send_fw[j])
        # Stage edges that carry no operator data (e.g. the chain edges of a sequential
        # pipeline whose consecutive stages are independent branches) still order tasks in
        # the simulator's semantics (fw(y, j) waits for fw(x, i), bw(x, j) for bw(y, i),
        # SPEC.md:436-441): they are realised as 4-byte token messages, sent when the
        # producing task ends and waited for before the consuming task's first op.
        data_pairs = {(self.owner[u], self.owner[v]) for u, v in g.edges
                      if u in self.owner and v in self.owner and self.owner[u] != self.owner[v]}
        self.tok_in = {j: [] for j in range(self.n)}   # fw: wait at task start; bw: send at task end
        self.tok_out = {j: [] for j in range(self.n)}  # fw: send at task end; bw: wait at task start
        for (a, b) in sorted(self.sg.edges):
            if (a, b) in data_pairs or st.id not in (a, b):
                continue
            seen = set()
            for pc in build_pieces(self.sg.by_id[a], self.sg.by_id[b], [-1], self.B):
                key = (pc.producer, pc.consumer, pc.p_task, pc.c_task)
                if key in seen:
                    continue
                seen.add(key)
                if b == st.id and pc.consumer == self.rank:
                    self.tok_in[pc.c_task].append(pc)
                if a == st.id and pc.producer == self.rank:
                    self.tok_out[pc.p_task].append(pc)
        for j in range(self.n):
            self.tok_in[j] = _order(self.tok_in[j])
            self.tok_out[j] = _order(self.tok_out[j])
        self.first_bw = next(t.index for t in st.schedule if t.direction == "bw")
        dense = [o for o in self.ops if self.wl.layers[o].kind == "dense"]
        self._next_dense = {a: b for a, b in zip(dense, dense[1:])}
        self._prev_dense = {b: a for a, b in zip(dense, dense[1:])}
        self.last_bw = [t.index for t in st.schedule if t.direction == "bw"][-1]

    def eff_act(self, u: int) -> str:
        spec = self.wl.layers[u]
        if spec.kind == "dense":
            return spec.act
        if spec.kind == "concat":
            acts = {self.eff_act(p) for p in self.wl.graph.predecessors(u)}
            if len(acts) != 1:
                raise NotImplementedError("concat of inputs with different activations")
            return acts.pop()
        return "none"

    # ---------------------------------------------------------------- memory
    def _alloc_params(self):
        specs = []
        total = 0
        self.tables: dict[int, torch.Tensor] = {}
        for o in self.ops:
            if self.layers[o].kind == "embbag":  # big sparse tables live outside the flat buffers
                self.tables[o] = init_table(self.layers[o], o, self.seed, self.dev)
                continue
            for name, t in init_params(self.layers[o], o, self.seed):
                specs.append((o, name, t))
                total += -(-t.numel() // _ALIGN) * _ALIGN
        # dense weights first: with the fused optimizer they are updated by their wgrad
        # epilogues and the flat SGD kernel only walks the remainder [rest_off:]
        from .mmt import WEIGHTS as MMT_WEIGHTS
        fusable = lambda o, name: (self.layers[o].kind == "dense" and name == "w") or (
            self.layers[o].kind == "mmt_layer" and name in MMT_WEIGHTS)
        specs.sort(key=lambda t: 0 if fusable(t[0], t[1]) else 1)
        total = max(total, _ALIGN)
        self.master = torch.zeros(total, dtype=torch.float32, device=self.dev)
        self.grad = torch.zeros(total, dtype=torch.float32, device=self.dev)
        self.shadow = torch.zeros(total, dtype=torch.bfloat16, device=self.dev) if self.dtype == torch.bfloat16 else None
        self.P: dict[tuple[int, str], torch.Tensor] = {}     # fp32 master views
        self.G: dict[tuple[int, str], torch.Tensor] = {}     # fp32 grad views
        self.W: dict[tuple[int, str], torch.Tensor] = {}     # compute-dtype weight views
        off = 0
        self.rest_off = None
        for o, name, t in specs:
            if self.rest_off is None and not fusable(o, name):
                self.rest_off = off
            n = t.numel()
            self.master[off:off + n].copy_(t.reshape(-1))
            self.P[(o, name)] = self.master[off:off + n].view(t.shape)
            self.G[(o, name)] = self.grad[off:off + n].view(t.shape)
            if self.shadow is not None:
                self.W[(o, name)] = self.shadow[off:off + n].view(t.shape)
            else:
                self.W[(o, name)] = self.P[(o, name)]
            off += -(-n // _ALIGN) * _ALIGN
        if self.rest_off is None:
            self.rest_off = off
        if self.shadow is not None:
            self.shadow.copy_(self.master.to(torch.bfloat16))
        for o, t in self.tables.items():
            self.P[(o, "table")] = t
        self.param_count = sum(t.numel() for _, _, t in specs)

    def _ring(self, shape, dtype=None):
        return [torch.zeros(shape, dtype=dtype or self.dtype, device=self.dev) for _ in range(self.ell)]

    def _alloc_buffers(self):
        m, g = self.m, self.wl.graph
        self.out, self.recv, self.gbuf, self.grecv, self.gsend, self.pre = {}, {}, {}, {}, {}, {}
        self.pred, self.dpred = {}, {}
        self.emb_grad, self.zbuf, self.dzbuf = {}, {}, {}
        self.mmt = {}
        for o in self.ops:
            spec = self.layers[o]
            if spec.kind in ("dense", "concat"):
                self.out[o] = self._ring((m, _width(spec)))
                if self.eff_act(o) == "gelu":  # GELU' needs the pre-activation downstream
                    self.pre[o] = self._ring((m, _width(spec)))
                if o in self.out_remote:
                    self.grecv[o] = self._ring((m, _width(spec)))
                elif g.successors(o):
                    self.gbuf[o] = self._ring((m, _width(spec)))
            elif spec.kind in ("mse_head", "bce_head"):
                self.pred[o] = self._ring((m,), torch.float32)
                self.dpred[o] = self._ring((m,), torch.float32)
            elif spec.kind == "ce_head":
                self.pred[o] = self._ring((m, spec.out_dim))
                self.dpred[o] = self._ring((m, spec.out_dim))
            elif spec.kind == "embbag":
                self.out[o] = self._ring((m, spec.out_dim))
                if o in self.out_remote:
                    self.grecv[o] = self._ring((m, spec.out_dim))
                elif g.successors(o):
                    self.gbuf[o] = self._ring((m, spec.out_dim))
                # pooled-output gradients of the whole iteration -> one sparse SGD scatter
                self.emb_grad[o] = torch.zeros((self.n * m, spec.out_dim), dtype=self.dtype, device=self.dev)
            elif spec.kind == "mmt_layer":
                from .mmt import MMTLayer
                self.out[o] = self._ring((m, spec.out_dim))
                if o in self.out_remote:
                    self.grecv[o] = self._ring((m, spec.out_dim))
                elif g.successors(o):
                    self.gbuf[o] = self._ring((m, spec.out_dim))
                self.mmt[o] = MMTLayer(self, o, spec)
            elif spec.kind == "interaction":
                F = spec.in_dim
                self.out[o] = self._ring((m, spec.out_dim))
                self.zbuf[o] = self._ring((m, F * 64))
                self.dzbuf[o] = torch.zeros((m, F * 64), dtype=self.dtype, device=self.dev)
                if o in self.out_remote:
                    self.grecv[o] = self._ring((m, spec.out_dim))
                elif g.successors(o):
                    self.gbuf[o] = self._ring((m, spec.out_dim))
            else:
                raise NotImplementedError(f"layer kind {spec.kind}")
        for u in self.in_remote:
            w = _width(self.wl.layers[u])
            self.recv[u] = self._ring((m, w))
            self.gsend[u] = self._ring((m, w))
        self.loss_acc = torch.zeros(1, dtype=torch.float32, device=self.dev)
        self._send_works: dict[tuple, list] = {}
        # ordering tokens of data-less stage edges (content irrelevant)
        self.tok_tx = torch.zeros(1, dtype=torch.float32, device=self.dev)
        self.tok_rx = torch.zeros(1, dtype=torch.float32, device=self.dev)

    # ------------------------------------------------------------ data access
    def local_rows(self, key_tensor_full: torch.Tensor) -> torch.Tensor:
        """This rank's rows of a full [B, ...] batch tensor, in (task, row) order."""
        b = self.stage.micro_batch
        idx = torch.cat([torch.arange(j * b + self.row_off, j * b + self.row_off + self.m) for j in range(self.n)])
        return key_tensor_full.index_select(0, idx)

    def data_keys(self) -> list[str]:
        keys = []
        for o in self.ops:
            s = self.layers[o]
            for k in (s.data_key, s.label_key):
                if k is not None:
                    keys.append(k)
        return keys

    def _x_of(self, u: int, slot: int) -> torch.Tensor:
        return self.out[u][slot] if u in self.out else self.recv[u][slot]

    def _input(self, o: int, j: int, slot: int, batch) -> torch.Tensor:
        spec = self.layers[o]
        if spec.data_key is not None:
            return batch[spec.data_key][j * self.m:(j + 1) * self.m]
        preds = self.wl.graph.predecessors(o)
        if len(preds) != 1:
            raise NotImplementedError(f"op {o} ({spec.kind}) needs exactly one input")
        return self._x_of(preds[0], slot)

    def _saved_for(self, u: int, x: torch.Tensor, slot: int):
        """act'-saved tensor of producer u: its output for RELU, its pre-activation for GELU."""
        act = self.eff_act(u)
        if act == "gelu":
            if u not in self.pre:
                raise NotImplementedError(f"GELU pre-activation of op {u} is not on this stage")
            return self.pre[u][slot], act
        return x, act

    def _dx_target(self, u: int, slot: int) -> torch.Tensor:
        return self.gbuf[u][slot] if u in self.gbuf else self.gsend[u][slot]

    def _dz_of(self, o: int, slot: int) -> torch.Tensor:
        return self.grecv[o][slot] if o in self.grecv else self.gbuf[o][slot]

    # ------------------------------------------------------------- transport
    def _irecv_many(self, items):
        return self.tp.irecv_many(items) if items else []

    def _isend_many(self, items):
        return self.tp.isend_many(items) if items else []

    def _wait_sends(self, key):
        for w in self._send_works.pop(key, []):
            w.wait()

    # ---------------------------------------------------------------- tasks
    def _fw(self, j: int, batch):
        be, slot = self.be, j % self.ell
        # receives are posted up front but waited for only by the first op consuming them,
        # so ops fed locally (e.g. this stage's own towers) overlap the transfer
        pending: dict[int, list] = {}
        rws = self._irecv_many([(self.recv[pc.tensor][slot][pc.c_row0:pc.c_row0 + pc.rows], pc.producer)
                                  for pc in self.recv_fw[j]])
        for pc, w in zip(self.recv_fw[j], rws):
            pending.setdefault(pc.tensor, []).append(w)
        for w in self._irecv_many([(self.tok_rx, pc.producer) for pc in self.tok_in[j]]):
            w.wait()
        self._wait_sends(("fw", slot))
        sends = _OrderedSends(self.send_fw[j], lambda pc: pc.consumer)
        post = lambda pcs: self._isend_many([(self.out[pc.tensor][slot][pc.p_row0:pc.p_row0 + pc.rows],
                                                pc.consumer) for pc in pcs])
        works = []
        scale = 1.0 / self.B
        for o in self.ops:
            spec = self.layers[o]
            for u in self.wl.graph.predecessors(o):
                for w in pending.pop(u, ()):
                    w.wait()
            if spec.kind == "dense":
                x = self._input(o, j, slot, batch)
                pre = self.pre[o][slot] if o in self.pre else None
                be.linear_fwd(self.out[o][slot], x, self.W[(o, "w")], self.P[(o, "b")], spec.act, pre=pre)
                if self.tap is not None:
                    self.tap[(o, j)] = self.out[o][slot].detach().clone()
            elif spec.kind == "concat":
                off, dst, src, pdst, psrc = 0, [], [], [], []
                for u in self.wl.graph.predecessors(o):
                    w_u = _width(self.wl.layers[u])
                    dst.append(self.out[o][slot][:, off:off + w_u])
                    src.append(self._x_of(u, slot))
                    if o in self.pre:
                        if u not in self.pre:
                            raise NotImplementedError(f"GELU pre-activation of op {u} is not on this stage")
                        pdst.append(self.pre[o][slot][:, off:off + w_u])
                        psrc.append(self.pre[u][slot])
                    off += w_u
                be.copy_rows_multi(dst, src)
                be.copy_rows_multi(pdst, psrc)
            elif spec.kind in ("mse_head", "bce_head"):
                x = self._input(o, j, slot, batch)
                y = batch[spec.label_key][j * self.m:(j + 1) * self.m]
                # head GEMV + loss + dLoss in one kernel
                be.rowdot_loss(self.pred[o][slot], self.dpred[o][slot], self.loss_acc, x, self.P[(o, "w")],
                               self.P[(o, "b")], y, "mse" if spec.kind == "mse_head" else "bce", scale)
            elif spec.kind == "mmt_layer":
                x = self._input(o, j, slot, batch)
                lay = self.mmt[o]
                lay.forward(x.reshape(lay.T, lay.d), self.out[o][slot], slot)
            elif spec.kind == "embbag":
                idx = batch[spec.data_key][j * self.m:(j + 1) * self.m]
                be.embbag_fwd(self.out[o][slot], self.tables[o], idx)
            elif spec.kind == "interaction":
                us = self.wl.graph.predecessors(o)
                be.copy_rows_multi([self.zbuf[o][slot][:, 64 * i:64 * (i + 1)] for i in range(len(us))],
                                   [self._x_of(u, slot) for u in us])
                be.interaction_fwd(self.out[o][slot], self.zbuf[o][slot], spec.in_dim, spec.out_dim)
            elif spec.kind == "ce_head":
                x = self._input(o, j, slot, batch)
                be.linear_fwd(self.pred[o][slot], x, self.W[(o, "w")], self.P[(o, "b")], "none")
                lab = batch[spec.label_key][j * self.m:(j + 1) * self.m]
                be.ce_loss(self.loss_acc, self.dpred[o][slot], self.pred[o][slot], lab, scale)
            sends.mark(o)  # o's output is final: ship its pieces now (cheap embedding bags
            if spec.kind != "embbag":  # batch up into one grouped transfer)
                works += sends.flush(post)
        for ws in pending.values():
            for w in ws:
                w.wait()
        works += sends.flush(post, everything=True)
        works += self._isend_many([(self.tok_tx, pc.consumer) for pc in self.tok_out[j]])
        if works:
            self._send_works[("fw", slot)] = works

    def _bw(self, j: int, batch, accumulate: bool):
        be, slot = self.be, j % self.ell
        pending: dict[int, list] = {}
        # grads come back along the forward pieces of task j
        rws = self._irecv_many([(self.grecv[pc.tensor][slot][pc.p_row0:pc.p_row0 + pc.rows], pc.consumer)
                                  for pc in self.send_fw[j]])
        for pc, w in zip(self.send_fw[j], rws):
            pending.setdefault(pc.tensor, []).append(w)
        for w in self._irecv_many([(self.tok_rx, pc.consumer) for pc in self.tok_out[j]]):
            w.wait()
        self._wait_sends(("bw", slot))
        # input gradients go back along task j's forward pieces as soon as they are final
        sends = _OrderedSends(self.recv_fw[j], lambda pc: pc.producer)
        post = lambda pcs: self._isend_many([(self.gsend[pc.tensor][slot][pc.c_row0:pc.c_row0 + pc.rows],
                                                pc.producer) for pc in pcs])
        works = []
        emb_dst, emb_src = [], []
        g = self.wl.graph
        for o in reversed(self.ops):
            spec = self.layers[o]
            preds = g.predecessors(o)
            for w in pending.pop(o, ()):
                w.wait()
            needs_dx = spec.data_key is None and len(preds) == 1
            if spec.kind == "dense":
                x = self._input(o, j, slot, batch)
                dz = self._dz_of(o, slot)
                # dgrad first: the fused update below rewrites the weights it reads
                if needs_dx:
                    u = preds[0]
                    saved, act = self._saved_for(u, x, slot)
                    be.linear_dgrad(self._dx_target(u, slot), dz, self.W[(o, "w")], saved, act)

                self.bias_queue.append((self.G[(o, "b")], dz))  # bias grads: one launch per task
                if self.d > 1 and j == self.last_bw:
                    # DP stage: this weight's gradient is final -> overlap its all-reduce
                    # with the rest of the backward pass (bucket = one layer's weight)
                    be.linear_wgrad(self.G[(o, "w")], None, dz, x, accumulate)
                    self._ar_handles.append(self.tp.allreduce_async(self.G[(o, "w")]))
                elif self.fuse and j == self.last_bw:
                    # weight gradient + SGD in one epilogue, the bias gradient summed in the same
                    # kernel (applied by the flat SGD later)
                    be.linear_wgrad_sgd(self.P[(o, "w")], self.W[(o, "w")] if self.shadow is not None else None,
                                        self.G[(o, "w")], dz, x, self.lr, accumulate, self.keep_grads)
                else:
                    be.linear_wgrad(self.G[(o, "w")], None, dz, x, accumulate)
            elif spec.kind == "mmt_layer":
                lay = self.mmt[o]
                x = self._input(o, j, slot, batch)
                dx = self._dx_target(preds[0], slot).reshape(lay.T, lay.d) if needs_dx else None
                lay.backward(self._dz_of(o, slot), x.reshape(lay.T, lay.d), dx, slot, accumulate,
                             j == self.last_bw)
            elif spec.kind == "embbag":  # gathered: one launch for all tables after the loop
                emb_dst.append(self.emb_grad[o][j * self.m:(j + 1) * self.m])
                emb_src.append(self._dz_of(o, slot))
            elif spec.kind == "interaction":
                us = list(preds)
                first_act = self.eff_act(us[0])
                if first_act not in ("none", "relu") or any(self.eff_act(u) != "none" for u in us[1:]):
                    raise NotImplementedError("interaction inputs: ReLU/none first feature, linear others")
                be.interaction_bwd(self.dzbuf[o], self._dz_of(o, slot), self.zbuf[o][slot], spec.in_dim,
                                   first_act == "relu")
                be.copy_rows_multi([self._dx_target(u, slot) for u in us],
                                   [self.dzbuf[o][:, 64 * i:64 * (i + 1)] for i in range(len(us))])
            elif spec.kind == "concat":
                dz = self._dz_of(o, slot)
                off, dst, src = 0, [], []
                for u in preds:
                    w_u = _width(self.wl.layers[u])
                    dst.append(self._dx_target(u, slot))
                    src.append(dz[:, off:off + w_u])
                    off += w_u
                be.copy_rows_multi(dst, src)
            elif spec.kind in ("mse_head", "bce_head"):
                x = self._input(o, j, slot, batch)
                u = preds[0] if needs_dx else None
                dx = self._dx_target(u, slot) if needs_dx else None
                saved, act = self._saved_for(u, x, slot) if needs_dx else (None, "none")
                be.rowdot_bwd(dx, self.G[(o, "w")], self.G[(o, "b")], self.dpred[o][slot], x,
                              self.P[(o, "w")], saved, act, accumulate)
            elif spec.kind == "ce_head":
                x = self._input(o, j, slot, batch)
                dl = self.dpred[o][slot]
                be.linear_wgrad(self.G[(o, "w")], None, dl, x, accumulate)
                self.bias_queue.append((self.G[(o, "b")], dl))
                if needs_dx:
                    u = preds[0]
                    saved, act = self._saved_for(u, x, slot)
                    be.linear_dgrad(self._dx_target(u, slot), dl, self.W[(o, "w")], saved, act)
            marked = False
            for u in preds:
                if u in self.gsend:
                    sends.mark(u)
                    marked = True
            if marked:
                works += sends.flush(post)
        be.copy_rows_multi(emb_dst, emb_src)  # embedding-bag output grads -> the SGD scatter's rows
        self._flush_bias(accumulate)
        for ws in pending.values():
            for w in ws:
                w.wait()
        works += sends.flush(post, everything=True)
        works += self._isend_many([(self.tok_tx, pc.producer) for pc in self.tok_in[j]])
        if works:
            self._send_works[("bw", slot)] = works

    def _flush_bias(self, accumulate: bool) -> None:
        """The task's queued bias gradients (column sums of each layer's output gradient) in
        as few launches as possible (per dtype), before the next task reuses the rings."""
        if not self.bias_queue:
            return
        by_dt: dict = {}
        for out, dz in self.bias_queue:
            by_dt.setdefault(dz.dtype, ([], []))
            by_dt[dz.dtype][0].append(out)
            by_dt[dz.dtype][1].append(dz)
        for outs, xs in by_dt.values():
            self.be.colsum_multi(outs, xs, accumulate)
        self.bias_queue = []

    # ------------------------------------------------------------ iteration
    def run_iteration(self, batch: dict[str, torch.Tensor], step_optimizer: bool = True):
        """One synchronous training iteration (all tasks of Pi, DP all-reduce, SGD).

        ``batch`` maps data keys to this rank's rows ([B/d, ...] on the device).
        Returns the device loss accumulator (head stages) or None.
        """
        if self.stage is None:
            return None
        self.loss_acc.zero_()
        self._ar_handles = []
        seen_bw = False
        # Sparse table updates (non-DP stages): a micro-batch's rows may be written only once
        # no forward of this iteration will read the table again, i.e. after the stage's
        # last fw -- from then on each finished bw's scatter overlaps the cool-down instead
        # of all of them piling up after the last task (exact: the same per-row sums).
        eager_sparse = step_optimizer and bool(self.tables) and self.d == 1
        fw_left = sum(1 for t in self.stage.schedule if t.direction == "fw")
        bw_done: list[int] = []
        mark = getattr(self.be, "set_task", None)  # measured task trace (runtime/trace.py)
        sid = self.stage.id
        if mark:
            mark(("iteration",))
        for t in self.stage.schedule:
            if mark:
                mark((sid, t.direction, t.index))
            if t.direction == "fw":
                self._fw(t.index, batch)
                fw_left -= 1
            else:
                self._bw(t.index, batch, accumulate=seen_bw)
                seen_bw = True
                bw_done.append(t.index)
            if eager_sparse and fw_left == 0:
                for j in bw_done:
                    self._sparse_update(batch, j)
                bw_done = []
        if mark:
            mark((sid, "opt", 0))
        for key in list(self._send_works):
            self._wait_sends(key)
        if self.d > 1:
            # the non-weight remainder (biases, heads) in one bucket, then join the DP stream
            if self.rest_off < self.grad.numel():
                self._ar_handles.append(self.tp.allreduce_async(self.grad[self.rest_off:]))
            self.tp.join(self._ar_handles)
            self._ar_handles = []
        if step_optimizer:
            jobs = []
            for o, table in self.tables.items() if not eager_sparse else ():
                idx = batch[self.layers[o].data_key]
                g_o = self.emb_grad[o]
                if self.d > 1:  # every replica applies every replica's sparse updates
                    gi = torch.empty((self.d * idx.shape[0], idx.shape[1]), dtype=idx.dtype, device=idx.device)
                    gg = torch.empty((self.d * g_o.shape[0], g_o.shape[1]), dtype=g_o.dtype, device=g_o.device)
                    self.tp.allgather(gi, idx.contiguous())
                    self.tp.allgather(gg, g_o)
                    idx, g_o = gi, gg
                jobs.append((table, g_o, idx))
            self._apply_sparse(jobs)
            if self.fuse:
                if self.rest_off < self.master.numel():
                    sh = self.shadow[self.rest_off:] if self.shadow is not None else None
                    self.be.sgd_step(self.master[self.rest_off:], sh, self.grad[self.rest_off:], self.lr)
            else:
                self.be.sgd_step(self.master, self.shadow, self.grad, self.lr)
        if mark:
            mark(None)
        return self.loss_acc

    def _sparse_update(self, batch, j: int) -> None:
        """Embedding-bag SGD for micro-batch j's rows of every table on this stage."""
        rows = slice(j * self.m, (j + 1) * self.m)
        self._apply_sparse([(table, self.emb_grad[o][rows], batch[self.layers[o].data_key][rows])
                            for o, table in self.tables.items()])

    def _apply_sparse(self, jobs) -> None:
        """Sparse SGD of several tables: the per-table fp32-atomic scatter (default), or with
        GPP_EMB_SGD=deterministic the multi-table kernel (counting sort by row, each row's sum
        in (sample, bag) order, bit-reproducible) in one call per 32 tables."""
        if not jobs:
            return
        if self._emb_atomic or not hasattr(self.be, "embbag_sgd_multi"):
            for table, g, idx in jobs:
                self.be.embbag_sgd(table, g, idx, self.lr)
            return
        for i in range(0, len(jobs), 32):
            ch = jobs[i:i + 32]
            self.be.embbag_sgd_multi([t for t, _, _ in ch], [g for _, g, _ in ch], [x for _, _, x in ch], self.lr)

    def stage_loss(self, loss: torch.Tensor) -> float:
        """Loss of the whole mini-batch on a head rank (sums the DP replicas' shares)."""
        l = loss.clone()
        if self.d > 1:
            self.tp.allreduce(l)
        return float(l.item())

    @property
    def is_head(self) -> bool:
        return self.stage is not None and any(self.layers[o].kind.endswith("_head") for o in self.ops)
