"""Stage-edge transport: P2P pieces between ranks and the DP all-reduce.

``NcclTransport`` (product, GPU): NCCL communicators created and driven through
libgpp_b200.so, one per ordered rank pair (forward and backward traffic on separate
communicators and streams, so they never serialise), one per DP stage.  Every
transfer forks a dedicated stream off the compute stream with an event and joins
back with another, so a whole rank iteration is capturable into a CUDA graph.

``TorchTransport`` (CPU tests): the same interface over ``torch.distributed``
(gloo), used to check the executor's host logic without GPUs.
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist


class _Done:
    __slots__ = ("ev",)

    def __init__(self, ev):
        self.ev = ev

    def wait(self):
        torch.cuda.current_stream().wait_event(self.ev)


class TorchTransport:
    name = "torch.distributed"

    def __init__(self, rank: int, pairs, dp_groups):
        self.rank = rank
        self.p2p = {}
        for (a, b) in sorted(pairs):
            self.p2p[(a, b)] = dist.new_group(ranks=sorted({a, b}))
        self.dp = None
        for devs in dp_groups:
            g = dist.new_group(ranks=sorted(devs))
            if rank in devs:
                self.dp = g

    def irecv(self, buf, src):
        return dist.irecv(buf, src=src, group=self.p2p[(src, self.rank)])

    def isend(self, buf, dst):
        return dist.isend(buf, dst=dst, group=self.p2p[(self.rank, dst)])

    def irecv_many(self, items):
        return [self.irecv(b, src) for b, src in items]

    def isend_many(self, items):
        return [self.isend(b, dst) for b, dst in items]

    def allreduce(self, t):
        dist.all_reduce(t, group=self.dp)

    def allreduce_async(self, t):
        dist.all_reduce(t, group=self.dp)
        return None

    def allgather(self, out, t):
        dist.all_gather_into_tensor(out, t, group=self.dp)

    def join(self, handles):
        pass


class NcclTransport:
    name = "nccl (libgpp_b200)"

    def __init__(self, rank: int, pairs, dp_groups, device: torch.device):
        from . import lib

        L = lib.load()
        if not L.gpp_nccl_available():
            raise RuntimeError("libnccl.so.2 not loadable by libgpp_b200")
        self.rank, self.device = rank, device
        specs = [("p2p", (a, b)) for (a, b) in sorted(pairs)] + [("dp", tuple(sorted(d))) for d in dp_groups]
        ids = None
        if rank == 0:
            ids = []
            for _ in specs:
                buf = ctypes.create_string_buffer(128)
                lib.call("gpp_nccl_unique_id", ctypes.cast(buf, ctypes.c_void_p))
                ids.append(bytes(buf.raw))
        box = [ids]
        dist.broadcast_object_list(box, src=0)
        ids = box[0]
        mine = []
        for i, (kind, members) in enumerate(specs):
            mem = sorted(set(members))
            if rank in mem:
                mine.append((i, kind, members, len(mem), mem.index(rank)))
        n = len(mine)
        handles = (ctypes.c_void_p * max(1, n))()
        if n:
            id_blob = b"".join(ids[i] for i, *_ in mine)
            nr = (ctypes.c_int * n)(*[m[3] for m in mine])
            rk = (ctypes.c_int * n)(*[m[4] for m in mine])
            lib.call("gpp_comm_init_group", n, ctypes.c_char_p(id_blob), nr, rk, handles)
        self.comms = {}
        self.streams = {}
        self.dp_comm = None
        for j, (i, kind, members, _, _) in enumerate(mine):
            if kind == "p2p":
                self.comms[members] = handles[j]
                self.streams[members] = torch.cuda.Stream(device)
            else:
                self.dp_comm = handles[j]
        self._lib = lib
        self.dp_stream = None

    @staticmethod
    def _peer(a: int, b: int, other: int) -> int:
        return 0 if other == min(a, b) else 1

    def _fork(self, key):
        s = self.streams[key]
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        s.wait_event(ev)
        return s

    def irecv(self, buf, src):
        key = (src, self.rank)
        s = self._fork(key)
        self._lib.call("gpp_recv", self.comms[key], buf.data_ptr(), buf.numel() * buf.element_size(),
                       self._peer(*key, src), s.cuda_stream)
        done = torch.cuda.Event()
        done.record(s)
        return _Done(done)

    def isend(self, buf, dst):
        key = (self.rank, dst)
        s = self._fork(key)
        self._lib.call("gpp_send", self.comms[key], buf.data_ptr(), buf.numel() * buf.element_size(),
                       self._peer(*key, dst), s.cuda_stream)
        done = torch.cuda.Event()
        done.record(s)
        return _Done(done)

    def _many(self, items, send: bool):
        """Several transfers in ONE NCCL group: one fork per pair stream, one kernel per
        communicator -- DLRM ships 26 embedding pieces per task to the same peer."""
        if len(items) == 1:
            b, peer = items[0]
            return [self.isend(b, peer) if send else self.irecv(b, peer)]
        keys = [((self.rank, peer) if send else (peer, self.rank)) for _, peer in items]
        streams = {k: self._fork(k) for k in dict.fromkeys(keys)}
        fn = "gpp_send" if send else "gpp_recv"
        self._lib.call("gpp_group_start")
        try:
            for (b, peer), k in zip(items, keys):
                self._lib.call(fn, self.comms[k], b.data_ptr(), b.numel() * b.element_size(),
                               self._peer(*k, peer), streams[k].cuda_stream)
        finally:
            self._lib.call("gpp_group_end")
        done = {}
        for k, st in streams.items():
            done[k] = torch.cuda.Event()
            done[k].record(st)
        return [_Done(done[k]) for k in keys]

    def irecv_many(self, items):
        return self._many(items, send=False) if items else []

    def isend_many(self, items):
        return self._many(items, send=True) if items else []

    def allreduce(self, t):
        self._lib.call("gpp_allreduce_f32", self.dp_comm, t.data_ptr(), t.numel(),
                       torch.cuda.current_stream().cuda_stream)

    def allreduce_async(self, t):
        """Bucket all-reduce on the DP stream, forked off the compute stream now (the
        gradient is final), so it overlaps the rest of the backward pass."""
        if self.dp_stream is None:
            self.dp_stream = torch.cuda.Stream(self.device)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.dp_stream.wait_event(ev)
        self._lib.call("gpp_allreduce_f32", self.dp_comm, t.data_ptr(), t.numel(), self.dp_stream.cuda_stream)
        done = torch.cuda.Event()
        done.record(self.dp_stream)
        return _Done(done)

    def allgather(self, out, t):
        self._lib.call("gpp_allgather", self.dp_comm, t.data_ptr(), out.data_ptr(), t.numel() * t.element_size(),
                       torch.cuda.current_stream().cuda_stream)

    def join(self, handles):
        for h in handles:
            if h is not None:
                h.wait()
