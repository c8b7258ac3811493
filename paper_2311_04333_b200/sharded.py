"""Vertex-range-sharded exact coreness across GPUs.

The reference computes coreness on one shared-memory machine
(core.cpp:89-119).  Here the dense-id range is cut into P contiguous ranges
with balanced arc counts (split points on the degree prefix sum; RMAT puts
hubs at low ids); shard r keeps the residual degrees and labels of its range.
Synchronous rounds stay bit-identical to the reference:

    round at bound b:
      every shard expands its frontier -> decrements of its own vertices in
      place (crossing b+1 -> b enrols them in the next frontier), decrements
      of remote vertices bucketed by owner;
      decrement all-to-all (counts, then ids) -> owners apply them with the
      same crossing rule;
      all-reduce(sum) of the next frontier sizes (one value per round);
    empty global frontier:
      all-reduce(min) of the min alive degree -> new bound (= label) ->
      every shard collects its alive vertices with degree <= bound.

peel_rounds counts non-empty global rounds; kmax = last label.  Labels are
all-gathered at the end.  The shard work runs in CUDA (`CudaShard`, the
`dg_shard_*` C ABI); the protocol only moves counts and id lists.  `Comm`
implementations: `TorchComm` (torch.distributed: NCCL on GPUs, gloo on CPU)
and `LocalComm` (all shards in one process -- used to validate the CUDA
shard kernels on a single GPU without ranks that wait on each other).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

import numpy as np

__all__ = ["partition", "TorchComm", "LocalComm", "CudaShard", "sharded_coreness",
           "coreness_local_shards", "coreness_distributed", "link", "link_local", "link_ipc"]


def partition(offs: np.ndarray, P: int) -> np.ndarray:
    """Split points b[0]=0 < ... < b[P]=n with ~equal arc counts per range."""
    offs = np.asarray(offs, dtype=np.uint64)
    n = len(offs) - 1
    total = int(offs[-1])
    targets = np.array([(total * r) // P for r in range(P + 1)], dtype=np.uint64)
    b = np.searchsorted(offs[:-1], targets, side="left").astype(np.uint64)
    b[0], b[-1] = 0, n
    return np.maximum.accumulate(np.minimum(b, n)).astype(np.uint64)


# ------------------------------------------------------------------ communicators
class TorchComm:
    """One shard per process over torch.distributed (NCCL: device tensors; gloo: CPU)."""

    def __init__(self, device):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.P = dist.get_world_size()
        self.rank = dist.get_rank()
        self.device = torch.device(device)

    def shards(self) -> List[int]:
        return [self.rank]

    def _scalar(self, x: int, op):
        t = self.torch.tensor([x], dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=op)
        return int(t.item())

    def allreduce_sum(self, x: int) -> int:
        return self._scalar(x, self.dist.ReduceOp.SUM)

    def allreduce_min(self, x: int) -> int:
        return self._scalar(x, self.dist.ReduceOp.MIN)

    def allreduce_max(self, x: int) -> int:
        return self._scalar(x, self.dist.ReduceOp.MAX)

    def allreduce_sum_tensor(self, t):
        t = t.clone()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t

    def allgather_counts(self, counts: Sequence[int]) -> List[int]:
        t = self.torch.tensor([int(counts[0])], dtype=self.torch.int64, device=self.device)
        out = [self.torch.empty_like(t) for _ in range(self.P)]
        self.dist.all_gather(out, t)
        return [int(x.item()) for x in out]

    def alltoall_counts(self, counts: Sequence[Sequence[int]]) -> List[List[int]]:
        t = self.torch.tensor(list(counts[0]), dtype=self.torch.int64, device=self.device)
        out = self.torch.empty_like(t)
        self.dist.all_to_all_single(out, t)
        return [out.tolist()]

    def alltoallv(self, sends, send_counts, recv_counts):
        out = self.torch.empty(sum(recv_counts[0]), dtype=sends[0].dtype, device=self.device)
        self.dist.all_to_all_single(out, sends[0], output_split_sizes=list(recv_counts[0]),
                                    input_split_sizes=list(send_counts[0]))
        if self.device.type == "cuda":
            self.torch.cuda.synchronize()
        return [out]

    def allgather(self, arr: np.ndarray) -> List[np.ndarray]:
        objs = [None] * self.P
        self.dist.all_gather_object(objs, arr)
        return objs

    def allgatherv(self, ts):
        """Variable-length all-gather of one tensor per local shard -> P tensors."""
        t = ts[0]
        sizes = self.allgather_counts([t.numel()])
        cap = max(sizes + [1])
        pad = self.torch.zeros(cap, dtype=t.dtype, device=self.device)
        pad[: t.numel()] = t
        out = [self.torch.empty_like(pad) for _ in range(self.P)]
        self.dist.all_gather(out, pad)
        return [o[:c] for o, c in zip(out, sizes)]


class LocalComm:
    """All P shards in this process (single-GPU validation of the shard kernels)."""

    def __init__(self, P: int, device="cuda"):
        import torch
        self.torch, self.P, self.device = torch, P, torch.device(device)

    def shards(self) -> List[int]:
        return list(range(self.P))

    def allreduce_sum(self, x: int) -> int:
        return x

    def allreduce_min(self, x: int) -> int:
        return x

    def allreduce_max(self, x: int) -> int:
        return x

    def allreduce_sum_tensor(self, t):
        return t.clone()

    def allgather_counts(self, counts: Sequence[int]) -> List[int]:
        return [int(c) for c in counts]

    def alltoall_counts(self, counts):
        return [[counts[s][d] for s in range(self.P)] for d in range(self.P)]

    def alltoallv(self, sends, send_counts, recv_counts):
        outs = []
        for d in range(self.P):
            parts = []
            for s in range(self.P):
                lo = sum(send_counts[s][:d])
                parts.append(sends[s][lo:lo + send_counts[s][d]])
            outs.append(self.torch.cat(parts) if parts else sends[0][:0])
        return outs

    def allgather(self, arrs):
        return arrs

    def allgatherv(self, ts):
        return list(ts)


# ------------------------------------------------------------------ CUDA shard engine
class CudaShard:
    """dg_shard_* over the C ABI; exchange buffers are torch CUDA tensors."""

    def __init__(self, g, bounds: np.ndarray, rank: int, rows=None):
        """Shard `rank` of `g` (its rows are copied: `g` may be freed), or --
        with g=None and rows=(n, offs, adj) -- from the rank's own rows only."""
        import torch
        from . import _chk
        from ._abi import LIB, u32p, u64p
        self.torch, self.LIB, self._chk, self.u32p, self.u64p = torch, LIB, _chk, u32p, u64p
        self.bounds = np.ascontiguousarray(bounds, dtype=np.uint64)
        self.P = len(self.bounds) - 1
        self.rank = rank
        self.lo, self.hi = int(self.bounds[rank]), int(self.bounds[rank + 1])
        h = C.c_void_p()
        if rows is None:
            _chk(LIB.dg_shard_create(g._h, self.bounds.ctypes.data_as(u64p), self.P, rank,
                                     C.byref(h)))
        else:
            n, offs, adj = rows
            if isinstance(offs, torch.Tensor) and offs.is_cuda:
                # device rows (sharded_build): int64 offsets, int32 holding uint32 ids
                offs = offs.to(torch.int64).contiguous()
                adj = adj.to(torch.int32).contiguous()
                torch.cuda.synchronize()  # produced on torch's stream, copied on the library's
                _chk(LIB.dg_shard_create_rows(n, self.bounds.ctypes.data_as(u64p), self.P, rank,
                                              C.cast(C.c_void_p(offs.data_ptr()), u64p),
                                              C.cast(C.c_void_p(adj.data_ptr()), u32p), 1,
                                              C.byref(h)))
                _chk(LIB.dg_synchronize())  # copies done before torch may reuse the memory
            else:
                offs = np.ascontiguousarray(np.asarray(offs), dtype=np.uint64)
                adj = np.ascontiguousarray(np.asarray(adj).astype(np.int64) & 0xFFFFFFFF,
                                           dtype=np.uint32)
                _chk(LIB.dg_shard_create_rows(n, self.bounds.ctypes.data_as(u64p), self.P, rank,
                                              offs.ctypes.data_as(u64p), adj.ctypes.data_as(u32p),
                                              0, C.byref(h)))
        self._h = h

    @classmethod
    def from_rows(cls, n: int, bounds, rank: int, offs, adj):
        """Rows [bounds[rank], bounds[rank+1]) only: offs has n_local + 1 entries."""
        return cls(None, bounds, rank, rows=(n, offs, adj))

    def __del__(self):
        if getattr(self, "_h", None):
            self.LIB.dg_shard_free(self._h)
            self._h = None

    @property
    def n_local(self) -> int:
        return self.hi - self.lo

    def min_alive(self) -> int:
        x = C.c_uint32()
        self._chk(self.LIB.dg_shard_min_alive(self._h, C.byref(x)))
        return x.value

    def collect(self, bound: int, label: int) -> int:
        x = C.c_uint64()
        self._chk(self.LIB.dg_shard_collect(self._h, bound, label, C.byref(x)))
        return x.value

    def count_remote(self) -> List[int]:
        c = np.zeros(self.P, np.uint64)
        self._chk(self.LIB.dg_shard_count_remote(self._h, c.ctypes.data_as(self.u64p)))
        return [int(x) for x in c]

    def expand(self, bound: int, label: int, counts: List[int]):
        displs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
        send = self.torch.empty(max(1, int(sum(counts))), dtype=self.torch.int32, device="cuda")
        # torch's allocator may hand out a block that pending work on torch's
        # stream still writes; the library writes it on its own stream
        self.torch.cuda.synchronize()
        self._chk(self.LIB.dg_shard_expand(self._h, bound, label,
                                           displs.ctypes.data_as(self.u64p),
                                           C.c_void_p(send.data_ptr())))
        return send[: int(sum(counts))]

    def apply(self, recv, bound: int, label: int) -> int:
        x = C.c_uint64()
        ptr = recv.data_ptr() if recv.numel() else 0
        self.torch.cuda.synchronize()  # recv comes from torch ops (LocalComm) or NCCL
        self._chk(self.LIB.dg_shard_apply(self._h, C.c_void_p(ptr), recv.numel(), bound, label,
                                          C.byref(x)))
        return x.value

    # -- peer mode (fused decrement exchange over peer memory, see dg_b200.h)
    def ipc_handle(self) -> bytes:
        buf = (C.c_ubyte * 64)()
        self._chk(self.LIB.dg_shard_ipc_handle(self._h, buf))
        return bytes(buf)

    def peer_open(self, rank: int, handle: bytes):
        buf = (C.c_ubyte * 64).from_buffer_copy(handle)
        self._chk(self.LIB.dg_shard_peer_open(self._h, rank, buf))

    def peer_link(self, rank: int, other: "CudaShard"):
        self._chk(self.LIB.dg_shard_peer_link(self._h, rank, other._h))

    def expand_peer(self, bound: int, label: int) -> int:
        x = C.c_uint64()
        self._chk(self.LIB.dg_shard_expand_peer(self._h, bound, label, C.byref(x)))
        return x.value

    def finish_round(self) -> int:
        x = C.c_uint64()
        self._chk(self.LIB.dg_shard_finish_round(self._h, C.byref(x)))
        return x.value

    def labels(self) -> np.ndarray:
        out = np.zeros(max(1, self.n_local), np.uint32)
        self._chk(self.LIB.dg_shard_labels(self._h, out.ctypes.data_as(self.u32p)))
        return out[: self.n_local]


# ------------------------------------------------------------------ protocol
UNSET = 0xFFFFFFFF


def link_local(shards: List):
    """Peer mode for shards of one process: map every shard's state into the others."""
    for s in shards:
        for r, o in enumerate(shards):
            if o is not s:
                s.peer_link(r, o)


def link_ipc(shard, comm):
    """Peer mode across processes: all-gather the CUDA IPC handles of the
    shards' state blocks and map the others' (NVLink peer memory)."""
    handles = comm.allgather(shard.ipc_handle())
    for r, h in enumerate(handles):
        if r != comm.rank:
            shard.peer_open(r, h)


def link(shards: List, comm):
    """Peer mode wiring for whichever communicator holds the shards."""
    if isinstance(comm, LocalComm):
        link_local(shards)
    else:
        for sh in shards:
            link_ipc(sh, comm)


def sharded_coreness(shards: List, comm, n_global: int, approx=None, peer: bool = False):
    """Coreness over the shards held by this process (core.cpp:89-119).

    approx=None is exact_coreness; approx=(c_num, c_den) is approx_coreness
    with geometric phases t_{i+1} = max(t_i + 1, ceil(c * t_i)).
    peer=True runs the fused rounds (dg_shard_expand_peer: decrements applied
    at the owners through peer memory, one all-reduce per round) on shards
    linked by link_local / link_ipc.
    Returns (labels of the local shards in order, kmax, peel_rounds).  Every
    rank executes the same control flow (all decisions come from collectives).
    """
    if approx is not None:
        c_num, c_den = approx
        if c_den == 0 or c_num <= c_den:
            raise ValueError("approx_coreness needs c > 1")
    remaining = comm.allreduce_sum(sum(s.n_local for s in shards))
    if remaining != n_global:
        raise ValueError("shards do not cover the graph")
    if n_global == 0:
        raise ValueError("coreness of empty graph")
    bound = label = 0
    t = 1
    kmax = rounds = 0
    nfront = [0] * len(shards)
    while remaining > 0:
        total = comm.allreduce_sum(sum(nfront))
        if total == 0:
            # every alive degree exceeds `bound` here; the reference's empty
            # drains (core.cpp:101-111) advance until bound >= min alive degree
            local_min = min([s.min_alive() for s in shards] + [UNSET])
            gmin = comm.allreduce_min(local_min)
            if gmin == UNSET:
                raise RuntimeError("frontier empty with vertices remaining")
            if approx is None:
                bound = label = max(bound, gmin)
            else:
                while bound < gmin:
                    label = t
                    nt = max(t + 1, -(-(t * c_num) // c_den))
                    bound, t = nt - 1, nt
            nfront = [s.collect(bound, label) for s in shards]
            total = comm.allreduce_sum(sum(nfront))
            if total == 0:
                raise RuntimeError("level advance produced an empty frontier")
        rounds += 1
        kmax = max(kmax, label)
        remaining -= total
        if peer:
            produced = [s.expand_peer(bound, label) for s in shards]
            comm.allreduce_sum(sum(produced))  # the round barrier
            nfront = [s.finish_round() for s in shards]
            continue
        counts = [s.count_remote() for s in shards]
        recv_counts = comm.alltoall_counts(counts)
        sends = [s.expand(bound, label, c) for s, c in zip(shards, counts)]
        recvs = comm.alltoallv(sends, counts, recv_counts)
        nfront = [s.apply(r, bound, label) for s, r in zip(shards, recvs)]
    return [s.labels() for s in shards], kmax, rounds


def sharded_coreness_persistent(shards: List, comm, n_global: int, approx=None):
    """The device-resident form of sharded_coreness(peer=True): every rank
    launches ONE persistent kernel serving its shards (dg_shard_coreness_
    persistent); rounds are separated by a cross-shard barrier in device
    memory, so the host does no per-round work.  Shards must be linked
    (link_local / link_ipc).  Returns (labels per local shard, kmax, rounds,
    kernel ms)."""
    from . import _chk
    from ._abi import LIB
    if approx is not None:
        c_num, c_den = approx
        if c_den == 0 or c_num <= c_den:
            raise ValueError("approx_coreness needs c > 1")
    else:
        c_num, c_den = 1, 1
    if comm.allreduce_sum(sum(s.n_local for s in shards)) != n_global:
        raise ValueError("shards do not cover the graph")
    if n_global == 0:
        raise ValueError("coreness of empty graph")
    for s in shards:
        if s.rank == 0:
            _chk(LIB.dg_shard_xctrl_reset(s._h))
    comm.allreduce_sum(0)  # nobody enters before shard 0's control block is reset
    hs = (C.c_void_p * len(shards))(*[s._h.value for s in shards])
    kmax, rounds, ms = C.c_uint32(), C.c_uint32(), C.c_float()
    _chk(LIB.dg_shard_coreness_persistent(hs, len(shards), 0 if approx is None else 1,
                                          c_num, c_den, C.byref(kmax), C.byref(rounds),
                                          C.byref(ms)))
    return [s.labels() for s in shards], kmax.value, rounds.value, ms.value


def _decomposition(labels, kmax, rounds, approx):
    from . import CoreDecomposition
    return CoreDecomposition(labels=labels, kmax=kmax, peel_rounds=rounds,
                             kind="exact" if approx is None else "approximate",
                             c_num=1 if approx is None else approx[0],
                             c_den=1 if approx is None else approx[1])


def coreness_local_shards(g, P: int, approx=None, peer: bool = False,
                          persistent: bool = False):
    """All P range shards of `g` on this GPU (validates the shard kernels).
    persistent=True: one cooperative launch, a group of CTAs per shard."""
    bounds = partition(g.offs, P)
    shards = [CudaShard(g, bounds, r) for r in range(P)]
    if peer or persistent:
        link_local(shards)
    if persistent:
        labs, kmax, rounds, _ = sharded_coreness_persistent(shards, LocalComm(P), g.n, approx)
        return _decomposition(np.concatenate(labs), kmax, rounds, approx)
    labs, kmax, rounds = sharded_coreness(shards, LocalComm(P), g.n, approx, peer)
    return _decomposition(np.concatenate(labs), kmax, rounds, approx)


def coreness_distributed(g, approx=None, peer: bool = True, persistent: bool = False):
    """One range shard per torch.distributed rank (NCCL); every rank gets all
    labels.  peer=True maps the other ranks' shard state by CUDA IPC (one
    node, NVLink) and runs the fused rounds; persistent=True runs them as one
    device-resident kernel per GPU (implies peer)."""
    import torch
    comm = TorchComm(torch.device("cuda", torch.cuda.current_device()))
    bounds = partition(g.offs, comm.P)
    shard = CudaShard(g, bounds, comm.rank)
    if peer or persistent:
        link_ipc(shard, comm)
    if persistent:
        labs, kmax, rounds, _ = sharded_coreness_persistent([shard], comm, g.n, approx)
        return _decomposition(np.concatenate(comm.allgather(labs[0])), kmax, rounds, approx)
    labs, kmax, rounds = sharded_coreness([shard], comm, g.n, approx, peer)
    return _decomposition(np.concatenate(comm.allgather(labs[0])), kmax, rounds, approx)
