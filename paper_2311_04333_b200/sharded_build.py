"""Distributed CSR build ("the CSR build shards the same way").

Every rank holds a slice of the sample pairs (u, v) -- e.g. its share of a
seeded generator's stream -- and ends with ITS rows of exactly the CSR that
parse_edge_list / dg_graph_build would build from all pairs on one machine
(io.cpp:51-92: loops dropped, duplicates merged, dense id = rank of the
original id among present ones, rows ascending).  Protocol (collectives over
`Comm`, the same objects as sharded.py, so NCCL on GPUs and gloo on CPU):

  1  canonical pairs, loops dropped (local)
  2  owner ranges of the ORIGINAL id space: all-reduced 4096-bucket histogram
     of arc endpoints -> split points balancing arcs per rank; the dense
     relabel is monotone, so original-id ranges are dense-id ranges
  3  both arc directions routed to the owner of their source (all-to-all)
  4  per rank: sort (src, dst), unique -> rows in ascending dst order; the
     present vertices are the distinct sources
  5  dense ids: exclusive scan of the per-rank vertex counts (all-gather)
  6  neighbour ids: the distinct dsts are sent to their owners, answered with
     dense ids (binary search in the owner's sorted vertices), returned
     (all-to-all twice)

Tensor work is torch on the device of the communicator (CUB sorts on GPUs).
Original ids must be below 2^32 (the generators' ranges).  Result: the
global vertex count n, the dense-id split points bounds[0..P] (numpy) and per
local shard (offs, adj, orig) as tensors on the communicator's device: offs
int64 rebased to 0 (n_r + 1 entries), adj = global dense ids (int32 holding
uint32 bits), orig int64 = original ids of the rank's vertices -- the input of
CudaShard.from_rows (dg_shard_create_rows, device pointers).
"""
from __future__ import annotations

import os

from typing import List, Sequence

import numpy as np

__all__ = ["build_shards", "coreness_from_pairs_distributed", "shard_get_core", "gather_rows",
           "prune_distributed", "run_distributed"]

NB = 4096  # endpoint histogram buckets
NONE32 = -1  # dropped vertex in a keep map (uint32 0xFFFFFFFF as int32)


def _ptr(t):
    import ctypes as C
    return C.c_void_p(t.data_ptr() if t.numel() else 0)


class CudaDistOps:
    """The per-rank device steps of the distributed build and of get_core on
    a shard: the library's kernels (csrc/dist_build.cu, dg_dist_* C ABI) on
    torch CUDA tensors used as buffers.  Every call synchronises torch's
    stream first (its tensors feed the library's stream) and the library
    returns with its stream drained."""

    def __init__(self, device):
        import torch
        from . import _chk
        from ._abi import LIB
        self.torch, self.LIB, self._chk, self.dev = torch, LIB, _chk, torch.device(device)

    def _sync(self):
        self.torch.cuda.synchronize(self.dev)

    def _empty(self, n, dtype):
        return self.torch.empty(max(1, int(n)), dtype=dtype, device=self.dev)

    def max_id(self, u, v) -> int:
        import ctypes as C
        self._sync()
        out = C.c_uint64()
        self._chk(self.LIB.dg_dist_max_id(_ptr(u), _ptr(v), u.numel(), C.byref(out)))
        return out.value

    def hist(self, u, v, shift, nb):
        import ctypes as C
        self._sync()
        h = np.zeros(nb, np.uint64)
        self._chk(self.LIB.dg_dist_endpoint_hist(_ptr(u), _ptr(v), u.numel(), shift, nb,
                                                 h.ctypes.data_as(C.POINTER(C.c_uint64))))
        return h.astype(np.int64)

    def route(self, u, v, bounds_id):
        import ctypes as C
        self._sync()
        P = len(bounds_id) - 1
        b = np.ascontiguousarray(bounds_id, dtype=np.uint64)
        cnt = np.zeros(P, np.uint64)
        keys = self._empty(2 * u.numel(), self.torch.int64)
        self._chk(self.LIB.dg_dist_route(_ptr(u), _ptr(v), u.numel(),
                                         b.ctypes.data_as(C.POINTER(C.c_uint64)), P, _ptr(keys),
                                         cnt.ctypes.data_as(C.POINTER(C.c_uint64))))
        return keys[: int(cnt.sum())], [int(c) for c in cnt]

    def rows(self, keys):
        import ctypes as C
        self._sync()
        n = keys.numel()
        offs = self._empty(n + 1, self.torch.int64)
        verts = self._empty(n, self.torch.int64)
        dst = self._empty(n, self.torch.int32)
        nv, m = C.c_uint64(), C.c_uint64()
        self._chk(self.LIB.dg_dist_rows(_ptr(keys), n, _ptr(offs), _ptr(verts), _ptr(dst),
                                        C.byref(nv), C.byref(m)))
        return offs[: nv.value + 1], verts[: nv.value], dst[: m.value]

    def unique(self, vals):
        import ctypes as C
        self._sync()
        n = vals.numel()
        uniq = self._empty(n, self.torch.int32)
        inv = self._empty(n, self.torch.int32)
        nu = C.c_uint64()
        self._chk(self.LIB.dg_dist_unique(_ptr(vals), n, _ptr(uniq), _ptr(inv), C.byref(nu)))
        return uniq[: nu.value], inv[:n]

    def bucket_counts(self, vals, bounds_id):
        import ctypes as C
        self._sync()
        P = len(bounds_id) - 1
        b = np.ascontiguousarray(bounds_id, dtype=np.uint64)
        cnt = np.zeros(P, np.uint64)
        self._chk(self.LIB.dg_dist_bucket_counts(_ptr(vals), vals.numel(),
                                                 b.ctypes.data_as(C.POINTER(C.c_uint64)), P,
                                                 cnt.ctypes.data_as(C.POINTER(C.c_uint64))))
        return [int(c) for c in cnt]

    def lookup(self, verts, asked, base):
        self._sync()
        out = self._empty(asked.numel(), self.torch.int32)
        self._chk(self.LIB.dg_dist_lookup(_ptr(verts), verts.numel(), _ptr(asked), asked.numel(),
                                          int(base), _ptr(out)))
        return out[: asked.numel()]

    def relabel(self, back, inv):
        self._sync()
        adj = self._empty(inv.numel(), self.torch.int32)
        self._chk(self.LIB.dg_dist_relabel(_ptr(back), _ptr(inv), inv.numel(), _ptr(adj)))
        return adj[: inv.numel()]

    def keep_map(self, labels, k, base):
        import ctypes as C
        self._sync()
        labels = labels.to(self.torch.int32).contiguous()
        m = self._empty(labels.numel(), self.torch.int32)
        kept = C.c_uint64()
        self._chk(self.LIB.dg_dist_keep_map(_ptr(labels), labels.numel(), int(k), int(base),
                                            _ptr(m), C.byref(kept)))
        return m[: labels.numel()], kept.value

    def core_rows(self, offs, adj, local_map, full_map):
        import ctypes as C
        self._sync()
        nl = offs.numel() - 1
        noffs = self._empty(nl + 1, self.torch.int64)
        nadj = self._empty(adj.numel(), self.torch.int32)
        kn, m = C.c_uint64(), C.c_uint64()
        self._chk(self.LIB.dg_dist_core_rows(_ptr(offs), _ptr(adj), nl, _ptr(local_map),
                                             _ptr(full_map), _ptr(noffs), _ptr(nadj),
                                             C.byref(kn), C.byref(m)))
        return noffs[: kn.value + 1], nadj[: m.value]

    def take(self, x, local_map, base, kept):
        self._sync()
        x = x.contiguous()
        out = self._empty(kept, x.dtype)
        self._chk(self.LIB.dg_dist_take(_ptr(x), _ptr(local_map), x.numel(), int(base),
                                        x.element_size(), _ptr(out)))
        return out[:kept]


def default_ops(device):
    import torch
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError("the distributed build runs on CUDA devices (pass ops= for host tests)")
    return CudaDistOps(dev)


def _alltoallv(comm, sends, send_counts):
    """all-to-all of one tensor per local shard, split by send_counts."""
    recv_counts = comm.alltoall_counts([list(map(int, c)) for c in send_counts])
    return comm.alltoallv(sends, [list(map(int, c)) for c in send_counts], recv_counts)


def build_shards(pairs: Sequence, comm, ops=None):
    """pairs: one (u, v) pair of int64 tensors per local shard (comm.shards()).
    Returns (n, bounds, [(offs, adj, orig) per local shard]).  `ops`: the
    per-rank steps (default: the library's CUDA kernels)."""
    import torch
    ops = ops or default_ops(pairs[0][0].device)
    P = comm.P
    pairs = [(u.to(torch.int64).contiguous(), v.to(torch.int64).contiguous()) for u, v in pairs]
    # 1-2  owner ranges of the original id space (balanced arc counts)
    idmax = comm.allreduce_max(max([ops.max_id(u, v) for u, v in pairs] + [0]))
    if idmax >= (1 << 32):
        raise ValueError("distributed build: original ids must be below 2^32")
    if idmax == 0:
        raise ValueError("no edges after removing self-loops and duplicates")
    shift = 0
    while (idmax >> shift) >= NB:
        shift += 1
    hist = sum(ops.hist(u, v, shift, NB) for u, v in pairs)
    hist = comm.allreduce_sum_tensor(torch.as_tensor(hist, device=comm.device)).cpu().numpy()
    cum = np.cumsum(hist)
    total = int(cum[-1])
    split = np.searchsorted(cum, [(total * r) // P for r in range(P)], side="right")
    split[0] = 0
    split = np.maximum.accumulate(split)
    bounds_id = np.array([int(x) << shift for x in split] + [idmax + 1], dtype=np.uint64)
    # 3  both arc directions routed to the owner of their source
    sends, counts = [], []
    for u, v in pairs:
        keys, c = ops.route(u, v, bounds_id)
        sends.append(keys)
        counts.append(c)
    recvd = _alltoallv(comm, sends, counts)
    del sends
    # 4  rows: sort + unique; present vertices = distinct sources
    rows = [ops.rows(k) for k in recvd]
    del recvd
    # 5  dense ids: exclusive scan of the vertex counts over ranks
    counts_v = comm.allgather_counts([int(verts.numel()) for _, verts, _ in rows])
    base = np.concatenate([[0], np.cumsum(counts_v)[:-1]]).astype(np.int64)
    # 6  neighbour ids: ask the owners for the dense ids of the distinct dsts
    qs, qcounts, inv = [], [], []
    for _, _, dst in rows:
        udst, iv = ops.unique(dst)
        qs.append(udst)
        qcounts.append(ops.bucket_counts(udst, bounds_id))  # udst ascending: grouped by owner
        inv.append(iv)
    asked = _alltoallv(comm, qs, qcounts)
    answers = [ops.lookup(rows[k][1], asked[k], base[r]) for k, r in enumerate(comm.shards())]
    back_counts = comm.alltoall_counts([list(map(int, c)) for c in qcounts])
    back = comm.alltoallv(answers, back_counts, [list(map(int, c)) for c in qcounts])
    out = []
    for k in range(len(rows)):
        offs, verts, _ = rows[k]
        out.append((offs, ops.relabel(back[k], inv[k]), verts))
    n = int(sum(counts_v))
    bounds = np.concatenate([base, [n]]).astype(np.uint64)
    return n, bounds, out


def coreness_from_pairs_distributed(u, v, approx=None):
    """One rank's slice of the sample pairs (CUDA tensors) -> distributed CSR
    build -> sharded coreness (NCCL).  Every rank gets all labels."""
    import torch
    from .sharded import CudaShard, TorchComm, _decomposition, sharded_coreness
    comm = TorchComm(torch.device("cuda", torch.cuda.current_device()))
    n, bounds, ((offs, adj, _orig),) = build_shards([(u, v)], comm)
    shard = CudaShard.from_rows(n, bounds, comm.rank, offs, adj)
    labs, kmax, rounds = sharded_coreness([shard], comm, n, approx)
    return _decomposition(np.concatenate(comm.allgather(labs[0])), kmax, rounds, approx)


# ------------------------------------------------------------------ per-shard get_core
def _dev(x, dev, dtype):
    import torch
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype)
    return torch.as_tensor(np.asarray(x).astype(np.int64), device=dev).to(dtype)


def shard_get_core(comm, bounds, rows, labels, k: int, ops=None):
    """get_core (core.cpp:133-140 -> induced_subgraph, graph.hpp:50-80) on the
    shards: each rank keeps its vertices with label >= k; new dense ids =
    exclusive scan of the kept counts over ranks (old order preserved); the
    old->new map is all-gathered (one id per vertex) so every rank renames its
    kept arcs locally.  rows / labels: per local shard (offs, adj, orig) and
    labels (tensors or numpy).  Returns (n', bounds', rows', labels') with
    rows' / labels' tensors on the communicator's device."""
    import torch
    dev = comm.device
    ops = ops or default_ops(dev)
    labs = [_dev(l, dev, torch.int64).to(torch.int32) for l in labels]
    counts = comm.allgather_counts([ops.keep_map(l, k, 0)[1] for l in labs])
    base = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    maps = [ops.keep_map(l, k, int(base[r]))[0] for l, r in zip(labs, comm.shards())]
    full = torch.cat(comm.allgatherv(maps))
    out_rows, out_labels = [], []
    for (offs, adj, orig), lab, m, r, c in zip(rows, labs, maps, comm.shards(),
                                               [counts[r] for r in comm.shards()]):
        offs = _dev(offs, dev, torch.int64).contiguous()
        adj = _dev(adj, dev, torch.int64).to(torch.int32).contiguous()
        noffs, nadj = ops.core_rows(offs, adj, m, full)
        norig = ops.take(_dev(orig, dev, torch.int64), m, int(base[r]), c)
        out_rows.append((noffs, nadj, norig))
        out_labels.append(ops.take(lab, m, int(base[r]), c).to(torch.int64))
    n2 = int(sum(counts))
    return n2, np.concatenate([base, [n2]]).astype(np.uint64), out_rows, out_labels


def gather_rows(comm, rows, labels):
    """All ranks get the whole (core) CSR as device tensors: offs (int64),
    adj (int32 holding uint32 bits), orig (int64), labels (int64)."""
    import torch
    dev = comm.device
    deg = torch.cat(comm.allgatherv([_dev(o, dev, torch.int64).diff() for o, _, _ in rows]))
    offs = torch.zeros(deg.numel() + 1, dtype=torch.int64, device=dev)
    offs[1:] = torch.cumsum(deg, 0)
    adj = torch.cat(comm.allgatherv([_dev(a, dev, torch.int32) for _, a, _ in rows]))
    orig = torch.cat(comm.allgatherv([_dev(o, dev, torch.int64) for _, _, o in rows]))
    lab = torch.cat(comm.allgatherv([_dev(l, dev, torch.int64) for l in labels]))
    return offs, adj, orig, lab


def prune_distributed(pairs, comm, make_shard, cfg, peer: bool = False, ops=None,
                      persistent: bool = False, timings=None):
    """framework.cpp:58-79 on the shards: distributed build, sharded coreness
    (exact, or approximate for approx/hybrid), first threshold, per-shard
    get_core, one gather.  Returns (core offs, adj, orig, core labels, kmax,
    peel_rounds) on every rank -- the input of run_pruned.
    make_shard(n, bounds, rank, offs, adj) -> a shard engine."""
    from . import Density, ceil_scaled
    from .sharded import link, sharded_coreness
    if cfg.pruning == "none":
        raise ValueError("the sharded pipeline prunes; use run() for pruning='none'")
    approx = None if cfg.pruning == "exact" else (cfg.c_num, cfg.c_den)
    import time
    t0 = time.perf_counter()
    n, bounds, rows = build_shards(pairs, comm, ops)
    t1 = time.perf_counter()
    shards = [make_shard(n, bounds, r, o, a) for r, (o, a, _) in zip(comm.shards(), rows)]
    if peer or persistent:
        link(shards, comm)
    kc_ms = None
    t2 = time.perf_counter()
    if persistent:
        from .sharded import sharded_coreness_persistent
        labs, kmax, rounds, kc_ms = sharded_coreness_persistent(shards, comm, n, approx)
    else:
        labs, kmax, rounds = sharded_coreness(shards, comm, n, approx, peer)
    t3 = time.perf_counter()
    del shards
    lower = Density(kmax, 2)
    thresh = ceil_scaled(lower, 1, 1) if approx is None else ceil_scaled(lower, cfg.c_den,
                                                                         cfg.c_num)
    _, _, crow, clab = shard_get_core(comm, bounds, rows, labs, thresh, ops)
    offs, adj, orig, lab = gather_rows(comm, crow, clab)
    if timings is not None:
        arcs = sum(int(o[-1]) for o, _, _ in rows)
        timings.update(n=n, m=comm.allreduce_sum(arcs) // 2, build_s=t1 - t0,
                       coreness_s=t3 - t2, coreness_kernel_ms=kc_ms,
                       get_core_gather_s=time.perf_counter() - t3)
    return offs, adj, orig, lab, kmax, rounds


def peer_capable() -> bool:
    """Every rank of the job on this node, and this GPU can map every other
    local GPU's memory (CUDA IPC over NVLink): the fused peer-memory exchange
    applies.  Otherwise (multi-node jobs, no P2P) the NCCL all-to-all rounds."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    local = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    if local != world or torch.cuda.device_count() < world:
        ok = False
    else:
        me = torch.cuda.current_device()
        ok = all(torch.cuda.can_device_access_peer(me, d)
                 for d in range(torch.cuda.device_count()) if d != me)
    t = torch.tensor([1 if ok else 0], device=torch.device("cuda", torch.cuda.current_device()))
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def run_distributed(u, v, cfg=None, peer=None, persistent: bool = True):
    """run() over torch.distributed ranks (NCCL): this rank's slice of the
    sample pairs (CUDA int64 tensors) -> distributed build -> sharded
    coreness -> per-shard compaction -> the core gathered to every rank ->
    Greedy++ replica (dg_run_pruned).  Same RunResult as run() on the graph
    of all pairs.  peer=None picks the peer-memory exchange when every rank
    can map every other's memory (peer_capable), else NCCL all-to-all;
    with peer memory the rounds run device-resident (one persistent kernel
    per GPU) unless persistent=False."""
    import torch
    from . import Graph, RunConfig, run_pruned
    from .sharded import CudaShard, TorchComm
    cfg = cfg or RunConfig()
    comm = TorchComm(torch.device("cuda", torch.cuda.current_device()))
    if peer is None:
        peer = peer_capable()
    offs, adj, orig, lab, kmax, rounds = prune_distributed(
        [(u, v)], comm, CudaShard.from_rows, cfg, peer=peer, persistent=persistent and peer)
    return run_pruned(Graph.from_device_csr(offs, adj, orig), lab.cpu().numpy(), kmax, rounds,
                      cfg)
