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


def _alltoallv(comm, sends, send_counts):
    """all-to-all of one int64 tensor per local shard, split by send_counts."""
    recv_counts = comm.alltoall_counts([list(map(int, c)) for c in send_counts])
    return comm.alltoallv(sends, [list(map(int, c)) for c in send_counts], recv_counts)


def build_shards(pairs: Sequence, comm):
    """pairs: one (u, v) pair of int64 tensors per local shard (comm.shards()).
    Returns (n, bounds, [(offs, adj, orig) numpy tuple per local shard])."""
    import torch
    P = comm.P
    dev = pairs[0][0].device
    # 1  canonical pairs, loops out
    can = []
    for u, v in pairs:
        u = u.to(torch.int64)
        v = v.to(torch.int64)
        keep = u != v
        a, b = torch.minimum(u, v)[keep], torch.maximum(u, v)[keep]
        if a.numel() and int(b.max()) >= (1 << 32):
            raise ValueError("distributed build: original ids must be below 2^32")
        can.append((a, b))
    # 2  owner ranges of the original id space
    local_max = max([int(b.max()) if b.numel() else 0 for _, b in can] + [0])
    idmax = comm.allreduce_max(local_max)
    shift = 0
    while (idmax >> shift) >= NB:
        shift += 1
    hist = torch.zeros(NB, dtype=torch.int64, device=dev)
    for a, b in can:
        hist += torch.bincount(a >> shift, minlength=NB)[:NB]
        hist += torch.bincount(b >> shift, minlength=NB)[:NB]
    hist = comm.allreduce_sum_tensor(hist)
    cum = torch.cumsum(hist, 0).cpu().numpy()
    total = int(cum[-1])
    if total == 0:
        raise ValueError("no edges after removing self-loops and duplicates")
    # split[r] = first bucket of rank r (balanced arc counts)
    split = np.searchsorted(cum, [(total * r) // P for r in range(P)], side="right")
    split[0] = 0
    split = np.maximum.accumulate(split)
    bounds_id = [int(s) << shift for s in split] + [idmax + 1]  # original-id ranges

    bnd = torch.tensor(bounds_id[1:-1], dtype=torch.int64, device=dev)

    def owner(x):
        return torch.bucketize(x, bnd, right=True)

    # 3  route both arc directions to the owner of their source
    sends, counts = [], []
    for a, b in can:
        src = torch.cat([a, b])
        dst = torch.cat([b, a])
        o = owner(src)
        # (src - 2^31) * 2^32 + dst: order-preserving in signed int64
        packed = ((src - (1 << 31)) << 32) | dst
        if P > 1:  # grouping only (the receiver sorts): a narrow key keeps the radix sort short
            packed = packed[torch.argsort(o.to(torch.int16), stable=True)]
        sends.append(packed)
        counts.append(torch.bincount(o, minlength=P).cpu().tolist())
    recvd = _alltoallv(comm, sends, counts)
    # 4  rows: sort + unique; present vertices = distinct sources
    rows = []
    for k, r in enumerate(comm.shards()):
        arcs = torch.unique(recvd[k])  # sorted, duplicates merged
        src = (arcs >> 32) + (1 << 31)
        dst = arcs & 0xFFFFFFFF
        verts, deg = torch.unique_consecutive(src, return_counts=True)
        rows.append((verts, deg, dst))
    # 5  dense ids: exclusive scan of the vertex counts over ranks
    counts_v = comm.allgather_counts([int(v.numel()) for v, _, _ in rows])
    base = np.concatenate([[0], np.cumsum(counts_v)[:-1]]).astype(np.int64)
    # 6  neighbour ids: ask the owners for the dense ids of the distinct dsts
    qs, qcounts, inv = [], [], []
    for verts, deg, dst in rows:
        udst, iv = torch.unique(dst, return_inverse=True)
        o = owner(udst)  # udst is sorted and owners ascend with ids: already grouped
        qs.append(udst)
        qcounts.append(torch.bincount(o, minlength=P).cpu().tolist())
        inv.append(iv)
    asked = _alltoallv(comm, qs, qcounts)
    answers = []
    for k, r in enumerate(comm.shards()):
        verts = rows[k][0]
        pos = torch.searchsorted(verts, asked[k])
        answers.append(pos + int(base[r]))
    # the answers go back along the reverse routes, in the askers' order
    back_counts = comm.alltoall_counts([list(map(int, c)) for c in qcounts])
    back = comm.alltoallv(answers, back_counts, [list(map(int, c)) for c in qcounts])
    out = []
    for k, r in enumerate(comm.shards()):
        verts, deg, dst = rows[k]
        dense = back[k][inv[k]]
        offs = torch.zeros(verts.numel() + 1, dtype=torch.int64, device=dev)
        offs[1:] = torch.cumsum(deg, 0)
        out.append((offs, dense.to(torch.int32), verts))
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


def shard_get_core(comm, bounds, rows, labels, k: int):
    """get_core (core.cpp:133-140 -> induced_subgraph, graph.hpp:50-80) on the
    shards: each rank keeps its vertices with label >= k; new dense ids =
    exclusive scan of the kept counts over ranks (old order preserved); the
    old->new map is all-gathered (one id per vertex) so every rank renames its
    kept arcs locally.  rows / labels: per local shard (offs, adj, orig) and
    labels (tensors or numpy).  Returns (n', bounds', rows', labels') with
    rows' / labels' tensors on the communicator's device."""
    import torch
    dev = comm.device
    labs = [_dev(l, dev, torch.int64) for l in labels]
    keeps = [l >= k for l in labs]
    counts = comm.allgather_counts([int(kp.sum()) for kp in keeps])
    base = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    maps_local = []
    for r, keep in zip(comm.shards(), keeps):
        new = torch.cumsum(keep.to(torch.int64), 0) - 1 + int(base[r])
        maps_local.append(torch.where(keep, new, torch.full_like(new, -1)))
    full = torch.cat(comm.allgatherv(maps_local))
    out_rows, out_labels = [], []
    for (offs, adj, orig), lab, keep in zip(rows, labs, keeps):
        offs = _dev(offs, dev, torch.int64)
        adj = _dev(adj, dev, torch.int64) & 0xFFFFFFFF
        nl = offs.numel() - 1
        row = torch.repeat_interleave(torch.arange(nl, device=dev), offs[1:] - offs[:-1],
                                      output_size=adj.numel())
        nadj = full[adj]
        ka = keep[row] & (nadj >= 0)
        deg = torch.bincount(row[ka], minlength=nl)[keep]
        noffs = torch.zeros(deg.numel() + 1, dtype=torch.int64, device=dev)
        noffs[1:] = torch.cumsum(deg, 0)
        out_rows.append((noffs, nadj[ka].to(torch.int32), _dev(orig, dev, torch.int64)[keep]))
        out_labels.append(lab[keep])
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


def prune_distributed(pairs, comm, make_shard, cfg, peer: bool = False):
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
    n, bounds, rows = build_shards(pairs, comm)
    shards = [make_shard(n, bounds, r, o, a) for r, (o, a, _) in zip(comm.shards(), rows)]
    if peer:
        link(shards, comm)
    labs, kmax, rounds = sharded_coreness(shards, comm, n, approx, peer)
    del shards
    lower = Density(kmax, 2)
    thresh = ceil_scaled(lower, 1, 1) if approx is None else ceil_scaled(lower, cfg.c_den,
                                                                         cfg.c_num)
    _, _, crow, clab = shard_get_core(comm, bounds, rows, labs, thresh)
    offs, adj, orig, lab = gather_rows(comm, crow, clab)
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


def run_distributed(u, v, cfg=None, peer=None):
    """run() over torch.distributed ranks (NCCL): this rank's slice of the
    sample pairs (CUDA int64 tensors) -> distributed build -> sharded
    coreness -> per-shard compaction -> the core gathered to every rank ->
    Greedy++ replica (dg_run_pruned).  Same RunResult as run() on the graph
    of all pairs.  peer=None picks the peer-memory exchange when every rank
    can map every other's memory (peer_capable), else NCCL all-to-all."""
    import torch
    from . import Graph, RunConfig, run_pruned
    from .sharded import CudaShard, TorchComm
    cfg = cfg or RunConfig()
    comm = TorchComm(torch.device("cuda", torch.cuda.current_device()))
    if peer is None:
        peer = peer_capable()
    offs, adj, orig, lab, kmax, rounds = prune_distributed([(u, v)], comm, CudaShard.from_rows,
                                                           cfg, peer=peer)
    return run_pruned(Graph.from_device_csr(offs, adj, orig), lab.cpu().numpy(), kmax, rounds,
                      cfg)
