"""Range-sharded coreness: protocol on CPU (numpy shards,
in-process and world_size-2 gloo), CUDA shard kernels on the GPU.  Every
case is checked against the oracle's og_coreness (core.cpp:89-119):
labels, kmax and peel_rounds bit-exact."""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch

from graphs import biclique_with_k4, clique, path_graph, star, triangle_pendant, uv
from shard_numpy import NumpyShard

from paper_2311_04333_b200.sharded import LocalComm, TorchComm, partition, sharded_coreness

APPROX = [None, (3, 2), (2, 1)]


def _graphs(orc):
    out = {}
    for name, e in [("path", path_graph(9)), ("clique", clique(7)), ("star", star(12)),
                    ("tri_pendant", triangle_pendant()), ("biclique_k4", biclique_with_k4())]:
        out[name] = orc.build(*uv(e))
    out["gnp"] = orc.build(*orc.gen_gnp(300, 40, 7))
    out["rmat10"] = orc.build(*orc.gen_rmat(10, 16 * 1024, 3))
    out["planted"] = orc.build(*orc.gen_er_planted(2000, 6000, 30, 5))
    return out


def _check(orc, g, labs, kmax, rounds, approx):
    if approx is None:
        lab, k, r = orc.coreness(g)
    else:
        lab, k, r = orc.coreness(g, True, *approx)
    np.testing.assert_array_equal(np.concatenate(labs).astype(np.uint32), lab)
    assert (kmax, rounds) == (k, r)


def test_partition_balanced(orc):
    g = orc.build(*orc.gen_rmat(12, 64 * 1024, 9))
    for P in (1, 2, 3, 8, 64):
        b = partition(g.offs, P)
        assert len(b) == P + 1 and b[0] == 0 and b[-1] == g.n
        assert np.all(np.diff(b.astype(np.int64)) >= 0)
        arcs = np.diff(g.offs[b.astype(np.int64)].astype(np.int64))
        # every range within one max-degree row of the ideal share
        assert arcs.max() <= int(g.offs[-1]) // P + g.max_degree() + 1


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_protocol_numpy_local(orc, P):
    for name, g in _graphs(orc).items():
        for approx in APPROX:
            b = partition(g.offs, P)
            shards = [NumpyShard(g.offs, g.adj, b, r) for r in range(P)]
            labs, kmax, rounds = sharded_coreness(shards, LocalComm(P, "cpu"), g.n, approx)
            _check(orc, g, labs, kmax, rounds, approx)


def test_protocol_rejects_bad_input(orc):
    g = orc.build(*uv(clique(4)))
    b = partition(g.offs, 2)
    shards = [NumpyShard(g.offs, g.adj, b, 0)]  # one of two shards missing
    with pytest.raises(ValueError):
        sharded_coreness(shards, LocalComm(2, "cpu"), g.n)
    with pytest.raises(ValueError):
        sharded_coreness([NumpyShard(g.offs, g.adj, b, r) for r in range(2)],
                         LocalComm(2, "cpu"), g.n, (1, 1))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, outdir):
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "oracle"))
    import torch.distributed as dist
    from oracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        res = {}
        for name, g in _graphs(orc).items():
            for ai, approx in enumerate(APPROX):
                b = partition(g.offs, world)
                comm = TorchComm("cpu")
                labs, kmax, rounds = sharded_coreness([NumpyShard(g.offs, g.adj, b, rank)],
                                                      comm, g.n, approx)
                full = np.concatenate(comm.allgather(labs[0]))
                res[f"{name}/{ai}"] = (full, kmax, rounds)
        if rank == 0:
            np.save(os.path.join(outdir, "res.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_gloo_world2(orc):
    """world_size-2 gloo run of the NCCL protocol (one shard per process)."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = np.load(os.path.join(d, "res.npy"), allow_pickle=True).item()
    gs = _graphs(orc)
    assert len(res) == len(gs) * len(APPROX)
    for name, g in gs.items():
        for ai, approx in enumerate(APPROX):
            full, kmax, rounds = res[f"{name}/{ai}"]
            _check(orc, g, [full], kmax, rounds, approx)


# ------------------------------------------------------------------ CUDA shard kernels
@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4, 7])
def test_cuda_shards_local(orc, dg, P):
    from paper_2311_04333_b200.sharded import coreness_local_shards
    for name, hg in _graphs(orc).items():
        g = dg.Graph.from_csr(hg.offs, hg.adj, hg.orig)
        for approx in APPROX:
            dec = coreness_local_shards(g, P, approx)
            _check(orc, hg, [dec.labels], dec.kmax, dec.peel_rounds, approx)


@pytest.mark.gpu
def test_cuda_shards_rmat16(orc, dg):
    """Larger graph: 8 shards vs the single-GPU kernel and the oracle."""
    from paper_2311_04333_b200.sharded import coreness_local_shards
    u, v = orc.gen_rmat(16, 16 << 16, 16)
    hg = orc.build(u, v)
    g = dg.Graph.from_csr(hg.offs, hg.adj, hg.orig)
    dec = coreness_local_shards(g, 8)
    one = dg.exact_coreness(g)
    np.testing.assert_array_equal(dec.labels, one.labels)
    assert (dec.kmax, dec.peel_rounds) == (one.kmax, one.peel_rounds)
    _check(orc, hg, [dec.labels], dec.kmax, dec.peel_rounds, None)


@pytest.mark.gpu
def test_cuda_shards_from_own_rows(orc, dg):
    """Memory-scaled shards: each is created from its own rows only (host
    slices of the CSR), or copies its rows from a graph that is then freed."""
    from paper_2311_04333_b200.sharded import CudaShard, LocalComm
    u, v = orc.gen_rmat(14, 16 << 14, 77)
    hg = orc.build(u, v)
    lab, kmax, rounds = orc.coreness(hg)
    for P in (1, 3, 5):
        b = partition(hg.offs, P)
        shards = []
        for r in range(P):
            lo, hi = int(b[r]), int(b[r + 1])
            offs = hg.offs[lo:hi + 1]
            adj = hg.adj[int(offs[0]):int(offs[-1])]
            shards.append(CudaShard.from_rows(hg.n, b, r, offs, adj))
        labs, k, rr = sharded_coreness(shards, LocalComm(P), hg.n)
        np.testing.assert_array_equal(np.concatenate(labs), lab)
        assert (k, rr) == (kmax, rounds)
    g = dg.Graph.from_csr(hg.offs, hg.adj, hg.orig)
    b = partition(hg.offs, 4)
    shards = [CudaShard(g, b, r) for r in range(4)]
    del g  # shards own their rows
    labs, k, rr = sharded_coreness(shards, LocalComm(4), hg.n)
    np.testing.assert_array_equal(np.concatenate(labs), lab)


# ------------------------------------------------------------------ peer mode (fused rounds)
@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_peer_protocol_numpy_local(orc, P):
    from shard_numpy import NumpyPeerShard
    from paper_2311_04333_b200.sharded import link_local
    for name, g in _graphs(orc).items():
        for approx in APPROX:
            b = partition(g.offs, P)
            shards = [NumpyPeerShard(g.offs, g.adj, b, r) for r in range(P)]
            link_local(shards)
            labs, kmax, rounds = sharded_coreness(shards, LocalComm(P, "cpu"), g.n, approx,
                                                  peer=True)
            _check(orc, g, labs, kmax, rounds, approx)


def _gloo_peer_worker(rank, world, port, outdir):
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "oracle"))
    import torch.distributed as dist
    from oracle import Oracle
    from shard_numpy import NumpyPeerShard
    from paper_2311_04333_b200.sharded import link_ipc

    class Serial(NumpyPeerShard):  # one rank at a time inside a round (any order is valid)
        def expand_peer(self, bound, label):
            made = 0
            for turn in range(world):
                if turn == rank:
                    made = super().expand_peer(bound, label)
                dist.barrier()
            return made

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        res = {}
        for name, g in _graphs(orc).items():
            for ai, approx in enumerate(APPROX):
                b = partition(g.offs, world)
                comm = TorchComm("cpu")
                shard = Serial(g.offs, g.adj, b, rank, shm=True)
                link_ipc(shard, comm)
                labs, kmax, rounds = sharded_coreness([shard], comm, g.n, approx, peer=True)
                full = np.concatenate(comm.allgather(labs[0]))
                dist.barrier()  # nobody maps this block any more
                shard.close()
                res[f"{name}/{ai}"] = (full, kmax, rounds)
        if rank == 0:
            np.save(os.path.join(outdir, "res.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_peer_gloo_world2(orc):
    """world_size-2 run of the fused protocol: the shard state blocks are
    shared memory mapped by the other process (the CPU stand-in for CUDA IPC
    over NVLink), one all-reduce per round."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_peer_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = np.load(os.path.join(d, "res.npy"), allow_pickle=True).item()
    gs = _graphs(orc)
    for name, g in gs.items():
        for ai, approx in enumerate(APPROX):
            full, kmax, rounds = res[f"{name}/{ai}"]
            _check(orc, g, [full], kmax, rounds, approx)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4, 7])
def test_cuda_shards_peer_local(orc, dg, P):
    """Peer-mode kernels: P shards on one GPU decrement each other's state
    blocks directly (the same kernel maps NVLink peer memory across GPUs)."""
    from paper_2311_04333_b200.sharded import coreness_local_shards
    for name, hg in _graphs(orc).items():
        g = dg.Graph.from_csr(hg.offs, hg.adj, hg.orig)
        for approx in APPROX:
            dec = coreness_local_shards(g, P, approx, peer=True)
            _check(orc, hg, [dec.labels], dec.kmax, dec.peel_rounds, approx)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 3, 4, 7, 16])
def test_cuda_shards_persistent_local(orc, dg, P):
    """The device-resident round loop (dg_shard_coreness_persistent): P
    shards served by P CTA groups of ONE cooperative launch, rounds separated
    by the cross-shard barrier in shard 0's control block, remote decrements
    and queue appends through the peer views -- the code path every GPU of a
    multi-GPU job runs with one group."""
    from paper_2311_04333_b200.sharded import coreness_local_shards
    for name, hg in _graphs(orc).items():
        g = dg.Graph.from_csr(hg.offs, hg.adj, hg.orig)
        for approx in APPROX:
            dec = coreness_local_shards(g, P, approx, persistent=True)
            _check(orc, hg, [dec.labels], dec.kmax, dec.peel_rounds, approx)


@pytest.mark.gpu
def test_cuda_shards_persistent_rmat(orc, dg):
    """RMAT-18 (hub rows cut into pieces): 1, 4 and 8 shards in one launch
    against the single-GPU kernel, exact and approximate."""
    from paper_2311_04333_b200.sharded import coreness_local_shards
    g = dg.Graph.generate_rmat(18, 16 << 18, 18)
    one = dg.exact_coreness(g)
    apx = dg.approx_coreness(g, 3, 2)
    for P in (1, 4, 8):
        dec = coreness_local_shards(g, P, persistent=True)
        np.testing.assert_array_equal(dec.labels, one.labels)
        assert (dec.kmax, dec.peel_rounds) == (one.kmax, one.peel_rounds)
        dec = coreness_local_shards(g, P, (3, 2), persistent=True)
        np.testing.assert_array_equal(dec.labels, apx.labels)
        assert (dec.kmax, dec.peel_rounds) == (apx.kmax, apx.peel_rounds)


def _ipc_worker(rank, world, port, outdir):
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "oracle"))
    import torch.distributed as dist
    from oracle import Oracle
    import paper_2311_04333_b200 as dg
    from paper_2311_04333_b200.sharded import CudaShard, link_ipc
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        res = {}
        gs = _graphs(orc)
        for name in ("rmat10", "planted", "tri_pendant"):
            hg = gs[name]
            g = dg.Graph.from_csr(hg.offs, hg.adj, hg.orig)
            b = partition(hg.offs, world)
            comm = TorchComm("cpu")
            shard = CudaShard(g, b, rank)
            link_ipc(shard, comm)  # the other process's state block, by CUDA IPC
            for ai, approx in enumerate(APPROX):
                if ai:  # fresh state per run
                    dist.barrier()
                    del shard
                    shard = CudaShard(g, b, rank)
                    link_ipc(shard, comm)
                labs, kmax, rounds = sharded_coreness([shard], comm, hg.n, approx, peer=True)
                res[f"{name}/{ai}"] = (np.concatenate(comm.allgather(labs[0])), kmax, rounds)
            dist.barrier()  # nobody maps the blocks any more
            del shard
        if rank == 0:
            np.save(os.path.join(outdir, "res.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_cuda_peer_ipc_two_processes(orc):
    """The IPC path of peer mode: two processes (gloo for the host
    collectives) map each other's shard state with cudaIpcOpenMemHandle and
    run the fused rounds.  Both processes share the one GPU here; no kernel
    waits on the other process (rounds are separated by the host all-reduce)."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_ipc_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = np.load(os.path.join(d, "res.npy"), allow_pickle=True).item()
    gs = _graphs(orc)
    for name in ("rmat10", "planted", "tri_pendant"):
        for ai, approx in enumerate(APPROX):
            full, kmax, rounds = res[f"{name}/{ai}"]
            _check(orc, gs[name], [full], kmax, rounds, approx)
