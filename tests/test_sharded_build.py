"""Distributed CSR build (sharded_build.py): every rank starts
from a slice of the sample pairs and ends with its rows of exactly the CSR the
oracle builds from all pairs (io.cpp:51-92: loops dropped, duplicates merged,
dense ids = rank of the original id).  CPU: in-process shards and a
world_size-2 gloo run, then coreness over the built shards vs the oracle;
GPU: the same on CUDA tensors feeding the CUDA shard kernels."""
import os
import sys
import tempfile

import numpy as np
import pytest
import torch

from dist_ops_torch import TorchDistOps
from shard_numpy import NumpyShard
from test_sharded import _free_port

from paper_2311_04333_b200.sharded import LocalComm, TorchComm, sharded_coreness
from paper_2311_04333_b200.sharded_build import build_shards


HOST = TorchDistOps()  # host restatement of the CUDA steps (tests only)


def _cases(orc):
    rng = np.random.default_rng(11)
    out = {
        "rmat12": orc.gen_rmat(12, 64 * 1024, 3),
        "chung_lu": orc.gen_chung_lu(3000, 20000, 5),
        "planted": orc.gen_er_planted(2000, 6000, 30, 5),
    }
    # duplicates (both orientations), self-loops and ids spread up to 2^32-1
    ids = np.unique(np.concatenate([rng.integers(0, 1 << 32, 400, dtype=np.uint64),
                                    np.array([0, (1 << 32) - 1], np.uint64)]))
    a = ids[rng.integers(0, len(ids), 3000)]
    b = ids[rng.integers(0, len(ids), 3000)]
    u = np.concatenate([a, b, a[:50], a[:40]])
    v = np.concatenate([b, a, b[:50], a[:40]])
    out["sparse_ids_dups_loops"] = (u, v)
    return out


def _split(u, v, P, skew=False):
    """Sample slices per rank; skew=True puts everything on the last rank."""
    if skew:
        cuts = [0] * P + [len(u)]
    else:
        cuts = np.linspace(0, len(u), P + 1).astype(int)
    return [(torch.from_numpy(np.asarray(u[cuts[i]:cuts[i + 1]], np.int64)),
             torch.from_numpy(np.asarray(v[cuts[i]:cuts[i + 1]], np.int64))) for i in range(P)]


def _np(t, dtype):
    """tensor (any device) -> numpy; ids are int32/int64 holding unsigned values."""
    a = t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
    if dtype == np.uint32:
        return (a.astype(np.int64) & 0xFFFFFFFF).astype(np.uint32)
    return a.astype(dtype)


def _assemble(sh):
    base, offs = 0, [np.zeros(1, np.uint64)]
    for o, _, _ in sh:
        o = _np(o, np.uint64)
        offs.append(o[1:] + np.uint64(base))
        base += int(o[-1])
    return (np.concatenate(offs), np.concatenate([_np(s[1], np.uint32) for s in sh]),
            np.concatenate([_np(s[2], np.uint64) for s in sh]))


def _check_csr(g, n, bounds, sh):
    offs, adj, orig = _assemble(sh)
    assert n == g.n and int(bounds[-1]) == n and bounds[0] == 0
    np.testing.assert_array_equal(offs, g.offs)
    np.testing.assert_array_equal(adj, g.adj)
    np.testing.assert_array_equal(orig, g.orig)


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
def test_build_local_matches_oracle(orc, P):
    for name, (u, v) in _cases(orc).items():
        g = orc.build(u, v)
        for skew in (False, True):
            n, bounds, sh = build_shards(_split(u, v, P, skew), LocalComm(P, "cpu"), HOST)
            _check_csr(g, n, bounds, sh)
            # coreness over the rank-owned rows = the oracle's
            shards = [NumpyShard.from_rows(n, bounds, r, sh[r][0], sh[r][1]) for r in range(P)]
            labs, kmax, rounds = sharded_coreness(shards, LocalComm(P, "cpu"), n)
            lab, k, rr = orc.coreness(g)
            np.testing.assert_array_equal(np.concatenate(labs), lab)
            assert (kmax, rounds) == (k, rr)


def test_build_balances_arcs(orc):
    u, v = orc.gen_rmat(14, 16 << 14, 8)
    g = orc.build(u, v)
    P = 4
    n, bounds, sh = build_shards(_split(u, v, P), LocalComm(P, "cpu"), HOST)
    arcs = np.array([int(_np(o, np.uint64)[-1]) for o, _, _ in sh])
    assert arcs.sum() == int(g.offs[-1])
    # bucket-granular split: within 25% of the ideal share on RMAT-14
    assert arcs.max() <= 1.25 * arcs.sum() / P


def test_build_rejects_bad_input():
    z = torch.zeros(0, dtype=torch.int64)
    with pytest.raises(ValueError, match="no edges"):
        build_shards([(torch.tensor([3, 4]), torch.tensor([3, 4])), (z, z)], LocalComm(2, "cpu"),
                     HOST)
    with pytest.raises(ValueError, match="2\\^32"):
        build_shards([(torch.tensor([0]), torch.tensor([1 << 32]))], LocalComm(1, "cpu"), HOST)
    with pytest.raises(ValueError, match="CUDA"):  # the product has no host path
        build_shards([(torch.tensor([0]), torch.tensor([1]))], LocalComm(1, "cpu"))


def _gloo_worker(rank, world, port, outdir):
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "oracle"))
    import torch.distributed as dist
    from oracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        res = {}
        for name, (u, v) in _cases(orc).items():
            comm = TorchComm("cpu")
            n, bounds, sh = build_shards([_split(u, v, world)[rank]], comm, TorchDistOps())
            shard = NumpyShard.from_rows(n, bounds, rank, sh[0][0], sh[0][1])
            labs, kmax, rounds = sharded_coreness([shard], comm, n)
            parts = comm.allgather((sh[0], labs[0]))
            res[name] = (n, bounds, [p[0] for p in parts], np.concatenate([p[1] for p in parts]),
                         kmax, rounds)
        if rank == 0:
            np.save(os.path.join(outdir, "res.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_build_gloo_world2(orc):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = np.load(os.path.join(d, "res.npy"), allow_pickle=True).item()
    for name, (u, v) in _cases(orc).items():
        g = orc.build(u, v)
        n, bounds, sh, labels, kmax, rounds = res[name]
        _check_csr(g, n, bounds, sh)
        lab, k, rr = orc.coreness(g)
        np.testing.assert_array_equal(labels, lab)
        assert (kmax, rounds) == (k, rr)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 3, 8])
def test_build_cuda_shards(orc, dg, P):
    """CUDA tensors through the build, rows into the CUDA shard kernels."""
    from paper_2311_04333_b200.sharded import CudaShard
    for name, (u, v) in _cases(orc).items():
        g = orc.build(u, v)
        pairs = [(a.cuda(), b.cuda()) for a, b in _split(u, v, P)]
        n, bounds, sh = build_shards(pairs, LocalComm(P))
        _check_csr(g, n, bounds, sh)
        shards = [CudaShard.from_rows(n, bounds, r, sh[r][0], sh[r][1]) for r in range(P)]
        labs, kmax, rounds = sharded_coreness(shards, LocalComm(P), n)
        lab, k, rr = orc.coreness(g)
        np.testing.assert_array_equal(np.concatenate(labs), lab)
        assert (kmax, rounds) == (k, rr)


@pytest.mark.gpu
def test_build_cuda_rmat18(orc, dg):
    u, v = orc.gen_rmat(18, 16 << 18, 21)
    g = orc.build(u, v)
    P = 4
    pairs = [(a.cuda(), b.cuda()) for a, b in _split(u, v, P)]
    n, bounds, sh = build_shards(pairs, LocalComm(P))
    _check_csr(g, n, bounds, sh)


# ------------------------------------------------------------------ sharded prune pipeline
PRUNINGS = ["exact", "approx", "hybrid"]


def _expected_core(orc, g, pruning, c_num=3, c_den=2):
    """framework.cpp:58-79 first prune on the whole graph (oracle)."""
    approx = pruning != "exact"
    lab, kmax, rounds = orc.coreness(g, approx, c_num, c_den) if approx else orc.coreness(g)
    num, den = (1, 1) if not approx else (c_den, c_num)
    p, q = kmax * num, 2 * den
    thresh = p // q + (p % q != 0)
    keep = lab >= thresh
    core, _ = orc.get_core(g, lab, thresh)
    return core, lab[keep], kmax, rounds


def _check_core(orc, g, pruning, got):
    offs, adj, orig, lab, kmax, rounds = got
    offs, adj, orig, lab = (_np(offs, np.uint64), _np(adj, np.uint32), _np(orig, np.uint64),
                            _np(lab, np.uint32))
    core, elab, ek, er = _expected_core(orc, g, pruning)
    np.testing.assert_array_equal(offs, core.offs)
    np.testing.assert_array_equal(adj, core.adj)
    np.testing.assert_array_equal(orig, core.orig)
    np.testing.assert_array_equal(lab, elab)
    assert (kmax, rounds) == (ek, er)


@pytest.mark.parametrize("P", [1, 2, 3])
def test_prune_local_matches_oracle(orc, P):
    from oracle import RunConfig
    from paper_2311_04333_b200.sharded_build import prune_distributed
    for name, (u, v) in _cases(orc).items():
        g = orc.build(u, v)
        for pruning in PRUNINGS:
            got = prune_distributed(_split(u, v, P), LocalComm(P, "cpu"), NumpyShard.from_rows,
                                    RunConfig(pruning=pruning), ops=HOST)
            _check_core(orc, g, pruning, got)


def test_prune_rejects_none(orc):
    from oracle import RunConfig
    from paper_2311_04333_b200.sharded_build import prune_distributed
    u, v = _cases(orc)["planted"]
    with pytest.raises(ValueError):
        prune_distributed(_split(u, v, 2), LocalComm(2, "cpu"), NumpyShard.from_rows,
                          RunConfig(pruning="none"), ops=HOST)


def _gloo_prune_worker(rank, world, port, outdir):
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "oracle"))
    import torch.distributed as dist
    from oracle import Oracle, RunConfig
    from paper_2311_04333_b200.sharded_build import prune_distributed
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        res = {}
        for name, (u, v) in _cases(orc).items():
            for pruning in PRUNINGS:
                res[f"{name}/{pruning}"] = prune_distributed(
                    [_split(u, v, world)[rank]], TorchComm("cpu"), NumpyShard.from_rows,
                    RunConfig(pruning=pruning), ops=TorchDistOps())
        np.save(os.path.join(outdir, f"res{rank}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_prune_gloo_world2(orc):
    """Every rank ends with the same gathered core (the Greedy++ replicas' input)."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_prune_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [np.load(os.path.join(d, f"res{r}.npy"), allow_pickle=True).item() for r in (0, 1)]
    for name, (u, v) in _cases(orc).items():
        g = orc.build(u, v)
        for pruning in PRUNINGS:
            for r in (0, 1):
                _check_core(orc, g, pruning, res[r][f"{name}/{pruning}"])


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 4])
def test_run_pruned_matches_run(orc, dg, P):
    """Sharded prune on CUDA shards + dg_run_pruned = run() on the whole graph
    = the oracle's run (best, witness, trace, final vertices, slack)."""
    from oracle import RunConfig as ORC
    from paper_2311_04333_b200.sharded import CudaShard
    from paper_2311_04333_b200.sharded_build import prune_distributed
    for name, (u, v) in _cases(orc).items():
        hg = orc.build(u, v)
        g = dg.Graph.from_csr(hg.offs, hg.adj, hg.orig)
        for pruning in PRUNINGS:
            for algorithm in ("peel", "sort"):
                cfg = dg.RunConfig(algorithm=algorithm, pruning=pruning, iterations=6)
                pairs = [(a.cuda(), b.cuda()) for a, b in _split(u, v, P)]
                offs, adj, orig, lab, kmax, rounds = prune_distributed(
                    pairs, LocalComm(P), CudaShard.from_rows, cfg, peer=(P > 1),
                    persistent=(P > 1))
                got = dg.run_pruned(dg.Graph.from_device_csr(offs, adj, orig),
                                    lab.cpu().numpy(), kmax, rounds, cfg)
                want = dg.run(g, cfg)
                ref = orc.run(hg, ORC(algorithm=algorithm, pruning=pruning, iterations=6))
                assert got.best == want.best
                assert (got.best.edges, got.best.verts) == tuple(ref.best)
                np.testing.assert_array_equal(got.witness, want.witness)
                assert got.witness_edges == want.witness_edges
                assert [(t.rho, t.n, t.m, t.width) for t in got.trace.iters] == \
                    [(t.rho, t.n, t.m, t.width) for t in want.trace.iters]
                np.testing.assert_array_equal(got.trace.final_vertices,
                                              want.trace.final_vertices)
                i, j = got.trace.init, want.trace.init
                assert (i.kmax, i.threshold, i.kmax_exact, i.pruned_n, i.pruned_m,
                        i.peel_rounds) == (j.kmax, j.threshold, j.kmax_exact, j.pruned_n,
                                           j.pruned_m, j.peel_rounds)
                assert got.trace.slack_violations == want.trace.slack_violations
                assert got.reprunes == want.reprunes
