"""Multi-GPU paths on >= 2 GPUs (skipped on a one-GPU box): one process per
GPU over NCCL, shards linked by CUDA IPC (NVLink peer memory), the
device-resident sharded k-core (one persistent kernel per GPU meeting the
others at the cross-GPU barrier), the distributed CSR build and per-shard
get_core, Greedy++ replicas -- against run() on one GPU; and `bench.py
--gpus 2` self-launching its ranks."""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


need2 = pytest.mark.skipif(_ngpus() < 2, reason="needs two GPUs")


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_2311_04333_b200 as dg
    from paper_2311_04333_b200.sharded_build import run_distributed
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dg.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        S = 16 << 16
        k0, k1 = S * rank // world, S * (rank + 1) // world
        u = torch.empty(k1 - k0, dtype=torch.int64, device="cuda")
        v = torch.empty(k1 - k0, dtype=torch.int64, device="cuda")
        dg.gen_rmat_range(16, k0, k1 - k0, 16, (u.data_ptr(), v.data_ptr()))
        out = {}
        for persistent in (True, False):
            r = run_distributed(u, v, dg.RunConfig(iterations=5), persistent=persistent)
            out[persistent] = ((r.best.edges, r.best.verts), r.witness.tolist(),
                               [(t.rho.edges, t.rho.verts, t.n, t.m, t.width)
                                for t in r.trace.iters],
                               r.trace.init.peel_rounds, r.trace.init.kmax)
        np.save(os.path.join(outdir, f"r{rank}.npy"), out, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@need2
def test_run_distributed_two_gpus(dg):
    import torch.multiprocessing as mp
    from test_sharded import _free_port
    g = dg.Graph.generate_rmat(16, 16 << 16, 16)
    want = dg.run(g, dg.RunConfig(iterations=5))
    w = ((want.best.edges, want.best.verts), want.witness.tolist(),
         [(t.rho.edges, t.rho.verts, t.n, t.m, t.width) for t in want.trace.iters],
         want.trace.init.peel_rounds, want.trace.init.kmax)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        for r in (0, 1):
            got = np.load(os.path.join(d, f"r{r}.npy"), allow_pickle=True).item()
            assert got[True] == w and got[False] == w


@need2
def test_bench_two_gpus():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--config", "rmat18", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["sharded"]["kcore_rounds"] > 0


def test_bench_sharded_pipeline_one_rank():
    """The multi-GPU pipeline's plumbing on one rank (its own process group)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--sharded",
                        "--config", "rmat18", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["scaling"] == "strong"
    assert line["sharded"]["best"][1] > 0 and line["kcore"]["value"] > 0
