#!/usr/bin/env python3
"""bench.py -- Greedy++ edges/s per iteration and k-core edges/s on B200.

Workload (BASELINE.json configs[1], the metric's N=1 config): RMAT scale 22,
edge factor 16 (67,108,864 seeded samples, a=.57 b=.19 c=.19 d=.05),
symmetrised / deduplicated / loop-free u32 CSR; exact k-core -> ceil(kmax/2)-core
-> Greedy++ T=20 (eps=0.05 is advisory: explicit T wins, framework.cpp:99-104)
with adaptive re-pruning -> witness.  One STEP = that whole hot path on the
resident CSR.  Inputs are synthetic (seeded generators; no dataset).

  value   Greedy++ edges/s per iteration = sum_it m_cur / sum_it t_iter over the
          timed steps, t_iter = CUDA-event time of ordering + Alg. 3
  kcore   k-core edges/s = m / t(k-core kernel), CUDA events
  e2e     the same numerator through the C ABI from pinned HOST buffers:
          H2D of the CSR + k-core + prune + T iterations + D2H of the results,
          wall-clocked -- every overhead is charged to the iterations
  roofline  dominant kernel (the Greedy++ batch-peel kernel) against the
          measured HBM copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline  the unmodified reference library (oracle/_ref) on this host

--impl reference runs only the reference library (rank 0), same metric.
Multi-GPU (torchrun): every rank runs the full step on its own GPU
("replicas", weak scaling), timing = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

METRIC = "Greedy++ edges/sec per iteration and k-core edges/sec; % of HBM roofline"
CONFIGS = {
    # BASELINE.json configs[1]
    "rmat22": dict(kind="rmat", scale=22, edge_factor=16, seed=22, T=20, eps=0.05),
    # configs[0] (ER n=100k m=1M + planted 300-block p=0.5), T=10
    "er_planted": dict(kind="er", n=100000, m=1000000, block=300, seed=1, T=10, eps=0.1),
    # configs[3]: RMAT-26, T=10
    "rmat26": dict(kind="rmat", scale=26, edge_factor=16, seed=26, T=10, eps=0.1),
    # configs[2]: Chung-Lu n=50M, 500M endpoint pairs, exponent 2.1, T=20
    "chunglu50m": dict(kind="cl", n=50_000_000, pairs=500_000_000, seed=50, T=20, eps=0.05),
    # configs[4]: RMAT-28 (4.3e9 samples), T=5 -- listed for 2-8 GPUs; fits one
    # B200 through the streamed build
    "rmat28": dict(kind="rmat", scale=28, edge_factor=16, seed=28, T=5, eps=0.1),
    # small config for quick checks / profiling
    "rmat18": dict(kind="rmat", scale=18, edge_factor=16, seed=18, T=20, eps=0.05),
}


def traffic():
    """DRAM bytes per launch of the hot kernels from the committed ncu captures."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.samples, self.proc, self.t = [], None, None
        self.window = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append((time.time(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0: float, t1: float):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inwin = [p for (t, p) in self.samples if t0 - 0.15 <= t <= t1 + 0.15] or \
                [p for (_, p) in self.samples]
        if not inwin:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = sorted(float(p[0]) for p in inwin if p[0].replace(".", "").isdigit())
        mx = max((float(p[1]) for p in inwin if p[1].replace(".", "").isdigit()), default=None)
        reasons = sorted({names[i] for p in inwin for i in range(4) if p[2 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(inwin)}


# ------------------------------------------------------------------ distributed plumbing
def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(n: int) -> int:
    """`bench.py --gpus N` without torchrun: launch N ranks of this same
    command line on this node (torchrun, 127.0.0.1) and return their status."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_init(force: bool = False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world == 1 and force:  # the sharded pipeline on one rank (its own process group)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(free_port()))
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    if world > 1 or force:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.barrier()
        torch.cuda.synchronize()


def allreduce(vals, op, world, local):
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.tolist()


# ------------------------------------------------------------------ inputs
def host_pairs(cfg):
    """Seeded pairs on the host (oracle generators; used by the reference arm)."""
    from oracle import Oracle
    orc = Oracle()
    if cfg["kind"] == "rmat":
        return orc.gen_rmat(cfg["scale"], cfg["edge_factor"] << cfg["scale"], cfg["seed"])
    if cfg["kind"] == "er":
        return orc.gen_er_planted(cfg["n"], cfg["m"], cfg["block"], cfg["seed"])
    return orc.gen_chung_lu(cfg["n"], cfg["pairs"], cfg["seed"])


def device_graph(dg, cfg):
    """The seeded graph built on the device straight from the generator
    (dg_graph_generate: no pair arrays, source-range parts)."""
    if cfg["kind"] == "er":
        u, v = host_pairs(cfg)
        return dg.Graph.from_pairs(u, v)
    if cfg["kind"] == "rmat":
        return dg.Graph.generate_rmat(cfg["scale"], cfg["edge_factor"] << cfg["scale"], cfg["seed"])
    return dg.Graph.generate_chung_lu(cfg["n"], cfg["pairs"], cfg["seed"])


def pinned_copy(a):
    import numpy as np
    import torch
    t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
    out = t.numpy().view(a.dtype)
    np.copyto(out, a)
    return out, t


# ------------------------------------------------------------------ reference arm
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_graph(cfg):
    """The seeded graph as a host CSR, built on the CPU (no GPU code): RMAT by
    the OpenMP builder og_par.c (checked equal to the oracle build and to the
    device CSR), the others by the sequential oracle build."""
    if cfg["kind"] == "rmat":
        from oracle import rmat_graph_par
        return rmat_graph_par(cfg["scale"], cfg["edge_factor"] << cfg["scale"], cfg["seed"])
    from oracle import Oracle
    u, v = host_pairs(cfg)
    return Oracle().build(u, v)


def run_reference(args, cfg, rank, world):
    """The reference's own CPU implementation (oracle/_ref = the unmodified
    densegraph library) on the same seeded graph, all host threads.

    A STEP is one Greedy++ iteration of the reference's run() (framework.cpp:
    105-153; IterRecord.ms = its ordering + Algorithm 3), the same unit our
    arm sums: run() is called ceil((W+K)/T) times back to back, the first W
    iterations are warm-up, the next K are timed; value = sum m_cur / sum
    IterRecord.ms.  k-core edges/s = m / one timed exact_coreness."""
    if rank != 0:
        return 0
    from oracle import Reference, RunConfig, reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference", "metric": METRIC,
                          "unavailable": "oracle/_ref/libdgref.so was not built (needs /root/reference at build time)"}))
        return 0
    ref = Reference()
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    t0 = time.perf_counter()
    h = host_graph(cfg)
    build_s = time.perf_counter() - t0
    n, m = h.n, h.m
    rg = ref.from_csr(h)
    del h
    t0 = time.perf_counter()
    ref.coreness(rg)
    kc_s = time.perf_counter() - t0
    T = cfg["T"]
    need = args.warmup + args.steps
    rcfg = RunConfig(iterations=T, epsilon=cfg["eps"])
    its, run_ms, last = [], [], None
    while len(its) < need:
        t0 = time.perf_counter()
        last = ref.run(rg, rcfg, threads=threads)
        run_ms.append((time.perf_counter() - t0) * 1e3)
        its += [(t[4], ms) for t, ms in zip(last.trace, last.iter_ms)]
    timed = its[args.warmup:need]
    edges = sum(e for e, _ in timed)
    ms = sum(x for _, x in timed)
    value = edges / (ms / 1e3)
    sample = (f"{args.steps} timed Greedy++ iterations (after {args.warmup} warm-up) of "
              f"{len(run_ms)} back-to-back reference run()s (T={T}), value = sum m_cur / "
              f"sum IterRecord.ms; k-core = one exact_coreness")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / len(timed), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(args.config, cfg, n, m, world),
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": threads, "kind": "reference",
                         "cpu": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "kcore": {"value": m / kc_s, "unit": "edges/s", "ms": kc_s * 1e3},
        "reference_detail": {"host_build_s": round(build_s, 2), "run_ms": run_ms,
                             "init_ms": last.times[1], "coreness_ms_incl_get_core": last.times[0],
                             "iter_ms": [round(x, 2) for _, x in its]},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(name, cfg, n, m, world):
    c = {"workload": f"{name}: exact k-core prune + Greedy++ T={cfg['T']} (eps={cfg['eps']} advisory)",
         "n": int(n), "m": int(m), "T": cfg["T"], "epsilon": cfg["eps"], "seed": cfg["seed"],
         "l2": "flushed between steps (256 MiB memset); CSR also exceeds L2",
         "parallelism": f"replicas x{world}" if world > 1 else "1 GPU"}
    if cfg["kind"] == "rmat":
        c.update(generator="RMAT a=.57 b=.19 c=.19 d=.05", scale=cfg["scale"],
                 samples=cfg["edge_factor"] << cfg["scale"])
    elif cfg["kind"] == "er":
        c.update(generator="ER + planted block p=0.5", block=cfg["block"])
    else:
        c.update(generator="Chung-Lu power law exponent 2.1", pairs=cfg["pairs"])
    return c


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg, rank, world, local):
    import numpy as np
    import paper_2311_04333_b200 as dg
    dg.set_device(local)
    hbm, peak_kind = peaks()
    g = device_graph(dg, cfg)
    n, m = g.n, g.m
    rcfg = dg.RunConfig(iterations=cfg["T"], epsilon=cfg["eps"])
    for _ in range(args.warmup):
        dg.run(g, rcfg)
    clocks = Clocks(local)
    time.sleep(0.25)
    res = []
    launches0 = dg.launch_count()
    barrier(world)
    dg.synchronize()
    t_start = time.time()
    for _ in range(args.steps):
        dg.flush_l2()
        res.append(dg.run(g, rcfg))
    dg.synchronize()
    barrier(world)
    t_end = time.time()
    launches = dg.launch_count() - launches0
    clk = clocks.summary(t_start, t_end)
    clocks.stop()

    iters = [it for r in res for it in r.trace.iters]
    edges = sum(it.m for it in iters)
    it_ms = sum(it.ms for it in iters)          # t_iter = ordering + Alg. 3 (CUDA events)
    order_ms = sum(it.order_ms for it in iters)
    batches = sum(it.batches for it in iters)
    # B_it = 8(n+1) offs + 8m adj + 16n loads r+w + 4n perm = 8m + 28n + 8
    it_bytes = sum(8 * (it.n + 1) + 8 * it.m + 16 * it.n + 4 * it.n for it in iters)
    # the peel kernel alone: offs + adj + loads read + perm + raw charges written
    peel_bytes = sum(8 * (it.n + 1) + 8 * it.m + 8 * it.n + 4 * it.n + 8 * it.n for it in iters)
    kc_ms = sum(r.trace.init.coreness_kernel_ms for r in res)
    dev_ms = sum(r.device_ms for r in res)
    # max over ranks for times, sum for work
    it_ms_max, kc_ms_max, dev_ms_max, order_ms_max = allreduce([it_ms, kc_ms, dev_ms, order_ms],
                                                               "max", world, local)
    edges_all, kc_edges_all = allreduce([float(edges), float(m * args.steps)], "sum", world, local)
    value = edges_all / (it_ms_max / 1e3)
    kcore_value = kc_edges_all / (kc_ms_max / 1e3)
    it_achieved = it_bytes / (it_ms / 1e3) / 1e9
    peel_achieved = peel_bytes / (order_ms / 1e3) / 1e9
    # B_kc = 8(n+1) offs + 8m adj + 4n degree init + 4n labels; the timed
    # region holds the degree-init kernel, the bitmap fill and the k-core kernel
    kc_bytes = 8 * m + 16 * n + 8
    kc_achieved = kc_bytes * args.steps / (kc_ms / 1e3) / 1e9
    big = max(iters, key=lambda it: it.n * 1.0 * it.ms)
    peel_kernel = "k_peel_cluster" if big.n > 16384 else "k_peel"
    tr = traffic()

    line = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": workload_config(args.config, cfg, n, m, world),
        "kcore": {"value": kcore_value, "unit": "edges/s",
                  "ms": kc_ms / args.steps, "peel_rounds": res[0].trace.init.peel_rounds,
                  "kmax": res[0].trace.init.kmax,
                  "roofline": {"bound": "hbm", "achieved": kc_achieved, "peak": hbm,
                               "unit": "GB/s", "frac": kc_achieved / hbm,
                               "algorithmic_bytes": kc_bytes, "peak_kind": peak_kind,
                               "kernel": "k_coreness (+ k_init_deg, bitmap fill)",
                               "traffic": tr.get(f"k_coreness_{args.config}", {}).get(
                                   "dram_bytes_per_launch")}},
        "roofline": {"bound": "hbm", "achieved": it_achieved, "peak": hbm, "unit": "GB/s",
                     "frac": it_achieved / hbm,
                     "traffic": tr.get(f"{peel_kernel}_{args.config}", {}).get("dram_bytes_per_launch"),
                     "traffic_note": tr.get(f"{peel_kernel}_{args.config}", {}).get("launch"),
                     "kernel": f"Greedy++ iteration: {peel_kernel} (batch peel, fused Alg.3 charges) + k_alg3",
                     "bytes_per_iteration": "8(n+1) offs + 8m adj + 16n loads r+w + 4n perm (SURVEY 8d)",
                     "time": "t_iter = CUDA events around ordering + Alg. 3, summed over the timed iterations",
                     "peel_kernel_only": {"achieved": peel_achieved, "frac": peel_achieved / hbm,
                                          "bytes": "8(n+1) + 8m + 8n loads + 4n perm + 8n raw charges",
                                          "time": "ordering events only"},
                     "peak_kind": peak_kind},
        "greedy": {"iterations": len(iters),
                   "batches_per_iter": batches / max(1, len(iters)),
                   "us_per_batch": order_ms * 1e3 / max(1, batches),
                   "order_ms_per_iter": order_ms / max(1, len(iters)),
                   "update_ms_per_iter": (it_ms - order_ms) / max(1, len(iters)),
                   "per_iteration": [[it.n, it.m, it.batches, round(it.ms, 3)]
                                     for it in res[0].trace.iters],
                   "core_n_m": [res[0].trace.init.pruned_n, res[0].trace.init.pruned_m],
                   "reprunes": res[0].reprunes,
                   "best": [res[0].best.edges, res[0].best.verts],
                   "witness_size": len(res[0].witness)},
        "gpu_launches": int(launches),
        "clocks": clk,
        # where one step's device time goes (ms, mean over the timed steps)
        "step_split": {
            "kcore_kernel": kc_ms / args.steps,
            "coreness_incl_get_core": sum(r.trace.init.coreness_ms for r in res) / args.steps,
            "init_total": sum(r.trace.init.init_ms for r in res) / args.steps,
            "iterations": it_ms / args.steps,
            "reprune": sum(r.reprune_ms for r in res) / args.steps,
            "host_total": sum(r.total_ms for r in res) / args.steps,
            "device_total": dev_ms / args.steps},
    }

    # ---- the GreedySorting++ variant on the same graph,
    # outside the timed region: informational, same edges/s definition
    sres = dg.run(g, dg.RunConfig(algorithm="sort", iterations=cfg["T"], epsilon=cfg["eps"]))
    s_edges = sum(it.m for it in sres.trace.iters)
    s_ms = sum(it.ms for it in sres.trace.iters)
    line["sort_variant"] = {"value": s_edges / (s_ms / 1e3), "unit": "edges/s",
                            "ms_per_iter": s_ms / max(1, len(sres.trace.iters)),
                            "best": [sres.best.edges, sres.best.verts],
                            "note": "algorithm=sort (refine.cpp:158-178), not the headline"}

    # ---- e2e through the C ABI from pinned host buffers
    offs, adj, orig = g.download()
    p_offs, _t1 = pinned_copy(offs)
    p_adj, _t2 = pinned_copy(adj)
    p_orig, _t3 = pinned_copy(orig)
    e2e_edges = e2e_s = 0.0
    d2h = 0
    e2e_steps = []
    for _ in range(max(1, min(args.steps, 5))):
        dg.flush_l2()
        dg.synchronize()
        t0 = time.perf_counter()
        g2 = dg.Graph.from_csr(p_offs, p_adj, p_orig)
        r = dg.run(g2, rcfg)
        del g2
        dt = time.perf_counter() - t0
        e2e_steps.append(round(1e3 * dt, 2))
        e2e_s += dt
        e2e_edges += sum(it.m for it in r.trace.iters)
        d2h = 8 * (len(r.witness) + len(r.trace.final_vertices)) + 80 * len(r.trace.iters) + 64
    e2e_s = allreduce([e2e_s], "max", world, local)[0]
    e2e_edges = allreduce([e2e_edges], "sum", world, local)[0]
    line["e2e"] = {"value": e2e_edges / e2e_s, "unit": "edges/s",
                   "h2d_bytes_per_step": int(p_offs.nbytes + p_adj.nbytes + p_orig.nbytes),
                   "d2h_bytes_per_step": int(d2h),
                   "step_ms": e2e_steps,
                   "includes": "H2D CSR + k-core + prune + T iterations + witness recount + D2H"}

    # ---- CPU baseline: the reference library on this host (rank 0, N=1)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, offs, adj, orig)
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm, N GPUs
def run_sharded(args, cfg, rank, world, local):
    """The multi-GPU pipeline on the SAME graph (strong scaling):
    every rank generates its slice of the seeded samples on its GPU ->
    distributed CSR build (library kernels + NCCL all-to-all) -> sharded exact
    k-core as ONE persistent kernel per GPU (peer memory over NVLink,
    device-side cross-GPU barrier) -> per-shard get_core -> the core
    all-gathered -> Greedy++ T iterations (replicated on every rank: one
    exact minimum per batch does not shard).  A step is the whole
    pipeline; times are CUDA events / device clocks, max over ranks."""
    import numpy as np
    import torch
    import paper_2311_04333_b200 as dg
    from paper_2311_04333_b200.sharded import CudaShard, TorchComm
    from paper_2311_04333_b200.sharded_build import peer_capable, prune_distributed
    if cfg["kind"] != "rmat":
        raise SystemExit("the multi-GPU pipeline generates RMAT slices per rank (rmat* configs)")
    dg.set_device(local)
    dev = torch.device("cuda", local)
    hbm, peak_kind = peaks()
    S = cfg["edge_factor"] << cfg["scale"]
    k0, k1 = S * rank // world, S * (rank + 1) // world
    peer = peer_capable() if world > 1 else True
    rcfg = dg.RunConfig(iterations=cfg["T"], epsilon=cfg["eps"])
    comm = TorchComm(dev)

    def step():
        u = torch.empty(k1 - k0, dtype=torch.int64, device=dev)
        v = torch.empty(k1 - k0, dtype=torch.int64, device=dev)
        dg.gen_rmat_range(cfg["scale"], k0, k1 - k0, cfg["seed"], (u.data_ptr(), v.data_ptr()))
        torch.cuda.synchronize(dev)
        tm = {}
        offs, adj, orig, lab, kmax, rounds = prune_distributed(
            [(u, v)], comm, CudaShard.from_rows, rcfg, peer=peer, persistent=peer, timings=tm)
        del u, v
        r = dg.run_pruned(dg.Graph.from_device_csr(offs, adj, orig), lab.cpu().numpy(), kmax,
                          rounds, rcfg)
        return r, tm

    for _ in range(args.warmup):
        step()
    clocks = Clocks(local)
    time.sleep(0.25)
    barrier(world)
    t_start = time.time()
    res, prune_s = [], []
    launches0 = dg.launch_count()
    for _ in range(args.steps):
        barrier(world)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r, tm = step()
        dg.synchronize()
        torch.cuda.synchronize(dev)
        e1.record()
        e1.synchronize()
        barrier(world)
        res.append((r, tm, e0.elapsed_time(e1) / 1e3))  # device-observed seconds
    t_end = time.time()
    clk = clocks.summary(t_start, t_end)
    clocks.stop()
    launches = dg.launch_count() - launches0
    iters = [it for r, _, _ in res for it in r.trace.iters]
    edges = sum(it.m for it in iters)
    it_ms = sum(it.ms for it in iters)
    step_s = sum(x for _, _, x in res)
    pr_s = sum(t["build_s"] + t["coreness_s"] + t["get_core_gather_s"] for _, t, _ in res)
    kc_ms = sum(t["coreness_kernel_ms"] or 0.0 for _, t, _ in res)
    bd_s = sum(t["build_s"] for _, t, _ in res)
    it_ms_max, step_max, pr_max, kc_max, bd_max = allreduce([it_ms, step_s, pr_s, kc_ms, bd_s],
                                                            "max", world, local)
    r0, t0_ = res[0][0], res[0][1]
    n, m = t0_["n"], t0_["m"]
    kc_bytes = 8 * m + 16 * n + 8
    line = {
        "metric": METRIC, "value": edges / (it_ms_max / 1e3), "unit": "edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": dict(workload_config(args.config, cfg, n, m, world),
                       parallelism=f"1D vertex-range shards x{world} (k-core), Greedy++ replicated",
                       pipeline="per-rank generation -> distributed CSR build -> persistent sharded "
                                "k-core -> per-shard get_core -> core all-gather -> Greedy++"),
        "kcore": {"value": m * args.steps / (kc_max / 1e3) if kc_max else None, "unit": "edges/s",
                  "ms": kc_max / args.steps,
                  "kernel": "k_shard_coreness (one persistent kernel per GPU)",
                  "roofline": {"bound": "hbm", "achieved": kc_bytes * args.steps / (kc_max / 1e3) / 1e9
                               / world if kc_max else None, "peak": hbm, "unit": "GB/s",
                               "frac": kc_bytes * args.steps / (kc_max / 1e3) / 1e9 / world / hbm
                               if kc_max else None, "peak_kind": peak_kind,
                               "note": "per GPU: algorithmic bytes / N / time"}},
        "sharded": {"time_to_solution_ms": 1e3 * step_max / args.steps,
                    "build_ms": 1e3 * bd_max / args.steps,
                    "build_kcore_prune_gather_ms": 1e3 * pr_max / args.steps,
                    "kcore_rounds": r0.trace.init.peel_rounds, "kmax": r0.trace.init.kmax,
                    "peer_memory": bool(peer),
                    "core_n_m": [r0.trace.init.pruned_n, r0.trace.init.pruned_m],
                    "best": [r0.best.edges, r0.best.verts]},
        "greedy": {"iterations": len(iters), "ms_per_iter": it_ms_max / max(1, len(iters))},
        # Greedy++ iteration roofline as at N=1 (8m + 28n + 8 bytes over t_iter)
        "roofline": {"bound": "hbm",
                     "achieved": sum(8 * it.m + 28 * it.n + 8 for it in iters) / (it_ms / 1e3) / 1e9,
                     "peak": hbm, "unit": "GB/s",
                     "frac": sum(8 * it.m + 28 * it.n + 8 for it in iters) / (it_ms / 1e3) / 1e9 / hbm,
                     "traffic": None, "peak_kind": peak_kind,
                     "kernel": "Greedy++ iteration (replicated): k_peel_cluster / k_peel + k_alg3"},
        # the sharded pipeline has no host input: every rank generates its slice of the
        # seeded samples on its GPU, so this is the whole pipeline (generation, build,
        # k-core, prune, gather, T iterations) timed on the device, not a host-buffer e2e
        "e2e": {"value": edges / step_max, "unit": "edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": int(4 * n),
                "includes": "per-rank generation + distributed build + sharded k-core + prune + "
                            "gather + T iterations; labels read back to the host"},
        "gpu_launches": int(launches),
        "clocks": clk,
        "value_note": "Greedy++ runs replicated on the gathered core: value counts one replica's "
                      "edges (the others are redundant), time = max over ranks",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(cfg, offs, adj, orig):
    from oracle import HostGraph, Reference, RunConfig, reference_available
    if not reference_available():
        return {"value": None, "unit": "edges/s", "cores": 0, "kind": "reference",
                "cpu": cpu_model(), "sample": "unavailable: oracle/_ref not built"}
    ref = Reference()
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    rg = ref.from_csr(HostGraph(offs, adj, orig))
    n, m, _ = rg.info()
    t0 = time.perf_counter()
    ref.coreness(rg)
    kc_s = time.perf_counter() - t0
    r = ref.run(rg, RunConfig(iterations=cfg["T"], epsilon=cfg["eps"]), threads=threads)
    edges = sum(t[4] for t in r.trace)
    return {"value": edges / (sum(r.iter_ms) / 1e3), "unit": "edges/s", "cores": threads,
            "kind": "reference", "cpu": cpu_model(),
            "sample": f"one full reference run() (T={cfg['T']}) + one exact_coreness on the same graph",
            "kcore_value": m / kc_s, "run_total_ms": r.times[2], "init_ms": r.times[1]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="rmat26", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--sharded", action="store_true",
                    help="run the multi-GPU pipeline even on one rank (tests its plumbing)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)
    sharded = args.impl == "ours" and (args.gpus > 1 or args.sharded)
    rank, world, local = dist_init(force=sharded)
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        rc = run_reference(args, cfg, rank, world)
    elif sharded:
        rc = run_sharded(args, cfg, rank, world, local)
    else:
        rc = run_ours(args, cfg, rank, world, local)
    if world > 1 or sharded:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
