"""End-to-end parity + timing on a BASELINE config, against the reference library.

usage: python tools/config_check.py CONFIG [--no-ref]
CONFIG in bench.CONFIGS (er_planted, rmat22, chunglu50m, rmat26, rmat18).
Builds the seeded graph on the GPU, runs dg.run(T), then (unless --no-ref)
runs the UNMODIFIED reference (oracle/_ref) on the downloaded CSR with all
host threads and compares best / witness / trace / final vertices and the
k-core labels bit for bit.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench  # noqa: E402
import paper_2311_04333_b200 as dg  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    name = sys.argv[1]
    cfg = bench.CONFIGS[name]
    t0 = time.time()
    g = bench.device_graph(dg, cfg)
    t_build = time.time() - t0
    dec = dg.exact_coreness(g)
    r = None
    for _ in range(2):
        r = dg.run(g, dg.RunConfig(iterations=cfg["T"]))
    out = {"config": name, "n": g.n, "m": g.m, "build_s": round(t_build, 2),
           "kmax": dec.kmax, "peel_rounds": dec.peel_rounds,
           "kcore_kernel_ms": round(r.trace.init.coreness_kernel_ms, 3),
           "core": [r.trace.init.pruned_n, r.trace.init.pruned_m],
           "best": [r.best.edges, r.best.verts], "witness": len(r.witness),
           "device_ms": round(r.device_ms, 2), "total_ms": round(r.total_ms, 2),
           "iters": [[it.n, it.m, it.batches, round(it.order_ms, 3)] for it in r.trace.iters]}
    if "--no-ref" not in sys.argv:
        from oracle import HostGraph, Reference, RunConfig
        ref = Reference()
        threads = os.cpu_count() or 1
        ref.set_threads(threads)
        offs, adj, orig = g.download()
        rg = ref.from_csr(HostGraph(offs, adj, orig))
        t = time.time()
        lab, kmax, rounds = ref.coreness(rg)
        out["ref_kcore_s"] = round(time.time() - t, 2)
        out["labels_equal"] = bool(np.array_equal(lab, dec.labels))
        out["kmax_rounds_equal"] = (kmax, rounds) == (dec.kmax, dec.peel_rounds)
        t = time.time()
        rr = ref.run(rg, RunConfig(iterations=cfg["T"]), threads=threads)
        out["ref_run_s"] = round(time.time() - t, 2)
        out["ref_iter_ms"] = [round(x, 1) for x in rr.iter_ms[:len(rr.trace)]]
        mine = [(it.iter, it.rho.edges, it.rho.verts, it.n, it.m, it.width) for it in r.trace.iters]
        out["trace_equal"] = mine == rr.trace
        out["best_equal"] = (r.best.edges, r.best.verts) == rr.best
        out["witness_equal"] = bool(np.array_equal(r.witness, rr.witness))
        out["final_equal"] = bool(np.array_equal(r.trace.final_vertices, rr.final_vertices))
        out["slack_equal"] = r.trace.slack_violations == rr.slack_violations
    print(json.dumps(out))


if __name__ == "__main__":
    main()
