"""GreedySorting++ (algorithm="sort", refine.cpp:158-178) on a BASELINE config:
per-iteration device time vs the reference library on the same CSR, and the
HBM roofline of an iteration (8m + 28n + 8 algorithmic bytes).

python tools/sort_probe.py [config]    (default rmat22)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2311_04333_b200 as dg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
cfg = bench.CONFIGS[name]
g = dg.Graph.generate_rmat(22, 16 << 22, 22) if name == "rmat22" else bench.device_graph(dg, cfg)
rc = dg.RunConfig(algorithm="sort", iterations=cfg["T"])
for _ in range(2):
    r = dg.run(g, rc)
its = r.trace.iters
hbm, _ = bench.peaks()
rows = []
for t in its:
    b = 8 * t.m + 28 * t.n + 8
    rows.append({"n": t.n, "m": t.m, "ms": round(t.ms, 4), "order_ms": round(t.order_ms, 4),
                 "update_ms": round(t.update_ms, 4), "GBps": round(b / (t.ms / 1e3) / 1e9, 1)})
out = {"config": name, "algorithm": "sort", "best": [r.best.edges, r.best.verts],
       "edges_per_s": sum(t.m for t in its) / (sum(t.ms for t in its) / 1e3),
       "iters": rows, "hbm_peak_GBps": hbm}
try:
    from oracle import Reference, RunConfig as ORC
    ref = Reference()
    offs, adj, orig = g.download()
    from oracle import HostGraph
    rg = ref.from_csr(HostGraph(offs=offs, adj=adj, orig=orig))
    ro = ref.run(rg, ORC(algorithm="sort", iterations=cfg["T"]), threads=ref.max_threads())
    out["reference_iter_ms"] = [round(x, 2) for x in ro.iter_ms] if hasattr(ro, "iter_ms") else None
    out["reference_best"] = list(ro.best)
    out["best_equal"] = tuple(ro.best) == (r.best.edges, r.best.verts)
    out["witness_equal"] = bool(np.array_equal(ro.witness, r.witness))
    out["reference_threads"] = ref.max_threads()
except Exception as e:  # reference not built on this host
    out["reference"] = f"unavailable: {e}"
print(json.dumps(out))
