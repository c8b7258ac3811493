"""One dg.run() on a bench config (profiling driver): python tools/run_once.py rmat26 [T]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2311_04333_b200 as dg  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1]]
T = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["T"]
g = bench.device_graph(dg, cfg)
r = dg.run(g, dg.RunConfig(iterations=T))
print(sys.argv[1], "best", r.best.edges, r.best.verts,
      [(it.n, it.m, it.batches, round(it.order_ms, 3)) for it in r.trace.iters])
