"""Breakdown of one bench e2e step (pinned-host CSR -> from_csr -> run -> free)."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_2311_04333_b200 as dg
import bench
u, v = dg.gen_rmat(22, 16 << 22, 22)
g = dg.Graph.from_pairs(u, v); del u, v
offs, adj, orig = g.download()
p_offs, _a = bench.pinned_copy(offs); p_adj, _b = bench.pinned_copy(adj); p_orig, _c = bench.pinned_copy(orig)
cfg = dg.RunConfig(iterations=20)
for k in range(4):
    dg.flush_l2(); dg.synchronize()
    t0 = time.perf_counter(); g2 = dg.Graph.from_csr(p_offs, p_adj, p_orig); dg.synchronize(); t1 = time.perf_counter()
    r = dg.run(g2, cfg); t2 = time.perf_counter()
    del g2; dg.synchronize(); t3 = time.perf_counter()
    print(f"from_csr {1e3*(t1-t0):.1f} ms  run {1e3*(t2-t1):.1f} ms (device {r.device_ms:.1f}, total {r.total_ms:.1f}, coreness {r.trace.init.coreness_ms:.1f})  free {1e3*(t3-t2):.1f} ms")
it = r.trace.iters
print(f"kcore kernel {r.trace.init.coreness_kernel_ms:.2f} ms; init {r.trace.init.init_ms:.1f} ms; "
      f"iter sum {sum(t.ms for t in it):.1f} ms (order {sum(t.order_ms for t in it):.1f}); "
      f"reprune {r.reprune_ms:.1f} ms x{r.reprunes}; it1 {it[0].ms:.2f} ms n={it[0].n}; "
      f"it2+ {sum(t.ms for t in it[1:]):.1f} ms")
