"""compute-sanitizer driver for the cluster Greedy++ kernel and its slice cache:
compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cluster.py [n] [avg_deg]
(a dense core forced into the cluster kernel, batch and one-at-a-time, checked
against the reference restatement)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2311_04333_b200 as dg  # noqa: E402
from oracle import Oracle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 600
orc = Oracle()
u, v = orc.gen_er_planted(n, n * deg // 2, 100, 5)
h = orc.build(u, v)
g = dg.Graph.from_csr(h.offs, h.adj, h.orig)
ld = np.random.default_rng(1).integers(0, 200, h.n).astype(np.uint64)
lh = ld.copy()
dg.set_peel_mode(2)
for it in range(2):
    p = dg.load_peel_order(g, ld).perm
    assert np.array_equal(p, orc.peel_order(h, lh, False)), it
    dg.density_and_load_update(g, p, ld)
    _, lh, _, _ = orc.density_update(h, p, lh)
p = dg.load_peel_order(g, ld, one_at_a_time=True).perm
assert np.array_equal(p, orc.peel_order(h, lh, True))
print("sanitize_cluster ok", h.n, h.m)
