"""Phase cycles of the cluster Greedy++ kernel on a large core:
python tools/cluster_probe.py [scale]  (RMAT; iteration 1's ceil(kmax/2)-core)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04333_b200 as dg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # the profile is the LAST launch's
g = dg.Graph.generate_rmat(scale, 16 << scale, scale)
r = None
for _ in range(2):
    try:
        r = dg.run(g, dg.RunConfig(iterations=iters))
    except dg.DensegraphError as e:  # timing experiments may break the charges
        print("run failed after the peel kernel:", e)
it = r.trace.iters[-1] if r else None
p = np.zeros(16, np.uint64)
dg.diag().dg_peel_profile(p.ctypes.data_as(C.POINTER(C.c_uint64)))
b = max(1, int(p[3]))
if it:
    print(f"core n={it.n} m={it.m} batches={it.batches} order={it.order_ms:.2f} ms "
          f"({1e3 * it.order_ms / it.batches:.2f} us/batch)")
print("profile words:", [int(x) for x in p[:14]])
print(f"cycles/batch S1={p[0] / b:.0f} S2={p[1] / b:.0f} S3={p[2] / b:.0f}")
print(f"members that were their CTA's candidate one batch earlier: simple batches {int(p[9])}/{int(p[10])}, "
      f"general batches (owner CTAs) {int(p[11])}/{int(p[12])}")
