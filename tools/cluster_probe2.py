"""Cluster Greedy++ kernel phase split (rank-0 thread-0 cycles per batch).

python tools/cluster_probe2.py [scale] [T...]   (dg_set_peel_mode(2))
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04333_b200 as dg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
Ts = [int(x) for x in sys.argv[2:]] or [1, 3]
g = dg.Graph.generate_rmat(scale, 16 << scale, scale)
dg.set_peel_mode(2)
for T in Ts:
    r = dg.run(g, dg.RunConfig(iterations=T))
    r = dg.run(g, dg.RunConfig(iterations=T))
    prof = np.zeros(16, np.uint64)
    dg.diag().dg_peel_profile(prof.ctypes.data_as(C.POINTER(C.c_uint64)))
    nb = max(1, int(prof[3]))
    it = r.trace.iters[-1]
    print(f"T={T} CS={prof[7]} n={it.n} batches={nb} simple={prof[4]} order={it.order_ms:.3f} ms "
          f"({1e3 * it.order_ms / nb:.2f} us/batch) cycles/batch S1={prof[0] / nb:.0f} "
          f"S2={prof[1] / nb:.0f} S3={prof[2] / nb:.0f}; batches beyond 32 members: {prof[5]} "
          f"({prof[8]} members, {prof[6] / max(1, int(prof[5])):.0f} cycles each)")
    if os.environ.get("DG_STAMPS"):
        ng = max(1, nb - int(prof[4]))
        print("  general batches: cycles per batch (owner loop, CTA barrier, member wait, removal):",
              [round(float(prof[12 + k]) / ng) for k in range(4)])
dg.set_peel_mode(0)
