"""Candidate-list peel statistics of the last launch: python tools/queue_stats.py [T] (RMAT-22)."""
import ctypes as C, numpy as np, sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04333_b200 as dg
u, v = dg.gen_rmat(22, 16 << 22, 22)
g = dg.Graph.from_pairs(u, v)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 3
r = dg.run(g, dg.RunConfig(iterations=T))
prof = np.zeros(16, np.uint64)
dg.diag().dg_peel_profile(prof.ctypes.data_as(C.POINTER(C.c_uint64)))
print("batches", prof[3], "rebases", prof[9], "full-scan batches", prof[10], "list batches", prof[11])
