"""Candidate-list peel statistics of the last launch (RMAT-22, T=3)."""
import ctypes as C, numpy as np, sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04333_b200 as dg
u, v = dg.gen_rmat(22, 16 << 22, 22)
g = dg.Graph.from_pairs(u, v)
r = dg.run(g, dg.RunConfig(iterations=3))
prof = np.zeros(16, np.uint64)
dg.LIB.dg_peel_profile(prof.ctypes.data_as(C.POINTER(C.c_uint64)))
print("batches", prof[3], "rebases", prof[9], "full-scan batches", prof[10], "list batches", prof[11])
