"""Latency floors on this B200 (dg_microbench): python tools/microbench.py"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04333_b200 as dg  # noqa: E402

NAMES = ["grid_barrier_ns", "cg_grid_sync_ns", "cluster8_sync_ns", "cta_syncthreads_ns",
         "dependent_load_4MiB_ns", "smem_atomic_per_warp_instr_ns",
         "smem_plain_rmw_per_warp_instr_ns", "dependent_load_64MiB_ns", "dependent_load_1GiB_ns",
         "cluster16_sync_ns", "cluster4_sync_ns", "smem_atom_ret_per_warp_instr_ns",
         "smem_lds_spread_per_warp_instr_ns", "smem_lds_dependent_ns", "redux_dependent_ns",
         "smem_atom_ret_dependent_ns", "smem_lds_random_tp_ns", "smem_red_random_tp_ns",
         "smem_atom_ret_random_tp_ns"]
ITERS = [20000, 20000, 100000, 1000000, 200000, 20000, 20000, 200000, 100000, 100000, 100000,
         20000, 20000, 200000, 200000, 200000, 5000, 5000, 5000]
out = {}
for i, (name, it) in enumerate(zip(NAMES, ITERS)):
    ns = C.c_double()
    st = dg.diag().dg_microbench(i, it, C.byref(ns))
    out[name] = round(ns.value, 2) if st == 0 else f"error {st}: {dg.LIB.dg_last_error().decode()}"
for i, name in zip(range(11, 19), NAMES[11:19]):  # the same in SM cycles
    v = C.c_double()
    if dg.diag().dg_microbench(100 + i, ITERS[i], C.byref(v)) == 0:
        out[name.replace("_ns", "_cycles")] = round(v.value, 2)
print(json.dumps(out))
