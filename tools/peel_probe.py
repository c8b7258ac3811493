"""Per-iteration Greedy++ timing probe: python tools/peel_probe.py [scale] [T]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04333_b200 as dg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
T = int(sys.argv[2]) if len(sys.argv) > 2 else 20
if os.environ.get("DG_PEEL_MODE"):  # e.g. 3: candidate-list kernel for every core
    dg.set_peel_mode(int(os.environ["DG_PEEL_MODE"]))
u, v = dg.gen_rmat(scale, 16 << scale, scale)
g = dg.Graph.from_pairs(u, v)
del u, v
for rep in range(2):
    r = dg.run(g, dg.RunConfig(iterations=T))
print(f"n={g.n} m={g.m} kmax={r.trace.init.kmax} rounds={r.trace.init.peel_rounds} "
      f"kcore_kernel_ms={r.trace.init.coreness_kernel_ms:.3f} coreness_ms={r.trace.init.coreness_ms:.3f} "
      f"device_ms={r.device_ms:.2f} total_ms={r.total_ms:.2f} reprune_ms={r.reprune_ms:.2f}")
import ctypes as C  # noqa: E402
import numpy as np  # noqa: E402
for it in r.trace.iters:
    print(f"it{it.iter:3d} n={it.n:7d} m={it.m:10d} batches={it.batches:6d} order={it.order_ms:8.3f}ms "
          f"upd={it.update_ms:6.3f}ms us/batch={1e3 * it.order_ms / max(1, it.batches):6.2f} "
          f"arcs/batch={2 * it.m / max(1, it.batches):8.0f}")

# instrumented rerun of the last iteration's core (cycle split; timeline window unreachable)
dg._chk(dg.diag().dg_peel_trace_arm(0xFFFFFFF0))
dg.run(g, dg.RunConfig(iterations=T))
dg._chk(dg.diag().dg_peel_trace_arm(0xFFFFFFFF))
prof = np.zeros(16, np.uint64)
dg.diag().dg_peel_profile(prof.ctypes.data_as(C.POINTER(C.c_uint64)))
tot = max(1, int(prof[:3].sum()))
print(f"last peel launch: batches={prof[3]} cycles/batch S1={prof[0]/max(1,prof[3]):.0f} "
      f"S2={prof[1]/max(1,prof[3]):.0f} S3={prof[2]/max(1,prof[3]):.0f} "
      f"(split {100*prof[0]/tot:.0f}/{100*prof[1]/tot:.0f}/{100*prof[2]/tot:.0f}%) "
      f"single-vertex batches={prof[5]} S3/single={prof[4]/max(1,prof[5]):.0f} "
      f"S3/multi={(prof[2]-prof[4])/max(1,prof[3]-prof[5]):.0f} big={prof[6]} table-path={prof[8]}")
if len(sys.argv) > 3:  # also time iteration 1's core with the other kernel mode
    mode = int(sys.argv[3])
    dg.set_peel_mode(mode)
    r = dg.run(g, dg.RunConfig(iterations=2))
    it = r.trace.iters[0]
    dg.diag().dg_peel_profile(prof.ctypes.data_as(C.POINTER(C.c_uint64)))
    print(f"mode {mode}: it1 n={it.n} batches={it.batches} order={it.order_ms:.3f}ms "
          f"us/batch={1e3 * it.order_ms / max(1, it.batches):.2f}")
    print(f"  last launch (it2) cycles/batch S1={prof[0]/max(1,prof[3]):.0f} "
          f"S2={prof[1]/max(1,prof[3]):.0f} S3={prof[2]/max(1,prof[3]):.0f} CS={prof[7]}")
    dg.set_peel_mode(0)
