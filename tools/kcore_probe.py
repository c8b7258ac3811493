"""k-core phase split: python tools/kcore_probe.py [scale | bench config name]"""
import ctypes as C
import os
os.environ["DG_KCORE_PROFILE"] = "1"  # the instrumented k-core variant
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04333_b200 as dg  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "22"
if arg.isdigit():
    scale = int(arg)
    g = dg.Graph.generate_rmat(scale, 16 << scale, scale)
else:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench  # noqa: E402
    g = bench.device_graph(dg, bench.CONFIGS[arg])
for _ in range(2):
    r = dg.run(g, dg.RunConfig(iterations=1))
p = np.zeros(8 + 6 * 4096, np.uint64)
dg.diag().dg_kcore_profile(p.ctypes.data_as(C.POINTER(C.c_uint64)))
ghz = 1.965e3
names = ["lvl_min", "lvl_sync", "collect", "expand", "flush", "exp_sync"]
print(f"n={g.n} m={g.m} rounds={r.trace.init.peel_rounds} kmax={r.trace.init.kmax} "
      f"kernel_ms={r.trace.init.coreness_kernel_ms:.3f} levels={p[6]} ovf_collects={p[7]}")
print("  " + " ".join(f"{k}={p[i] / ghz / 1e3:.3f}ms" for i, k in enumerate(names)))

R = int(r.trace.init.peel_rounds)
tr = p[8:8 + 3 * min(R, 4096)].reshape(-1, 3).astype(np.int64)
cyc, fc, ftot = tr[:, 0], tr[:, 1] & 0xffffffff, tr[:, 2]
alive = tr[:, 1] >> 32
order = np.argsort(-cyc)
print(f"  per-round expand: mean {cyc.mean()/ghz:.2f}us median {np.median(cyc)/ghz:.2f}us; "
      f"top-20 rounds hold {100*cyc[order[:20]].sum()/cyc.sum():.1f}% of expand time")
for i in order[:8]:
    print(f"    round {i+1}: {cyc[i]/ghz:.1f}us Fc={fc[i]} arcs={ftot[i]} alive={alive[i]}")
for A in (16384, 32768, 65536, 131072):
    sel = alive <= A
    print(f"  rounds with <= {A} alive: {sel.sum()} taking {cyc[sel].sum()/ghz/1e3:.2f}ms expand, "
          f"{ftot[sel].sum()/1e6:.0f}M arcs")
for lim in (1024, 4096, 16384, 65536, 262144):
    sel = ftot < lim
    print(f"  rounds with < {lim} arcs: {sel.sum()} ({cyc[sel].sum()/ghz/1e3:.2f} ms expand)")
print("  by round size (arcs): rounds, expand ms, us/round, G arcs/s")
for lo in (0, 1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24, 1 << 26):
    sel = (ftot >= lo) & (ftot < lo * 4 if lo else ftot < (1 << 12))
    if sel.any():
        t = cyc[sel].sum() / ghz / 1e3
        print(f"    [{lo:>9}, x4): {sel.sum():5d} {t:7.3f} ms {1e3 * t / sel.sum():8.2f} us "
              f"{ftot[sel].sum() / max(t, 1e-9) / 1e6:7.1f}")
small = ftot < 4096
print(f"  rounds with < 4096 arcs: {small.sum()} taking {cyc[small].sum()/ghz/1e3:.2f}ms "
      f"({cyc[small].mean()/ghz:.2f}us each); others {(~small).sum()} taking {cyc[~small].sum()/ghz/1e3:.2f}ms")

L = int(p[6])
lt = p[8 + 3 * 4096: 8 + 3 * 4096 + 3 * min(L, 4096)].reshape(-1, 3).astype(np.int64)
lc, ll, lsp = lt[:, 0], lt[:, 1], lt[:, 2]
full = (lsp >> 40) & 1 == 1
lsp = lsp & ((1 << 40) - 1)
print(f"  level passes: {L}, sum {lc.sum()/ghz/1e3:.3f}ms, entries scanned {ll.sum()/1e6:.1f}M, "
      f"spilled {lsp.sum()/1e6:.2f}M")
print(f"    full passes (live list): {full.sum()}, {lc[full].sum()/ghz/1e3:.3f}ms, "
      f"{ll[full].sum()/1e6:.1f}M entries; low-list passes: {(~full).sum()}, "
      f"{lc[~full].sum()/ghz/1e3:.3f}ms, {ll[~full].sum()/1e6:.1f}M entries")
for i in np.nonzero(full)[0][:12]:
    print(f"      full pass {i}: {lc[i]/ghz:.1f}us entries={ll[i]}")
for lo, hi in ((0, 10), (10, 50), (50, 200), (200, 100000)):
    sel = slice(lo, min(hi, L))
    if lo < L:
        print(f"    passes {lo}-{min(hi, L)}: {lc[sel].sum()/ghz/1e3:.3f}ms, mean live "
              f"{ll[sel].mean():.0f}, mean {lc[sel].mean()/ghz:.2f}us/pass")
