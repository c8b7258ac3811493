"""Per-warp timeline of the single-CTA Greedy++ peel (dg_peel_trace_*).

python tools/peel_trace.py [scale] [first_batch]

Runs RMAT-`scale` with T=3 (the trace keeps the last launch: the pruned core
of iteration 3) and prints, per traced batch, the critical path between the
three CTA barriers: last arrival and first departure at A / B / C, with the
warp that arrived last, in SM cycles.
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04333_b200 as dg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
first = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
u, v = dg.gen_rmat(scale, 16 << scale, scale)
g = dg.Graph.from_pairs(u, v)
del u, v
mode = int(sys.argv[3], 0) if len(sys.argv) > 3 else 0
dg.set_peel_mode(mode)
dg._chk(dg.diag().dg_peel_trace_arm(first))
T = int(os.environ.get("DG_TRACE_T", "3"))  # 1: iteration 1's core
r = dg.run(g, dg.RunConfig(iterations=T))
tr = np.zeros(8 * 32 * 12, np.uint64)
dg._chk(dg.diag().dg_peel_trace_read(tr.ctypes.data_as(C.POINTER(C.c_uint64))))
dg._chk(dg.diag().dg_peel_trace_arm(0xFFFFFFFF))  # disarm
tr = tr.reshape(8, 32, 12).astype(np.int64)
print(f"core n={r.trace.iters[-1].n} batches={r.trace.iters[-1].batches}")
hdr = ("batch  top->A(last w)  A wait  S2(last w)  B wait  S3(last w)  C wait | total")
print(hdr)
tot = np.zeros(7)
for b in range(7):
    t = tr[b]
    nxt = tr[b + 1]
    top = t[:, 0].min()
    a_last, a_w = t[:, 1].max(), int(t[:, 1].argmax())
    a_rel = t[t[:, 2] > 0, 2].min()
    b_last, b_w = t[:, 3].max(), int(t[:, 3].argmax())
    has3 = t[:, 4] > 0
    b_rel = t[has3, 4].min() if has3.any() else b_last
    c_last = t[has3, 5].max() if has3.any() else b_rel
    c_w = int(np.where(has3, t[:, 5], 0).argmax())
    c_rel = nxt[:, 0].min()
    seg = np.array([a_last - top, a_rel - a_last, b_last - a_rel, b_rel - b_last,
                    c_last - b_rel, c_rel - c_last, c_rel - top])
    tot += seg
    print(f"{first + b:5d}  {seg[0]:6d} (w{a_w:2d})  {seg[1]:6d}  {seg[2]:6d} (w{b_w:2d})  "
          f"{seg[3]:6d}  {seg[4]:6d} (w{c_w:2d})  {seg[5]:6d} | {seg[6]:6d}")
print("mean   " + "  ".join(f"{x:8.0f}" for x in tot / 7))
# S3 detail: per-warp S3 durations of the last traced batch
b = 5
print("S3 per warp (batch %d):" % (first + b),
      [int(tr[b, w, 5] - tr[b, w, 4]) if tr[b, w, 4] else None for w in range(32)])
# generic segment medians (both stamps set, same warp): see the stamp map in
# the kernels (peel_kernel.cuh / peel_queue.cuh, PK_STAMP / PQ_STAMP)
for a_, b_ in ((0, 6), (6, 7), (7, 8), (8, 9), (8, 1), (9, 1), (1, 2), (2, 3), (3, 4), (4, 5), (6, 8)):
    x = sorted(int(tr[b, w, b_] - tr[b, w, a_]) for b in range(7) for w in range(32)
               if tr[b, w, a_] and tr[b, w, b_] and tr[b, w, b_] >= tr[b, w, a_])
    if x:
        print(f"  stamp {a_}->{b_}: n={len(x)} median {x[len(x) // 2]} p90 {x[9 * len(x) // 10]}")
print("S1 per warp (batch %d):" % (first + b),
      [int(tr[b, w, 1] - tr[b, w, 0]) if tr[b, w, 1] else None for w in range(32)])
