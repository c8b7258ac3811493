"""Per-CTA timeline of the cluster Greedy++ kernel (DG_PEEL_PROF build):
python tools/cluster_timeline.py [scale] [T] [first_batch]
Prints, for 8 batches of the last launch, every CTA's SM cycles in: scan +
push, waiting for the 16 summaries, decode + removal, tail (barrier)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04333_b200 as dg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
T = int(sys.argv[2]) if len(sys.argv) > 2 else 2
first = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
g = dg.Graph.generate_rmat(scale, 16 << scale, scale)
dg.run(g, dg.RunConfig(iterations=T))
dg.diag().dg_peel_trace_arm(first)
r = dg.run(g, dg.RunConfig(iterations=T))
dg.diag().dg_peel_trace_arm(0xFFFFFFFF)
buf = np.zeros(8 * 32 * 12, np.uint64)
dg.diag().dg_peel_trace_read(buf.ctypes.data_as(C.POINTER(C.c_uint64)))
t = buf[: 8 * 16 * 12].reshape(8, 16, 12).astype(np.int64)
it = r.trace.iters[-1]
print(f"scale {scale} T={T}: last iteration n={it.n} batches={it.batches} "
      f"{1e3 * it.order_ms / it.batches:.2f} us/batch; batches {first}..{first + 7}")
phases = ["push", "wait", "remove", "tail", "total", "scan", "bar", "w0red", "send", "decode", "rm_rows"]
acc = np.zeros((16, 11))
nsimple = 0
for b in range(8):
    row = []
    simple = all(t[b, q, 3] > t[b, q, 2] for q in range(16))
    nsimple += simple
    for q in range(16):
        s = t[b, q]
        d = [s[1] - s[0], s[2] - s[1], (s[3] - s[2]) if simple else 0, (s[4] - s[3]) if simple else 0,
             s[4] - s[0], s[5] - s[0], s[6] - s[5], s[7] - s[6], s[1] - s[7],
             (s[8] - s[2]) if simple else 0, (s[3] - s[8]) if simple else 0]
        if simple:
            acc[q] += d
        row.append(d)
    print(f"batch {first + b} ({'simple' if simple else 'general'}): per CTA push/wait/remove/tail/total:")
    for q in range(16):
        print(f"   CTA {q:2d}: " + " ".join(f"{x:6d}" for x in row[q]))
if nsimple:
    print("mean over simple batches, per CTA:", phases)
    for q in range(16):
        print(f"   CTA {q:2d}: " + " ".join(f"{x / nsimple:7.0f}" for x in acc[q]))
