"""Split an ncu SASS source page into segments delimited by clock reads
(CS2R SR_CLOCKLO) and report samples / instructions / top stalls per segment.
usage: python tools/ncu_segments.py report.ncu-rep [batches]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
batches = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
si, wi, ii = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[wi] or 0) for r in data)
seg, segs, start = 0, {}, {}
for idx, r in enumerate(data):
    if "SR_CLOCKLO" in r[si]:
        seg += 1
        start[seg] = idx
    d = segs.setdefault(seg, {"samples": 0.0, "inst": 0.0, **{c: 0.0 for c in reasons}})
    d["samples"] += float(r[wi] or 0)
    d["inst"] += float(r[ii] or 0)
    for c in reasons:
        d[c] += float(r[h.index(c)] or 0)
for k, d in segs.items():
    top = sorted(((v, c) for c, v in d.items() if c.startswith("stall_")), reverse=True)[:5]
    print(f"seg{k} @{start.get(k)} {100 * d['samples'] / tot:5.1f}% warp-inst/batch="
          f"{d['inst'] / batches:8.0f} " + " ".join(f"{c[6:]}={int(v)}" for v, c in top))
