"""Summaries of ncu output for profiles/ (run here, no GPU needed).

python tools/ncu_report.py launches <launches.csv> "<command line>"   -> per-kernel shares
python tools/ncu_report.py full <report.ncu-rep> "<command line>"     -> details page + DRAM bytes
"""
import csv
import io
import subprocess
import sys


def launches(path, cmd):
    rows = []
    with open(path) as f:
        text = f.read()
    text = text[text.index('"ID"'):] if '"ID"' in text else text
    for r in csv.DictReader(io.StringIO(text)):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "nsecond": 1e-6, "second": 1e3}.get(unit, 1e-6)
        rows.append((r["Kernel Name"], v * scale))
    agg = {}
    for name, ms in rows:
        a = agg.setdefault(name, [0.0, 0])
        a[0] += ms
        a[1] += 1
    tot = sum(a[0] for a in agg.values())
    out = [f"ncu --metrics gpu__time_duration.sum --clock-control none  {cmd}",
           "(cold-cache serialised launches: compare SHARES, not absolutes)",
           f"total kernel time {tot:.1f} ms over {len(rows)} launches", "",
           f"{'ms':>10} {'share':>6} {'launches':>8}  kernel"]
    for name, (ms, k) in sorted(agg.items(), key=lambda x: -x[1][0]):
        out.append(f"{ms:10.3f} {100 * ms / tot:5.1f}% {k:8d}  {name[:110]}")
    print("\n".join(out))


def full(rep, cmd):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True,
                         text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h = r[0]
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__warps_eligible.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
            "launch__grid_size", "launch__block_size"]
    print(f"ncu --set full --clock-control none --import-source on  {cmd}\n")
    for li, v in enumerate(r[2:]):
        print(f"-- launch {li}")
        for k in keys:
            if k in h:
                print(f"{k}: {v[h.index(k)]} {r[1][h.index(k)]}")
        print()
    print(det)


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
