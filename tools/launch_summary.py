"""Per-kernel launch counts, times and shares from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file f.csv <command>`).
usage: python tools/launch_summary.py launches.csv[.gz] "title line" > profiles/<tag>_launch_summary.md"""
import csv
import gzip
import io
import sys
from collections import defaultdict

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
lines = [ln for ln in raw.splitlines() if ln.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
per = defaultdict(list)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1e-3)
    name = r[ki].split("(")[0].replace("sfk::", "").replace("(int)", "").replace("(bool)", "")
    per[name].append(v * scale)
tot = sum(sum(v) for v in per.values())
print(f"# {title}")
print()
print("ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold-cache per-launch times:")
print("a kernel's SHARE is the comparable number, not its absolute time).")
print()
print("| kernel | launches | total ms | mean us | share |")
print("|---|---:|---:|---:|---:|")
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    print(f"| `{k}` | {len(v)} | {sum(v) / 1e3:.1f} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
print()
print(f"{sum(len(v) for v in per.values())} launches, {tot / 1e3:.1f} ms of kernel time.")
