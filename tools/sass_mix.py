"""Opcode mix and stall hot spots from `ncu --page source --csv --print-source sass`."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
mix, stall = Counter(), Counter()
lines = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ex = float(r[ix["Instructions Executed"]] or 0)
    smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    mix[op] += ex
    stall[op] += smp
    lines.append((smp, r[ix["Address"]], src, ex))
tot = sum(mix.values())
print(f"total warp instructions {tot:.3e}")
for op, n in mix.most_common(25):
    print(f"  {op:10s} {n:12.0f} {100*n/tot:5.1f}%   stall samples {stall[op]:.0f}")
print("top stall lines:")
for smp, addr, src, ex in sorted(lines, reverse=True)[:25]:
    print(f"  {smp:7.0f} {addr} {src[:70]:70s} exec={ex:.0f}")
