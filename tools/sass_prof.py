"""Per-opcode executed-instruction / stall-sample breakdown of an ncu
source page (--page source --csv --print-source sass). Optional address
ranges split the kernel into regions: python tools/sass_prof.py f.csv [lo:hi ...]"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        addr = int(r[ix["Address"]], 16)
    except ValueError:
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    recs.append((addr, op, src, int(r[ix["Instructions Executed"]] or 0),
                 int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
base = recs[0][0]
tot_i = sum(r[3] for r in recs)
tot_s = sum(r[4] for r in recs)
print(f"total warp inst {tot_i:.4e}  samples {tot_s}")
by = defaultdict(lambda: [0, 0])
for a, op, s, n, st in recs:
    by[op.split('.')[0]][0] += n
    by[op.split('.')[0]][1] += st
for op, (n, st) in sorted(by.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{op:12s} inst {n/tot_i*100:5.1f}%  stall {st/tot_s*100:5.1f}%")
print("top stall instructions:")
for a, op, s, n, st in sorted(recs, key=lambda r: -r[4])[:25]:
    print(f"  {a-base:6x} {st:6d} {n:9d} {s[:70]}")
