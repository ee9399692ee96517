"""Top SASS lines per stall reason from one kernel's section of
`ncu --page source --csv --print-source sass` (development aid).
usage: python tools/stall_top.py section.csv [reason ...]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
reasons = sys.argv[2:] or ["stall_long_sb", "stall_wait", "stall_short_sb", "stall_barrier", "stall_math"]
tot = {k: sum(float(r[ix[k]] or 0) for r in body) for k in hdr if k.startswith("stall_") and "Not" not in k}
print("totals:", sorted(((round(v), k) for k, v in tot.items()), reverse=True)[:10])
for k in reasons:
    print("==", k)
    top = sorted(body, key=lambda r: -float(r[ix[k]] or 0))[:8]
    for r in top:
        print(f"  {float(r[ix[k]] or 0):7.0f} {r[ix['Address']][-5:]} {r[ix['Source']][:90]}")
