"""Top SASS lines by warp-stall samples, per kernel section of
`ncu -i report.ncu-rep --page source --csv --print-source sass` (development aid).
usage: python tools/stall_top.py full.sass.csv [lines per kernel]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
heads = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
for si, h in enumerate(heads):
    hdr = rows[h]
    ix = {k: i for i, k in enumerate(hdr)}
    end = heads[si + 1] - 1 if si + 1 < len(heads) else len(rows)
    body = [r for r in rows[h + 1:end] if len(r) == len(hdr) and r[0].startswith("0x")]
    if not body:
        continue
    name = rows[h - 1][1] if h > 0 and len(rows[h - 1]) > 1 else "?"
    stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
    allk = "Warp Stall Sampling (All Samples)"
    tot = Counter()
    for r in body:
        for k in stalls:
            tot[k] += float(r[ix[k]] or 0)
    samples = sum(float(r[ix[allk]] or 0) for r in body)
    print(f"== {name[:90]}: {len(body)} instructions, {int(samples)} samples")
    print("   " + ", ".join(f"{k[6:]} {int(v)}" for k, v in tot.most_common(8)))
    for r in sorted(body, key=lambda r: -float(r[ix[allk]] or 0))[:top_n]:
        st = sorted(((k, float(r[ix[k]] or 0)) for k in stalls), key=lambda x: -x[1])[:2]
        print(f"{int(float(r[ix[allk]] or 0)):7d} {r[0][-5:]} {r[ix['Source']].strip()[:66]:66s} "
              f"{st[0][0][6:]}:{int(st[0][1])} {st[1][0][6:]}:{int(st[1][1])}")
