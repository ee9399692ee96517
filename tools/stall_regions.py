"""Stall-reason totals per code region of an ncu SASS source page
(--page source --csv --print-source sass). Regions are split at markers:
python tools/stall_regions.py f.csv"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for r in rows[2:]:
    try:
        a = int(r[ix["Address"]], 16)
    except ValueError:
        continue
    recs.append((a, r[ix["Source"]].strip(), int(r[ix["Instructions Executed"]] or 0),
                 {k: int(r[ix[k]] or 0) for k in reasons}))
base = recs[0][0]
split = [a for a, s, n, st in recs if "TRY_ALLOC" in s][0]
# B region: classify by a simple state machine: y-pass from a TRYWAIT on xb_full to the
# SYNCS.ARRIVE on xb_empty; everything else in B is 'epilogue/other'
reg = defaultdict(Counter)
inst = Counter()
state = "A"
for a, s, n, st in recs:
    if a >= split and state == "A":
        state = "B-other"
    if state != "A":
        if "SYNCS.PHASECHK" in s and state == "B-other" and "0x36f9" in s:
            state = "B-ypass"
        elif "SYNCS.ARRIVE" in s and state == "B-ypass":
            reg[state].update(st)
            inst[state] += n
            state = "B-other"
            continue
    reg[state].update(st)
    inst[state] += n
for k, c in reg.items():
    tot = sum(c.values())
    print(f"{k:10s} inst {inst[k]:.3e} samples {tot}")
    for rr, v in c.most_common(8):
        print(f"     {rr:24s} {v:6d} {v / max(1, tot) * 100:5.1f}%")
