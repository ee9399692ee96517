"""Warp-stall samples of an ncu SASS source page (--page source --csv
--print-source sass), summed between synchronisation landmarks (development aid).
usage: python tools/stall_segments.py full.sass.csv [min_exec] [kernel section index]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
minex = float(sys.argv[2]) if len(sys.argv) > 2 else 1000
heads = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
sec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hi = heads[sec]
end = heads[sec + 1] - 1 if sec + 1 < len(heads) else len(rows)
hdr = rows[hi]
ix = {k: i for i, k in enumerate(hdr)}
body = [r for r in rows[hi + 1:end] if len(r) == len(hdr) and r[0].startswith("0x")]
allk = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ix[allk]] or 0) for r in body)
print("total samples", tot, "instructions", len(body))
seg_s = seg_n = 0
start = 0
for i, r in enumerate(body):
    src = r[ix["Source"]].strip()
    s = float(r[ix[allk]] or 0)
    ex = float(r[ix["Instructions Executed"]] or 0)
    mark = any(m in src for m in ("SYNCS.PHASECHK", "SYNCS.ARRIVE", "BAR.SYNC", "UTMALDG", "UTMASTG")) and ex >= minex
    if mark:
        print(f"   [{start:5d}-{i:5d}) n={seg_n:4d} samples={seg_s:6.0f}")
        print(f"{i:5d} {r[0][-5:]} {src[:64]:64s} samples={s:5.0f} exec={ex:.0f}")
        seg_s = seg_n = 0
        start = i + 1
    else:
        seg_s += s
        seg_n += 1
print(f"   [{start:5d}-end) n={seg_n:4d} samples={seg_s:6.0f}")
