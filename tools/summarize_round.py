"""Turns gpurun_out/prof_<TAG>/ (tools/profile_round.sh) into committed
evidence under profiles/:
  <TAG>_bench_c1_{fast,exact}.json     the bench lines
  <TAG>_launches_c1_fast.csv           ncu launch list of the bench command
  <TAG>_launch_summary.md              per-kernel counts / times / shares
  <TAG>_ncu_full_c1_{fast,exact}.txt   key metrics of one --set full capture
  traffic_c1_{fast,exact}.json         DRAM bytes per fused launch (bench.py reads it)
usage: python tools/summarize_round.py r01"""
import csv
import io
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
TAG = sys.argv[1] if len(sys.argv) > 1 else "dev"
SRC = ROOT / "gpurun_out" / f"prof_{TAG}"
DST = ROOT / "profiles"
DST.mkdir(exist_ok=True)

for a in ("fast", "exact"):
    f = SRC / f"bench_{a}.json"
    if f.exists():
        shutil.copy(f, DST / f"{TAG}_bench_c1_{a}.json")

# launch list
lf = SRC / "launches_fast.csv"
if lf.exists():
    text = lf.read_text()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    (DST / f"{TAG}_launches_c1_fast.csv").write_text("\n".join(lines) + "\n")
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    per = defaultdict(list)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1e-3)
        per[r[ki].split("(")[0]].append(v * scale)
    tot = sum(sum(v) for v in per.values())
    out = [f"# {TAG}: ncu launch list of `python bench.py --steps 5 --warmup 3 --arith fast`",
           "", "ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold-cache",
           "per-launch times: the kernel's SHARE of the step is the comparable number).", "",
           "| kernel | launches | total us | mean us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.2f} | {sum(v) / tot * 100:.1f}% |")
    (DST / f"{TAG}_launch_summary.md").write_text("\n".join(out) + "\n")
    print("\n".join(out))

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "lts__t_sector_hit_rate.pct", "sm__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "smsp__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second",
]
for a in ("fast", "exact"):
    rep = SRC / f"full_{a}.ncu-rep"
    rawf = SRC / f"full_{a}.raw.csv"  # exported on the box (tools/profile_round.sh)
    if rawf.exists():
        raw = rawf.read_text()
    elif rep.exists():
        raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    else:
        continue
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    lines = [f"# {TAG}: ncu --set full --clock-control none, fused kernel, c1, {a.upper()}",
             "# (python tools/prof_run.py --iters 3 --arith " + a + "; launch 2 of the solve)", ""]
    for k in KEYS:
        if k in d:
            lines.append(f"{k:66s} {d[k][0]} {d[k][1]}")
    stalls = [(h[len("smsp__average_warp_latency_issue_stalled_"):].split(".")[0], float(v.replace(",", "")))
              for h, (v, u) in d.items()
              if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")
              and v not in ("", "n/a")]
    if stalls:
        lines += ["", "stall cycles per issued instruction:"]
        for n, v in sorted(stalls, key=lambda kv: -kv[1])[:10]:
            lines.append(f"   {n:28s} {v:.3f}")
    (DST / f"{TAG}_ncu_full_c1_{a}.txt").write_text("\n".join(lines) + "\n")

    def num(k):
        v, u = d[k]
        x = float(v.replace(",", ""))
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    (DST / f"traffic_c1_{a}.json").write_text(json.dumps({
        "kernel": d["Kernel Name"][0], "dram_bytes_per_launch": traffic,
        "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
        "source": f"profiles/{TAG}_ncu_full_c1_{a}.txt"}, indent=1) + "\n")
    print("\n".join(lines))
