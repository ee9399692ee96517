"""Summarise `ncu --page raw --csv` (one row per captured launch) into the
numbers the roofline and DESIGN.md cite (reads here, no GPU).
usage: python tools/ncu_raw_summary.py raw.csv [voxels_per_launch] > summary.txt"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
vox = float(sys.argv[2]) if len(sys.argv) > 2 else None
KEYS = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("-" * 78)
    for k in KEYS:
        if k in d:
            print(f"{k:62s} {d[k]} {units[hdr.index(k)]}")
    if vox:
        b = sum(float(d[k].replace(",", "")) * SCALE.get(units[hdr.index(k)], 1.0)
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        x = float(d["l1tex__m_xbar2l1tex_read_bytes.sum"].replace(",", "")) * \
            SCALE.get(units[hdr.index("l1tex__m_xbar2l1tex_read_bytes.sum")], 1.0)
        print(f"{'DRAM bytes per voxel (this launch)':62s} {b / vox:.2f}")
        print(f"{'L2->SM bytes per voxel (this launch)':62s} {x / vox:.2f}")
    st = [(h, float(d[h].replace(",", ""))) for h in hdr
          if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
          and d[h]]
    st.sort(key=lambda x: -x[1])
    print("stalls per issued instruction:",
          ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
                    f" {v:.2f}" for h, v in st[:8]))
