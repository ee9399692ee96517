#!/bin/bash
# ncu evidence for the multi-channel FAST kernels (fused_mc.cuh) on a c4 crop:
# plain run, then one --set full capture of the 2nd iteration's launches.
# usage (GPU box): tools/prof_mc.sh TAG [config] [frames]
set -u
TAG=${1:-dev}; CFG=${2:-4}; FR=${3:-64}
OUT=gpurun_out/prof_$TAG
mkdir -p "$OUT"
timeout 300 python tools/prof_run.py --config $CFG --frames $FR --iters 3 --arith fast > "$OUT/plain.log" 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_step_mc -s 2 -c 2 \
  -o "$OUT/full" python tools/prof_run.py --config $CFG --frames $FR --iters 3 --arith fast > "$OUT/ncu_full.log" 2>&1 || echo "capture failed"
if [ -f "$OUT/full.ncu-rep" ]; then
  ncu -i "$OUT/full.ncu-rep" --page raw --csv > "$OUT/full.raw.csv" 2>/dev/null
  ncu -i "$OUT/full.ncu-rep" --page source --csv --print-source sass > "$OUT/full.sass.csv" 2>/dev/null
  [ "${KEEP_REPS:-0}" = 1 ] || rm -f "$OUT/full.ncu-rep"
fi
ls -la "$OUT"
