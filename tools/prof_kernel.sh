#!/bin/bash
# One ncu --set full capture of a fused kernel on a BASELINE config (after a
# plain run of the same command exits 0), exported as raw + SASS-source CSV.
# usage (GPU box): tools/prof_kernel.sh TAG CONFIG FRAMES ARITH REGEX [SKIP] [COUNT]
set -u
TAG=$1; CFG=$2; FR=$3; AR=$4; RX=$5; SKIP=${6:-1}; CNT=${7:-1}
OUT=gpurun_out/prof_$TAG
mkdir -p "$OUT"
FA=""; [ "$FR" != "0" ] && FA="--frames $FR"
timeout 300 python tools/prof_run.py --config $CFG $FA --iters 3 --arith $AR > "$OUT/plain.log" 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s $SKIP -c $CNT \
  -o "$OUT/full" python tools/prof_run.py --config $CFG $FA --iters 3 --arith $AR > "$OUT/ncu_full.log" 2>&1 || echo "capture failed"
if [ -f "$OUT/full.ncu-rep" ]; then
  ncu -i "$OUT/full.ncu-rep" --page raw --csv > "$OUT/full.raw.csv" 2>/dev/null
  ncu -i "$OUT/full.ncu-rep" --page source --csv --print-source sass > "$OUT/full.sass.csv" 2>/dev/null
  [ "${KEEP_REPS:-0}" = 1 ] || rm -f "$OUT/full.ncu-rep"
fi
ls -la "$OUT"
