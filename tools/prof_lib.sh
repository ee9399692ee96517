#!/bin/bash
# ncu --set full capture of one fused kernel for a library build, with tight
# timeouts (a kernel that hangs under replay must not eat the GPU budget).
# usage (GPU box): tools/prof_lib.sh TAG LIB CONFIG FRAMES ARITH REGEX [SKIP] [COUNT]
set -u
TAG=$1; export SFSEG_CUDA_LIB=$2; CFG=$3; FR=$4; AR=$5; RX=$6; SKIP=${7:-1}; CNT=${8:-1}
OUT=gpurun_out/prof_$TAG
mkdir -p "$OUT"
FA=""; [ "$FR" != "0" ] && FA="--frames $FR"
timeout 120 python tools/prof_run.py --config $CFG $FA --iters 3 --arith $AR > "$OUT/plain.log" 2>&1 || { echo "plain run failed"; exit 1; }
timeout 240 ncu --set full --clock-control none --import-source on -k regex:$RX -s $SKIP -c $CNT \
  -o "$OUT/full" python tools/prof_run.py --config $CFG $FA --iters 3 --arith $AR > "$OUT/ncu_full.log" 2>&1 || echo "capture failed"
if [ -f "$OUT/full.ncu-rep" ]; then
  ncu -i "$OUT/full.ncu-rep" --page raw --csv > "$OUT/full.raw.csv" 2>/dev/null
  ncu -i "$OUT/full.ncu-rep" --page source --csv --print-source sass > "$OUT/full.sass.csv" 2>/dev/null
  rm -f "$OUT/full.ncu-rep"
fi
ls "$OUT"
