#!/bin/bash
# Regenerates the measurement evidence of a round in ONE gpurun call:
#   bench lines (fast/exact), the ncu launch list of the bench command
#   (gpu__time_duration.sum, --clock-control none), and one ncu --set full
#   capture of the fused kernel per arithmetic mode.
# usage (on the GPU box): tools/profile_round.sh r01   -> gpurun_out/prof_r01/
# then here:              python tools/summarize_round.py r01  -> profiles/
set -u
TAG=${1:-dev}
OUT=gpurun_out/prof_$TAG
mkdir -p "$OUT"
for a in fast exact; do
  timeout 300 python bench.py --steps 5 --warmup 3 --arith $a > "$OUT/bench_$a.json" 2> "$OUT/bench_$a.err" || { echo "bench $a failed"; tail -5 "$OUT/bench_$a.err"; exit 1; }
done
# launch list of the same command (only after it exited 0 without ncu)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches_fast.csv" python bench.py --steps 5 --warmup 3 --arith fast \
  --no-cpu-baseline > "$OUT/bench_under_ncu.log" 2>&1 || echo "launch list failed"
for a in fast exact; do
  timeout 200 python tools/prof_run.py --iters 3 --arith $a > "$OUT/plain_$a.log" 2>&1 && \
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:fused_step_ -s 1 -c 1 \
    -o "$OUT/full_$a" python tools/prof_run.py --iters 3 --arith $a > "$OUT/ncu_full_$a.log" 2>&1 || echo "full capture $a failed"
done
# the .ncu-rep files are ~20 MB each and gpurun_out/ travels back only under
# 64 MiB: export the raw pages (and the SASS source page of the FAST kernel)
# here and drop the reports unless KEEP_REPS=1
for a in fast exact; do
  [ -f "$OUT/full_$a.ncu-rep" ] || continue
  ncu -i "$OUT/full_$a.ncu-rep" --page raw --csv > "$OUT/full_$a.raw.csv" 2>/dev/null
  [ "$a" = fast ] && ncu -i "$OUT/full_$a.ncu-rep" --page source --csv --print-source sass > "$OUT/full_$a.sass.csv" 2>/dev/null
  [ "${KEEP_REPS:-0}" = 1 ] || rm -f "$OUT/full_$a.ncu-rep"
done
ls -la "$OUT"
