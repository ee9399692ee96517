#!/bin/bash
# End-of-round evidence in one gpurun call: GPU suite, default bench line,
# reference arm, ncu launch list of the bench command.
# usage (GPU box): tools/evidence_round.sh TAG   -> gpurun_out/TAG/
TAG=${1:-dev}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
(time timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -8) > "$OUT/gpu_tests.log" 2>&1
timeout 600 python bench.py > "$OUT/bench_default.json" 2> "$OUT/bench_default.err" || echo "bench failed"
timeout 600 python bench.py --impl reference > "$OUT/bench_reference_arm.json" 2> "$OUT/bench_reference_arm.err" || echo "reference arm failed"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches_default.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > "$OUT/bench_under_ncu.log" 2>&1 || echo "launch list failed"
gzip -f "$OUT/launches_default.csv"
tail -4 "$OUT/gpu_tests.log"; tail -c 300 "$OUT/bench_default.json"; ls -la "$OUT"
