#!/bin/bash
# One GPU iteration: parity tests, both benches, ncu of the FAST kernel.
# usage: tools/gpu_cycle.sh TAG
TAG=${1:-dev}
timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for a in exact fast; do
  timeout 150 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --arith $a > gpurun_out/bench_${a}_$TAG.json 2> gpurun_out/bench_${a}_$TAG.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${a}_$TAG.json'));r=d['roofline'];print('$a', '%.3e'%d['value'], 'launch_ms=%.4f'%r['avg_launch_ms'], 'frac=%.3f'%r['frac'], 'e2e=%.3e'%d['e2e']['value'], d['clocks'])" || tail -5 gpurun_out/bench_${a}_$TAG.err
done
timeout 100 python tools/prof_run.py --iters 3 --arith fast > gpurun_out/plain.log 2>&1 && timeout 300 ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o gpurun_out/prof_c1_fast_$TAG python tools/prof_run.py --iters 3 --arith fast > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log
