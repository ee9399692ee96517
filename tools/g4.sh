mkdir -p gpurun_out
timeout 100 python tools/prof_run.py --iters 3 --arith fast > gpurun_out/plain.log 2>&1 && timeout 400 ncu --set full --clock-control none --import-source on -k regex:fused_step_rs -s 1 -c 1 -o gpurun_out/rs_v3 python tools/prof_run.py --iters 3 --arith fast > gpurun_out/ncu.log 2>&1; tail -2 gpurun_out/ncu.log
