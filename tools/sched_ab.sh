for s in lockstep even lockstep even; do
  for c in 1 2; do
    SFSEG_SCHED=$s timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/sched_${s}_c$c.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/sched_${s}_c$c.json'));r=d['roofline'];print('$s c$c', '%.4e'%d['value'], 'launch_ms=%.4f'%r['avg_launch_ms'], 'frac=%.3f'%r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], 'exact', d.get('other_arith',{}).get('avg_launch_ms'))"
  done
done
SFSEG_SCHED=even timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
