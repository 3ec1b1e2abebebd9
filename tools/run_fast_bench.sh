#!/bin/bash
set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -s -k fast 2>&1 | grep -E "via|passed|failed|rror|sweep" | tail -8
for c in ${CONFIGS:-c3 c5}; do
  st=20; [ $c = c5 ] && st=5; [ $c = c2 ] && st=200
  timeout 900 python bench.py --config $c --mode ${MODE:-tf32x3} --steps $st --warmup 3 --no-cpu > gpurun_out/bench_${c}_${MODE:-tf32x3}.json 2> gpurun_out/bench_${c}.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_${c}_${MODE:-tf32x3}.json')); r=d['roofline']; print('$c', d['config']['mode'], round(d['value'],2), 'evals/s', round(d['ms_per_step'],3), 'ms; kernel', round(r['kernel_avg_ms'],3), 'ms', r['bound'], round(r['achieved'],1), r['unit'], 'frac', round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/bench_${c}.err
done
