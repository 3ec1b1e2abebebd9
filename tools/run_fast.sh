#!/bin/bash
set -u
timeout 900 python -m pytest tests -x -q -m gpu -s 2>&1 | grep -E "via|passed|failed|rror|assert|sweep" | tail -30
for c in c3 c5 c2; do
  st=20; [ $c = c5 ] && st=5; [ $c = c2 ] && st=200
  timeout 900 python bench.py --config $c --mode tf32x3 --steps $st --warmup 3 --no-cpu > gpurun_out/bench_${c}_tf32.json 2> gpurun_out/bench_${c}_tf32.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_${c}_tf32.json')); r=d['roofline']; print('$c tf32x3', round(d['value'],2), 'evals/s', round(d['ms_per_step'],3), 'ms; kernel', round(r['kernel_avg_ms'],3), 'ms', r['bound'], round(r['achieved'],1), r['unit'], 'frac', round(r['frac'],3), d['clocks'])" || tail -3 gpurun_out/bench_${c}_tf32.err
done
