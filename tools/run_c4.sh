#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -s -k "configs_vs or sweep or permutation or parts" 2>&1 | grep -E "X\|\|\^2|passed|failed|rror" | tail -8
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; python -c "
import json; d=json.load(open('gpurun_out/bench_c4.json')); r=d['roofline']; print('c4', round(d['ms_per_step'],2), 'ms', r['kernel'], round(r['achieved'],2), 'TF', round(r['frac'],3), d['value_check'])"
