#!/bin/bash
# Round-end bench lines for every config (run under gpurun): profiles/<round>/bench_*.json
set -u
R=${R:-r01}
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench_c2.json 2> gpurun_out/final/bench_c2.err
python bench.py --config c1 --steps 200 --warmup 10 > gpurun_out/final/bench_c1.json 2> gpurun_out/final/bench_c1.err
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err
python bench.py --config c3 --mode tf32x3 --steps 20 --warmup 3 --no-cpu > gpurun_out/final/bench_c3_tf32.json 2> gpurun_out/final/bench_c3_tf32.err
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/final/bench_c4.json 2> gpurun_out/final/bench_c4.err
python bench.py --config c5 --mode tf32x3 --steps 4 --warmup 3 --no-cpu > gpurun_out/final/bench_c5_tf32.json 2> gpurun_out/final/bench_c5_tf32.err
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/final/bench_c5.json 2> gpurun_out/final/bench_c5.err
