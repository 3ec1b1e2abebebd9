#!/bin/bash
# One pass over the BASELINE configs (never the driver's bench line): c1, c3, c4, c5 timings.
set -u
mkdir -p gpurun_out
timeout 300 python bench.py --config c1 --steps 500 --warmup 20 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; tail -c 600 gpurun_out/bench_c1.json
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 900 gpurun_out/bench_c3.json; tail -2 gpurun_out/bench_c3.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json; tail -2 gpurun_out/bench_c4.err
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 900 gpurun_out/bench_c5.json; tail -2 gpurun_out/bench_c5.err
