#!/bin/bash
# K1X iteration on the GPU box: parity tests, c3 / c5 bench lines, optional ncu capture.
#   tools/run_k1x.sh [ncu]
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_k1x.py -x -q -s -p no:cacheprovider > gpurun_out/k1x_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/k1x_tests.txt
timeout 300 python bench.py --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 400 python bench.py --config c5 --no-cpu --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
if [ "$1" = ncu ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1 --launch-skip 1 \
    --launch-count 1 -o gpurun_out/k1w_c3 python tools/prof_k1.py --config c3 --p 1000000 --evals 3 \
    > gpurun_out/ncu_k1w.log 2>&1
fi
