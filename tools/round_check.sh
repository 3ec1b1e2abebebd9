#!/bin/bash
# Round-end style checks on the GPU box: the -m gpu suite, the default bench (c3 FP64) with its
# CPU baseline and the reference arm, other configs, and ncu captures of the dominant kernels.
#   tools/round_check.sh [tests] [bench] [ncu] [small]
mkdir -p gpurun_out
for what in "$@"; do
case $what in
tests)
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
  echo "rc=$?" >> gpurun_out/pytest_gpu.txt ;;
bench)
  timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
  timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err
  timeout 300 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
  timeout 600 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
  timeout 600 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
  timeout 600 python bench.py --config c3 --mode tf32x3 > gpurun_out/bench_c3t.json 2> gpurun_out/bench_c3t.err
  timeout 600 python bench.py --config c5 --mode tf32x3 --steps 5 --warmup 3 > gpurun_out/bench_c5t.json 2> gpurun_out/bench_c5t.err ;;
ncu)
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k" -c 200 --csv \
    --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1x --launch-skip 1 \
    --launch-count 1 -o gpurun_out/k1x_c3 python tools/prof_k1.py --config c3 --evals 3 > gpurun_out/ncu_k1x.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1t2 --launch-skip 1 \
    --launch-count 1 -o gpurun_out/k1t2_c5 python tools/prof_k1.py --config c5 --mode tf32x3 --evals 2 > gpurun_out/ncu_k1t2.log 2>&1
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:k1z --launch-skip 2 \
    --launch-count 1 -o gpurun_out/k1z_t2 python tools/prof_k1z.py --shape 500,10,3,1000 > gpurun_out/ncu_k1z.log 2>&1 ;;
small)
  python tools/sweep_small.py > gpurun_out/sweep_small.txt 2>&1
  timeout 600 python tools/bench_adam.py --epochs 10 --cpu-epochs 1 > gpurun_out/adam_t2.txt 2>&1 ;;
esac
done
