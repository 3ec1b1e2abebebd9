#!/bin/bash
# Round profile set (run under gpurun): bench lines, the c2 launch list, one ncu --set full
# capture each of the c2 FP64 kernel (K1Q) and the c3 fast-mode kernel (K1T2).
set -u
NCU=/usr/local/cuda/bin/ncu
R=${R:-r01}
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
$NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k1q_fg_pairs -s 3 -c 1 \
  -o gpurun_out/k1q_c2_$R -f python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_k1q.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k1t2_fg_tf32 -s 2 -c 1 \
  -o gpurun_out/k1t2_c3_$R -f python bench.py --config c3 --mode tf32x3 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_k1t2.log 2>&1
python bench.py --config c3 --mode tf32x3 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c3_tf32.json 2> gpurun_out/bench_c3_tf32.err
