#!/bin/bash
# Multi-rank bench flow on ONE GPU (test mode: both ranks on cuda:0 over gloo), with Python
# tracebacks on a hang:  tools/sd_debug.sh CONFIG [extra bench args]
mkdir -p gpurun_out
cfg=$1; shift
port=$((29500 + RANDOM % 1000))
for r in 0 1; do
  MASTER_ADDR=127.0.0.1 MASTER_PORT=$port WORLD_SIZE=2 RANK=$r LOCAL_RANK=$r MCP_BENCH_SAME_DEVICE=1 \
    timeout -s ABRT 240 python -X faulthandler bench.py --gpus 2 --config $cfg --no-cpu "$@" \
    > gpurun_out/sd_${cfg}_r$r.out 2> gpurun_out/sd_${cfg}_r$r.err &
done
wait
