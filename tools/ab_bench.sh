#!/bin/bash
# A/B bench lines over library variants: tools/ab_bench.sh "<bench args>" tag1 tag2 ...
# ("default" = the product build).  Lines go to gpurun_out/ab_<tag>_<n>.json.
args="$1"; shift
for rep in $(seq 1 ${ROUNDS:-1}); do
  for v in "$@"; do
    if [ "$v" = default ]; then lib=""; else lib=$PWD/paper_1911_03813_b200/_lib/variants/libmomentcp_b200_$v.so; fi
    MCP_LIBRARY=$lib timeout 600 python bench.py $args --no-cpu > gpurun_out/ab_${v}_$rep.json 2> gpurun_out/ab_${v}_$rep.err
  done
done
