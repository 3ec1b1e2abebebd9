#!/bin/bash
# A/B of K1Z launch / barrier variants at c1 (bench value = L2-flushed device-resident step)
mkdir -p gpurun_out
V=paper_1911_03813_b200/_lib/variants
for tag in default z_nopdl z_prof nosmall; do   # tags built with tools/build_variant.py
  if [ $tag = default ]; then unset MCP_LIBRARY; elif [ $tag = nosmall ]; then export MCP_LIBRARY=$PWD/$V/libmomentcp_b200_z_nosmall.so; else export MCP_LIBRARY=$PWD/$V/libmomentcp_b200_$tag.so; fi
  [ -n "$MCP_LIBRARY" ] && [ ! -f "$MCP_LIBRARY" ] && continue
  for cfg in "$@"; do
    timeout 300 python bench.py --config $cfg --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$tag', '$cfg', 'step_us', round(1e3*d['ms_per_step'],2), 'k1_us', round(1e3*d['roofline']['kernel_avg_ms'],2), 'e2e', round(d['e2e']['value'],1), d['kernel'])
" 2>&1 | tail -1
  done
done
