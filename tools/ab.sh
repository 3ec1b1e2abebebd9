#!/bin/bash
# A/B the c2 bench over library variants: tools/ab.sh [bench args] -- tag1 tag2 ...
# ("default" = the product build).  Prints ms_per_step, roofline frac, e2e per variant.
args=()
while [ "$1" != "--" ] && [ -n "$1" ]; do args+=("$1"); shift; done
shift
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=$PWD/paper_1911_03813_b200/_lib/variants/libmomentcp_b200_$v.so; fi
  MCP_LIBRARY=$lib python bench.py "${args[@]}" > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    print(v, d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"], d["config"].get("k1_variant"))
except Exception as e:
    print(v, "FAILED", open(f"gpurun_out/ab_{v}.err").read()[-400:])
PY
done
