#!/bin/bash
# Alternate library variants on the device-resident loop: tools/ab_libs.sh "<p_sweep args>" tag1 tag2 ...
# ("default" = the product build); two rounds so clock drift shows up as spread.
args="$1"; shift
for rep in $(seq 1 ${ROUNDS:-2}); do
  for v in "$@"; do
    if [ "$v" = default ]; then lib=""; else lib=$PWD/paper_1911_03813_b200/_lib/variants/libmomentcp_b200_$v.so; fi
    echo "== $v (round $rep)"
    MCP_LIBRARY=$lib python tools/p_sweep.py $args 2>&1 | grep -v Warn
  done
done
