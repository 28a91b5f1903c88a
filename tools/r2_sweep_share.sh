#!/bin/bash
# Throughput-mode grid sharing vs streams at config 3 (4 frames per launch).
cd "$(dirname "$0")/.."
for e in "PK_X=0" "PK_FSYM_SHARE=1" "PK_FSYM_SHARE=4" "PK_SYM_GRID=444" "PK_SYM_GRID=296"; do
  for st in 2 4 6; do
    v=$(env $e timeout 300 python bench.py --steps 40 --streams $st --no-ncu --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;print(round(json.load(sys.stdin)['value'],1))")
    echo "cfg3 [$e] streams $st: $v"
  done
done
