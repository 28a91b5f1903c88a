#!/bin/bash
# frames/s vs batch (frames per launch) and streams: cfg4 sequence, cfg2 and cfg3 single-frame workloads
cd "$(dirname "$0")/.."
for c in "cfg4 4 4" "cfg4 4 8" "cfg4 4 12" "cfg4 2 8" "cfg2 4 4" "cfg2 4 8" "cfg3 2 4" "cfg3 4 4" "cfg3 1 4"; do
  set -- $c
  timeout 300 python bench.py --config $1 --batch $2 --streams $3 --steps 20 --warmup 3 --no-cpu --no-e2e --no-ncu 2>/dev/null > gpurun_out/sw_$1_b$2_s$3.json
  echo "$1 batch $2 streams $3: $(python -c "import json;print(round(json.load(open('gpurun_out/sw_$1_b$2_s$3.json'))['value'],1))" 2>&1 | tail -1)"
done
