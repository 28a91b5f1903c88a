#!/bin/bash
# config 3 frames/s vs concurrent streams (4 frames per launch), short runs
cd "$(dirname "$0")/.."
for ss in 2 3 4 6 8; do
  timeout 300 python bench.py --streams $ss --steps 40 --no-cpu --no-e2e --no-ncu --no-fp64 > gpurun_out/ss_$ss.json 2>/dev/null
  echo "streams $ss: $(python -c "import json;print(round(json.load(open('gpurun_out/ss_$ss.json'))['value'],1))" 2>&1 | tail -1)"
done
