#!/bin/bash
# config 3 throughput against the number of streams (one throughput-mode plan each)
cd "$(dirname "$0")/.."
for s in ${@:-3 4 5 6 8}; do
  timeout 200 python bench.py --no-cpu --no-e2e --streams $s --steps ${STEPS:-200} 2>/dev/null > gpurun_out/sw_$s.json
  echo "streams $s $(python -c 'import json,sys;print(round(json.load(open(sys.argv[1]))["value"],1))' gpurun_out/sw_$s.json)"
done
