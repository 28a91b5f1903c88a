#!/bin/bash
# cfg4 (1024-frame sequence at 256^2) throughput against streams and batch (GPU box)
cd "$(dirname "$0")/.."
for sb in "4 1" "8 1" "16 1" "4 2" "8 2" "4 4"; do
  set -- $sb
  timeout 300 python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu --no-e2e --streams $1 --batch $2 \
    2>/dev/null > gpurun_out/cfg4_s$1_b$2.json
  echo "streams $1 batch $2: $(python -c 'import json,sys;print(round(json.load(open(sys.argv[1]))["value"],1))' gpurun_out/cfg4_s$1_b$2.json)"
done
