#!/bin/bash
# Throughput sweep (streams x batch) of the small configs with the product library.
cd "$(dirname "$0")/.."
for sb in "4 1" "8 1" "4 4" "8 4" "12 4" "8 2" "16 4"; do
  set -- $sb
  v=$(timeout 600 python bench.py --config cfg4 --steps 2 --warmup 3 --streams $1 --batch $2 --no-ncu --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;print(round(json.load(sys.stdin)['value'],1))")
  echo "cfg4 streams $1 batch $2: $v"
done
for sb in "4 1" "8 1" "4 4" "8 4" "8 2"; do
  set -- $sb
  v=$(timeout 600 python bench.py --config cfg2 --steps 40 --warmup 5 --streams $1 --batch $2 --no-ncu --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;print(round(json.load(sys.stdin)['value'],1))")
  echo "cfg2 streams $1 batch $2: $v"
done
