#!/bin/bash
# throughput-mode projector grid share: cfg4 / cfg2 / cfg3 frames/s with PK_FSYM_SHARE = 1, 2, 4
cd "$(dirname "$0")/.."
for sh in 1 2 4; do
  for c in cfg4 cfg2 cfg3; do
    st=4; [ $c = cfg4 ] && st=8
    PK_FSYM_SHARE=$sh timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e --no-ncu --streams $st 2>/dev/null > gpurun_out/share_${c}_$sh.json
    echo "share $sh $c: $(python -c 'import json,sys;d=json.load(open(sys.argv[1]));print(round(d["value"],1))' gpurun_out/share_${c}_$sh.json)"
  done
done
