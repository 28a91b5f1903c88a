#!/bin/bash
# projector warps-per-CTA variants at cfg3 (1 frame) and cfg2 (4 frames), warm kernel times
cd "$(dirname "$0")/.."
for c in "cfg3 1" "cfg2 4"; do
  set -- $c
  for v in "PK_FSYM_NW=32" "PK_FSYM_NW=16 PK_FSYM_PERSM=1" "PK_FSYM_NW=16"; do
    env $v timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/wn.csv python tools/profile_kernels.py --config $1 --iterations 10 --reps 2 --frames $2 > /dev/null 2>&1
    echo "== $1 frames $2 $v: $(python tools/warm_summary.py gpurun_out/wn.csv | grep fp_sym_f32)"
  done
done
