#!/bin/bash
# Warm projector/back-projector times of one config under env settings.
# Usage: tools/k2_sweep_cfg.sh "cfg2 --frames 4" "PK_FSYM_LW=184" "PK_FSYM_T=64 PK_FSYM_LW=320" ...
cd "$(dirname "$0")/.."
cfg=$1; shift
for e in "$@"; do
  env $e timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/sw.csv python tools/profile_kernels.py --config $cfg --iterations 10 --reps 2 > /dev/null 2>&1
  echo "$cfg [$e] $(python tools/warm_summary.py gpurun_out/sw.csv | grep 'fp_sym_f32\|bp_sym_f32' | awk '{print $2, $(NF-4)}' | tr '\n' ' ')"
done
