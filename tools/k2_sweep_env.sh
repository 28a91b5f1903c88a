#!/bin/bash
# Warm projector time per config for env settings (PK_LIB + "VAR=value" list).
# Usage: tools/k2_sweep_env.sh LIBSUFFIX "PK_X=1" "PK_X=2" ...
cd "$(dirname "$0")/.."
lib=paper_2404_10928_b200/libpactgpu${1:+_v$1}.so; shift
for cfg in "cfg3" "cfg2" "cfg2 --frames 4"; do
  for e in "$@"; do
    env PK_LIB=$lib $e timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file gpurun_out/sw.csv python tools/profile_kernels.py --config $cfg --iterations 10 --reps 2 > /dev/null 2>&1
    echo "$cfg [$e] $(python tools/warm_summary.py gpurun_out/sw.csv | grep fp_sym_f32 | awk "{print \$(NF-4)}")"
  done
done
