#!/bin/bash
# Compare warm per-kernel times of the product library and experiment builds (PK_LIB variants)
# at config 3, config 2 and config 2 x 4 frames.  Usage: tools/k2_cmp.sh v1 v2 ...  ("" = product)
cd "$(dirname "$0")/.."
for cfg in "cfg3" "cfg2" "cfg2 --frames 4"; do
  for v in "$@"; do
    lib=paper_2404_10928_b200/libpactgpu${v:+_v$v}.so
    PK_LIB=$lib timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file gpurun_out/cmp.csv python tools/profile_kernels.py --config $cfg --iterations 10 --reps 2 > /dev/null 2>&1
    echo "== $cfg [${v:-product}]"; python tools/warm_summary.py gpurun_out/cmp.csv | grep "fp_sym_f32\|bp_sym\|finalize_sym"
  done
done
