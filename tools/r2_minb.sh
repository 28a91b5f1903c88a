#!/bin/bash
# back-projector register cap variants (experiment builds via PK_LIB): warm K1s time at config 3
cd "$(dirname "$0")/.."
for v in "PK_LIB=paper_2404_10928_b200/libpactgpu.so" "PK_LIB=paper_2404_10928_b200/libpactgpu_minb4.so PK_SYM_NBUF=3" "PK_LIB=paper_2404_10928_b200/libpactgpu_minb4.so PK_SYM_NBUF=4" "PK_LIB=paper_2404_10928_b200/libpactgpu.so PK_SYM_NBUF=3"; do
  env $v timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/wm.csv python tools/profile_kernels.py --iterations 10 --reps 2 > /dev/null 2>&1
  echo "== $v: $(python tools/warm_summary.py gpurun_out/wm.csv | grep 'bp_sym_f32')"
done
