#!/bin/bash
# Multi-strip epilogue compiled for 1 / 6 / 8 CTAs per SM (libpactgpu_ve*.so from tools/k2v.sh): warm times at 1 and 4 frames
cd "$(dirname "$0")/.."
for v in e1 e6 e8 e1 e6 e8; do for fr in 1 4; do
  PK_LIB=paper_2404_10928_b200/libpactgpu_v$v.so timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"epik" --csv \
    --log-file gpurun_out/epv_${v}_$fr.csv python tools/profile_kernels.py --iterations 10 --reps 2 --frames $fr > /dev/null 2>&1
  echo "== $v frames $fr: $(python tools/warm_summary.py gpurun_out/epv_${v}_$fr.csv | grep epik)"
done; done
