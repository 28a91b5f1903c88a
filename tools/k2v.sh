#!/bin/bash
# Build / time variants of the library given as "name:-DFLAG=V -DFLAG2=W" (K2V_BUILD=1 builds
# here; without it, times the projector of each variant on the GPU box with warm caches).
set -e
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  if [ "$K2V_BUILD" = 1 ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include -shared \
      -Xcompiler -fPIC -lpthread $flags -o paper_2404_10928_b200/libpactgpu_v$name.so \
      paper_2404_10928_b200/csrc/pactgpu.cu &
  else
    echo "== $name ($flags)"
    PK_LIB=paper_2404_10928_b200/libpactgpu_v$name.so timeout 240 ncu --metrics gpu__time_duration.sum \
      --clock-control none --cache-control none -k regex:"fp_sym_f32|bp_sym|finalize" --csv \
      --log-file gpurun_out/v$name.csv python tools/profile_kernels.py --iterations 10 --reps 2 > /dev/null 2>&1 || true
    python tools/warm_summary.py gpurun_out/v$name.csv | grep -v "init\|maxabs\|table" || true
  fi
done
wait
