#!/bin/bash
# Build timing-only variants of the symmetric projector (PK_K2X, pk_kernels.cuh) and print
# the warm per-launch time of each (K2X_BUILD=1: build here; then run on the GPU box):
#   0 product, 1 no shared atomics, 2 records from registers (no LDS), 3 no sqrt, 4 one atomic/pair,
#   6 no window store, 7 no counts load (timings r01d: DESIGN.md, K2s)
set -e
cd "$(dirname "$0")/.."
if [ "$K2X_BUILD" = 1 ]; then
for v in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include -shared \
    -Xcompiler -fPIC -lpthread -DPK_K2X=$v -o paper_2404_10928_b200/libpactgpu_k2x$v.so \
    paper_2404_10928_b200/csrc/pactgpu.cu
done
exit 0
fi
for v in "$@"; do
  echo "== PK_K2X=$v"
  PK_LIB=paper_2404_10928_b200/libpactgpu_k2x$v.so timeout 240 ncu --metrics gpu__time_duration.sum \
    --clock-control none --cache-control none -k regex:fp_sym_f32 --csv --log-file gpurun_out/k2x$v.csv \
    python tools/profile_kernels.py --iterations 10 --reps 2 > /dev/null 2>&1 || true
  python tools/warm_summary.py gpurun_out/k2x$v.csv | grep fp_sym_f32 || true
done
