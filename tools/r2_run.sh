#!/bin/bash
# Round-2 evidence run on the GPU box: fast parity subset, the default bench line, dense-mode
# timings, and an ncu --set full capture (with source) of one launch of each solver kernel.
# Usage: tools/r2_run.sh TAG [skip-tests]
set -u
TAG=${1:-r02x}
cd "$(dirname "$0")/.."
if [ "${2:-}" != "skip-tests" ]; then
  timeout 600 python -m pytest tests/test_gpu_symmetry.py tests/test_gpu_parity.py -m gpu -q -x \
    -k "not cfg5 and not concurrent" > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_$TAG.log
fi
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 200 python tools/time_dense.py > gpurun_out/dense_$TAG.txt 2>&1
timeout 400 ncu --set full --clock-control none --import-source on \
  -k regex:"fp_sym_f32|bp_sym|finalize_kernel" -s 8 -c 4 -o gpurun_out/prof_$TAG \
  python tools/profile_kernels.py --iterations 3 --reps 1 > gpurun_out/prof_$TAG.log 2>&1
ls gpurun_out | grep $TAG
