#!/bin/bash
# Final round-2 evidence on the GPU box: launch list of the default bench (4 frames per
# launch), ncu --set full of one launch of each solver kernel at config 3 (one frame and four
# frames per launch).  PK_SYM_WDIAG pins the back-projector's cut weight to the value the
# unprofiled plans choose at config 3 (under a profiler the plan-setup timing of the
# candidates would be the tool's, and its launches would be the ones captured).
set -u
TAG=${1:-r02h}
cd "$(dirname "$0")/.."
PK_SYM_WDIAG=24 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"fp_sym_f32|bp_sym|finalize|table_kernel|init_kernel|copy_out" -s 250 -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --streams 1 --no-e2e --no-cpu --no-ncu > /dev/null 2>&1
PK_SYM_WDIAG=24 timeout 400 ncu --set full --clock-control none --import-source on \
  -k regex:"fp_sym_f32|bp_sym|finalize" -s 4 -c 4 -o gpurun_out/prof_$TAG \
  python tools/profile_kernels.py --iterations 3 --reps 1 > gpurun_out/prof_$TAG.log 2>&1
PK_SYM_WDIAG=24 timeout 400 ncu --set full --clock-control none --import-source on \
  -k regex:"fp_sym_f32|bp_sym|finalize" -s 4 -c 4 -o gpurun_out/prof_${TAG}_b4 \
  python tools/profile_kernels.py --iterations 3 --reps 1 --frames 4 > gpurun_out/prof_${TAG}_b4.log 2>&1
ls -la gpurun_out | grep $TAG
