#!/bin/bash
# One round's evidence on the GPU box: bench line, launch list of the bench command, and an
# ncu --set full capture of one launch of each solver kernel (cfg3).  Usage: tools/profile_round.sh TAG
set -u
TAG=${1:-rXX}
cd "$(dirname "$0")/.."
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"fp_sym_f32|bp_sym|finalize|table_kernel|init_kernel|copy_out" -s 250 -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --streams 1 --no-e2e --no-cpu --no-ncu > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on \
  -k regex:"fp_sym_f32|bp_sym|finalize" -s 4 -c 4 -o gpurun_out/prof_$TAG \
  python tools/profile_kernels.py --iterations 3 --reps 1 > gpurun_out/prof_$TAG.log 2>&1
ls -la gpurun_out | grep $TAG
