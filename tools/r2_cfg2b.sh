#!/bin/bash
# cfg2 batched (frames 4) projector variants + an ncu capture of the default
cd "$(dirname "$0")/.."
for v in "PK_FSYM=1"; do
  env $v timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/wb.csv python tools/profile_kernels.py --config cfg2 --iterations 10 --reps 2 --frames 4 > /dev/null 2>&1
  echo "== $v"; python tools/warm_summary.py gpurun_out/wb.csv | grep "fp_sym_f32"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"fp_sym_f32|bp_sym_f32" -s 2 -c 2 -o gpurun_out/prof_c2b python tools/profile_kernels.py --config cfg2 --iterations 3 --reps 1 --frames 4 > /dev/null 2>&1
ls gpurun_out/prof_c2b*
