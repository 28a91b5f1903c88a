#!/bin/bash
# Projector phase traces (-DPK_FS_TRACE build, libpactgpu_vtr.so) at configs 2 and 3, 1 and 4 frames per launch.
cd "$(dirname "$0")/.."
for c in "cfg2 4" "cfg2 1" "cfg3 4"; do set -- $c
  echo "=== $1 frames $2"
  PK_LIB=paper_2404_10928_b200/libpactgpu_vtr.so timeout 200 python tools/k2_trace.py --config $1 --frames $2 2>&1 | tail -30
done > gpurun_out/k2trace_r02n.txt
cat gpurun_out/k2trace_r02n.txt
