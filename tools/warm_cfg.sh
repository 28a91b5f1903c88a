#!/bin/bash
# warm per-launch kernel times of one config under env settings:
#   tools/warm_cfg.sh cfg2 "PK_FIN_CHUNKS=1" "PK_FIN_CHUNKS=2" ...
cd "$(dirname "$0")/.."
C=$1; shift
for e in "$@"; do
  echo "== $C $e"
  env $e timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/warm_$C.csv python tools/profile_kernels.py --config $C --iterations 10 --reps 2 > /dev/null 2>&1
  python tools/warm_summary.py gpurun_out/warm_$C.csv | grep -v "init\|maxabs\|table\|hold\|_lo_\|count"
done
