#!/bin/bash
# per-kernel device times of the cfg3 solve under plan-tuning environment variables
# usage: tools/sweep.sh "ENV=.. ENV2=.." "..." ...
cd "$(dirname "$0")/.."
for e in "$@"; do
  echo "== $e"
  env $e timeout 120 python tools/profile_kernels.py --config ${CFG:-cfg3} --iterations 10 --reps 3 2>&1 | grep -v Warn | tail -1
done
