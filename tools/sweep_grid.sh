#!/bin/bash
# bench throughput against the back-projector's persistent grid (PK_SYM_GRID):
#   tools/sweep_grid.sh CONFIG STREAMS GRID...   (GRID "default" = the plan's choice)
cd "$(dirname "$0")/.."
C=$1; S=$2; shift 2
for g in "$@"; do
  if [ $g = default ]; then E=""; else E="PK_SYM_GRID=$g"; fi
  env $E timeout 300 python bench.py --config $C --steps ${STEPS:-2} --warmup 3 --no-cpu --no-e2e --streams $S \
    2>/dev/null > gpurun_out/grid_${C}_s${S}_g$g.json
  echo "$C streams $S grid $g: $(python -c 'import json,sys;print(round(json.load(open(sys.argv[1]))["value"],1))' gpurun_out/grid_${C}_s${S}_g$g.json)"
done
