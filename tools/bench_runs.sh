#!/bin/bash
# N default bench runs (config 3), one summary line each: run-to-run variance
cd "$(dirname "$0")/.."
for i in $(seq 1 ${1:-3}); do
  timeout 300 python bench.py --no-cpu 2>/dev/null > gpurun_out/run_$i.json
  python - "$i" gpurun_out/run_$i.json <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
print(f"run {sys.argv[1]} value {d['value']:.1f} e2e {d['e2e']['value']:.1f} ms/iter {d['ms_per_iteration']:.4f} "
      f"K2 frac {d['roofline']['frac']:.3f} smem {d['roofline']['smem_pipe_frac']:.3f} "
      f"clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
done
