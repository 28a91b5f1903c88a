#!/bin/bash
# one bench line per BASELINE config (our arm, one GPU): tools/bench_configs.sh [configs...]
cd "$(dirname "$0")/.."
for c in ${@:-cfg1 cfg2 cfg3 cfg5}; do
  timeout 400 python bench.py --config $c --no-cpu --steps ${STEPS:-50} 2>/dev/null > gpurun_out/cfg_$c.json
  python - "$c" gpurun_out/cfg_$c.json <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
print(f"{sys.argv[1]} value {d['value']:.1f} e2e {d['e2e']['value']:.1f} ms/iter {d['ms_per_iteration']:.4f} "
      f"frac {d['roofline']['frac']:.3f} ({d['roofline']['kernel'][:2]})")
PY
done
