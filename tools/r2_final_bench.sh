#!/bin/bash
# Final round-2 evidence: GPU suite, the default bench line (with its ncu traffic capture),
# one line per other BASELINE config, two more default lines for the spread.
set -u
TAG=${1:-r02j}
cd "$(dirname "$0")/.."
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 1200 -p no:cacheprovider > gpurun_out/gputests_$TAG.log 2>&1
echo "tests rc=$?" >> gpurun_out/gputests_$TAG.log
tail -3 gpurun_out/gputests_$TAG.log
timeout 400 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
for c in cfg1 cfg2 cfg4 cfg5; do
  st=20; [ $c = cfg5 ] && st=3; [ $c = cfg4 ] && st=3
  timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-ncu > gpurun_out/bench_${TAG}_$c.json 2>/dev/null
done
for r in 1 2; do timeout 300 python bench.py --no-cpu --no-ncu > gpurun_out/bench_${TAG}_run$r.json 2>/dev/null; done
for f in gpurun_out/bench_${TAG}*.json; do python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[1], round(d['value'],1), 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None, 'lat', round(d.get('latency_ms_per_frame') or 0, 4), 'frac', round(d['roofline']['frac'], 3) if d.get('roofline') else None)" $f; done
