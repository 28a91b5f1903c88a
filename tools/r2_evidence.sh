#!/bin/bash
# Round-2 evidence: full GPU suite, the default bench line + launch list + ncu capture
# (tools/profile_round.sh), one bench line per BASELINE config, bench spread at config 3.
set -u
TAG=${1:-r02}
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/gputests_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_$TAG.log
tail -3 gpurun_out/gputests_$TAG.log
bash tools/profile_round.sh $TAG
for c in cfg1 cfg2 cfg4 cfg5; do
  st=20; [ $c = cfg5 ] && st=3; [ $c = cfg4 ] && st=3
  timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-ncu > gpurun_out/bench_${TAG}_$c.json 2>/dev/null
done
for r in 1 2; do timeout 300 python bench.py --no-cpu --no-ncu > gpurun_out/bench_${TAG}_run$r.json 2>/dev/null; done
for f in gpurun_out/bench_${TAG}*.json; do python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[1], round(d['value'],1), 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None, 'lat', d.get('latency_ms_per_frame'))" $f; done
