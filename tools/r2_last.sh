#!/bin/bash
# Final evidence of the round (TAG): GPU suite, default bench, one line per other config,
# launch list + ncu --set full of the solver kernels (tools/r2_final.sh).
cd "$(dirname "$0")/.."
TAG=${1:-r02q}
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputests_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_$TAG.log
tail -3 gpurun_out/gputests_$TAG.log
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python tools/bsum.py gpurun_out/bench_$TAG.json
for c in cfg1 cfg2 cfg4 cfg5; do
  timeout 400 python bench.py --config $c --no-cpu --steps 30 > gpurun_out/bench_${TAG}_$c.json 2>/dev/null
  python tools/bsum.py gpurun_out/bench_${TAG}_$c.json
done
bash tools/r2_final.sh $TAG
