#!/bin/bash
# HEAD check: GPU suite, smoke(), default bench (TAG)
cd "$(dirname "$0")/.."
TAG=${1:-head}
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputests_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_$TAG.log
tail -3 gpurun_out/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log; tail -3 gpurun_out/smoke_$TAG.log
timeout 400 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
python tools/bsum.py gpurun_out/bench_$TAG.json
