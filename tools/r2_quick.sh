#!/bin/bash
# Quick GPU check of a kernel change: symmetric-path parity tests, warm per-kernel timings for
# the given env variants (tools/warm.sh), one default bench line.
# Usage: tools/r2_quick.sh TAG [ENV=VALUE ...]
set -u
TAG=${1:-q}; shift
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_symmetry.py tests/test_gpu_parity.py tests/test_gpu_census.py -m gpu -q -x \
  -k "not cfg5" -p no:cacheprovider > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_$TAG.log
tail -3 gpurun_out/t_$TAG.log
bash tools/warm.sh "$@" > gpurun_out/warm_$TAG.txt 2>&1; cat gpurun_out/warm_$TAG.txt
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print('bench',d['value'],'e2e',d['e2e']['value'],'lat',d['latency_ms_per_frame'],{k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})"
