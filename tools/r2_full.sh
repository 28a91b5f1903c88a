#!/bin/bash
# Full GPU test suite + default bench line + smoke (round-end style check of a change).
# Usage: tools/r2_full.sh TAG
set -u
TAG=${1:-f}
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests_$TAG.log
tail -4 gpurun_out/tests_$TAG.log
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print('bench',d['value'],'e2e',d['e2e']['value'],'lat',d['latency_ms_per_frame'],{k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()}, d['roofline']['frac'])"
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
