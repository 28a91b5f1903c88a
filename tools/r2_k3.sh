#!/bin/bash
# K3 change check: symmetric-path parity tests, warm kernel times at 1 and 4 frames per launch, bench.
set -u
TAG=${1:-k3}
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_symmetry.py tests/test_gpu_parity.py tests/test_gpu_census.py -m gpu -q -x \
  -p no:cacheprovider > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_$TAG.log
tail -3 gpurun_out/t_$TAG.log
for fr in 1 4; do
  timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/warm_${TAG}_$fr.csv \
    python tools/profile_kernels.py --iterations 10 --reps 2 --frames $fr > /dev/null 2>&1
  echo "== frames $fr"; python tools/warm_summary.py gpurun_out/warm_${TAG}_$fr.csv | grep -v "init\|maxabs\|table"
done
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python tools/bsum.py gpurun_out/bench_$TAG.json
