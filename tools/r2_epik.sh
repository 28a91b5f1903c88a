#!/bin/bash
# Epilogue strips-per-CTA check: symmetry / parity tests, warm epilogue times for PK_SYM_EPIK=1/2/4 at 1 and 4 frames, bench.
cd "$(dirname "$0")/.."
TAG=${1:-epik}
timeout 900 python -m pytest tests/test_gpu_symmetry.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_$TAG.log
tail -2 gpurun_out/t_$TAG.log
for fr in 1 4; do for ks in 1 2 4; do
  PK_SYM_EPIK=$ks timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"epi|finalize" --csv \
    --log-file gpurun_out/w_${TAG}_${fr}_$ks.csv python tools/profile_kernels.py --iterations 10 --reps 2 --frames $fr > /dev/null 2>&1
  echo "== frames $fr ks $ks"; python tools/warm_summary.py gpurun_out/w_${TAG}_${fr}_$ks.csv | grep "epi"
done; done
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python tools/bsum.py gpurun_out/bench_$TAG.json
