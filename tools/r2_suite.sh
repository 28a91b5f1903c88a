set -u
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputests_r02m.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_r02m.log
tail -3 gpurun_out/gputests_r02m.log
timeout 400 python bench.py > gpurun_out/bench_r02m.json 2> gpurun_out/bench_r02m.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_r02m.json
