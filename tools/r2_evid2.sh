#!/bin/bash
# End-of-round evidence on the final build: sanitizers (racecheck / synccheck / memcheck),
# one bench line per BASELINE config, the reference arm at config 3, the fp64 mode line.
cd "$(dirname "$0")/.."
bash tools/sanitize.sh r02n
STEPS=30 bash tools/bench_configs.sh cfg1 cfg2 cfg4 cfg5
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_r02n.json 2>gpurun_out/ref_r02n.err; tail -c 400 gpurun_out/ref_r02n.json
