#!/bin/bash
# cfg4 / cfg2 small-frame state: warm per-kernel times at cfg2 and cfg4 throughput vs streams
cd "$(dirname "$0")/.."
timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/warm_cfg2.csv python tools/profile_kernels.py --config cfg2 --iterations 10 --reps 2 > /dev/null 2>&1
python tools/warm_summary.py gpurun_out/warm_cfg2.csv | grep -v "init\|maxabs\|table\|hold"
for s in 4 8 16; do
  timeout 300 python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu --no-e2e --no-ncu --streams $s 2>/dev/null > gpurun_out/cfg4_s$s.json
  echo "cfg4 streams $s: $(python -c 'import json,sys;d=json.load(open(sys.argv[1]));print(round(d["value"],1), d.get("ms_per_step"))' gpurun_out/cfg4_s$s.json)"
done
timeout 300 python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu --no-e2e --no-ncu 2>/dev/null > gpurun_out/cfg2_b.json
python -c 'import json;d=json.load(open("gpurun_out/cfg2_b.json"));print("cfg2", round(d["value"],1), {k:round(v["ms_per_launch"]*1e3,1) for k,v in d["kernels"].items()}, d["roofline"]["frac"])'
