for s in 3 4 6 8; do
  timeout 200 python bench.py --no-cpu --no-e2e --streams $s --steps 100 2>/dev/null > gpurun_out/sw_$s.json
  echo "streams $s $(python -c 'import json,sys;print(json.load(open(sys.argv[1]))["value"])' gpurun_out/sw_$s.json)"
done
timeout 200 python bench.py --no-cpu --no-e2e --streams 4 --batch 2 --steps 50 2>/dev/null > gpurun_out/sw_b2.json
echo "batch2 $(python -c 'import json,sys;print(json.load(open(sys.argv[1]))["value"])' gpurun_out/sw_b2.json)"
