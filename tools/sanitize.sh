#!/bin/bash
# compute-sanitizer (racecheck / synccheck / memcheck) of the solver kernels at a small
# configuration: K1s (mbarrier producer/consumer ring), its epilogue, K2s, K3 (last-block
# counters), the PDL chain of the captured solve, and the peer barrier (2 in-process ranks).
# Usage: tools/sanitize.sh TAG   (logs into gpurun_out/sanitize_TAG_*.log)
set -u
TAG=${1:-r02}
cd "$(dirname "$0")/.."
CS=compute-sanitizer
for tool in memcheck racecheck synccheck; do
  # (no --leak-check: torch's caching allocator keeps its blocks until exit, which a leak
  # check reports as leaks; memcheck still reports every invalid or misaligned access)
  extra=""
  timeout 900 $CS --tool $tool $extra --error-exitcode 99 --print-limit 50 \
    python tools/sanitize_driver.py > gpurun_out/sanitize_${TAG}_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_${TAG}_$tool.log
done
grep -H "ERROR SUMMARY\|rc=" gpurun_out/sanitize_${TAG}_*.log
