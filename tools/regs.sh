#!/bin/bash
# Registers / spills of the kernels matching $1 (nvcc -Xptxas=-v of libpactgpu, output to /tmp).
cd "$(dirname "$0")/.."
python - "$1" <<'PY'
import subprocess, sys
sys.path.insert(0, '.')
from paper_2404_10928_b200 import _native as n
r = subprocess.run(n.nvcc_command('/tmp/regs_probe.so') + ['-Xptxas=-v'], capture_output=True, text=True)
if r.returncode: print(r.stderr[-3000:]); sys.exit(1)
print(subprocess.run([sys.executable, 'tools/ptxas_regs.py', sys.argv[1]], input=r.stderr, capture_output=True, text=True).stdout)
PY
