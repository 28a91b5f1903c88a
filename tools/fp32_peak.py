"""The FP32 roofline denominator, measured once per box and committed (profiles/fp32_peak.json):
the FFMA microkernel of pk_measure_fp32_peak (8 independent chains per thread, 148 x 4 CTAs),
best of 20, with nvidia-smi SM clocks sampled while it runs and the theoretical
148 SMs x 128 FP32 lanes x 2 flops x clock for comparison.

    python tools/fp32_peak.py > profiles/fp32_peak.json
"""
import ctypes
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2404_10928_b200 import _native as N  # noqa: E402

lib = N.load()
smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                        "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
vals = []
for _ in range(20):
    v = ctypes.c_double()
    N.check(lib.pk_measure_fp32_peak(0, ctypes.byref(v)))
    vals.append(v.value)
smi.terminate()
out, _ = smi.communicate(timeout=5)
rows = [ln.split(",") for ln in out.strip().splitlines() if ln.count(",") >= 2]
sm = sorted(float(r[0]) for r in rows) if rows else []
mx = max(float(r[1]) for r in rows) if rows else None
name = subprocess.run(["nvidia-smi", "--query-gpu=name", "--format=csv,noheader"], capture_output=True,
                      text=True).stdout.strip()
rec = {"fp32_tflops": max(vals), "fp32_tflops_median": sorted(vals)[len(vals) // 2],
       "samples": len(vals), "sm_mhz_median": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
       "theoretical_tflops_at_max_clock": 148 * 128 * 2 * (mx or 1965.0) * 1e6 / 1e12,
       "gpu": name, "how": "pk_measure_fp32_peak (FFMA, 8 chains/thread, 592 CTAs x 256 threads, "
       "4096 x 16 x 8 FFMA per thread), best of 20 with CUDA events",
       "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
print(json.dumps(rec, indent=1))
