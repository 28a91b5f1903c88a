"""Public-call wall time of the fp32 solver right after the harness's fp64 solves, with and
without a pause, and with the SM clock read around it:  python tools/api_slow_probe.py"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200.harness import _scene  # noqa: E402

n, M, Q = 512, 512, 2048
grid, ring, ac, ph, K, y, cfg = _scene(n, M, Q, 0, pk.ReconConfig(iterations=10), 0)
f32, f64 = pk.CudaPool(0, "float32"), pk.CudaPool(0, "float64")


def clk():
    q = "clocks.sm,power.draw,clocks_event_reasons.active"
    return subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader"],
                          capture_output=True, text=True).stdout.strip()


def t(pool, k=5):
    out = []
    for _ in range(k):
        t0 = time.perf_counter()
        pk.iterative_reconstruct(K, y, cfg, pool=pool)
        out.append((time.perf_counter() - t0) * 1e3)
    return " ".join(f"{v:.2f}" for v in out)


print("f32", t(f32), clk())
for pause in (0.0, 0.0, 0.5, 2.0):
    r = pk.iterative_reconstruct(K, y, cfg, pool=f64)
    print("f64x6", t(f64, 6), clk())
    time.sleep(pause)
    print(f"f32 after {pause}s", t(f32), clk())
