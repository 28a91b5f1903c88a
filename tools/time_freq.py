"""Device time of the matrix-free frequency-domain products (build_freq_matrix) against the
FP32 FMA roofline: per product 8 flops per (sensor, pixel, wavenumber) -- a complex
multiply-add for the accumulation (forward) / Horner step (adjoint), the phase recurrence
of the forward counted alongside.

    python tools/time_freq.py [--n 128 --sensors 128 --samples 1024 --qn 1024]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200 import _native as N  # noqa: E402
from paper_2404_10928_b200.measurement import device_operator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--sensors", type=int, default=128)
ap.add_argument("--samples", type=int, default=1024)
ap.add_argument("--qn", type=int, default=1024)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
grid, ring, ac, ph = pk.make_scene(a.n, a.sensors, a.samples, seed=0)
ac = pk.AcousticConfig(c=ac.c, dt=ac.dt, q_s=ac.q_s, q_n=a.qn)
K = pk.build_freq_matrix(grid, ring, ac)
op = device_operator(K, pk.CudaPool(0, "float32"))
x = torch.tensor(ph.values, device="cuda", dtype=torch.float32)
y = op.matvec(x)
peak = ctypes.c_double()
N.check(N.load().pk_measure_fp32_peak(0, ctypes.byref(peak)))
flops = 8.0 * a.sensors * grid.size * a.qn
for name, fn in (("forward", lambda: op.matvec(x)), ("adjoint", lambda: op.adjoint(y))):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / a.reps * 1e-3
    ach = flops / t / 1e12
    print(f"{name}: {t * 1e3:.3f} ms, {ach:.1f} TFLOP/s = {ach / peak.value:.2f} of the measured FFMA peak "
          f"({peak.value:.1f})")
