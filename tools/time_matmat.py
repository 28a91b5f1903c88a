"""Explicit-matrix mode on the tensor cores: frame-batched products K X and K^T Y
(pk_dense_matmat / pk_dense_rmatmat: tcgen05 kind::tf32 with the 3xTF32 split) at BASELINE
config 1's dense K (131072 x 16384 fp32, formed on the device), against F streaming GEMVs.

    python tools/time_matmat.py [--frames 8 16 32 64 128]

Algorithmic flops 2 R C F per product (the 3xTF32 split issues 3x that on the tensor
cores); bytes of K streamed once per product.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_10928_b200 as pk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, nargs="+", default=[8, 16, 32, 64, 128])
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
peaks = json.load(open(mp)) if os.path.exists(mp) else {}
hbm = float(peaks.get("hbm_gbs", 6650.0))
tc = float(peaks.get("bf16_tflops", peaks.get("dense_bf16_tflops", 0.0)) or 0.0)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


g, ring, ac, ph = pk.make_scene(128, 128, 1024, seed=0)
Kd = pk.dense_time_matrix(g, ring, ac, pk.CudaPool(0, "float32"))
op = Kd.dense_operator
R, C = Kd.rows, Kd.cols
kbytes = 4.0 * R * C
rng = np.random.default_rng(0)
x1 = torch.tensor(ph.values, device="cuda", dtype=torch.float32)
t_mv = timed(lambda: op.matvec(x1), a.reps)
print(f"K {R} x {C} fp32 ({kbytes / 1e9:.1f} GB); GEMV {t_mv * 1e3:.3f} ms = {kbytes / t_mv / 1e9:.0f} GB/s "
      f"({kbytes / t_mv / 1e9 / hbm:.2f} of {hbm:.0f} GB/s)")
for F in a.frames:
    X = torch.tensor(rng.random((F, C)), device="cuda", dtype=torch.float32)
    Y = torch.tensor(rng.standard_normal((F, R)), device="cuda", dtype=torch.float32)
    t_f = timed(lambda: op.matmat(X), a.reps)
    t_a = timed(lambda: op.rmatmat(Y), a.reps)
    fl = 2.0 * R * C * F
    print(f"F {F:4d}: K X {t_f * 1e3:7.3f} ms ({fl / t_f / 1e12:6.1f} TFLOP/s algorithmic, "
          f"{3 * fl / t_f / 1e12:6.1f} issued, K at {kbytes / t_f / 1e9:5.0f} GB/s; {F} GEMVs {F * t_mv * 1e3:7.2f} ms)  "
          f"K^T Y {t_a * 1e3:7.3f} ms ({fl / t_a / 1e12:6.1f} TFLOP/s)")
op.close()
