"""Explicit-matrix mode timings (pk_dense_*) at BASELINE config 1's dense K (131072 x 16384):
forward GEMV, adjoint GEMV^H, and the 10-iteration device solve, fp32 and fp64, with the
bytes of K each streams against the measured HBM copy bandwidth (MEASURED_PEAKS.json).

    python tools/time_dense.py [--reps 5]
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
from paper_2404_10928_b200.workloads import PINNED  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best


g, ring, ac, ph = pk.make_scene(128, 128, 1024, seed=0)
y = pk.forward_project(pk.build_time_matrix(g, ring, ac), ph, pool=pk.CudaPool(0, "float64"))
alpha, beta, step = PINNED["cfg1"]
cfg = pk.ReconConfig(alpha, beta, 10, step)
out = {}
for dt in ("float32", "float64"):
    pool = pk.CudaPool(0, dt)
    K = pk.dense_time_matrix(g, ring, ac, pool)
    op = K.dense_operator
    kbytes = op.rows * op.cols * (4 if dt == "float32" else 8)
    x = torch.tensor(ph.values, device="cuda", dtype=op.rdtype)
    r = torch.tensor(y.values, device="cuda", dtype=op.rdtype)
    t_fwd = timed(lambda: op.matvec(x), a.reps)
    t_adj = timed(lambda: op.adjoint(r), a.reps)
    params = pk.solver.solver_params(cfg, alpha, beta, step)
    t_solve = timed(lambda: op.reconstruct(r, params, 128, 128), a.reps)
    passes = 11 if op.info.fused else 21  # K passes per 10-iteration solve (init + per iteration)
    res = {"K_GB": kbytes / 1e9, "fused": int(op.info.fused),
           "forward_ms": t_fwd * 1e3, "forward_GBs": kbytes / t_fwd / 1e9,
           "adjoint_ms": t_adj * 1e3, "adjoint_GBs": kbytes / t_adj / 1e9,
           "solve_ms": t_solve * 1e3, "solve_frames_per_s": 1.0 / t_solve,
           "solve_K_passes": passes, "solve_GBs": passes * kbytes / t_solve / 1e9,
           "hbm_peak_GBs": peak}
    for k in ("forward", "adjoint", "solve"):
        res[k + "_frac"] = res[k + "_GBs"] / peak
    out[dt] = res
    print(dt, json.dumps(res), flush=True)
    op.close()
    del K, op
    torch.cuda.empty_cache()
print(json.dumps(out))
