"""Device time of the standalone products (pk_matvec / pk_adjoint_matvec) on controlled
inputs, with CUDA events: phantom (sparse), dense random, and the iterate of a 10-iteration
solve (what the solver's projector actually sees).

    python tools/time_products.py [--config cfg3] [--reps 20]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
cfg = CONFIGS[a.config]
grid, ring, ac, ph = pk.make_scene(cfg.n, cfg.sensors, cfg.samples, seed=0)
pool = pk.CudaPool(0, "float32")
op = pk.operator_for(grid, ring, ac, pool)
K = pk.build_time_matrix(grid, ring, ac)
y = op.matvec(ph.values)
cfgp = pk.ReconConfig(alpha=8.8e-8, beta=8.8e-10, iterations=10, step=333.0)
res = pk.iterative_reconstruct(K, pk.SensorData("time", cfg.sensors, cfg.samples, y.double().cpu().numpy()),
                               cfgp, pool=pool)
xi = torch.tensor(res.image.values, device="cuda", dtype=torch.float32)
rng = np.random.default_rng(0)
inputs = {
    "phantom": torch.tensor(ph.values, device="cuda", dtype=torch.float32),
    "dense": torch.tensor(rng.random(cfg.pixels), device="cuda", dtype=torch.float32),
    "iterate": xi,
}


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / a.reps


for name, x in inputs.items():
    nnz = float((x != 0).float().mean())
    t_fp = timed(lambda: op.matvec(x))
    yy = op.matvec(x)
    t_bp = timed(lambda: op.adjoint(yy))
    print(f"{name:8s} nnz {nnz:6.3f}  matvec {t_fp:7.1f} us  adjoint {t_bp:7.1f} us")
