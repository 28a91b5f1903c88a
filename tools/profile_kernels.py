"""Launch the solver kernels of one configuration un-graphed (for ncu).

    python tools/profile_kernels.py [--config cfg3] [--iterations 2] [--dtype float32]

Runs pk_profile_iterations once (init, table, then iterations x (K1, K2, K3)) after a
warm-up, so `ncu -k regex:bp_f32|fp_f32 -s <skip> -c <n>` can select single launches.
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
from paper_2404_10928_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--iterations", type=int, default=2)
ap.add_argument("--dtype", default="float32")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--frames", type=int, default=1, help="batched plan (1, 2, 4 frames per launch)")
a = ap.parse_args()
cfg = CONFIGS[a.config]
grid, ring, ac, ph = pk.make_scene(cfg.n, cfg.sensors, cfg.samples, seed=0)
op = pk.operator_for(grid, ring, ac, pk.CudaPool(0, a.dtype), frames=a.frames)
y = op.matvec(np.tile(ph.values, a.frames))
params1 = N.SolverParams(alpha=8.8e-8, beta=8.8e-10, step=333.0, tv_epsilon=1e-3, tolerance=0.0,
                        iterations=a.iterations, nonneg=0)
params = (N.SolverParams * a.frames)(*([params1] * a.frames))
lib = N.load()
ms = (ctypes.c_float * 3)()
n = ctypes.c_int32()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
best = [1e30] * 3
for _ in range(a.reps):
    N.check(lib.pk_profile_iterations(op.handle, params, y.data_ptr(), ms, ctypes.byref(n), s))
    best = [min(b, v) for b, v in zip(best, ms)]
torch.cuda.synchronize()
us = [1e3 * v / a.iterations for v in best]
print("per-launch us: K1 %.1f  K2 %.1f  K3 %.1f  (sum %.1f; launches %d)" % (us[0], us[1], us[2], sum(us), n.value))
