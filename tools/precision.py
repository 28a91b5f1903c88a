"""fp32 path precision vs the fp64 validation mode (itself checked against the CPU oracle),
per configuration and back-projector table layout (PK_BP_ATRICK=0/1).

    python tools/precision.py [cfg3 cfg5 ...] [--iterations N]
"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2404_10928_b200 as pk
from paper_2404_10928_b200 import _native as N
from paper_2404_10928_b200.workloads import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["cfg3"])
ap.add_argument("--iterations", type=int, default=0)
a = ap.parse_args()
out = []
for name in a.configs:
    cfg = CONFIGS[name]
    iters = a.iterations or cfg.iterations
    g, ring, ac, ph = pk.make_scene(cfg.n, cfg.sensors, cfg.samples, seed=0)
    K = pk.build_time_matrix(g, ring, ac)
    f64 = pk.CudaPool(0, "float64")
    t0 = time.time()
    y = pk.forward_project(K, ph, pool=f64)
    pinned = pk.resolve_config(pk.ReconConfig(iterations=iters), K, y, pool=f64)
    ref = pk.iterative_reconstruct(K, y, pinned, pool=f64)
    t_ref = time.time() - t0
    rec = {"config": name, "iterations": iters, "pinned": [pinned.alpha, pinned.beta, pinned.step],
           "fp64_seconds": t_ref, "ref_iterations_run": ref.iterations_run}
    for at in ("0", "1"):
        os.environ["PK_BP_ATRICK"] = at
        pk.clear_plan_cache()
        res = pk.iterative_reconstruct(K, y, pinned, pool=pk.CudaPool(0, "float32"))
        err = float(np.linalg.norm(res.image.values - ref.image.values) / np.linalg.norm(ref.image.values))
        hist = float(np.max(np.abs(res.objective_history / ref.objective_history - 1)))
        op = pk.operator_for(g, ring, ac, pk.CudaPool(0, "float32"))
        params = pk.solver.solver_params(pinned, pinned.alpha, pinned.beta, pinned.step)
        yt = op.tensor(y.values)
        ms = (ctypes.c_float * 3)()
        nl = ctypes.c_int32()
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        tot = np.zeros(3)
        for _ in range(3):
            N.check(N.load().pk_profile_iterations(op.handle, ctypes.byref(params), yt.data_ptr(), ms, ctypes.byref(nl), st))
            tot += np.array(ms[:])
        rec[f"atrick{at}"] = {"rel_l2": err, "max_rel_objective_dev": hist,
                              "ms_per_launch": list(tot / (3 * iters))}
    print(json.dumps(rec), flush=True)
