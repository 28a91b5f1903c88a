"""One-rank NCCL check that the speculative sensor-sharded solve captures into a CUDA graph
with its all-reduces (the multi-GPU bench path), and matches the graph solver.

    python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 tools/nccl_capture_check.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200.sharded import DeviceShardOps, SpeculativeShardSolve  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
g, ring, ac, ph = pk.make_scene(512, 512, 2048, seed=0)
F32 = pk.CudaPool(0, "float32")
op = pk.operator_for(g, ring, ac, F32)
y = op.matvec(ph.values)
cfg = pk.ReconConfig(8.8e-8, 8.8e-10, 10, 333.0)
K = pk.build_time_matrix(g, ring, ac)
ref = pk.iterative_reconstruct(K, pk.SensorData("time", 512, 2048, y.double().cpu().numpy()), cfg, pool=F32)
ops = DeviceShardOps(g, ring, ac, F32, 0, 512)
for graph in (False, True):
    sol = SpeculativeShardSolve(ops, 10, graph=graph)
    res = sol.solve(y, cfg, cfg.alpha, cfg.beta, cfg.step)
    err = np.abs(res.image - ref.image.values).max() / np.abs(ref.image.values).max()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        sol.solve(y, cfg, cfg.alpha, cfg.beta, cfg.step)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"graph={graph}: max rel diff vs graph solver {err:.2e}, {dt * 1e3:.2f} ms/frame (incl. D2H + host stop rules)")
dist.destroy_process_group()
