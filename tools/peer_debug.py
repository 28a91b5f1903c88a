"""Debug the in-process peer exchange: launch `world` ranks on one device, then poll the
flag/epoch words of every rank's block from a side stream instead of synchronising."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200.sharded import PeerShardSolve  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
graph = len(sys.argv) > 2 and sys.argv[2] == "graph"
F32 = pk.CudaPool(0, "float32")
g, ring, ac, ph = pk.make_scene(64, 32, 128, seed=3)
full = pk.operator_for(g, ring, ac, F32)
yt = full.matvec(ph.values)
cfg = pk.ReconConfig(1e-6, 1e-8, 10, 1000.0)
ranks = [PeerShardSolve(g, ring, ac, F32, world, r, 10, graph=graph) for r in range(world)]
for r in ranks:
    r.connect([q.handle for q in ranks])
for r in ranks:
    r.prepare(cfg, 1e-6, 1e-8, 1000.0)
torch.cuda.synchronize()
print("prepared", flush=True)
streams = [torch.cuda.Stream() for _ in ranks]
print("streams", [hex(s.cuda_stream) for s in streams], flush=True)
Q = ac.q_s
for r, s in zip(ranks, streams):
    with torch.cuda.stream(s):
        r.launch(yt[r.m0 * Q:r.m1 * Q], cfg, 1e-6, 1e-8, 1000.0)
    print("launched rank", r.rank, flush=True)
import os  # noqa: E402

for t in range(12):
    done = [s.query() for s in streams]
    print(f"t={t * 0.5:.1f}s done={done}", flush=True)
    if all(done):
        print("OK", [r.x[-1].abs().sum().item() for r in ranks])
        break
    time.sleep(0.5)
else:
    print("STUCK", flush=True)
    os._exit(3)
