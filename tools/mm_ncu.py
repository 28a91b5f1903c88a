import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2404_10928_b200 as pk
g, ring, ac, ph = pk.make_scene(128, 128, 1024, seed=0)
Kd = pk.dense_time_matrix(g, ring, ac, pk.CudaPool(0, "float32"))
op = Kd.dense_operator
X = torch.rand((32, Kd.cols), device="cuda", dtype=torch.float32)
for _ in range(3):
    op.matmat(X)
torch.cuda.synchronize()
