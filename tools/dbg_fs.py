import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2404_10928_b200 as pk
from oracle import pyoracle as O
F32 = pk.CudaPool(0, "float32")
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for (n, M, Q) in [(64, 32, 128), (96, 64, 512), (128, 128, 1024)]:
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=2)
    o = O.Operator.of(O.make_scene(n, M, Q, 2))
    pk.clear_plan_cache()
    op = pk.operator_for(g, ring, ac, F32)
    x = ph.values + 0.05 * np.random.default_rng(9).random(g.size)
    yd = op.matvec(x).double().cpu().numpy(); yo = o.forward(x)
    err = np.abs(yd - yo).reshape(M, Q)
    print(n, M, Q, "sym", op.info.symmetric, "tile", op.info.fp_tile, "fwd rel", rel(yd, yo),
          "worst sensors", np.argsort(err.max(1))[-4:], "worst samples", np.argsort(err.max(0))[-4:])
