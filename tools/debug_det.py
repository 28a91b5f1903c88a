"""Determinism / sanitizer driver: two projections of the same image must be bitwise equal."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2404_10928_b200 as pk

n, M, Q, seed = [int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (64, 32, 128, 1))]
g, ring, ac, ph = pk.make_scene(n, M, Q, seed=seed)
K = pk.build_time_matrix(g, ring, ac)
for dtype in ("float32", "float64"):
    pool = pk.CudaPool(0, dtype)
    op = pk.operator_for(g, ring, ac, pool)
    print(dtype, "plan info: fp_tile", op.info.fp_tile, "fp_window", op.info.fp_window, "bits", op.info.fp_bits,
          "bp_window", op.info.bp_window, "bp_chunk", op.info.bp_chunk)
    ys = [pk.forward_project(K, ph, pool=pool).values for _ in range(4)]
    for k in range(1, 4):
        d = np.flatnonzero(ys[k] != ys[0])
        print(f"  run {k}: {d.size} differing samples", (d[:10], ys[0][d[:5]], ys[k][d[:5]]) if d.size else "")
    rng = np.random.default_rng(0)
    r = rng.standard_normal(M * Q)
    a = [op.adjoint(r).double().cpu().numpy() for _ in range(3)]
    print("  adjoint equal:", all(np.array_equal(a[0], b) for b in a[1:]))
