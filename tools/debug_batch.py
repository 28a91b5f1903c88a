import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2404_10928_b200 as pk
from oracle import pyoracle as O
F32 = pk.CudaPool(0, "float32")
n, M, Q = 256, 256, 2048
grid, ring, ac, _ = pk.make_scene(n, M, Q, 0)
K = pk.build_time_matrix(grid, ring, ac)
o = O.Operator.of(O.make_scene(n, M, Q, 0))
def rel(a,b): return float(np.linalg.norm(np.ravel(a)-np.ravel(b))/np.linalg.norm(np.ravel(b)))
for batch in (2, 4):
    op = pk.operator_for(grid, ring, ac, F32, frames=batch)
    print("batch", batch, "sym", op.info.symmetric, "bp_split", op.info.bp_split)
    rng = np.random.default_rng(5)
    xs = rng.random((batch, n*n))
    yb = op.matvec(xs.ravel()).double().cpu().numpy().reshape(batch, -1)
    rb = rng.standard_normal((batch, M*Q))
    gb = op.adjoint(rb.ravel()).double().cpu().numpy().reshape(batch, -1)
    for f in range(batch):
        print("  f", f, "fwd", rel(yb[f], o.forward(xs[f])), "adj", rel(gb[f], o.adjoint(rb[f])))
    alpha, beta, step = 2.0817e-8, 2.0817e-10, 2651.30
    ys = []
    for f in range(batch):
        ph = pk.make_vessel_phantom(grid, 10 + f).values * (1.0 + f)
        ys.append(pk.SensorData("time", M, Q, o.forward(ph)))
    for N in (1, 2, 4):
        cfg = pk.ReconConfig(alpha, beta, N, step)
        many = pk.reconstruct_frames(K, ys, cfg, pool=F32, batch=batch, pinned=(alpha, beta, step))
        singles = [pk.iterative_reconstruct(K, y, cfg, pool=F32) for y in ys]
        print("  N", N, [round(rel(a.image.values, b.image.values), 8) for a, b in zip(many, singles)],
              [ (a.objective_history[-1], b.objective_history[-1]) for a,b in zip(many[:1], singles[:1])])
    pk.clear_plan_cache()
