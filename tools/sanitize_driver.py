"""Small workload for compute-sanitizer (tools/sanitize.sh): every fp32 solver kernel of the
symmetric path (K1s + epilogue, K2s, K3, table/init/copy-out) through one captured solve and
one un-graphed profile pass, the generic and fp64 kernels, the dense kernels, and the
peer-memory barrier with 2 in-process ranks."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

os.environ.setdefault("PK_FSYM", "1")  # the rotation-symmetric projector even at this small size

import paper_2404_10928_b200 as pk  # noqa: E402
from paper_2404_10928_b200 import measurement as meas  # noqa: E402

F32, F64 = pk.CudaPool(0, "float32"), pk.CudaPool(0, "float64")
# 128^2 / 64 sensors / 512 samples: symmetric back-projector and projector both active
g, ring, ac, ph = pk.make_scene(128, 64, 512, seed=1)
K = pk.build_time_matrix(g, ring, ac)
y = pk.forward_project(K, ph, pool=F64)
cfg = pk.resolve_config(pk.ReconConfig(iterations=4), K, y, pool=F64)
for pool in (F32, F64):
    op = pk.operator_for(g, ring, ac, pool)
    print(pool.dtype, "symmetric flags", op.info.symmetric)
    res = pk.iterative_reconstruct(K, y, cfg, pool=pool)
    res = pk.iterative_reconstruct(K, y, cfg, pool=pool)  # graph replay
    op.profile_iterations(y.values, pk.solver.solver_params(cfg, cfg.alpha, cfg.beta, cfg.step))
    print(pool.dtype, "iterations", res.iterations_run)
# batched symmetric plan (2 frames per launch): frame-major chunks, segments, residual CTAs
opb = pk.operator_for(g, ring, ac, F32, frames=2)
pb = pk.solver.solver_params(cfg, cfg.alpha, cfg.beta, cfg.step)
yb = np.concatenate([y.values, 0.5 * y.values])
for _ in range(2):
    opb.reconstruct(yb, pb)
torch.cuda.synchronize()
print("batched symmetric flags", opb.info.symmetric, "frames", opb.info.frames)
# generic (non-symmetric) kernels: off-centre ring
g2 = pk.make_grid(48, 40, 1e-4, (-2.4e-3, -2.0e-3))
ring2 = pk.make_ring(24, 6e-3, (0.3e-3, -0.2e-3), g2)
ac2 = pk.AcousticConfig(c=1500.0, dt=1.6e-7, q_s=128, q_n=128)
K2 = pk.build_time_matrix(g2, ring2, ac2)
y2 = pk.forward_project(K2, pk.make_vessel_phantom(g2, 2), pool=F64)
pk.iterative_reconstruct(K2, y2, pk.ReconConfig(iterations=3), pool=F32)
# dense explicit-matrix kernels (fused and two-pass)
A = pk.build_time_matrix(*pk.make_scene(32, 16, 64, seed=3)[:3]).entries
for pool in (F32, F64):
    Kd = pk.MeasurementMatrix("time", A, {"grid": pk.make_scene(32, 16, 64, seed=3)[0]})
    yd = pk.SensorData("time", 16, 64, A @ pk.make_scene(32, 16, 64, seed=3)[3].values)
    pk.iterative_reconstruct(Kd, yd, pk.ReconConfig(iterations=3), pool=pool)
    meas.device_operator(Kd, pool).adjoint(np.ones(A.shape[0]) + 1j)
# peer barrier: 2 ranks in one process (tests/test_gpu_peer.py's in-process harness)
from paper_2404_10928_b200.sharded import PeerShardSolve, shard_range  # noqa: E402

solvers = [PeerShardSolve(g, ring, ac, F32, 2, r, 3, graph=False) for r in range(2)]
handles = [s.handle for s in solvers]
for s in solvers:
    s.connect(handles)
streams = [torch.cuda.Stream() for _ in range(2)]
yl = []
for r, s in enumerate(solvers):
    m0, m1 = shard_range(64, r, 2)
    yl.append(torch.tensor(y.values[m0 * 512:m1 * 512], device="cuda", dtype=torch.float32))
for s in solvers:
    s.prepare(cfg, cfg.alpha, cfg.beta, cfg.step)
torch.cuda.synchronize()
for r, s in enumerate(solvers):
    with torch.cuda.stream(streams[r]):
        s.launch(yl[r], cfg, cfg.alpha, cfg.beta, cfg.step)
torch.cuda.synchronize()
print("peer data terms", [float(s.local_data_terms()[0]) for s in solvers])
# shards listing whole D4 orbits keep the symmetric kernels (pk_geometry_desc.sensor_list)
from paper_2404_10928_b200.sharded import shard_sensors  # noqa: E402

for r in range(2):
    lst = shard_sensors(64, r, 2)
    op = pk.DeviceOperator(g, ring, ac, F32, sensor_list=lst)
    print("shard", r, "symmetric flags", op.info.symmetric)
    rr = torch.tensor(np.random.default_rng(r).standard_normal(len(lst) * 512), device="cuda",
                      dtype=torch.float32)
    op.adjoint(rr)
    op.matvec(ph.values)
    op.close()
for s in solvers:
    s.op.close()
pk.clear_plan_cache()
meas._dense_cache.clear()
torch.cuda.synchronize()
print("sanitize driver done")
