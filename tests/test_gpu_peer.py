"""Sensor-sharded solve with the gradient exchanged over peer memory (pk_peer_*,
sharded.PeerShardSolve): ranks on one device (plans in this process on separate streams, or
two processes mapping each other's blocks over CUDA IPC) against the single-rank solver."""

import os
import socket

import numpy as np
import pytest

import paper_2404_10928_b200 as pk

pytestmark = pytest.mark.gpu

F32 = pk.CudaPool(0, "float32")
SCENE = (64, 32, 128, 3)


def _problem(oracle):
    n, M, Q, seed = SCENE
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=seed)
    o = oracle.Operator.of(oracle.make_scene(n, M, Q, seed))
    y = o.forward(ph.values)
    alpha, beta = oracle.resolve_regularization(o, y)
    step = oracle.resolve_step(o, beta, 1e-3)
    return g, ring, ac, y, alpha, beta, step


def _reference(g, ring, ac, y, cfg):
    K = pk.build_time_matrix(g, ring, ac)
    return pk.iterative_reconstruct(K, pk.SensorData("time", ring.count, ac.q_s, y), cfg, pool=F32)


def _check(res, ref):
    assert res.iterations_run == ref.iterations_run
    assert res.stopped_by == ref.stopped_by
    scale = np.abs(ref.image.values).max()
    np.testing.assert_allclose(res.image, ref.image.values, rtol=0, atol=2e-5 * scale)
    np.testing.assert_allclose(res.history[:, 0], ref.objective_history, rtol=1e-4)


@pytest.mark.parametrize("world,graph", [(2, False), (2, True), (3, False), (4, True)])
def test_peer_shards_in_process(oracle, world, graph):
    """`world` plans on cuda:0, one stream each, enqueued back to back: the device barrier
    orders them; x is bit-identical on every rank and matches the single-rank solve."""
    import torch

    from paper_2404_10928_b200.sharded import PeerShardSolve

    g, ring, ac, y, alpha, beta, step = _problem(oracle)
    cfg = pk.ReconConfig(alpha, beta, 10, step)
    ref = _reference(g, ring, ac, y, cfg)
    Q = ac.q_s
    ranks = [PeerShardSolve(g, ring, ac, F32, world, r, cfg.iterations, graph=graph) for r in range(world)]
    handles = [r.handle for r in ranks]
    for r in ranks:
        r.connect(handles)
    for r in ranks:
        r.prepare(cfg, alpha, beta, step)
    streams = [torch.cuda.Stream() for _ in ranks]
    yt = torch.tensor(y, device="cuda", dtype=torch.float32)
    for rep in range(2):  # epochs keep advancing across solves (and graph replays)
        for r, s in zip(ranks, streams):
            with torch.cuda.stream(s):
                r.launch(r.local_y(yt), cfg, alpha, beta, step)
        torch.cuda.synchronize()
        data = sum(r.local_data_terms() for r in ranks)
        res = [r.finish(data) for r in ranks]
        for q in res[1:]:
            assert np.array_equal(q.image, res[0].image)  # replicated x stays bit-identical
        for r in ranks:
            assert torch.equal(r.x, ranks[0].x)
        _check(res[0], ref)


def test_peer_api_errors():
    import ctypes

    from paper_2404_10928_b200 import _native as N
    from paper_2404_10928_b200.device import DeviceOperator

    g, ring, ac, _ = pk.make_scene(32, 16, 64, seed=0)
    op = DeviceOperator(g, ring, ac, F32, 0, 8)
    with pytest.raises(ValueError):
        op.peer_buffer(0)  # no block yet
    h = op.peer_handle()
    assert len(h) == N.PK_PEER_HANDLE_BYTES
    assert op.peer_buffer(1) > op.peer_buffer(0)
    with pytest.raises(ValueError):
        op.peer_buffer(2)
    with pytest.raises(ValueError):
        op.peer_connect(2, 0, [h])  # wrong count
    with pytest.raises(ValueError):
        op.peer_connect(9, 0, [h] * 9)  # world above PK_PEER_MAX
    other = DeviceOperator(g, ring, ac, F32, 8, 16)
    h2 = other.peer_handle()
    with pytest.raises(ValueError):
        op.peer_connect(2, 0, [h2, h])  # handles[rank] must be this plan's
    params = N.SolverParams(alpha=0.0, beta=0.0, step=1.0, tv_epsilon=1e-3, tolerance=0.0,
                            iterations=1, nonneg=0)
    lib = N.load()
    rc = lib.pk_peer_grad_update(op.handle, ctypes.byref(params), op.peer_buffer(0), 0,
                                 op.peer_buffer(1), op.peer_buffer(1), None)
    assert rc == N.PK_ERR_INVALID  # not connected


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, y, cfgv, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_10928_b200.sharded import PeerShardSolve

        n, M, Q, seed = SCENE
        g, ring, ac, _ = pk.make_scene(n, M, Q, seed=seed)
        alpha, beta, step = cfgv
        cfg = pk.ReconConfig(alpha, beta, 10, step)
        s = PeerShardSolve(g, ring, ac, F32, world, rank, cfg.iterations)
        s.connect_distributed()
        res = s.solve(s.local_y(y), cfg, alpha, beta, step)
        # three frames through two pipelined instances (graph-captured), each on its stream
        from paper_2404_10928_b200.sharded import PipelinedShardSolve

        inst = [PeerShardSolve(g, ring, ac, F32, world, rank, cfg.iterations, graph=True) for _ in range(2)]
        for q in inst:
            q.connect_distributed()
        frames = PipelinedShardSolve(inst).solve_frames([s.local_y(y)] * 3, cfg, alpha, beta, step)
        same = all(np.array_equal(fr.image, res.image) for fr in frames)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), image=res.image, hist=res.history,
                 meta=np.array([res.iterations_run, int(same)]))
        dist.barrier()  # keep every block mapped until all ranks are done
    finally:
        dist.destroy_process_group()


def test_peer_shards_two_processes_ipc(oracle, tmp_path):
    """Two processes on cuda:0 map each other's blocks through CUDA IPC (the one-process-
    per-GPU production layout, here time-sliced on one device); handles go over gloo.  Each
    rank then runs three frames through two pipelined, graph-captured instances."""
    import torch.multiprocessing as mp

    g, ring, ac, y, alpha, beta, step = _problem(oracle)
    cfg = pk.ReconConfig(alpha, beta, 10, step)
    ref = _reference(g, ring, ac, y, cfg)
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, y, (alpha, beta, step), str(tmp_path)))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert codes == [0, 0], codes
    a, b = (np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(2))
    assert np.array_equal(a["image"], b["image"])
    assert a["meta"][1] == 1 and b["meta"][1] == 1  # pipelined frames == the single solve
    from paper_2404_10928_b200.sharded import ShardResult

    _check(ShardResult(a["image"], a["hist"], int(a["meta"][0]), ref.stopped_by), ref)


_TIMEOUT_SCRIPT = r"""
import sys
import torch
sys.path.insert(0, sys.argv[1])
import paper_2404_10928_b200 as pk
from paper_2404_10928_b200.sharded import PeerShardSolve
F32 = pk.CudaPool(0, "float32")
g, ring, ac, ph = pk.make_scene(32, 16, 64, seed=0)
ranks = [PeerShardSolve(g, ring, ac, F32, 2, r, 2) for r in range(2)]
for r in ranks:
    r.connect([q.handle for q in ranks])
cfg = pk.ReconConfig(1e-6, 1e-8, 2, 100.0)
for r in ranks:
    r.prepare(cfg, 1e-6, 1e-8, 100.0)
y = torch.zeros(8 * 64, device="cuda")
ranks[0].launch(y, cfg, 1e-6, 1e-8, 100.0)  # rank 1 never arrives
torch.cuda.synchronize()
assert ranks[0].op.peer_timed_out()
assert not ranks[1].op.peer_timed_out()
assert torch.isnan(ranks[0].x[1]).all()
try:
    ranks[0].finish([0.0, 0.0, 0.0])
except RuntimeError as e:
    assert "timed out" in str(e)
    print("TIMEOUT-OK")
"""


def test_peer_barrier_times_out_without_hanging():
    """A rank whose peer never arrives gives up after PK_PEER_TIMEOUT_S instead of hanging
    the device; the update is poisoned with NaN and finish() raises."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PK_PEER_TIMEOUT_S="1")
    r = subprocess.run([sys.executable, "-c", _TIMEOUT_SCRIPT, root], env=env, capture_output=True,
                       text=True, timeout=240)
    assert r.returncode == 0 and "TIMEOUT-OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("world", [2, 4, 8])
def test_orbit_shards_run_symmetric_kernels(oracle, world, monkeypatch):
    """Sensor shards of whole D4 orbits (shard_sensors, pk_geometry_desc.sensor_list) keep the
    D4 back-projector and the rotation-symmetric projector on every rank (info.symmetric == 3);
    at 2 / 4 / 8 in-process ranks x stays bit-identical across ranks and the solve matches
    the fp64 oracle's reconstruction (recon.py:286-377) within the fp32 tolerance."""
    import torch

    from paper_2404_10928_b200.sharded import PeerShardSolve

    monkeypatch.setenv("PK_FSYM", "1")  # (small shards: the projector's unit count is low)
    pk.clear_plan_cache()
    n, M, Q, seed = 128, 64, 512, 2
    g, ring, ac, ph = pk.make_scene(n, M, Q, seed=seed)
    o = oracle.Operator.of(oracle.make_scene(n, M, Q, seed))
    y = o.forward(ph.values)
    alpha, beta = oracle.resolve_regularization(o, y)
    step = oracle.resolve_step(o, beta, 1e-3)
    cfg = pk.ReconConfig(alpha, beta, 10, step)
    ref = oracle.reconstruct(o, y, alpha, beta, step, 10)
    ranks = [PeerShardSolve(g, ring, ac, F32, world, r, cfg.iterations, graph=True) for r in range(world)]
    assert sorted(sum((r.sensor_ids for r in ranks), [])) == list(range(M))
    assert all(r.op.info.symmetric == 3 for r in ranks), [r.op.info.symmetric for r in ranks]
    handles = [r.handle for r in ranks]
    for r in ranks:
        r.connect(handles)
    for r in ranks:
        r.prepare(cfg, alpha, beta, step)
    streams = [torch.cuda.Stream() for _ in ranks]
    yt = torch.tensor(y, device="cuda", dtype=torch.float32)
    for r, s in zip(ranks, streams):
        with torch.cuda.stream(s):
            r.launch(r.local_y(yt), cfg, alpha, beta, step)
    torch.cuda.synchronize()
    data = sum(r.local_data_terms() for r in ranks)
    res = [r.finish(data) for r in ranks]
    for q in res[1:]:
        assert np.array_equal(q.image, res[0].image)
    assert res[0].iterations_run == 10
    err = float(np.linalg.norm(res[0].image - ref["image"]) / np.linalg.norm(ref["image"]))
    print(f"{world} orbit shards: rel L2 vs oracle {err:.3e}")
    assert err <= 1e-4
    np.testing.assert_allclose(res[0].history[:, 0], ref["objective_history"], rtol=1e-4)
    pk.clear_plan_cache()
