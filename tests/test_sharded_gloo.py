"""World-size-2 test of the sensor-sharded driver on CPU (gloo).

The production per-rank ops are CUDA kernels; here a CPU implementation built on the
oracle is substituted so the driver logic itself -- shard ranges, the all-reduce of the
partial gradient and of the data term, identical updates on every rank, the stopping
rules -- runs for real across two processes.  The sharded result must equal the
unsharded oracle reconstruction (to summation-order rounding).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_10928_b200.sharded import SensorShardedSolver, shard_range
from paper_2404_10928_b200.solver import ReconConfig


class OracleShardOps:
    """CPU stand-in for DeviceShardOps (tests only)."""

    def __init__(self, scene, m0, m1):
        from oracle import pyoracle as O

        self.O = O
        self.op = O.Operator(scene.xx, scene.yy, scene.pos, scene.c, scene.dt, scene.Q, m0, m1)
        self.shape = (scene.ny, scene.nx)
        self.pixels = scene.P
        self.r = None

    def zeros_image(self):
        return torch.zeros(self.pixels, dtype=torch.float64)

    def residual(self, x, y_local):
        self.r = self.op.forward(np.asarray(x)) - y_local
        return torch.tensor([float(self.r @ self.r)], dtype=torch.float64)

    def backproject(self):
        return torch.from_numpy(2.0 * self.op.adjoint(self.r))

    def update(self, params, x, grad):
        O = self.O
        xv = np.asarray(x, dtype=np.float64)
        g = grad.numpy().copy()
        if params.beta > 0:
            g += params.beta * O.tv_gradient(xv.reshape(self.shape), params.tv_epsilon).reshape(-1)
        xn = O.soft_threshold(xv - params.step * g, params.step * params.alpha)
        if params.nonneg:
            xn = np.maximum(xn, 0.0)
        sums = torch.tensor([np.abs(xn).sum(), O.tv_value(xn.reshape(self.shape)),
                             float(np.count_nonzero(~np.isfinite(xn))), 0.0], dtype=torch.float64)
        return torch.from_numpy(xn), sums


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q, cfg_kw):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as O

        s = O.make_scene(32, 16, 64, 3)
        full = O.Operator.of(s)
        y = full.forward(s.phantom)
        alpha, beta = O.resolve_regularization(full, y)
        step = O.resolve_step(full, beta, 1e-3)
        m0, m1 = shard_range(s.M, rank, world)
        ops = OracleShardOps(s, m0, m1)
        cfg = ReconConfig(alpha=alpha, beta=beta, step=step, **cfg_kw)
        res = SensorShardedSolver(ops).solve(y[m0 * s.Q : m1 * s.Q], cfg, alpha, beta,
                                             step if "step" not in cfg_kw else cfg_kw["step"])
        out_q.put((rank, res.image, res.history, res.iterations_run, res.stopped_by))
    finally:
        dist.destroy_process_group()


def _run(cfg_kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, cfg_kw)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(outs, key=lambda t: t[0])


def test_shard_range_partitions():
    for count in (7, 8, 512, 1000):
        for world in (1, 2, 3, 8):
            if count < world:
                continue
            spans = [shard_range(count, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(3, 0, 4)


@pytest.mark.parametrize("cfg_kw", [dict(iterations=10), dict(iterations=40, tolerance=0.2),
                                    dict(iterations=10, nonneg=True)],
                         ids=["plain", "tolerance", "nonneg"])
def test_sensor_sharded_equals_unsharded(oracle, cfg_kw):
    outs = _run(cfg_kw)
    (r0, img0, h0, n0, sb0), (r1, img1, h1, n1, sb1) = outs
    # the all-reduced gradient makes every rank apply the identical update
    assert np.array_equal(img0, img1)
    assert n0 == n1 and sb0 == sb1
    s = oracle.make_scene(32, 16, 64, 3)
    full = oracle.Operator.of(s)
    y = full.forward(s.phantom)
    alpha, beta = oracle.resolve_regularization(full, y)
    step = oracle.resolve_step(full, beta, 1e-3)
    ref = oracle.reconstruct(full, y, alpha, beta, step, cfg_kw["iterations"],
                             nonneg=cfg_kw.get("nonneg", False),
                             tolerance=cfg_kw.get("tolerance", 0.0))
    assert n0 == ref["iterations_run"] and sb0 == ref["stopped_by"]
    assert oracle.rel_l2(img0, ref["image"]) <= 1e-12
    np.testing.assert_allclose(h0[:, 0], ref["objective_history"], rtol=1e-12)


# --------------------------------------------------------------------------- device-resident
# drivers (SpeculativeShardSolve, PeerShardSolve) on CPU: an oracle-backed stand-in for the
# DeviceOperator they drive, with the peer exchange emulated by an all_gather in rank order


class OracleDeviceOp:
    """The DeviceOperator surface the sharded drivers use, on the CPU oracle (tests only):
    residual_into / adjoint_residual / grad_update_into, and the peer entry points with the
    device barrier + rank-ordered slot sum of pk_peer_grad_update emulated over gloo."""

    def __init__(self, scene, ids):
        from oracle import pyoracle as O

        self.O = O
        self.sensor_ids = list(ids)
        pos = np.ascontiguousarray(scene.pos[self.sensor_ids])
        self.o = O.Operator(scene.xx, scene.yy, pos, scene.c, scene.dt, scene.Q)
        self.shape = (scene.ny, scene.nx)
        self.P, self.sensors, self.samples = scene.P, len(ids), scene.Q
        self.device, self.tdtype = torch.device("cpu"), torch.float64
        self.r = None
        self._slots = None

    # the plain sharded pieces
    def residual_into(self, x, y, sumsq, r=None):
        self.r = self.o.forward(x.numpy()) - y.numpy()
        sumsq[0] = float(self.r @ self.r)

    def adjoint_residual(self, scale=1.0, out=None):
        g = torch.from_numpy(scale * self.o.adjoint(self.r))
        if out is None:
            return g
        out.copy_(g)
        return out

    def grad_update_into(self, params, x, grad, xo, sums):
        O, xv = self.O, x.numpy()
        g = grad.numpy().copy()
        if params.beta > 0:
            g += params.beta * O.tv_gradient(xv.reshape(self.shape), params.tv_epsilon).reshape(-1)
        xn = O.soft_threshold(xv - params.step * g, params.step * params.alpha)
        if params.nonneg:
            xn = np.maximum(xn, 0.0)
        xo.copy_(torch.from_numpy(xn))
        sums.copy_(torch.tensor([np.abs(xn).sum(), O.tv_value(xn.reshape(self.shape)),
                                 float(np.count_nonzero(~np.isfinite(xn))), 0.0], dtype=torch.float64))

    # peer exchange
    def peer_handle(self):
        self._slots = [torch.zeros(self.P, dtype=torch.float64) for _ in range(2)]
        return f"rank{dist.get_rank()}".encode().ljust(64, b"\0")

    def peer_buffer(self, slot):
        return self._slots[slot]

    def peer_connect(self, world, rank, handles):
        assert len(handles) == world and handles[rank].startswith(f"rank{rank}".encode())

    def adjoint_residual_to(self, scale, slot_tensor):
        slot_tensor.copy_(torch.from_numpy(scale * self.o.adjoint(self.r)))

    def peer_grad_update_into(self, params, x, slot, xo, sums):
        parts = [torch.empty(self.P, dtype=torch.float64) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, self._slots[slot])  # the barrier + every rank's slot
        grad = parts[0].clone()
        for p in parts[1:]:  # rank order, as the fused update kernel sums them
            grad += p
        self.grad_update_into(params, x, grad, xo, sums)

    def peer_timed_out(self):
        return False


def _device_driver_worker(rank, world, port, out_q, kind, cfg_kw):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as O
        from paper_2404_10928_b200.sharded import (DeviceShardOps, PeerShardSolve, SpeculativeShardSolve,
                                                    local_traces, shard_sensors)

        s = O.make_scene(32, 16, 64, 3)
        full = O.Operator.of(s)
        y = full.forward(s.phantom)
        alpha, beta = O.resolve_regularization(full, y)
        step = cfg_kw.pop("step", None) or O.resolve_step(full, beta, 1e-3)
        cfg = ReconConfig(alpha=alpha, beta=beta, step=step, **cfg_kw)
        ids = shard_sensors(s.M, rank, world)
        op = OracleDeviceOp(s, ids)
        yl = torch.from_numpy(local_traces(y, ids, s.Q).copy())
        if kind == "speculative":
            ops = DeviceShardOps.__new__(DeviceShardOps)  # the stand-in op, no plan
            ops.op, ops.pixels, ops.sensor_ids = op, s.P, ids
            res = SpeculativeShardSolve(ops, cfg.iterations, graph=False).solve(yl, cfg, alpha, beta, step)
        else:
            class _G:  # grid / ring stand-ins: only .size and .count are read
                size = s.P
                count = s.M
            sol = PeerShardSolve(_G, _G, None, None, world, rank, cfg.iterations, op=op)
            sol.connect_distributed()
            res = sol.solve(yl, cfg, alpha, beta, step)
        out_q.put((rank, ids, res.image, res.history, res.iterations_run, res.stopped_by))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["speculative", "peer"])
@pytest.mark.parametrize("cfg_kw", [dict(iterations=10), dict(iterations=40, tolerance=0.2),
                                    dict(iterations=12, step=0.5)],
                         ids=["plain", "tolerance", "divergence"])
def test_device_resident_shard_drivers(oracle, kind, cfg_kw):
    """The drivers the bench runs -- SpeculativeShardSolve (NCCL all-reduce) and PeerShardSolve
    (peer-slot sum in rank order) -- on 2 gloo ranks over D4-orbit shards: all iterations are
    enqueued, the stopping rules are applied afterwards to the recorded terms (stop_point),
    and the accepted iterate equals the unsharded oracle reconstruction on both ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_device_driver_worker, args=(r, 2, port, q, kind, dict(cfg_kw)))
             for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, ids0, img0, h0, n0, sb0), (_, ids1, img1, h1, n1, sb1) = outs
    assert sorted(ids0 + ids1) == list(range(16)) and not set(ids0) & set(ids1)
    assert np.array_equal(img0, img1) and n0 == n1 and sb0 == sb1
    s = oracle.make_scene(32, 16, 64, 3)
    full = oracle.Operator.of(s)
    y = full.forward(s.phantom)
    alpha, beta = oracle.resolve_regularization(full, y)
    step = cfg_kw.get("step") or oracle.resolve_step(full, beta, 1e-3)
    ref = oracle.reconstruct(full, y, alpha, beta, step, cfg_kw["iterations"],
                             tolerance=cfg_kw.get("tolerance", 0.0))
    assert n0 == ref["iterations_run"] and sb0 == ref["stopped_by"], (n0, sb0, ref["stopped_by"])
    if sb0 != "divergence":
        assert oracle.rel_l2(img0, ref["image"]) <= 1e-12
    np.testing.assert_allclose(h0[:, 0], ref["objective_history"], rtol=1e-12)


def test_shard_sensors_whole_d4_orbits():
    """shard_sensors: a partition of the ring into whole D4 orbits (closed under m -> m + M/4
    and m -> -m), balanced to within one orbit, identical on every rank."""
    from paper_2404_10928_b200.sharded import d4_orbits, shard_sensors

    for M in (16, 32, 64, 128, 512, 1024):
        q = M // 4
        assert sorted(sum(d4_orbits(M), [])) == list(range(M))
        for world in (1, 2, 3, 4, 8):
            if len(d4_orbits(M)) < world:
                continue
            shards = [shard_sensors(M, r, world) for r in range(world)]
            assert sorted(sum(shards, [])) == list(range(M))
            for sh in shards:
                st = set(sh)
                assert all((m + q) % M in st and (-m) % M in st for m in sh)
            sizes = [len(sh) for sh in shards]
            assert max(sizes) - min(sizes) <= 8
    assert shard_sensors(30, 1, 2) == list(range(15, 30))  # no D4: contiguous ranges
