"""Multi-GPU drivers: one process per GPU, torch.distributed (NCCL) for the plumbing.

Two natural shardings of the hot path:

* ``SensorShardedSolver`` -- one large frame, sensors split across ranks.  Rank g owns
  sensors [g*M/G, (g+1)*M/G) and its slice of y and r; x is replicated.  Per iteration:
  local back-projection (partial 2 K_g^T r_g) -> all-reduce(sum) of the image-sized
  gradient -> identical update on every rank -> local projection and residual ->
  all-reduce of the data-term scalar.  This is the only exchange the algorithm has.
* ``FrameShardedSolver`` -- a dynamic sequence: independent frames per rank, no
  collective at all (weak scaling).

The per-rank compute goes through an ``ops`` object; the production one is
``DeviceShardOps`` (C ABI kernels on the rank's GPU).  Tests substitute a CPU
implementation to exercise the sharding / reduction / stopping logic with gloo.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .device import CudaPool, operator_for
from .solver import DIVERGENCE_STREAK, ReconConfig, solver_params

__all__ = ["shard_range", "shard_sensors", "d4_orbits", "local_traces", "DeviceShardOps", "SensorShardedSolver", "SpeculativeShardSolve",
           "PeerShardSolve", "PipelinedShardSolve", "FrameShardedSolver", "stop_point"]


def shard_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced split of [0, count) -- sizes differ by at most one."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world of {world}")
    if count < world:
        raise ValueError(f"cannot split {count} sensors over {world} ranks")
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def d4_orbits(count: int) -> list[list[int]]:
    """Orbits of the ring indices under the ring's D4 symmetry (rotation m -> m + M/4,
    reflection m -> -m), sorted by their smallest member; M % 4 == 0."""
    if count % 4:
        raise ValueError(f"a ring of {count} sensors has no D4 symmetry")
    q = count // 4
    return [sorted({(sgn * b + k * q) % count for sgn in (1, -1) for k in range(4)})
            for b in range(q // 2 + 1)]


def shard_sensors(count: int, rank: int, world: int) -> list[int]:
    """Rank `rank`'s sensors when the ring is split into whole D4 orbits (rotation-closed and
    reflection-closed shards), balanced by sensor count: each rank's plan keeps the symmetric
    back-projector and projector (one delay per 8 / 4 pairs), with every rank's traces a
    list of ring indices (pk_geometry_desc.sensor_list).  Orbits go, largest first, to the
    rank with the fewest sensors (ties: lowest rank) -- deterministic on every rank.  A ring
    without D4 symmetry (M % 4 != 0) falls back to the contiguous shard_range."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world of {world}")
    if count % 4:
        lo, hi = shard_range(count, rank, world)
        return list(range(lo, hi))
    orbits = d4_orbits(count)
    if len(orbits) < world:
        raise ValueError(f"cannot split {len(orbits)} D4 orbits over {world} ranks")
    load, own = [0] * world, [[] for _ in range(world)]
    for orb in sorted(orbits, key=lambda o: (-len(o), o[0])):
        r = min(range(world), key=lambda k: (load[k], k))
        own[r].extend(orb)
        load[r] += len(orb)
    return sorted(own[rank])


def local_traces(y_full, sensor_ids, samples: int):
    """Rows `sensor_ids` (ring indices, in order) of a whole-ring trace vector [M*Q]: a
    contiguous slice for a range shard, a gather for a D4-orbit shard (tensor or array)."""
    ids = list(sensor_ids)
    if ids == list(range(ids[0], ids[0] + len(ids))):
        return y_full[ids[0] * samples:(ids[-1] + 1) * samples]
    try:
        import torch

        if isinstance(y_full, torch.Tensor):
            idx = torch.tensor(ids, device=y_full.device)
            return y_full.view(-1, samples).index_select(0, idx).reshape(-1).contiguous()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(y_full).reshape(-1, samples)[ids].reshape(-1)


class DeviceShardOps:
    """Per-rank kernels (C ABI) for a sensor shard: a contiguous range [m0, m1) or, with
    ``sensors``, a list of ring indices (e.g. shard_sensors' D4-closed shards)."""

    def __init__(self, grid, ring, acoustic, pool: CudaPool, m0: int = 0, m1: int | None = None,
                 sensors=None):
        self.op = operator_for(grid, ring, acoustic, pool, m0, m1, sensor_list=sensors)
        self.pixels = grid.size
        self.sensor_ids = self.op.sensor_ids

    def zeros_image(self):
        import torch

        return torch.zeros(self.pixels, device=self.op.device, dtype=self.op.tdtype)

    def residual(self, x, y_local):
        """r = K_g x - y_g kept on the device for the next back-projection; returns sum r^2
        as a 1-element fp64 tensor."""
        _, ss = self.op.residual(x, y_local)
        return ss

    def backproject(self):
        """2 K_g^T r_g (partial data gradient)."""
        return self.op.adjoint_residual(2.0)

    def update(self, params, x, grad):
        """x' = prox(x - eta (grad + beta tv_grad x)); returns (x', [sum|x'|, TV(x'), #nonfinite])."""
        return self.op.grad_update(params, x, grad)


@dataclass
class ShardResult:
    image: np.ndarray
    history: np.ndarray  # (n, 4): total, data, l1, tv
    iterations_run: int
    stopped_by: str


class SensorShardedSolver:
    """iterative_reconstruct (recon.py:286-377) over sensor shards with an all-reduce."""

    def __init__(self, ops, group=None):
        self.ops = ops
        self.group = group

    def _allreduce(self, t):
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(t, group=self.group)
        return t

    def solve(self, y_local, config: ReconConfig, alpha: float, beta: float, step: float) -> ShardResult:
        import torch

        params = solver_params(config, alpha, beta, step)
        x = self.ops.zeros_image()
        ss = self.ops.residual(x, y_local)  # r0 = -y
        f_prev = float(self._allreduce(ss.clone())[0])
        hist = []
        stopped_by = "max_iterations"
        grow = 0
        for _ in range(config.iterations):
            grad = self.ops.backproject()
            self._allreduce(grad)
            x_new, sums = self.ops.update(params, x, grad)
            ss = self.ops.residual(x_new, y_local)
            data = float(self._allreduce(ss.clone())[0])
            s = sums.double().cpu().numpy()
            l1, tvv, bad = alpha * float(s[0]), beta * float(s[1]), float(s[2])
            total = data + l1 + tvv
            if not math.isfinite(total) or bad > 0:
                stopped_by = "divergence"
                # the residual kept by the device is r(x_new); x stays the last accepted one
                break
            hist.append((total, data, l1, tvv))
            x = x_new
            grow = grow + 1 if total > f_prev else 0
            if grow >= DIVERGENCE_STREAK:
                stopped_by = "divergence"
                break
            rel = abs(total - f_prev) / max(abs(f_prev), 1e-300)
            f_prev = total
            if config.tolerance > 0 and rel < config.tolerance:
                stopped_by = "tolerance"
                break
        img = x.double().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x, dtype=np.float64)
        return ShardResult(img, np.array(hist, dtype=np.float64).reshape(-1, 4), len(hist), stopped_by)


def stop_point(hist_raw, f0: float, alpha: float, beta: float, tolerance: float):
    """The stopping rules of recon.py:346-363 applied after the fact to per-iteration
    (data, sum|x|, TV, #nonfinite) rows: returns (iterations_run, stopped_by, history)."""
    hist = []
    f_prev, grow = f0, 0
    for data, l1s, tvs, bad in hist_raw:
        l1, tvv = alpha * l1s, beta * tvs
        total = data + l1 + tvv
        if not math.isfinite(total) or bad > 0:
            return len(hist), "divergence", hist
        hist.append((total, data, l1, tvv))
        grow = grow + 1 if total > f_prev else 0
        if grow >= DIVERGENCE_STREAK:
            return len(hist), "divergence", hist
        rel = abs(total - f_prev) / max(abs(f_prev), 1e-300)
        f_prev = total
        if tolerance > 0 and rel < tolerance:
            return len(hist), "tolerance", hist
    return len(hist), "max_iterations", hist


class SpeculativeShardSolve:
    """Device-resident sensor-sharded solve: all N iterations are enqueued without a host
    round trip (iterates kept on the device), the stopping rules are applied afterwards to
    the recorded objective terms, and the accepted iterate is returned -- the same result as
    ``SensorShardedSolver.solve``, with iterations past a stop computed but discarded.  With
    static buffers the whole solve, NCCL all-reduces included, is captured once into a CUDA
    graph (``graph=True``) and replayed per frame."""

    def __init__(self, ops: "DeviceShardOps", iterations: int, graph: bool = False, group=None):
        import torch

        self.ops, self.n, self.group = ops, iterations, group
        op = ops.op
        P = ops.pixels
        self.y = torch.zeros(op.sensors * op.samples, device=op.device, dtype=op.tdtype)
        self.x = torch.zeros(iterations + 1, P, device=op.device, dtype=op.tdtype)
        self.grad = torch.empty(P, device=op.device, dtype=op.tdtype)
        self.ss = torch.zeros(iterations + 1, 1, device=op.device, dtype=torch.float64)
        self.sums = torch.zeros(iterations, 4, device=op.device, dtype=torch.float64)
        self.graph = None
        self._use_graph = graph
        self._params = None

    def _allreduce(self, t):
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(t, group=self.group)

    def _body(self):
        ops, p = self.ops, self._params
        ops.op.residual_into(self.x[0], self.y, self.ss[0])  # r0 = -y
        self._allreduce(self.ss[0])
        for it in range(self.n):
            ops.op.adjoint_residual(2.0, out=self.grad)
            self._allreduce(self.grad)
            ops.op.grad_update_into(p, self.x[it], self.grad, self.x[it + 1], self.sums[it])
            ops.op.residual_into(self.x[it + 1], self.y, self.ss[it + 1])
            self._allreduce(self.ss[it + 1])

    def solve(self, y_local, config: ReconConfig, alpha: float, beta: float, step: float) -> ShardResult:
        import torch

        params = solver_params(config, alpha, beta, step)
        key = (params.alpha, params.beta, params.step, params.tv_epsilon, params.nonneg)
        self.y.copy_(y_local)
        if self._params is None or self._key != key:
            self._params, self._key, self.graph = params, key, None
        if self._use_graph and self.graph is None:
            self._body()  # warm-up: plan workspaces, parameter upload, NCCL communicators
            torch.cuda.current_stream().synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._body()
            self.graph = g
        if self.graph is not None:
            self.graph.replay()
        else:
            self._body()
        ss = self.ss[:, 0].cpu().numpy()
        sums = self.sums.cpu().numpy()
        rows = [(float(ss[i + 1]), float(sums[i, 0]), float(sums[i, 1]), float(sums[i, 2]))
                for i in range(self.n)]
        k, stopped_by, hist = stop_point(rows, float(ss[0]), alpha, beta, config.tolerance)
        img = self.x[k].double().cpu().numpy()
        return ShardResult(img, np.array(hist, dtype=np.float64).reshape(-1, 4), k, stopped_by)


class PeerShardSolve:
    """Sensor-sharded solve with the gradient exchanged over peer memory (NVLink /
    NVSwitch) instead of an NCCL all-reduce: per iteration

        pk_adjoint_residual  -> this rank's partial 2 K_g^T r_g into its peer slot (it & 1)
        pk_peer_grad_update  -> device barrier of the world, grad = sum of all ranks' slots in
                                rank order (peer loads) fused with the TV + prox update
        pk_residual          -> r_g = K_g x' - y_g and its sum of squares

    so the only collective is fused into the update kernel and x stays bit-identical on every
    rank.  Like ``SpeculativeShardSolve`` all N iterations are enqueued without a host round
    trip (optionally as one CUDA graph); the per-rank data terms are summed once at the end
    and the stopping rules applied afterwards (``stop_point``).

    One instance per rank (process or, for tests, plan on a shared device).  Handles are
    exchanged with ``connect`` (``handles`` in rank order) or, in a torch.distributed job,
    with ``connect_distributed``."""

    def __init__(self, grid, ring, acoustic, pool: CudaPool, world: int, rank: int,
                 iterations: int, graph: bool = False, layout: str = "orbits", op=None):
        import torch

        from .device import DeviceOperator

        self.world, self.rank, self.n = int(world), int(rank), int(iterations)
        M = int(ring.count)
        if op is not None:  # an operator with the same interface (tests: a CPU stand-in)
            self.op = op
            self.sensor_ids = list(op.sensor_ids)
        elif layout == "orbits":  # whole D4 orbits: the shard keeps the symmetric kernels
            self.sensor_ids = shard_sensors(M, rank, world)
            self.op = op = DeviceOperator(grid, ring, acoustic, pool, sensor_list=self.sensor_ids)
        elif layout == "contiguous":
            m0, m1 = shard_range(M, rank, world)
            self.sensor_ids = list(range(m0, m1))
            self.op = op = DeviceOperator(grid, ring, acoustic, pool, m0, m1)
        else:
            raise ValueError(f"layout must be 'orbits' or 'contiguous', got {layout!r}")
        op = self.op
        P = grid.size
        self.y = torch.zeros(op.sensors * op.samples, device=op.device, dtype=op.tdtype)
        self.x = torch.zeros(iterations + 1, P, device=op.device, dtype=op.tdtype)
        self.ss = torch.zeros(iterations + 1, device=op.device, dtype=torch.float64)
        self.sums = torch.zeros(iterations, 4, device=op.device, dtype=torch.float64)
        self.handle = op.peer_handle()
        self.slots = (op.peer_buffer(0), op.peer_buffer(1))
        self._use_graph, self.graph, self._key, self._params = graph, None, None, None
        self._stream = None
        self._alpha = self._beta = 0.0
        self._tol = 0.0

    def local_y(self, y_full):
        """This rank's traces of a whole-ring measurement [M*Q] (trace order of the plan)."""
        return local_traces(y_full, self.sensor_ids, self.op.samples)

    def connect(self, handles) -> None:
        self.op.peer_connect(self.world, self.rank, handles)

    def connect_distributed(self, group=None) -> None:
        """Exchange handles with all_gather_object and connect (then a barrier, so no rank
        signals a peer block before that peer has mapped the world)."""
        import torch.distributed as dist

        import torch

        handles = [None] * self.world
        dist.all_gather_object(handles, self.handle, group=group)
        err = None
        try:
            self.connect(handles)
        except Exception as e:  # e.g. no peer access between two devices of this node
            err = e
        # every rank learns whether any rank failed, so all raise together (none is left
        # waiting in a collective of a solve the others abandoned)
        dev = torch.device("cuda", self.op.pool.device) if dist.get_backend(group) == "nccl" else "cpu"
        bad = torch.tensor([1 if err is not None else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=group)
        if int(bad.item()):
            raise RuntimeError(f"peer exchange unavailable on rank {self.rank}: "
                               f"{err if err is not None else 'another rank failed to connect'}")
        dist.barrier(group=group)

    def _body(self):
        op, p = self.op, self._params
        op.residual_into(self.x[0], self.y, self.ss[0:1])  # r0 = -y
        for it in range(self.n):
            slot = it & 1
            op.adjoint_residual_to(2.0, self.slots[slot])
            op.peer_grad_update_into(p, self.x[it], slot, self.x[it + 1], self.sums[it])
            op.residual_into(self.x[it + 1], self.y, self.ss[it + 1:it + 2])

    def prepare(self, config: ReconConfig, alpha: float, beta: float, step: float) -> None:
        """Upload the solver parameters and (graph mode) capture the solve.  Capturing does
        not run it, so the barrier epochs advance only on replay, identically on every rank.
        Ranks sharing one device in one process must all prepare before any launches (the
        capture synchronises the device)."""
        import torch

        params = solver_params(config, alpha, beta, step)
        key = (params.alpha, params.beta, params.step, params.tv_epsilon, params.nonneg)
        self._alpha, self._beta, self._tol = alpha, beta, config.tolerance
        if self._key == key:
            return
        self._params, self._key, self.graph = params, key, None
        # parameter upload outside any capture, and one pass over every kernel of the body:
        # under lazy module loading a first launch waits for the device to drain, which never
        # happens while another rank of this process spins in its barrier (scratch results)
        op = self.op
        op.grad_update_into(params, self.x[0], self.x[0], self.x[1], self.sums[0])
        op.residual_into(self.x[0], self.y, self.ss[0:1])
        op.adjoint_residual_to(2.0, self.slots[0])
        if self._use_graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._body()
            self.graph = g

    def launch(self, y_local, config: ReconConfig, alpha: float, beta: float, step: float) -> None:
        """Enqueue the whole solve on the current stream (returns without synchronising)."""
        import torch

        self.prepare(config, alpha, beta, step)
        self._stream = torch.cuda.current_stream(self.y.device) if self.y.is_cuda else None
        self.y.copy_(torch.as_tensor(y_local).to(self.y.device, self.y.dtype), non_blocking=True)
        if self.graph is not None:
            self.graph.replay()
        else:
            self._body()

    def local_data_terms(self):
        """This rank's sum r_g^2 after 0..N iterations (waits for the launch's stream)."""
        if self._stream is not None:
            self._stream.synchronize()
        return self.ss.cpu().numpy()

    def finish(self, data_terms=None) -> ShardResult:
        """Apply the stopping rules.  ``data_terms`` = the world's summed data terms (N+1
        values); default: all-reduce of the local ones over torch.distributed."""
        if data_terms is None:
            data_terms = _allreduce_host(self.local_data_terms())
        if self.op.peer_timed_out():
            raise RuntimeError(f"rank {self.rank}: peer barrier timed out (a rank did not arrive)")
        ss = np.asarray(data_terms, dtype=np.float64)
        sums = self.sums.cpu().numpy()
        rows = [(float(ss[i + 1]), float(sums[i, 0]), float(sums[i, 1]), float(sums[i, 2]))
                for i in range(self.n)]
        k, stopped_by, hist = stop_point(rows, float(ss[0]), self._alpha, self._beta, self._tol)
        img = self.x[k].double().cpu().numpy()
        return ShardResult(img, np.array(hist, dtype=np.float64).reshape(-1, 4), k, stopped_by)

    def solve(self, y_local, config: ReconConfig, alpha: float, beta: float, step: float) -> ShardResult:
        self.launch(y_local, config, alpha, beta, step)
        return self.finish()


class PipelinedShardSolve:
    """Several independent frames of a sensor-sharded solve in flight at once (SURVEY 8(e):
    one frame's exchange overlaps another frame's compute): S ``PeerShardSolve`` instances,
    each with its own plan, peer block and CUDA stream; frame f runs on instance f % S, and
    its result is collected once frame f + S - 1 has been enqueued.  Every rank must call
    ``solve_frames`` with the same number of frames (the per-frame data-term all-reduces are
    collectives)."""

    def __init__(self, solvers):
        import torch

        self.solvers = list(solvers)
        dev = self.solvers[0].y.device
        self.streams = [torch.cuda.Stream(dev) for _ in self.solvers]

    def solve_frames(self, ys, config: ReconConfig, alpha: float, beta: float, step: float):
        import torch

        S, out, pending = len(self.solvers), [], []
        for s in self.solvers:  # parameter upload / graph capture before anything is in flight
            s.prepare(config, alpha, beta, step)
        for f, y in enumerate(ys):
            q = f % S
            if len(pending) == S:  # instance q is about to be reused: collect its frame
                out.append(pending.pop(0).finish())
            self.streams[q].wait_stream(torch.cuda.current_stream(self.streams[q].device))
            with torch.cuda.stream(self.streams[q]):
                self.solvers[q].launch(y, config, alpha, beta, step)
            pending.append(self.solvers[q])
        out.extend(s.finish() for s in pending)
        return out


def _allreduce_host(a: np.ndarray) -> np.ndarray:
    """Sum a small host array over the torch.distributed world (any backend)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return a
    t = torch.as_tensor(np.asarray(a, dtype=np.float64))
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t)
    return t.cpu().numpy()


class FrameShardedSolver:
    """Independent frames of a dynamic sequence on this rank (no collective)."""

    def __init__(self, grid, ring, acoustic, pool: CudaPool):
        self.op = operator_for(grid, ring, acoustic, pool)

    @staticmethod
    def frames_of(total: int, rank: int, world: int) -> range:
        lo, hi = shard_range(total, rank, world)
        return range(lo, hi)

    def solve(self, y, config: ReconConfig, alpha: float, beta: float, step: float):
        params = solver_params(config, alpha, beta, step)
        return self.op.reconstruct(y, params)
