"""Back-projection and the compressed-sensing iterative reconstruction, on the device.

Public surface of the reference's ``pactkit.recon`` (pkg/src/pactkit/recon.py:24-40) with
the same signatures, argument meaning, error behaviour and result types.  The hot loop
(recon.py:318-363) runs entirely on the B200 through ``pk_reconstruct``: one fused
back-projection + TV + soft-threshold (+ non-negativity) kernel, one projection kernel and
one residual/objective kernel per iteration, with the stopping rules evaluated on the
device and the whole solve replayed from a captured CUDA graph.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _native as N
from .device import CudaPool, DeviceOperator
from .measurement import (DenseOperator, FreqOperator, SensorData, _as_pool, device_operator,
                          geometry_path)
from .scene import ImageField

__all__ = [
    "ReconConfig",
    "ReconResult",
    "ObjectiveParts",
    "back_project",
    "data_gradient",
    "soft_threshold",
    "tv_value",
    "tv_gradient",
    "objective",
    "estimate_lipschitz",
    "iterative_reconstruct",
    "resolve_regularization",
    "resolve_config",
    "solver_params",
    "reconstruct_frames",
    "rmse",
    "psnr",
]

DIVERGENCE_STREAK = 5  # recon.py:42-43


@dataclass(frozen=True)
class ReconConfig:
    """Solver settings (recon.py:46-79): alpha/beta None -> calibrated from the data,
    step "auto" -> 1/(2 sigma_max^2 + 8 beta/eps), tolerance 0 -> run all iterations."""

    alpha: float | None = None
    beta: float | None = None
    iterations: int = 90
    step: float | str = "auto"
    tv_epsilon: float = 1e-3
    nonneg: bool = False
    tolerance: float = 0.0

    def __post_init__(self):
        if self.alpha is not None and self.alpha < 0:
            raise ValueError(f"alpha must be >= 0, got {self.alpha}")
        if self.beta is not None and self.beta < 0:
            raise ValueError(f"beta must be >= 0, got {self.beta}")
        if self.iterations < 1:
            raise ValueError(f"iterations must be >= 1, got {self.iterations}")
        if not self.tv_epsilon > 0:
            raise ValueError(f"tv_epsilon must be > 0, got {self.tv_epsilon}")
        if self.tolerance < 0:
            raise ValueError(f"tolerance must be >= 0, got {self.tolerance}")
        if isinstance(self.step, str):
            if self.step != "auto":
                raise ValueError(f"step must be a positive number or 'auto', got {self.step!r}")
        elif not self.step > 0:
            raise ValueError(f"step must be > 0, got {self.step}")


@dataclass(frozen=True)
class ReconResult:
    image: ImageField
    objective_history: np.ndarray
    data_term_history: np.ndarray
    l1_history: np.ndarray
    tv_history: np.ndarray
    iterations_run: int
    stopped_by: str  # "max_iterations" | "tolerance" | "divergence"
    alpha_used: float = 0.0
    beta_used: float = 0.0
    step_used: float = 0.0


class ObjectiveParts(NamedTuple):
    total: float
    data: float
    l1: float
    tv: float


# ---------------------------------------------------------------------------
# argument checks (recon.py:103-116)


def _grid_of(K, grid):
    g = grid or getattr(K, "grid", None)
    if g is None:
        raise ValueError("matrix carries no grid; pass grid= explicitly")
    if g.size != K.cols:
        raise ValueError(f"grid {g.nx}x{g.ny} does not match matrix columns {K.cols}")
    return g


def _check_pair(K, y):
    if K.domain != y.domain:
        raise ValueError(f"domain mismatch: matrix is {K.domain}, signal is {y.domain}")
    if K.rows != y.length:
        raise ValueError(f"matrix has {K.rows} rows but signal has {y.length} values")


def _real(t):
    return t.real if t.is_complex() else t


# ---------------------------------------------------------------------------
# products


def back_project(K, y, grid=None, pool=None) -> ImageField:
    """Re(K^H y) scaled to unit peak (an all-zero signal stays zero) -- recon.py:119-136."""
    g = _grid_of(K, grid)
    _check_pair(K, y)
    op = device_operator(K, pool)
    x = _real(op.adjoint(y.values, 1.0)).double()
    peak = x.abs().max()
    x = x / peak if float(peak) > 0 else x
    return ImageField(g, x.cpu().numpy())


def _data_gradient_dev(op, xv, yv):
    if isinstance(op, DeviceOperator):
        op.residual(xv, yv)
        return op.adjoint_residual(2.0)
    r = op.matvec(xv) - op.tensor(yv)
    return 2.0 * _real(op.adjoint(r, 1.0))


def data_gradient(K, x, y, pool=None) -> ImageField:
    """2 Re(K^H (K x - y)) -- recon.py:146-155."""
    g = _grid_of(K, x.grid)
    _check_pair(K, y)
    op = device_operator(K, pool)
    return ImageField(g, _data_gradient_dev(op, x.values, y.values).double().cpu().numpy())


# ---------------------------------------------------------------------------
# small host utilities of the public API (not on the device loop; recon.py:158-189)


def soft_threshold(v: ImageField, lam: float) -> ImageField:
    if lam < 0:
        raise ValueError(f"lambda must be >= 0, got {lam}")
    a = v.values
    return ImageField(v.grid, np.sign(a) * np.maximum(np.abs(a) - lam, 0.0))


def _tv_of(img: np.ndarray) -> float:
    return float(np.abs(np.diff(img, axis=1)).sum() + np.abs(np.diff(img, axis=0)).sum())


def tv_value(x: ImageField) -> float:
    """Anisotropic total variation (recon.py:169-175)."""
    return _tv_of(x.image)


def _tv_grad_np(img: np.ndarray, eps: float) -> np.ndarray:
    h = np.diff(img, axis=1)
    v = np.diff(img, axis=0)
    wh = h / np.sqrt(h * h + eps * eps)
    wv = v / np.sqrt(v * v + eps * eps)
    out = np.zeros_like(img)
    out[:, :-1] -= wh
    out[:, 1:] += wh
    out[:-1, :] -= wv
    out[1:, :] += wv
    return out


def tv_gradient(x: ImageField, epsilon: float) -> ImageField:
    if not epsilon > 0:
        raise ValueError(f"epsilon must be > 0, got {epsilon}")
    return ImageField(x.grid, _tv_grad_np(x.image, epsilon).reshape(-1))


# ---------------------------------------------------------------------------
# calibration (recon.py:199-283)


def resolve_regularization(config: ReconConfig, K, y, pool=None) -> tuple[float, float]:
    """alpha = 1e-3 max|2 Re(K^H y)| unless given, beta = 1e-2 alpha unless given."""
    alpha = config.alpha
    if alpha is None:
        op = device_operator(K, pool)
        alpha = 1e-3 * float(_real(op.adjoint(y.values, 2.0)).abs().max())
    beta = config.beta
    if beta is None:
        beta = 1e-2 * alpha
    return float(alpha), float(beta)


def estimate_lipschitz(K, iterations: int = 50, seed: int = 0, pool=None) -> float:
    """Power iteration for sigma_max(K)^2 (recon.py:236-261), products on the device.

    Same seeded start vector as the reference (numpy default_rng(seed)); norms in fp64.
    Accepts a MeasurementMatrix or a plain 2-D array.
    """
    import torch

    if iterations < 1:
        raise ValueError(f"iterations must be >= 1, got {iterations}")
    op = device_operator(K, pool)
    cols = op.pixels if isinstance(op, DeviceOperator) else op.cols
    rng = np.random.default_rng(seed)
    is_cplx = isinstance(op, (DenseOperator, FreqOperator)) and op.tdtype.is_complex
    v = rng.standard_normal(cols) + 1j * rng.standard_normal(cols) if is_cplx else rng.standard_normal(cols)
    nrm = np.linalg.norm(v)
    if nrm == 0:
        return 0.0
    vt = op.tensor(v / nrm)
    zero_seen = torch.zeros((), dtype=torch.bool, device=vt.device)
    for _ in range(iterations):
        w = op.adjoint(op.matvec(vt), 1.0)
        n = torch.linalg.vector_norm(w.to(torch.complex128 if w.is_complex() else torch.float64))
        zero_seen |= n == 0
        vt = w / n.to(w.dtype)
    if bool(zero_seen):
        return 0.0
    kv = op.matvec(vt)
    return float(torch.linalg.vector_norm(kv.to(torch.complex128 if kv.is_complex() else torch.float64)) ** 2)


def _resolve_step(config: ReconConfig, K, beta: float, pool=None) -> float:
    if config.step != "auto":
        return float(config.step)
    sigma_sq = estimate_lipschitz(K, iterations=50, seed=0, pool=pool)
    lipschitz = 2.0 * sigma_sq + beta * 8.0 / config.tv_epsilon
    return 1.0 / lipschitz if lipschitz > 0 else 1.0


def resolve_config(config: ReconConfig, K, y, pool=None) -> ReconConfig:
    """Pin auto alpha/beta/step to the values the solver would use (recon.py:272-283)."""
    alpha, beta = resolve_regularization(config, K, y, pool)
    return ReconConfig(
        alpha=alpha,
        beta=beta,
        iterations=config.iterations,
        step=_resolve_step(config, K, beta, pool),
        tv_epsilon=config.tv_epsilon,
        nonneg=config.nonneg,
        tolerance=config.tolerance,
    )


def solver_params(config: ReconConfig, alpha: float, beta: float, step: float) -> N.SolverParams:
    return N.SolverParams(
        alpha=float(alpha), beta=float(beta), step=float(step),
        tv_epsilon=float(config.tv_epsilon), tolerance=float(config.tolerance),
        iterations=int(config.iterations), nonneg=1 if config.nonneg else 0,
    )


# ---------------------------------------------------------------------------
# objective (recon.py:212-227)


def _parts_dev(r, x, shape, alpha, beta) -> ObjectiveParts:
    import torch

    r64 = r.to(torch.complex128) if r.is_complex() else r.double()
    data = float(torch.real(torch.vdot(r64, r64)))
    xi = x.double().reshape(shape)
    l1 = alpha * float(xi.abs().sum())
    tvv = float((xi[:, 1:] - xi[:, :-1]).abs().sum() + (xi[1:, :] - xi[:-1, :]).abs().sum())
    tv = beta * tvv
    return ObjectiveParts(data + l1 + tv, data, l1, tv)


def objective(K, x, y, config: ReconConfig, pool=None) -> ObjectiveParts:
    g = _grid_of(K, x.grid)
    _check_pair(K, y)
    alpha, beta = resolve_regularization(config, K, y, pool)
    op = device_operator(K, pool)
    if isinstance(op, DeviceOperator):
        r, _ = op.residual(x.values, y.values)
    else:
        r = op.matvec(x.values) - op.tensor(y.values)
    xt = op.tensor(x.values)
    return _parts_dev(r, _real(xt), (g.ny, g.nx), alpha, beta)


# ---------------------------------------------------------------------------
# the solver


_spec_graphs: dict = {}


def _speculative_loop(op, yv, alpha, beta, eta, config, shape):
    """Frequency-domain (matrix-free) operator: the loop of recon.py:318-363 with no host
    round trip per iteration.  All N iterations are enqueued (iterates and the per-iteration
    data / l1 / TV / non-finite terms kept on the device), captured once into a CUDA graph
    per (operator, N, parameters) and replayed; the stopping rules are applied afterwards to
    the recorded terms (sharded.stop_point) and the accepted iterate returned -- the
    reference's result, with iterations past a stop computed and discarded."""
    import torch

    from .sharded import stop_point

    ny, nx = shape
    N, P = config.iterations, nx * ny
    rdt = torch.float64 if op.pool.dtype == "float64" else torch.float32
    key = (id(op), N, P, float(alpha), float(beta), float(eta), float(config.tv_epsilon),
           bool(config.nonneg))
    st = _spec_graphs.get(key)
    if st is None or st["op"] is not op:
        y_s = op.tensor(np.zeros(op.rows, dtype=np.complex128))
        st = {"op": op, "y": y_s, "xs": torch.zeros(N + 1, P, dtype=rdt, device=op.device),
              "rows": torch.zeros(N, 4, dtype=torch.float64, device=op.device),
              "f0": torch.zeros((), dtype=torch.float64, device=op.device), "graph": None}
        eps2 = config.tv_epsilon ** 2

        def body():
            y, xs, rows = st["y"], st["xs"], st["rows"]
            r = -y
            r64 = r.to(torch.complex128) if r.is_complex() else r.double()
            st["f0"].copy_(torch.real(torch.vdot(r64, r64)))
            for it in range(N):
                x = xs[it]
                grad = 2.0 * _real(op.adjoint(r, 1.0)).to(rdt)
                if beta > 0:
                    img = x.reshape(ny, nx)
                    h = img[:, 1:] - img[:, :-1]
                    v = img[1:, :] - img[:-1, :]
                    wh = h / torch.sqrt(h * h + eps2)
                    wv = v / torch.sqrt(v * v + eps2)
                    t = torch.zeros_like(img)
                    t[:, :-1] -= wh
                    t[:, 1:] += wh
                    t[:-1, :] -= wv
                    t[1:, :] += wv
                    grad = grad + beta * t.reshape(-1)
                z = x - eta * grad
                xn = torch.sign(z) * torch.clamp_min(z.abs() - eta * alpha, 0.0)
                if config.nonneg:
                    xn = torch.clamp_min(xn, 0.0)
                xs[it + 1].copy_(xn)
                r = op.matvec(xn) - y
                r64 = r.to(torch.complex128) if r.is_complex() else r.double()
                xd = xn.double().reshape(ny, nx)
                rows[it, 0] = torch.real(torch.vdot(r64, r64))
                rows[it, 1] = xd.abs().sum()
                rows[it, 2] = (xd[:, 1:] - xd[:, :-1]).abs().sum() + (xd[1:, :] - xd[:-1, :]).abs().sum()
                rows[it, 3] = (~torch.isfinite(xn)).sum()

        st["body"] = body
        _spec_graphs.clear()
        _spec_graphs[key] = st
    st["y"].copy_(op.tensor(yv))
    with torch.cuda.device(op.device):
        if st["graph"] is None:
            st["body"]()  # warm-up: operator workspaces, kernels loaded
            torch.cuda.current_stream(op.device).synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                st["body"]()
            st["graph"] = g
        st["graph"].replay()
    rows = st["rows"].cpu().numpy()
    f0 = float(st["f0"].cpu())
    k, stopped_by, hist = stop_point([tuple(float(v) for v in r) for r in rows], f0, alpha, beta,
                                     config.tolerance)
    h = np.array(hist, dtype=np.float64).reshape(-1, 4)
    return st["xs"][k].double().cpu().numpy(), h, stopped_by


def _dense_loop(op, yv, alpha, beta, eta, config, shape):
    """The loop with device products and host stopping checks (kept as the reference-shaped
    path for operators without a device-resident solve)."""
    import torch

    dev = op.device
    rdt = torch.float64 if op.pool.dtype == "float64" else torch.float32
    y = op.tensor(yv)
    x = torch.zeros(op.cols, dtype=rdt, device=dev)
    r = -y.clone()
    r64 = r.to(torch.complex128) if r.is_complex() else r.double()
    f_prev = float(torch.real(torch.vdot(r64, r64)))  # fp64 like every later objective
    hist = []
    stopped_by = "max_iterations"
    grow = 0
    ny, nx = shape
    for _ in range(config.iterations):
        grad = 2.0 * _real(op.adjoint(r, 1.0)).to(rdt)
        if beta > 0:
            img = x.reshape(ny, nx)
            h = img[:, 1:] - img[:, :-1]
            v = img[1:, :] - img[:-1, :]
            wh = h / torch.sqrt(h * h + config.tv_epsilon**2)
            wv = v / torch.sqrt(v * v + config.tv_epsilon**2)
            t = torch.zeros_like(img)
            t[:, :-1] -= wh
            t[:, 1:] += wh
            t[:-1, :] -= wv
            t[1:, :] += wv
            grad = grad + beta * t.reshape(-1)
        z = x - eta * grad
        x_new = torch.sign(z) * torch.clamp_min(z.abs() - eta * alpha, 0.0)
        if config.nonneg:
            x_new = torch.clamp_min(x_new, 0.0)
        r_new = op.matvec(x_new) - y
        parts = _parts_dev(r_new, x_new, shape, alpha, beta)
        if not (math.isfinite(parts.total) and bool(torch.isfinite(x_new).all())):
            stopped_by = "divergence"
            break
        hist.append(parts)
        x, r = x_new, r_new
        grow = grow + 1 if parts.total > f_prev else 0
        if grow >= DIVERGENCE_STREAK:
            stopped_by = "divergence"
            break
        rel = abs(parts.total - f_prev) / max(abs(f_prev), 1e-300)
        f_prev = parts.total
        if config.tolerance > 0 and rel < config.tolerance:
            stopped_by = "tolerance"
            break
    h = np.array(hist, dtype=np.float64).reshape(-1, 4)
    return x.double().cpu().numpy(), h, stopped_by


_stage_split: dict = {}


def _book_stages(times: dict, wall: float, op, yv, config, alpha, beta, eta) -> None:
    """Apportion a graph solve's wall time over the reference's stage keys by the plan's
    device-time split (see iterative_reconstruct)."""
    key = (id(op), float(alpha), float(beta), float(eta), int(config.iterations))
    split = _stage_split.get(key)
    if split is None:
        bp, upd, fp, fin = op.profile_stages(yv, solver_params(config, alpha, beta, eta))
        tot = max(bp + upd + fp + fin, 1e-30)
        split = ((bp + fp) / tot, upd / tot, fin / tot)
        _stage_split[key] = split
    prod, upd, obj = split
    times["gradient_products"] += wall * prod
    times["tv_gradient" if beta > 0 else "prox"] += wall * upd
    times["objective"] += wall * obj


def iterative_reconstruct(K, y, config: ReconConfig, grid=None, pool=None,
                          stage_seconds: dict | None = None) -> ReconResult:
    """Proximal-gradient minimisation of ||Kx-y||^2 + alpha||x||_1 + beta TV(x)
    (recon.py:286-377), x0 = 0, on the device.

    stage_seconds, if given, accumulates wall time under the reference's keys
    (recon.py:303-347).  The solve is one captured graph, so its wall time is apportioned by
    the plan's per-kernel device times (pk_profile_stages, one un-graphed replay per plan and
    parameter set, cached): "gradient_products" <- back-projection + projection, "tv_gradient"
    <- the update kernel (TV gradient fused with the soft threshold and non-negativity; with
    beta = 0 it is booked under "prox"), "objective" <- the residual/objective kernel.  Other
    operators (explicit, frequency-domain) book the whole solve under "gradient_products".
    """
    g = _grid_of(K, grid)
    _check_pair(K, y)
    pool = _as_pool(pool)
    alpha, beta = resolve_regularization(config, K, y, pool)
    eta = _resolve_step(config, K, beta, pool)
    times = stage_seconds if stage_seconds is not None else {}
    for key in ("gradient_products", "tv_gradient", "prox", "objective"):
        times.setdefault(key, 0.0)
    op = device_operator(K, pool)
    t0 = time.perf_counter()
    if isinstance(op, DeviceOperator):
        params = solver_params(config, alpha, beta, eta)
        x, hist, status = op.reconstruct(y.values, params)
        status = status.cpu().numpy()[0]
        n = int(status[0])
        h = hist.cpu().numpy()[0][:, :n].T
        stopped_by = N.STOPPED_BY[int(status[1])]
        xv = x[0].double().cpu().numpy()
    elif isinstance(op, DenseOperator):  # explicit K: the device loop of pk_dense_reconstruct
        x, hist, status = op.reconstruct(y.values, solver_params(config, alpha, beta, eta), g.nx, g.ny)
        status = status.cpu().numpy()
        n = int(status[0])
        h = hist.cpu().numpy()[:, :n].T
        stopped_by = N.STOPPED_BY[int(status[1])]
        xv = x.double().cpu().numpy()
    else:  # frequency-domain operator: speculative device loop, one graph replay
        xv, h, stopped_by = _speculative_loop(op, y.values, alpha, beta, eta, config, (g.ny, g.nx))
        n = h.shape[0]
    wall = time.perf_counter() - t0
    if stage_seconds is not None and isinstance(op, DeviceOperator):
        _book_stages(times, wall, op, y.values, config, alpha, beta, eta)
    else:
        times["gradient_products"] += wall
    return ReconResult(
        image=ImageField(g, xv),
        objective_history=h[:, 0].copy(),
        data_term_history=h[:, 1].copy(),
        l1_history=h[:, 2].copy(),
        tv_history=h[:, 3].copy(),
        iterations_run=n,
        stopped_by=stopped_by,
        alpha_used=alpha,
        beta_used=beta,
        step_used=eta,
    )


# ---------------------------------------------------------------------------
# metrics (recon.py:380-394)


def rmse(a: ImageField, b: ImageField) -> float:
    if a.grid != b.grid:
        raise ValueError("fields live on different grids")
    return float(np.sqrt(np.mean((a.values - b.values) ** 2)))


def psnr(a: ImageField, b: ImageField, peak: float) -> float:
    if a.grid != b.grid:
        raise ValueError("fields live on different grids")
    mse = float(np.mean((a.values - b.values) ** 2))
    if mse == 0:
        return math.inf
    return 10.0 * math.log10(peak * peak / mse)


# ---------------------------------------------------------------------------
# dynamic sequences: many frames on one geometry (BASELINE config 4)


def reconstruct_frames(K, ys, config: ReconConfig, pool=None, batch: int = 4,
                       pinned: tuple[float, float, float] | None = None) -> list[ReconResult]:
    """iterative_reconstruct for a sequence of frames sharing one geometry.

    Frames are solved ``batch`` at a time (1, 2 or 4) by plans that evaluate each
    sensor-pixel delay once for the whole batch.  Each frame's result equals its
    single-frame solve (per-frame alpha/beta/step, stopping rules and histories).
    ``pinned`` = (alpha, beta, step) applies one calibration to every frame (config 4's
    protocol: pinned once from frame 0); otherwise every frame is calibrated like
    iterative_reconstruct does.
    """
    from .device import operator_for

    pool = _as_pool(pool)
    if batch not in (1, 2, 4):
        raise ValueError(f"batch must be 1, 2 or 4, got {batch}")
    if pool.dtype != "float32" and batch != 1:
        raise ValueError("batched frames run in float32")
    ys = list(ys)
    if not ys:
        return []
    g = _grid_of(K, None)
    for y in ys:
        _check_pair(K, y)
    prov = getattr(K, "provenance", {}) or {}
    if geometry_path(K) != "time":  # explicit or frequency-domain K: one solve per frame
        return [iterative_reconstruct(K, y, config, pool=pool) for y in ys]
    cal = []
    for y in ys:
        if pinned is not None:
            cal.append(tuple(float(v) for v in pinned))
        else:
            a, b = resolve_regularization(config, K, y, pool)
            cal.append((a, b, _resolve_step(config, K, b, pool)))
    out: list[ReconResult] = []
    for s in range(0, len(ys), batch):
        chunk = list(range(s, min(len(ys), s + batch)))
        nb = batch if len(chunk) == batch else 1
        groups = [chunk] if nb == batch else [[c] for c in chunk]
        for grp in groups:
            op = operator_for(prov["grid"], prov["ring"], prov["acoustic"], pool, frames=len(grp))
            params = [solver_params(config, *cal[c]) for c in grp]
            yv = np.concatenate([np.asarray(ys[c].values, dtype=np.float64) for c in grp])
            x, hist, status = op.reconstruct(yv, params)
            x = x.double().cpu().numpy()
            hist = hist.cpu().numpy()
            status = status.cpu().numpy()
            for q, c in enumerate(grp):
                n = int(status[q, 0])
                h = hist[q][:, :n].T
                out.append(ReconResult(
                    image=ImageField(g, x[q]),
                    objective_history=h[:, 0].copy(), data_term_history=h[:, 1].copy(),
                    l1_history=h[:, 2].copy(), tv_history=h[:, 3].copy(),
                    iterations_run=n, stopped_by=N.STOPPED_BY[int(status[q, 1])],
                    alpha_used=cal[c][0], beta_used=cal[c][1], step_used=cal[c][2]))
    return out
