"""Acoustics, the (lazy) measurement operator, sensor data and projection.

Mirror of the reference's ``pactkit.forward`` public surface (pkg/src/pactkit/forward.py)
for the hot path.  The difference is the operator: ``build_time_matrix`` returns a
geometry-backed ``MeasurementMatrix`` whose products run matrix-free on the B200
(``DeviceOperator``); the dense (M*Q, P) array of forward.py:185-194 -- 2.2 TB at
512^2 x 512 x 2048 -- is only formed if ``.entries`` is explicitly requested.

Explicit matrices (``MeasurementMatrix(domain, entries)`` without provenance, e.g. read
from a PACTMAT file) are supported through ``DenseOperator`` -- hand-written streaming
GEMV kernels and a device-resident solver loop (pk_dense_*).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np

from .device import CudaPool, operator_for, resolve_pool
from .scene import GeometryError, ImageField, check_enclosure

__all__ = [
    "AcousticConfig",
    "MeasurementMatrix",
    "SensorData",
    "TruncationWarning",
    "DenseOperator",
    "build_time_matrix",
    "build_freq_matrix",
    "FreqOperator",
    "forward_project",
    "add_noise",
    "device_operator",
    "DeviceMatrix",
    "dense_time_matrix",
]

DEFAULT_SOUND_SPEED = 1500.0  # m/s (forward.py:32)


class TruncationWarning(UserWarning):
    """Some acoustic delays fall outside the acquisition window (forward.py:35-36)."""


@dataclass(frozen=True)
class AcousticConfig:
    """Sound speed c, sample spacing dt, q_s time samples, q_n wavenumbers (forward.py:39-67)."""

    c: float = DEFAULT_SOUND_SPEED
    dt: float = 1e-7
    q_s: int = 64
    q_n: int = 64

    def __post_init__(self):
        if not (self.c > 0 and self.dt > 0):
            raise ValueError(f"c and dt must be > 0, got c={self.c}, dt={self.dt}")
        if self.q_s < 1 or self.q_n < 1:
            raise ValueError(f"sample counts must be >= 1, got q_s={self.q_s}, q_n={self.q_n}")

    @property
    def k_values(self) -> np.ndarray:
        n = np.arange(1, self.q_n + 1, dtype=np.float64)
        return 2.0 * np.pi * n / (self.q_s * self.dt) / self.c

    @property
    def window(self) -> float:
        return self.q_s * self.dt


@dataclass(frozen=True)
class SensorData:
    """Stacked per-sensor traces; sensor m owns [m*samples, (m+1)*samples) (forward.py:124-150)."""

    domain: str
    sensors: int
    samples: int
    values: np.ndarray

    def __post_init__(self):
        if self.domain not in ("time", "frequency"):
            raise ValueError(f"unknown domain {self.domain!r}")
        want = np.complex128 if self.domain == "frequency" else np.float64
        v = np.ascontiguousarray(np.asarray(self.values).ravel(), dtype=want)
        if v.size != self.sensors * self.samples:
            raise ValueError(
                f"signal length {v.size} != sensors*samples = {self.sensors * self.samples}"
            )
        if not np.all(np.isfinite(v.view(np.float64))):
            raise ValueError("sensor data must be finite")
        v.setflags(write=False)
        object.__setattr__(self, "values", v)

    @property
    def length(self) -> int:
        return self.values.size


@dataclass(frozen=True, eq=False, init=False)
class MeasurementMatrix:
    """The discretised operator K.

    Geometry-backed (``provenance`` holds grid / ring / acoustic, as build_time_matrix
    records them, forward.py:207-215): products run matrix-free on the device and
    ``entries`` is materialised only on request.  Explicit (``entries`` given): the dense
    array is the operator.

    The constructor is the reference's, ``MeasurementMatrix(domain, entries, provenance)``
    (forward.py:70-91), positionally or by keyword (``entries=``); ``entries=None`` with
    grid/ring/acoustic provenance is the lazy form.  The dense array is held in the field
    ``entries_`` (the ``entries`` property materialises it), so ``dataclasses.replace(K,
    entries=...)`` works too.
    """

    domain: str
    entries_: np.ndarray | None = None
    provenance: dict = field(default_factory=dict)

    def __init__(self, domain, entries=None, provenance=None, *, entries_=None):
        object.__setattr__(self, "domain", domain)
        object.__setattr__(self, "entries_", entries if entries is not None else entries_)
        object.__setattr__(self, "provenance", {} if provenance is None else provenance)
        self.__post_init__()

    def __post_init__(self):
        if self.domain not in ("time", "frequency"):
            raise ValueError(f"unknown domain {self.domain!r}")
        if self.entries_ is not None:
            want = np.complex128 if self.domain == "frequency" else np.float64
            e = np.ascontiguousarray(np.asarray(self.entries_), dtype=want)
            if e.ndim != 2:
                raise ValueError("matrix entries must be 2-D")
            e.setflags(write=False)
            object.__setattr__(self, "entries_", e)
        elif not self.geometry_backed:
            raise ValueError("a MeasurementMatrix needs entries or grid/ring/acoustic provenance")

    @property
    def geometry_backed(self) -> bool:
        p = self.provenance
        return self.entries_ is None and all(p.get(k) is not None for k in ("grid", "ring", "acoustic"))

    @property
    def grid(self):
        return self.provenance.get("grid")

    @property
    def ring(self):
        return self.provenance.get("ring")

    @property
    def acoustic(self):
        return self.provenance.get("acoustic")

    @property
    def rows(self) -> int:
        if self.entries_ is not None:
            return self.entries_.shape[0]
        q = self.acoustic.q_s if self.domain == "time" else self.acoustic.q_n
        return self.ring.count * q

    @property
    def cols(self) -> int:
        if self.entries_ is not None:
            return self.entries_.shape[1]
        return self.grid.size

    def layout(self) -> tuple[int, int]:
        """(sensor count, samples per sensor); needs builder provenance (forward.py:114-121)."""
        ring, ac = self.ring, self.acoustic
        if ring is None or ac is None:
            raise ValueError("matrix has no builder provenance; pass the layout explicitly")
        return ring.count, (ac.q_s if self.domain == "time" else ac.q_n)

    @property
    def entries(self) -> np.ndarray:
        """Dense K.  Geometry-backed matrices materialise it from the device's fp64 index
        dump (pk_index_dump, the same s0/frac the reference computes) -- small scenes only."""
        if self.entries_ is not None:
            return self.entries_
        cached = self.__dict__.get("_materialised")
        if cached is not None:  # kept apart from entries_: K stays geometry-backed
            return cached
        if self.domain == "frequency":
            return self._freq_entries()
        M, Q = self.ring.count, self.acoustic.q_s
        P = self.grid.size
        if M * Q * P > 64 * 1024 * 1024:
            raise MemoryError(f"refusing to materialise a {M * Q} x {P} dense matrix")
        op = operator_for(self.grid, self.ring, self.acoustic, CudaPool(dtype="float64"))
        s0, fr = op.index_dump()
        s0 = s0.cpu().numpy()
        fr = fr.cpu().numpy()
        w = 1.0 / (2.0 * np.pi * self.acoustic.c)
        K = np.zeros((M * Q, P))
        cols = np.broadcast_to(np.arange(P), s0.shape)
        m_idx = np.arange(M)[:, None]
        lo_ok = (s0 >= 1) & (s0 <= Q)
        hi_ok = (s0 >= 0) & (s0 <= Q - 1)
        K[(m_idx * Q + s0 - 1)[lo_ok], cols[lo_ok]] = (1.0 - fr[lo_ok]) * w
        K[(m_idx * Q + s0)[hi_ok], cols[hi_ok]] = fr[hi_ok] * w
        K.setflags(write=False)
        object.__setattr__(self, "_materialised", K)
        return K


    def _freq_entries(self) -> np.ndarray:
        """Dense i c k_n exp(-i k_n d) / d (forward.py:218-234) on the host -- small scenes
        only; the device products never form it."""
        M, Qn, P = self.ring.count, self.acoustic.q_n, self.grid.size
        if M * Qn * P > 16 * 1024 * 1024:
            raise MemoryError(f"refusing to materialise a {M * Qn} x {P} dense complex matrix")
        pix = self.grid.pixel_coords()
        pos = np.asarray(self.ring.positions)
        d = np.hypot(pix[None, :, 0] - pos[:, 0:1], pix[None, :, 1] - pos[:, 1:2])
        k = self.acoustic.k_values
        K = np.empty((M * Qn, P), dtype=np.complex128)
        for m in range(M):
            blk = (1j * self.acoustic.c * k)[:, None] * np.exp(-1j * k[:, None] * d[m][None, :])
            blk /= d[m][None, :]
            K[m * Qn:(m + 1) * Qn] = blk
        K.setflags(write=False)
        object.__setattr__(self, "_materialised", K)
        return K


# ---------------------------------------------------------------------------
# operators


class FreqOperator:
    """Frequency-domain operator (forward.py:218-234) run matrix-free on the device
    (pk_freq_matvec / pk_freq_adjoint): no (M*q_n, P) complex matrix is formed."""

    def __init__(self, grid, ring, acoustic, pool: CudaPool):
        self.dev_op = operator_for(grid, ring, acoustic, pool)
        self.q_n = int(acoustic.q_n)
        self.pool = pool
        self.device = self.dev_op.device
        self.tdtype = self.dev_op.cdtype
        self.rows, self.cols = ring.count * self.q_n, grid.size

    def tensor(self, a):
        import torch

        if isinstance(a, torch.Tensor):
            return a.to(device=self.device, dtype=self.tdtype)
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(self.device, self.tdtype)

    def matvec(self, x):
        """K_f x; a complex x is applied as K_f Re(x) + i K_f Im(x)."""
        import torch

        if isinstance(x, torch.Tensor) and x.is_complex() or (not isinstance(x, torch.Tensor) and np.iscomplexobj(x)):
            xt = self.tensor(x)
            re = self.dev_op.freq_matvec(xt.real.contiguous(), self.q_n)
            im = self.dev_op.freq_matvec(xt.imag.contiguous(), self.q_n)
            return re + 1j * im
        return self.dev_op.freq_matvec(x, self.q_n)

    def adjoint(self, y, scale: float = 1.0):
        return self.dev_op.freq_adjoint(y, self.q_n, scale)


class DenseOperator:
    """Explicit matrix on the device: the C ABI's pk_dense_* -- K held in
    HBM in the pool's dtype, hand-written streaming GEMV / GEMV^H kernels, and the whole
    solver loop on the device (``reconstruct``; one pass over K per iteration for real fp32
    K).  Replaces the reference's numba GEMV cores for a K given by its entries
    (kernels.py:195-225, read_matrix forward.py:303-312)."""

    def __init__(self, entries: np.ndarray | None, pool: CudaPool, shape=None, cplx: bool = False):
        import ctypes

        import torch

        from . import _native as N
        from .device import _require_cuda

        _require_cuda(pool.device)
        self._N, self._lib = N, N.load()
        self.pool = pool
        self.device = torch.device("cuda", pool.device)
        self.cplx = bool(np.iscomplexobj(entries)) if entries is not None else bool(cplx)
        if pool.dtype == "float32":
            self.rdtype = torch.float32
            self.tdtype = torch.complex64 if self.cplx else torch.float32
        else:
            self.rdtype = torch.float64
            self.tdtype = torch.complex128 if self.cplx else torch.float64
        self.rows, self.cols = entries.shape if entries is not None else shape
        h = ctypes.c_void_p()
        N.check(self._lib.pk_dense_create(self.rows, self.cols, pool.pk_dtype, int(self.cplx),
                                          pool.device, ctypes.byref(h)))
        self._h = h
        if entries is not None:
            e = np.ascontiguousarray(entries, dtype=np.complex128 if self.cplx else np.float64)
            with torch.cuda.device(self.device):
                N.check(self._lib.pk_dense_set_entries(self._h, e.ctypes.data, 0, self._stream()))
                torch.cuda.current_stream(self.device).synchronize()
        info = N.DenseInfo()
        N.check(self._lib.pk_dense_get_info(self._h, ctypes.byref(info)))
        self.info = info

    @classmethod
    def from_geometry(cls, grid, ring, acoustic, pool: CudaPool) -> "DenseOperator":
        """The time-domain K of build_time_matrix (forward.py:167-194) formed on the device
        (pk_dense_from_plan): fp64 entries bit-identical to the reference's dense K, without a
        host copy (config 1's K is 17.2 GB)."""
        import torch

        op = cls(None, pool, shape=(ring.count * acoustic.q_s, grid.size))
        plan = operator_for(grid, ring, acoustic, CudaPool(pool.device, "float64"))
        with torch.cuda.device(op.device):
            op._N.check(op._lib.pk_dense_from_plan(op._h, plan.handle, op._stream()))
            torch.cuda.current_stream(op.device).synchronize()
        return op

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.pk_dense_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def _stream(self):
        import ctypes

        import torch

        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def tensor(self, a):
        import torch

        if isinstance(a, torch.Tensor):
            return a.to(device=self.device, dtype=self.tdtype).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a)).to(self.device, self.tdtype)

    def _vec(self, a, n: int, what: str):
        """Device vector in the plan's real or complex dtype (complex only if a is complex)."""
        import torch

        if isinstance(a, torch.Tensor):
            t = a
        else:
            with warnings.catch_warnings():  # read-only reference containers: only copied
                warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
                t = torch.from_numpy(np.ascontiguousarray(a))
        c = t.is_complex()
        t = t.to(device=self.device, dtype=(torch.complex64 if self.rdtype == torch.float32
                                            else torch.complex128) if c else self.rdtype).contiguous()
        if t.numel() != n:
            raise ValueError(f"matrix has {n} {what} but vector has {t.numel()} values")
        return t, c

    def _frames(self, a, n: int, what: str):
        """[frames, n] real fp32 device matrix of a frame batch (tensor-core products)."""
        import torch

        if self.cplx or self.rdtype != torch.float32:
            raise ValueError("frame-batched products need a real float32 matrix")
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        if t.is_complex():
            raise ValueError("frame-batched products take real frames")
        t = t.to(device=self.device, dtype=torch.float32).reshape(-1, n).contiguous() if t.numel() % n == 0 else None
        if t is None or not 1 <= t.shape[0] <= 128:
            raise ValueError(f"expected 1..128 frames of {n} {what}")
        return t

    def matmat(self, xs):
        """K x for a batch of frames, xs [frames, cols] -> [frames, rows] (pk_dense_matmat:
        tcgen05 tensor cores, 3xTF32, fp32 accuracy)."""
        import torch

        xt = self._frames(xs, self.cols, "columns")
        out = torch.empty((xt.shape[0], self.rows), device=self.device, dtype=torch.float32)
        with torch.cuda.device(self.device):
            self._N.check(self._lib.pk_dense_matmat(self._h, xt.shape[0], xt.data_ptr(), out.data_ptr(),
                                                    self._stream()))
        return out

    def rmatmat(self, ys):
        """K^T y for a batch of frames, ys [frames, rows] -> [frames, cols] (pk_dense_rmatmat)."""
        import torch

        yt = self._frames(ys, self.rows, "rows")
        out = torch.empty((yt.shape[0], self.cols), device=self.device, dtype=torch.float32)
        with torch.cuda.device(self.device):
            self._N.check(self._lib.pk_dense_rmatmat(self._h, yt.shape[0], yt.data_ptr(), out.data_ptr(),
                                                     self._stream()))
        return out

    def matvec(self, x):
        import torch

        xt, xc = self._vec(x, self.cols, "columns")
        cd = torch.complex64 if self.rdtype == torch.float32 else torch.complex128
        out = torch.empty(self.rows, device=self.device, dtype=cd if (self.cplx or xc) else self.rdtype)
        with torch.cuda.device(self.device):
            self._N.check(self._lib.pk_dense_matvec(self._h, xt.data_ptr(), int(xc), out.data_ptr(),
                                                    self._stream()))
        return out

    def adjoint(self, y, scale: float = 1.0):
        import torch

        yt, yc = self._vec(y, self.rows, "rows")
        oc = self.cplx or yc
        cd = torch.complex64 if self.rdtype == torch.float32 else torch.complex128
        out = torch.empty(self.cols, device=self.device, dtype=cd if oc else self.rdtype)
        with torch.cuda.device(self.device):
            self._N.check(self._lib.pk_dense_adjoint(self._h, yt.data_ptr(), int(yc), out.data_ptr(),
                                                     float(scale), self._stream()))
        return out

    def reconstruct(self, y, params, nx: int, ny: int):
        """Device-resident solve (pk_dense_reconstruct): (x [P], history [4, N], status [2])."""
        import ctypes

        import torch

        yt, yc = self._vec(y, self.rows, "rows")
        if yc != self.cplx:
            raise ValueError("signal and matrix must both be real or both complex")
        n = int(params.iterations)
        x = torch.empty(self.cols, device=self.device, dtype=self.rdtype)
        hist = torch.zeros(4 * n, device=self.device, dtype=torch.float64)
        status = torch.zeros(2, device=self.device, dtype=torch.int32)
        with torch.cuda.device(self.device):
            self._N.check(self._lib.pk_dense_reconstruct(
                self._h, int(nx), int(ny), ctypes.byref(params), yt.data_ptr(), x.data_ptr(),
                hist.data_ptr(), status.data_ptr(), self._stream()))
        return x, hist.view(4, n), status


class DeviceMatrix:
    """An explicit K resident on the device (its entries are never on the host): the
    MeasurementMatrix surface the public API reads (domain, rows, cols, grid, layout) over a
    DenseOperator.  ``dense_time_matrix`` makes one from a geometry."""

    def __init__(self, op: DenseOperator, domain: str, grid=None, layout=None):
        self.dense_operator = op
        self.domain = domain
        self.rows, self.cols = op.rows, op.cols
        self.provenance = {"grid": grid} if grid is not None else {}
        self._layout = layout

    @property
    def grid(self):
        return self.provenance.get("grid")

    def layout(self) -> tuple[int, int]:
        if self._layout is None:
            raise ValueError("matrix has no builder provenance; pass the layout explicitly")
        return self._layout


def dense_time_matrix(grid, ring, acoustic, pool: CudaPool) -> DeviceMatrix:
    """build_time_matrix's explicit dense K (forward.py:167-215), formed on the device in the
    pool's dtype; its products and solves run the explicit-matrix kernels (pk_dense_*)."""
    check_enclosure(grid, ring)
    op = DenseOperator.from_geometry(grid, ring, acoustic, pool)
    return DeviceMatrix(op, "time", grid, (ring.count, acoustic.q_s))


_dense_cache: dict = {}
_freq_cache: dict = {}


def _as_pool(pool) -> CudaPool:
    """The device policy for a ``pool`` argument (see ``device.resolve_pool``)."""
    return resolve_pool(pool)


def geometry_path(K) -> str | None:
    """'time' / 'frequency' when K's products run matrix-free from its grid/ring/acoustic
    provenance (no explicit entries), else None (an explicit matrix: dense products)."""
    if isinstance(K, np.ndarray):
        return None
    prov = getattr(K, "provenance", {}) or {}
    has_geo = all(prov.get(k) is not None for k in ("grid", "ring", "acoustic"))
    explicit = getattr(K, "entries_", None) if isinstance(K, MeasurementMatrix) else None
    if has_geo and explicit is None and K.domain in ("time", "frequency"):
        return K.domain
    return None


def device_operator(K, pool=None):
    """DeviceOperator (geometry-backed) or DenseOperator (explicit) for K.

    Accepts this package's MeasurementMatrix and the reference's own
    ``pactkit.forward.MeasurementMatrix`` (duck-typed on .provenance / .entries).
    """
    pool = _as_pool(pool)
    dense = getattr(K, "dense_operator", None)
    if dense is not None:  # device-resident explicit K (DeviceMatrix)
        return dense
    prov = getattr(K, "provenance", {}) or {}
    if geometry_path(K) == "time":
        return operator_for(prov["grid"], prov["ring"], prov["acoustic"], pool)
    if geometry_path(K) == "frequency":
        fk = (id(operator_for(prov["grid"], prov["ring"], prov["acoustic"], pool)), int(prov["acoustic"].q_n))
        fo = _freq_cache.get(fk)
        if fo is None or fo.dev_op is not operator_for(prov["grid"], prov["ring"], prov["acoustic"], pool):
            fo = FreqOperator(prov["grid"], prov["ring"], prov["acoustic"], pool)
            _freq_cache[fk] = fo
        return fo
    entries = K.entries if not isinstance(K, np.ndarray) else K
    key = (id(entries), pool)
    op = _dense_cache.get(key)
    if op is None or op[0] is not entries:
        op = (entries, DenseOperator(entries, pool))
        _dense_cache.clear()
        _dense_cache[key] = op
    return op[1]


# ---------------------------------------------------------------------------
# building the operator


def _pair_bounds(grid, ring, acoustic):
    """Per-sensor min/max delay in samples over the grid rectangle (host, O(M))."""
    xs, ys = grid.axis_vectors() if hasattr(grid, "axis_vectors") else (
        grid.origin[0] + np.arange(grid.nx) * grid.dx, grid.origin[1] + np.arange(grid.ny) * grid.dx)
    pos = np.asarray(ring.positions)
    cx = np.clip(pos[:, 0], xs[0], xs[-1])
    cy = np.clip(pos[:, 1], ys[0], ys[-1])
    dmin = np.hypot(cx - pos[:, 0], cy - pos[:, 1])
    fx = np.maximum(np.abs(xs[0] - pos[:, 0]), np.abs(xs[-1] - pos[:, 0]))
    fy = np.maximum(np.abs(ys[0] - pos[:, 1]), np.abs(ys[-1] - pos[:, 1]))
    cdt = acoustic.c * acoustic.dt
    return dmin / cdt, np.hypot(fx, fy) / cdt


def _count_truncated(grid, ring, acoustic) -> int:
    """Exact truncated-pair count of forward.py:196-198.  Only evaluated when the O(M)
    bounds say truncation is possible; uses the reference's own arithmetic (np.hypot)."""
    lo, hi = _pair_bounds(grid, ring, acoustic)
    q = acoustic.q_s
    if lo.min() >= 1.0 + 1e-9 and hi.max() < q - 1 - 1e-9:
        return 0
    pix = grid.pixel_coords()
    cdt = acoustic.c * acoustic.dt
    total = 0
    for m0 in range(0, ring.count, 64):
        pos = ring.positions[m0 : m0 + 64]
        d = np.hypot(pix[None, :, 0] - pos[:, 0:1], pix[None, :, 1] - pos[:, 1:2])
        u = d / cdt
        s0 = np.floor(u).astype(np.int64)
        frac = u - s0
        in0 = (s0 >= 1) & (s0 <= q)
        in1 = (s0 + 1 >= 1) & (s0 + 1 <= q)
        total += int(np.count_nonzero(~in0 | (~in1 & (frac > 0.0))))
    return total


def build_time_matrix(grid, ring, acoustic) -> MeasurementMatrix:
    """Time-domain operator of forward.py:167-215, without forming the dense matrix.

    Same validation (ring must enclose the grid, no sensor on a pixel centre) and the same
    TruncationWarning / ``truncated_pairs`` provenance.
    """
    check_enclosure(grid, ring)
    xs = grid.origin[0] + np.arange(grid.nx) * grid.dx
    ys = grid.origin[1] + np.arange(grid.ny) * grid.dx
    pos = np.asarray(ring.positions)
    hit = np.isin(pos[:, 0], xs) & np.isin(pos[:, 1], ys)
    if hit.any():
        m = int(np.flatnonzero(hit)[0])
        i = int(np.flatnonzero(xs == pos[m, 0])[0])
        j = int(np.flatnonzero(ys == pos[m, 1])[0])
        raise GeometryError(f"sensor {m} coincides with pixel index {j * grid.nx + i}")
    truncated = _count_truncated(grid, ring, acoustic)
    if truncated:
        warnings.warn(
            f"{truncated} pixel-sensor delays fall (partly) outside the "
            f"{acoustic.window:g} s acquisition window; their weights are dropped",
            TruncationWarning,
            stacklevel=2,
        )
    return MeasurementMatrix(
        "time",
        None,
        provenance={"grid": grid, "ring": ring, "acoustic": acoustic, "truncated_pairs": truncated},
    )


def build_freq_matrix(grid, ring, acoustic) -> MeasurementMatrix:
    """Frequency-domain operator of forward.py:218-234 (Eq. 7), geometry-backed: products run
    matrix-free on the device, the dense complex matrix only forms if ``.entries`` is asked
    for.  Same validation as the reference (ring encloses the grid, no sensor on a pixel)."""
    check_enclosure(grid, ring)
    xs = grid.origin[0] + np.arange(grid.nx) * grid.dx
    ys = grid.origin[1] + np.arange(grid.ny) * grid.dx
    pos = np.asarray(ring.positions)
    hit = np.isin(pos[:, 0], xs) & np.isin(pos[:, 1], ys)
    if hit.any():
        m = int(np.flatnonzero(hit)[0])
        i = int(np.flatnonzero(xs == pos[m, 0])[0])
        j = int(np.flatnonzero(ys == pos[m, 1])[0])
        raise GeometryError(f"sensor {m} coincides with pixel index {j * grid.nx + i}")
    return MeasurementMatrix("frequency", None, provenance={"grid": grid, "ring": ring, "acoustic": acoustic})


def _grid_values(x):
    return np.asarray(getattr(x, "values", x))


def forward_project(K, x, pool=None) -> SensorData:
    """y = K vec(x) on the device (forward.py:253-261)."""
    grid = getattr(x, "grid", None)
    if grid is not None and K.cols != grid.size:
        raise ValueError(f"matrix has {K.cols} columns but field has {grid.size} pixels")
    sensors, samples = K.layout()
    op = device_operator(K, pool)
    y = op.matvec(_grid_values(x))
    yv = y.detach().cpu().numpy()
    if K.domain == "time":
        yv = yv.astype(np.float64)
    else:
        yv = yv.astype(np.complex128)
    return SensorData(K.domain, sensors, samples, yv)


def add_noise(y: SensorData, sigma: float, seed: int) -> SensorData:
    """Seeded i.i.d. Gaussian noise (forward.py:264-275); host-side input preparation."""
    if sigma < 0:
        raise ValueError(f"sigma must be >= 0, got {sigma}")
    if sigma == 0:
        return y
    rng = np.random.default_rng(seed)
    if y.domain == "frequency":
        noise = rng.normal(0.0, sigma, y.length) + 1j * rng.normal(0.0, sigma, y.length)
    else:
        noise = rng.normal(0.0, sigma, y.length)
    return SensorData(y.domain, y.sensors, y.samples, y.values + noise)


def make_image(grid, values) -> ImageField:
    return ImageField(grid, values)
