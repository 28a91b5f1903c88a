"""Device policy and the geometry-backed operator (one ``pk_plan`` per geometry).

``CudaPool`` takes the place of the reference's ``kernels.WorkerPool`` in the ``pool``
slot of every public function (pkg/src/pactkit/kernels.py:55-73): it names the CUDA
device and the arithmetic type (``resolve_pool`` maps None / WorkerPool to fp64).  ``DeviceOperator`` wraps the C ABI plan built from the
provenance a reference ``MeasurementMatrix`` carries (grid / ring / acoustic,
forward.py:70-121) -- the dense matrix is never formed.

Host buffers cross the boundary as torch tensors (device memory, streams); torch is
plumbing here, the arithmetic is in libpactgpu.so.
"""

from __future__ import annotations

import ctypes
import warnings
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N

__all__ = ["CudaPool", "DeviceOperator", "operator_for", "clear_plan_cache", "default_pool",
           "resolve_pool", "set_default_pool"]


@dataclass(frozen=True)
class CudaPool:
    """Execution policy for the device path.

    dtype "float32" is the production mode (fp32 storage and arithmetic, fp64 reductions);
    "float64" is the validation mode (fp64 delays evaluated exactly like the reference).
    """

    device: int = 0
    dtype: str = "float32"

    def __post_init__(self):
        if self.dtype not in ("float32", "float64"):
            raise ValueError(f"dtype must be 'float32' or 'float64', got {self.dtype!r}")
        if self.device < 0:
            raise ValueError(f"device must be >= 0, got {self.device}")

    @property
    def pk_dtype(self) -> int:
        return N.PK_F32 if self.dtype == "float32" else N.PK_F64


_default_pool: CudaPool | None = None


def set_default_pool(pool: CudaPool | None) -> None:
    """Policy used where a public call passes ``pool=None`` (None restores the built-in
    default, ``CudaPool(0, "float64")``)."""
    if pool is not None and not isinstance(pool, CudaPool):
        raise TypeError(f"expected a CudaPool or None, got {type(pool).__name__}")
    global _default_pool
    _default_pool = pool


def default_pool() -> CudaPool:
    return _default_pool if _default_pool is not None else CudaPool(0, "float64")


def resolve_pool(pool) -> CudaPool:
    """The device policy for the ``pool`` argument of the public API.

    * ``CudaPool(device, dtype)``: used as given -- ``dtype="float32"`` is the production
      mode, the only way to select fp32 arithmetic;
    * ``None`` (the reference's serial fp64 kernels, kernels.py:304-350): ``default_pool()``,
      the fp64 validation mode on cuda:0 unless ``set_default_pool`` chose otherwise;
    * a reference ``kernels.WorkerPool`` (parallel fp64 CPU kernels, kernels.py:55-73):
      ``CudaPool(0, "float64")`` -- the same fp64 numerics (<= 1e-12 of the reference), on
      the device; its worker count has no device meaning and is ignored.
    Anything else raises TypeError.  There is no CPU path.
    """
    if isinstance(pool, CudaPool):
        return pool
    if pool is None:
        return default_pool()
    if type(pool).__name__ == "WorkerPool" and hasattr(pool, "worker_count"):
        return CudaPool(0, "float64")
    raise TypeError(f"pool must be a CudaPool, a reference WorkerPool or None, got {type(pool).__name__}")


def _torch():
    import torch

    return torch


def _require_cuda(device: int):
    torch = _torch()
    if not torch.cuda.is_available():
        raise N.NativeUnavailable("no CUDA device visible: the device path has no CPU fallback")
    if device >= torch.cuda.device_count():
        raise ValueError(f"CUDA device {device} not present")


class DeviceOperator:
    """K restricted to sensors [sensor_begin, sensor_end) of a ring, on one device."""

    def __init__(self, grid, ring, acoustic, pool: CudaPool, sensor_begin=0, sensor_end=None,
                 frames: int = 1, concurrency: int = 1, sensor_list=None):
        _require_cuda(pool.device)
        lib = N.load()
        self.grid, self.ring, self.acoustic, self.pool = grid, ring, acoustic, pool
        self.frames = int(frames)
        M = int(ring.count)
        self.sensor_list = None if sensor_list is None else [int(v) for v in sensor_list]
        self.sensor_begin = int(sensor_begin) if self.sensor_list is None else 0
        self.sensor_end = (M if sensor_end is None else int(sensor_end)) if self.sensor_list is None \
            else len(self.sensor_list)
        xx = np.ascontiguousarray(grid.origin[0] + np.arange(grid.nx) * grid.dx, dtype=np.float64)
        yy = np.ascontiguousarray(grid.origin[1] + np.arange(grid.ny) * grid.dx, dtype=np.float64)
        pos = np.ascontiguousarray(ring.positions, dtype=np.float64)
        self._keep = (xx, yy, pos)
        dp = ctypes.POINTER(ctypes.c_double)
        desc = N.GeometryDesc(
            nx=grid.nx, ny=grid.ny,
            pixel_x=xx.ctypes.data_as(dp), pixel_y=yy.ctypes.data_as(dp),
            sensors=M, sensor_xy=pos.ctypes.data_as(dp),
            sensor_begin=self.sensor_begin, sensor_end=self.sensor_end,
            samples=int(acoustic.q_s), c=float(acoustic.c), dt=float(acoustic.dt),
            dtype=pool.pk_dtype, device=pool.device, frames=self.frames,
            concurrency=int(concurrency),
        )
        if self.sensor_list is not None:
            lst = np.ascontiguousarray(self.sensor_list, dtype=np.int32)
            self._keep = self._keep + (lst,)
            desc.sensor_list = lst.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            desc.sensor_list_len = int(lst.size)
        handle = ctypes.c_void_p()
        N.check(lib.pk_plan_create(ctypes.byref(desc), ctypes.byref(handle)))
        self._h = handle
        self._lib = lib
        info = N.PlanInfo()
        N.check(lib.pk_plan_get_info(self._h, ctypes.byref(info)))
        self.info = info
        torch = _torch()
        self.device = torch.device("cuda", pool.device)
        self.tdtype = torch.float32 if pool.dtype == "float32" else torch.float64
        self._pin, self._pin_evt, self._stage_lock = None, None, threading.Lock()

    # -- bookkeeping --------------------------------------------------------------
    @property
    def handle(self):
        return self._h

    @property
    def sensors(self) -> int:
        return self.sensor_end - self.sensor_begin

    @property
    def sensor_ids(self) -> list[int]:
        """Ring indices of this operator's traces, in trace order."""
        if self.sensor_list is not None:
            return list(self.sensor_list)
        return list(range(self.sensor_begin, self.sensor_end))

    @property
    def samples(self) -> int:
        return int(self.acoustic.q_s)

    @property
    def pixels(self) -> int:
        return self.grid.size

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.pk_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def stream(self):
        torch = _torch()
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def tensor(self, a) -> "object":
        """Upload a host array (or move a tensor) to this operator's device and dtype."""
        torch = _torch()
        if isinstance(a, torch.Tensor):
            return a.to(device=self.device, dtype=self.tdtype).contiguous()
        h = np.asarray(a)
        if h.dtype == np.float64 and h.size * 8 >= self._STAGE_MIN_BYTES:
            return self._upload_staged(h)
        h = np.ascontiguousarray(h, dtype=np.float64)
        with warnings.catch_warnings():
            # the reference's containers are read-only (forward.py:145); the tensor is only
            # read (copied to the device), so no host copy is made to silence torch
            warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
            t = torch.from_numpy(h)
        return t.to(device=self.device, dtype=self.tdtype).contiguous()

    _STAGE_MIN_BYTES = 1 << 20

    def _upload_staged(self, h: np.ndarray):
        """Large fp64 host arrays go through one pinned staging buffer per operator in the
        plan's dtype: a multi-threaded host copy (fp32 plans convert on the way, halving the
        DMA) into page-locked memory and an asynchronous DMA.  Pageable copies of config 3's
        8 MB traces took ~1 ms and up to 8 ms after other large host traffic.  The buffer is
        reused once the previous upload from it has completed (an event on the stream)."""
        torch = _torch()
        with self._stage_lock:
            n = h.size
            if self._pin is None or self._pin.numel() < n:
                self._pin = torch.empty(n, dtype=self.tdtype, pin_memory=True)
                self._pin_evt = None
            if self._pin_evt is not None:
                self._pin_evt.synchronize()
            buf = self._pin[:n].view(h.shape)
            with warnings.catch_warnings():
                warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
                buf.copy_(torch.from_numpy(h))
            with torch.cuda.device(self.device):
                t = buf.to(device=self.device, non_blocking=True)
                self._pin_evt = torch.cuda.Event()
                self._pin_evt.record(torch.cuda.current_stream(self.device))
            return t

    def empty(self, n: int):
        torch = _torch()
        return torch.empty(n, device=self.device, dtype=self.tdtype)

    # -- the seam: forward._matvec / forward._adjoint_matvec ----------------------
    def matvec(self, x):
        """(K x) restricted to this operator's sensors, as a device tensor."""
        xt = self.tensor(x)
        if xt.numel() != self.pixels * self.frames:
            raise ValueError(f"matrix has {self.pixels} columns but vector has {xt.numel()}")
        out = self.empty(self.sensors * self.samples * self.frames)
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_matvec(self._h, xt.data_ptr(), out.data_ptr(), self.stream()))
        return out

    def adjoint(self, y, scale: float = 1.0):
        """scale * K^T y for y on this operator's sensors, as a device tensor."""
        yt = self.tensor(y)
        if yt.numel() != self.sensors * self.samples * self.frames:
            raise ValueError(
                f"matrix has {self.sensors * self.samples} rows but signal has {yt.numel()} values"
            )
        out = self.empty(self.pixels * self.frames)
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_adjoint_matvec(self._h, yt.data_ptr(), out.data_ptr(),
                                                float(scale), self.stream()))
        return out

    def residual(self, x, y):
        """(r = K x - y, sum r^2 as a 1-element fp64 device tensor); keeps r for adjoint_residual."""
        torch = _torch()
        xt, yt = self.tensor(x), self.tensor(y)
        r = self.empty(self.sensors * self.samples * self.frames)
        ss = torch.empty(self.frames, device=self.device, dtype=torch.float64)
        with torch.cuda.device(self.device):
            N.check(self._lib.pk_residual(self._h, xt.data_ptr(), yt.data_ptr(), r.data_ptr(),
                                          ss.data_ptr(), self.stream()))
        return r, ss

    def adjoint_residual(self, scale: float = 1.0, out=None):
        out = self.empty(self.pixels * self.frames) if out is None else out
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_adjoint_residual(self._h, out.data_ptr(), float(scale),
                                                  self.stream()))
        return out

    def residual_into(self, x, y, sumsq, r=None):
        """pk_residual into caller buffers (no allocation: usable under graph capture)."""
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_residual(self._h, x.data_ptr(), y.data_ptr(),
                                          None if r is None else r.data_ptr(),
                                          sumsq.data_ptr(), self.stream()))

    def grad_update_into(self, params: "N.SolverParams", x, grad, xo, sums):
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_grad_update(self._h, ctypes.byref(params), x.data_ptr(),
                                             grad.data_ptr(), xo.data_ptr(), sums.data_ptr(),
                                             self.stream()))

    # -- peer exchange of the sensor-sharded gradient (pk_peer_*) --------------------
    def peer_handle(self) -> bytes:
        """Allocate the plan's peer-visible block; its 64-byte handle for pk_peer_connect."""
        buf = ctypes.create_string_buffer(N.PK_PEER_HANDLE_BYTES)
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_peer_handle(self._h, buf))
        return buf.raw

    def peer_connect(self, world: int, rank: int, handles) -> None:
        handles = [bytes(h) for h in handles]
        if len(handles) != world or any(len(h) != N.PK_PEER_HANDLE_BYTES for h in handles):
            raise ValueError(f"need {world} handles of {N.PK_PEER_HANDLE_BYTES} bytes")
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_peer_connect(self._h, int(world), int(rank), b"".join(handles)))

    def peer_buffer(self, slot: int) -> int:
        """Device address of this rank's gradient slot (0 or 1)."""
        ptr = ctypes.c_void_p()
        N.check(self._lib.pk_peer_buffer(self._h, int(slot), ctypes.byref(ptr)))
        return int(ptr.value)

    def adjoint_residual_to(self, scale: float, ptr: int) -> None:
        """scale * K^T r into a raw device address (a peer gradient slot)."""
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_adjoint_residual(self._h, ptr, float(scale), self.stream()))

    def peer_timed_out(self) -> bool:
        """True once a barrier of this plan gave up waiting for a peer (synchronous)."""
        v = ctypes.c_int32()
        N.check(self._lib.pk_peer_status(self._h, ctypes.byref(v)))
        return bool(v.value)

    def peer_grad_update_into(self, params: "N.SolverParams", x, slot: int, xo, sums) -> None:
        """World barrier, grad = sum of every rank's slot (rank order), then the update."""
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_peer_grad_update(self._h, ctypes.byref(params), x.data_ptr(),
                                                  int(slot), xo.data_ptr(), sums.data_ptr(),
                                                  self.stream()))

    def grad_update(self, params: "N.SolverParams", x, grad):
        """x_out = prox(x - eta*(grad + beta*tv_grad(x))) and [sum|x_out|, TV(x_out), #nonfinite]."""
        torch = _torch()
        xo = self.empty(self.pixels)
        sums = torch.zeros(4, device=self.device, dtype=torch.float64)
        with torch.cuda.device(self.device):
            N.check(self._lib.pk_grad_update(self._h, ctypes.byref(params), x.data_ptr(),
                                             grad.data_ptr(), xo.data_ptr(), sums.data_ptr(),
                                             self.stream()))
        return xo, sums

    def _check_y(self, yt):
        """The C ABI reads frames*M*Q values from a raw pointer: a short y must fail here
        (ValueError, like matvec / adjoint) instead of reading out of bounds on the device."""
        want = self.frames * self.sensors * self.samples
        if yt.numel() != want:
            raise ValueError(f"expected {want} measurement values ({self.frames} frame(s) x "
                             f"{self.sensors} sensors x {self.samples} samples), got {yt.numel()}")
        return yt

    def _params(self, params):
        """ctypes array of `frames` SolverParams (one struct is broadcast to all frames)."""
        if isinstance(params, N.SolverParams):
            params = [params] * self.frames
        if len(params) != self.frames:
            raise ValueError(f"need {self.frames} parameter sets, got {len(params)}")
        if getattr(self, "_params_t", None) is None:  # one ctypes array type per operator
            self._params_t = N.SolverParams * self.frames  # (a new type per call is cyclic garbage)
        arr = self._params_t(*params)
        return arr, int(params[0].iterations)

    def reconstruct(self, y, params):
        """Device-resident iterative_reconstruct of the plan's `frames` frames.

        y: [frames * M * Q] (frame-major).  Returns (x [frames, P], history [frames, 4, N],
        status [frames, 2]) device tensors."""
        torch = _torch()
        arr, n = self._params(params)
        yt = self._check_y(self.tensor(y))
        F = self.frames
        x = self.empty(self.pixels * F)
        hist = torch.zeros(4 * n * F, device=self.device, dtype=torch.float64)
        status = torch.zeros(2 * F, device=self.device, dtype=torch.int32)
        with torch.cuda.device(self.device):
            N.check(self._lib.pk_reconstruct(self._h, arr, yt.data_ptr(), x.data_ptr(),
                                             hist.data_ptr(), status.data_ptr(), self.stream()))
        return x.view(F, self.pixels), hist.view(F, 4, n), status.view(F, 2)

    def profile_iterations(self, y, params):
        """Un-graphed solver kernels with CUDA events around each launch (pk_profile_iterations):
        summed device seconds of K1 (back-projection with the fused TV/prox update), K2
        (projection), K3 (residual/objective), and the number of launches."""
        arr, _ = self._params(params)
        yt = self._check_y(self.tensor(y))
        ms = (ctypes.c_float * 3)()
        n = ctypes.c_int32()
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_profile_iterations(self._h, arr, yt.data_ptr(), ms, ctypes.byref(n),
                                                    self.stream()))
        return [v * 1e-3 for v in ms], int(n.value)

    def profile_stages(self, y, params):
        """Device seconds of the solver's stages over one un-graphed replay
        (pk_profile_stages): back-projection, update (TV gradient + prox), projection,
        residual/objective."""
        arr, _ = self._params(params)
        yt = self._check_y(self.tensor(y))
        ms = (ctypes.c_float * 4)()
        n = ctypes.c_int32()
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_profile_stages(self._h, arr, yt.data_ptr(), ms, ctypes.byref(n),
                                                self.stream()))
        return [v * 1e-3 for v in ms]

    def reconstruct_host(self, y_host: np.ndarray, params):
        """The C-ABI host-buffer entry (pk_reconstruct_host): fp64 in, fp64 out, synchronous."""
        arr, n = self._params(params)
        F = self.frames
        y = np.ascontiguousarray(y_host, dtype=np.float64).ravel()
        if y.size != F * self.sensors * self.samples:
            raise ValueError(f"expected {F * self.sensors * self.samples} measurement values, got {y.size}")
        x = np.empty(self.pixels * F)
        hist = np.empty(4 * n * F)
        status = np.zeros(2 * F, dtype=np.int32)
        dp = ctypes.POINTER(ctypes.c_double)
        with _torch().cuda.device(self.device):
            N.check(self._lib.pk_reconstruct_host(
                self._h, arr, y.ctypes.data_as(dp), x.ctypes.data_as(dp),
                hist.ctypes.data_as(dp), status.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                self.stream()))
        return x.reshape(F, self.pixels), hist.reshape(F, 4, n), status.reshape(F, 2)

    # -- frequency-domain operator (build_freq_matrix, forward.py:218-234) ------------
    @property
    def cdtype(self):
        torch = _torch()
        return torch.complex64 if self.tdtype == torch.float32 else torch.complex128

    def freq_matvec(self, x, q_n: int):
        """K_f x for a real image x: complex [sensors * q_n] device tensor."""
        torch = _torch()
        xt = self.tensor(x)
        if xt.numel() != self.pixels:
            raise ValueError(f"matrix has {self.pixels} columns but vector has {xt.numel()}")
        out = torch.empty(self.sensors * q_n, device=self.device, dtype=self.cdtype)
        with torch.cuda.device(self.device):
            N.check(self._lib.pk_freq_matvec(self._h, int(q_n), xt.data_ptr(), out.data_ptr(),
                                             self.stream()))
        return out

    def freq_adjoint(self, y, q_n: int, scale: float = 1.0):
        """scale * K_f^H y for complex y [sensors * q_n]: complex [P] device tensor."""
        torch = _torch()
        if isinstance(y, torch.Tensor):
            yt = y.to(device=self.device, dtype=self.cdtype).contiguous()
        else:
            yt = torch.from_numpy(np.ascontiguousarray(y, dtype=np.complex128)).to(
                device=self.device, dtype=self.cdtype).contiguous()
        if yt.numel() != self.sensors * q_n:
            raise ValueError(f"matrix has {self.sensors * q_n} rows but signal has {yt.numel()} values")
        out = torch.empty(self.pixels, device=self.device, dtype=self.cdtype)
        with torch.cuda.device(self.device):
            N.check(self._lib.pk_freq_adjoint(self._h, int(q_n), yt.data_ptr(), out.data_ptr(),
                                              float(scale), self.stream()))
        return out

    def delay_census(self, rule: int, ma: int = 0, mb: int | None = None):
        """fp32 (s0, frac) of the production kernels' delay rule (0 generic, 1 D4-symmetric
        back-projector, 2 rotation-symmetric projector) for local sensors [ma, mb), as device
        tensors [(mb-ma), P] (verification: pk_delay_census_f32)."""
        torch = _torch()
        mb = self.sensors if mb is None else mb
        n = (mb - ma) * self.pixels
        s0 = torch.empty(n, device=self.device, dtype=torch.int32)
        fr = torch.empty(n, device=self.device, dtype=torch.float32)
        with torch.cuda.device(self.device):
            N.check(self._lib.pk_delay_census_f32(self._h, int(rule), ma, mb, s0.data_ptr(),
                                                  fr.data_ptr(), self.stream()))
        return s0.view(mb - ma, self.pixels), fr.view(mb - ma, self.pixels)

    def index_dump(self, ma: int = 0, mb: int | None = None):
        """fp64 (s0, frac) for local sensors [ma, mb) as device tensors [(mb-ma), P]."""
        torch = _torch()
        mb = self.sensors if mb is None else mb
        n = (mb - ma) * self.pixels
        s0 = torch.empty(n, device=self.device, dtype=torch.int64)
        fr = torch.empty(n, device=self.device, dtype=torch.float64)
        with torch.cuda.device(self.device):
            N.check(self._lib.pk_index_dump(self._h, ma, mb, s0.data_ptr(), fr.data_ptr(),
                                            self.stream()))
        return s0.view(mb - ma, self.pixels), fr.view(mb - ma, self.pixels)


_cache: dict = {}
_cache_lock = threading.Lock()


def _key(grid, ring, acoustic, pool, m0, m1, frames=1, slot=0, concurrency=1, sensor_list=None):
    return (int(frames), int(slot), int(concurrency),
        None if sensor_list is None else tuple(int(v) for v in sensor_list),
        int(grid.nx), int(grid.ny), float(grid.dx), tuple(float(v) for v in grid.origin),
        int(ring.count), float(ring.radius), tuple(float(v) for v in ring.center),
        float(acoustic.c), float(acoustic.dt), int(acoustic.q_s),
        pool.device, pool.dtype, int(m0), int(m1),
    )


def operator_for(grid, ring, acoustic, pool: CudaPool, sensor_begin=0, sensor_end=None,
                 frames: int = 1, slot: int = 0, concurrency: int = 1, sensor_list=None):
    """Cached DeviceOperator for a geometry (plans are reused across calls and frames).

    ``slot`` selects independent plans for the same geometry (one per CUDA stream when
    frames are streamed concurrently); ``concurrency`` > 1 plans for that throughput mode
    (a smaller persistent back-projector grid; rounding-level differences)."""
    m1 = int(ring.count) if sensor_end is None else int(sensor_end)
    k = _key(grid, ring, acoustic, pool, sensor_begin, m1, frames, slot, concurrency, sensor_list)
    with _cache_lock:
        op = _cache.get(k)
        if op is None:
            op = DeviceOperator(grid, ring, acoustic, pool, sensor_begin, m1, frames, concurrency,
                                sensor_list=sensor_list)
            _cache[k] = op
        return op


def clear_plan_cache():
    with _cache_lock:
        for op in _cache.values():
            op.close()
        _cache.clear()
