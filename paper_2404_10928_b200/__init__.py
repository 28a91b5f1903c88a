"""B200-native iterative photoacoustic reconstruction (hot path of arXiv 2404.10928).

Drop-in for the reference package ``pactkit``'s reconstruction / projection API
(pkg/src/pactkit/__init__.py:10-78, hot-path subset): the same names, signatures and
result types, with every product running matrix-free in sm_100a CUDA kernels behind the
C ABI of include/pactgpu.h.  Pass ``pool=CudaPool(device, "float32")`` where the reference
takes a ``WorkerPool`` to select the fp32 production mode.  ``pool=None`` and a reference
``WorkerPool`` keep the reference's fp64 numerics (the device's fp64 validation mode,
``device.resolve_pool``); ``set_default_pool`` changes what ``None`` means.
"""

from .device import (CudaPool, DeviceOperator, clear_plan_cache, default_pool, operator_for,
                     resolve_pool, set_default_pool)
from .measurement import (
    AcousticConfig,
    DenseOperator,
    DeviceMatrix,
    MeasurementMatrix,
    SensorData,
    TruncationWarning,
    FreqOperator,
    add_noise,
    build_freq_matrix,
    build_time_matrix,
    dense_time_matrix,
    forward_project,
)
from .scene import (
    GeometryError,
    ImageField,
    ImagingGrid,
    TransducerRing,
    centered_grid,
    check_enclosure,
    field_from_image,
    make_grid,
    make_point_phantom,
    make_ring,
    make_vessel_phantom,
)
from .solver import (
    ObjectiveParts,
    ReconConfig,
    ReconResult,
    back_project,
    data_gradient,
    estimate_lipschitz,
    iterative_reconstruct,
    objective,
    psnr,
    reconstruct_frames,
    resolve_config,
    resolve_regularization,
    rmse,
    soft_threshold,
    tv_gradient,
    tv_value,
)
from .fileio import read_matrix, read_signal, write_matrix, write_signal
from .harness import BenchEntry, BenchReport, bench_recon, profile_breakdown
from .workloads import CONFIGS, make_scene

__version__ = "1.0.0"
