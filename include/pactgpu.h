/*
 * pactgpu.h -- C ABI of the B200-native iterative photoacoustic reconstruction
 * hot path (arXiv 2404.10928's `pactkit`).
 *
 * The reference has no FFI: its hot products go through the Python seam
 *   forward._matvec(K, x, pool)          pkg/src/pactkit/forward.py:237-241
 *   forward._adjoint_matvec(K, y, pool)  pkg/src/pactkit/forward.py:244-250
 * into numba GEMV cores (pkg/src/pactkit/kernels.py:185-225), driven by
 *   recon.iterative_reconstruct          pkg/src/pactkit/recon.py:286-377.
 * The entry points below are what a binding of that seam needs: an operator
 * "plan" built from the geometry the reference's MeasurementMatrix carries in
 * its provenance (grid / ring / acoustic, forward.py:70-121), the two
 * products, the device-resident solver loop, and the sensor-sharded pieces.
 *
 * Conventions
 *   - every call returns an int status: PK_OK (0) or a negative PK_ERR_*;
 *     pk_last_error() gives a thread-local message for the last failure.
 *   - no torch / C++ types: plain pointers and sizes.  `*_dev` pointers are
 *     caller-owned device buffers on the plan's device; `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).
 *   - element type of every image / trace buffer is the plan's dtype
 *     (PK_F32: float, PK_F64: double) unless stated otherwise.
 *   - no host synchronisation and no allocation inside the hot calls
 *     (pk_matvec, pk_adjoint_matvec, pk_reconstruct, pk_grad_update);
 *     all workspace is owned by the plan.  One plan may be used by one stream
 *     at a time.
 *   - image layout: row-major, index j*nx + i (geometry.py:59-68).
 *     trace layout: sensor-major, index (m - sensor_begin)*samples + s
 *     (forward.py:124-128, MeasurementMatrix rows m*Q + s, forward.py:70-76).
 */
#ifndef PACTGPU_H
#define PACTGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PK_OK 0
#define PK_ERR_INVALID -1     /* bad argument (the reference raises ValueError) */
#define PK_ERR_CUDA -2        /* CUDA runtime error */
#define PK_ERR_UNSUPPORTED -3 /* geometry/config the kernels do not handle */
#define PK_ERR_GEOMETRY -4    /* sensor coincides with a pixel (GeometryError, forward.py:161-163) */

#define PK_F32 0
#define PK_F64 1

/* stopped_by codes (ReconResult.stopped_by, recon.py:82-93) */
#define PK_STOP_MAX_ITERATIONS 0
#define PK_STOP_TOLERANCE 1
#define PK_STOP_DIVERGENCE 2

typedef struct pk_geometry_desc {
    int32_t nx, ny;          /* ImagingGrid.nx / .ny */
    const double* pixel_x;   /* host [nx]: origin[0] + i*dx  (geometry.py:61-63) */
    const double* pixel_y;   /* host [ny]: origin[1] + j*dx  (geometry.py:62-64) */
    int32_t sensors;         /* TransducerRing.count */
    const double* sensor_xy; /* host [sensors*2]: TransducerRing.positions (geometry.py:96-102) */
    int32_t sensor_begin;    /* this plan's shard of sensors [begin, end) */
    int32_t sensor_end;      /*   (whole ring: 0, sensors) */
    int32_t samples;         /* AcousticConfig.q_s */
    double c, dt;            /* AcousticConfig.c, .dt (forward.py:39-57) */
    int32_t dtype;           /* PK_F32 or PK_F64 */
    int32_t device;          /* CUDA device ordinal */
    int32_t frames;          /* frames reconstructed together on this geometry: 0/1 = one,
                                2 or 4 = batched (PK_F32 only).  Every image / trace buffer of
                                the entry points below then holds `frames` consecutive frames
                                (frame-major), and params points to `frames` structs. */
    int32_t concurrency;     /* plans the caller runs concurrently on this device (streams):
                                0/1 = latency (full persistent back-projector grid); > 1 =
                                throughput (at most half the occupancy-limited grid: fewer
                                partial slots, the other streams fill the SMs).  Each plan is deterministic; the two
                                modes sum the back-projector's partials in a different grouping
                                (fp32 rounding-level differences). */
    const int32_t* sensor_list; /* optional host [sensor_list_len]: this plan's sensors as a list
                                of ring indices (strictly increasing) instead of [begin, end);
                                traces are then stored in list order.  A list closed under the
                                ring's D4 symmetry (rotation m -> m + M/4, reflection m -> -m)
                                keeps the symmetric kernels on a sensor shard. */
    int32_t sensor_list_len;
} pk_geometry_desc;

typedef struct pk_plan pk_plan;

typedef struct pk_plan_info {
    int32_t local_sensors;   /* sensor_end - sensor_begin */
    int32_t pixels;          /* nx * ny */
    int32_t dtype;
    int32_t may_truncate;    /* 1 if some delay may leave the 1..q_s window (forward.py:196-205) */
    double c_dt;             /* c*dt as the reference forms it (forward.py:180) */
    double weight;           /* 1/(2*pi*c) (forward.py:183) */
    int32_t bp_tile, bp_window, bp_chunk, bp_buffers; /* back-projector tiling */
    int32_t fp_tile, fp_window, fp_bits;              /* projector tiling (symmetric: quadrant
                                                         tile side, window slots), fixed-point bits */
    int64_t device_bytes;    /* workspace held by the plan */
    int32_t frames;          /* frames per call */
    int32_t bp_split;        /* sensor slices per back-projector tile (symmetric: partial slots) */
    int32_t symmetric;       /* bit 0: D4-symmetric back-projector (one delay per 8 pairs);
                                bit 1: rotation-symmetric projector (one delay per 4 pairs) */
} pk_plan_info;

typedef struct pk_solver_params {
    double alpha, beta;      /* pinned ReconConfig.alpha / .beta (recon.py:46-79) */
    double step;             /* pinned eta */
    double tv_epsilon;
    double tolerance;
    int32_t iterations;
    int32_t nonneg;
} pk_solver_params;

/* Build the operator for one geometry (replaces build_time_matrix, forward.py:167-215,
 * without materialising K).  Uploads geometry, sizes tiles, allocates workspace. */
int pk_plan_create(const pk_geometry_desc* desc, pk_plan** out);
int pk_plan_destroy(pk_plan* plan);
int pk_plan_get_info(const pk_plan* plan, pk_plan_info* out);

/* out_dev[(m-begin)*Q + s] = (K x)[m*Q + s] for the plan's sensors.
 * Replaces forward._matvec (forward.py:237-241) -> kernels.matvec_parallel. */
int pk_matvec(pk_plan* plan, const void* x_dev, void* out_dev, void* stream);

/* out_dev[p] = scale * sum_{m in shard} sum_s K[m*Q+s, p] * y[(m-begin)*Q + s].
 * scale = 1 replaces forward._adjoint_matvec (forward.py:244-250); scale = 2 gives the
 * data gradient 2 K^T r of recon.py:139-143 (summed over shards by the caller). */
int pk_adjoint_matvec(pk_plan* plan, const void* y_dev, void* out_dev, double scale, void* stream);

/* The whole proximal-gradient loop of iterative_reconstruct (recon.py:318-363) on the
 * device, for a plan that owns all sensors: x0 = 0, r = -y, per iteration the fused
 * back-projection + TV + soft-threshold (+ nonneg) update, the projection + residual,
 * the objective and the stopping rules (non-finite, 5-streak, tolerance).
 *   params         [frames] structs (per-frame alpha/beta/step; iterations, tv_epsilon,
 *                  tolerance and nonneg are taken from params[0])
 *   y_dev          [frames][M*Q] measurements (plan dtype)
 *   x_out_dev      [frames][P] final images (plan dtype)
 *   history_dev    [frames][4][iterations] double: objective, data, l1, tv per accepted iteration
 *   status_dev     [frames][2] int32: iterations_run, stopped_by (PK_STOP_*)
 * Asynchronous on `stream`; captured into a CUDA graph on first use per iteration count. */
int pk_reconstruct(pk_plan* plan, const pk_solver_params* params, const void* y_dev,
                   void* x_out_dev, double* history_dev, int32_t* status_dev, void* stream);

/* Same with host buffers: y_host is double [M*Q] (SensorData.values), x_out_host double [P],
 * history_host double [4*iterations], status_host int32 [2].  Copies in, solves, copies out,
 * synchronises the stream.  Pinned host memory gives asynchronous copies. */
int pk_reconstruct_host(pk_plan* plan, const pk_solver_params* params, const double* y_host,
                        double* x_out_host, double* history_host, int32_t* status_host,
                        void* stream);

/* Asynchronous form of pk_reconstruct_host for streaming many frames: enqueues H2D, solve
 * and D2H on `stream` and returns; the host buffers must stay valid (and should be pinned)
 * until the stream has completed.  Plans are independent, so one plan per stream overlaps
 * copies and kernels of consecutive frames. */
int pk_reconstruct_host_async(pk_plan* plan, const pk_solver_params* params,
                              const double* y_host, double* x_out_host, double* history_host,
                              int32_t* status_host, void* stream);

/* Sensor-sharded building block: given the globally reduced gradient
 * grad_dev = 2 K^T r (summed over all shards), apply recon.py:330-338
 *   x_out = S_{eta*alpha}(x - eta*(grad + beta*tv_grad(x)))   (+ max(.,0) if nonneg)
 * and write sums_dev[3] (double): sum|x_out|, TV(x_out), non-finite count. */
int pk_grad_update(pk_plan* plan, const pk_solver_params* params, const void* x_dev,
                   const void* grad_dev, void* x_out_dev, double* sums_dev, void* stream);

/* Residual of the shard: r_out = K_shard x - y_shard (trace layout) and
 * sumsq_dev[0] = sum r^2 (double).  The plan keeps r for the next pk_adjoint_residual. */
int pk_residual(pk_plan* plan, const void* x_dev, const void* y_dev, void* r_out_dev,
                double* sumsq_dev, void* stream);
/* out_dev = scale * K_shard^T r for the residual kept by the last pk_residual. */
int pk_adjoint_residual(pk_plan* plan, void* out_dev, double scale, void* stream);

/* Peer-memory exchange for sensor-sharded solves: one process (or plan) per GPU
 * of one node with peer access over NVLink / NVSwitch.  Replaces the all-reduce of the
 * image-sized gradient between pk_adjoint_residual and pk_grad_update (the NCCL
 * dist.all_reduce of the gradient in sharded.SensorShardedSolver) with peer loads fused into
 * the update: every rank reads all ranks' partial gradients in rank order, so x stays bit
 * identical across ranks.
 *   pk_peer_handle   allocates the plan's peer-visible block (flags + two gradient slots)
 *                    and writes its 64-byte handle (cudaIpcMemHandle_t) to handle_out.
 *   pk_peer_connect  maps the world's blocks (handles[world][64], rank order; handles of
 *                    plans in this process are resolved without IPC).  All ranks must have
 *                    connected before any rank's first pk_peer_grad_update (a host barrier).
 *                    Plans of one process that share a device must each have run every
 *                    kernel of their solve once before any of them waits in a barrier: a
 *                    first (lazily loaded) launch waits for the device to drain.
 *   pk_peer_buffer   device pointer of this rank's gradient slot (0 or 1): the `out_dev` of
 *                    pk_adjoint_residual.
 *   pk_peer_grad_update  device barrier of the world (every rank calls it equally often;
 *                    a device-side epoch makes it graph-capturable), then
 *                    grad = sum_r slot buffer of rank r, and the update of pk_grad_update.
 *                    Alternate the slot per iteration (a rank may run one barrier ahead).
 * A barrier that waits longer than PK_PEER_TIMEOUT_S seconds (default 60; a dead rank) gives
 * up: the update writes NaN, and pk_peer_status reports timed_out = 1 (synchronous query). */
#define PK_PEER_MAX 8
#define PK_PEER_HANDLE_BYTES 64
int pk_peer_handle(pk_plan* plan, void* handle_out);
int pk_peer_connect(pk_plan* plan, int32_t world, int32_t rank, const void* handles);
int pk_peer_buffer(pk_plan* plan, int32_t slot, void** ptr_out);
int pk_peer_grad_update(pk_plan* plan, const pk_solver_params* params, const void* x_dev,
                        int32_t slot, void* x_out_dev, double* sums_dev, void* stream);
int pk_peer_status(pk_plan* plan, int32_t* timed_out);

/* Frequency-domain operator of build_freq_matrix (forward.py:218-234), matrix-free:
 *   K_f[m*q_n + (n-1), p] = i c k_n exp(-i k_n d_mp) / d_mp,  k_n = 2 pi n / (samples dt c).
 * Complex buffers are interleaved (re, im) in the plan dtype (complex64 / complex128).
 * pk_freq_matvec:  y_dev[(m-begin)*q_n + n-1] = (K_f x)[...]   (x real, [P])
 * pk_freq_adjoint: out_dev[p] = scale * (K_f^H y)[p]           (y complex [M*q_n], out complex [P])
 * Replaces forward._matvec / _adjoint_matvec for frequency-domain K (forward.py:237-250).
 * The forward keeps a partial-sum workspace in the plan, allocated on the first call for a
 * given q_n (the only allocation outside pk_plan_create). */
int pk_freq_matvec(pk_plan* plan, int32_t q_n, const void* x_dev, void* y_dev, void* stream);
int pk_freq_adjoint(pk_plan* plan, int32_t q_n, const void* y_dev, void* out_dev, double scale,
                    void* stream);

/* Index dump (verification): for local sensors [ma, mb) (relative to sensor_begin),
 * s0_dev[(m-ma)*P + p] = floor(hypot(px - sx, py - sy) / (c*dt)) and frac_dev likewise,
 * evaluated in fp64 exactly as forward.py:157-182 (s0 int64, frac double; frac may be NULL). */
int pk_index_dump(pk_plan* plan, int32_t ma, int32_t mb, int64_t* s0_dev, double* frac_dev,
                  void* stream);

/* fp32 delay census (verification of the production kernels' index rule): for local sensors
 * [ma, mb), s0_dev[(m-ma)*P + p] (int32) and frac_dev (float) exactly as the fp32 kernels
 * evaluate the delay of pair (p, m): rule 0 the generic back-projector / projector, rule 1 the
 * D4-symmetric back-projector (the representative pair's delay), rule 2 the rotation-symmetric
 * projector.  s0 + frac is the fp32 delay u; compare with pk_index_dump / np.hypot. */
int pk_delay_census_f32(pk_plan* plan, int32_t rule, int32_t ma, int32_t mb, int32_t* s0_dev,
                        float* frac_dev, void* stream);

/* Profiling hook (bench.py roofline): run the solver's kernels un-graphed on `stream`
 * for params->iterations iterations, with CUDA events around every launch.
 * ms_out[0..2] = summed device milliseconds of K1 (fused back-projection update),
 * K2 (projection) and K3 (residual/objective); launches_out[0] = kernels launched.
 * Synchronises the stream. */
int pk_profile_iterations(pk_plan* plan, const pk_solver_params* params, const void* y_dev,
                          float* ms_out, int32_t* launches_out, void* stream);

/* The same un-graphed replay with the symmetric back-projector's update kernel timed on its
 * own (replaces the stage accounting of iterative_reconstruct, recon.py:303-347):
 * ms_out[0..3] = summed device milliseconds of the back-projection (K^T r), the update
 * (TV gradient + soft threshold + non-negativity, recon.py:330-338), the projection and the
 * residual/objective kernel; plans without a separate update report it inside ms_out[0] and
 * ms_out[1] = 0.  Synchronises the stream. */
int pk_profile_stages(pk_plan* plan, const pk_solver_params* params, const void* y_dev,
                      float* ms_out, int32_t* launches_out, void* stream);

/* FP32 roofline denominator: FFMA throughput of `device` measured with a dependent-chain
 * microkernel (8 independent chains per thread, 148*4 CTAs), in TFLOP/s. */
int pk_measure_fp32_peak(int32_t device, double* tflops_out);

/* Explicit-matrix mode: a MeasurementMatrix given by its entries
 * (read_matrix / PACTMAT, forward.py:70-121, 297-330) rather than by geometry.  Replaces the
 * reference's numba GEMV cores for such a K: matvec_parallel / matvec_adjoint_parallel
 * (kernels.py:195-202, 215-225, 319-350) and iterative_reconstruct's loop (recon.py:286-377).
 * K is held on the device in the plan dtype (PK_F32 halves the bytes streamed per product);
 * complex entries (frequency-domain K) are interleaved (re, im).
 *   pk_dense_create        rows x cols operator; cols must fill whole 16-byte rows
 *                          (PK_ERR_UNSUPPORTED otherwise)
 *   pk_dense_set_entries   row-major fp64 (complex128) entries, host (on_device = 0) or
 *                          device memory; converted to the plan dtype on the device
 *   pk_dense_matvec        y = K x (x real, or complex if x_complex; y complex iff K or x is)
 *   pk_dense_adjoint       out = scale K^H y (out complex iff K or y is)
 *   pk_dense_reconstruct   the whole solve on the device (one captured graph, no host sync):
 *                          y [rows] plan dtype (complex interleaved for complex K), x_out [nx*ny]
 *                          real, hist [4][iterations] double, status [2] int32 (as pk_reconstruct).
 *                          A real PK_F32 operator reads K once per iteration (the residual
 *                          and the next gradient from one pass); otherwise two passes. */
typedef struct pk_dense pk_dense;
typedef struct pk_dense_info {
    int64_t rows, cols;
    int32_t dtype, complex_entries;
    int32_t fused;           /* 1: one pass over K per solver iteration */
    int32_t splits;          /* row splits of the adjoint's column partials */
    int64_t device_bytes;
} pk_dense_info;
int pk_dense_create(int64_t rows, int64_t cols, int32_t dtype, int32_t complex_entries,
                    int32_t device, pk_dense** out);
int pk_dense_destroy(pk_dense* op);
int pk_dense_get_info(const pk_dense* op, pk_dense_info* out);
int pk_dense_set_entries(pk_dense* op, const double* entries, int32_t on_device, void* stream);
/* Multi-frame products on the tensor cores (tcgen05 kind::tf32, 3xTF32 split: fp32
 * accuracy, ~2e-6 relative), real fp32 matrices: y[f] = K x[f] (x [frames][cols], y
 * [frames][rows]) and g[f] = K^T y[f] (g [frames][cols]; K^T is built in HBM on the first
 * call), 1 <= frames <= 128, cols (and rows, for the adjoint) multiples of 4.  The
 * reference's per-frame GEMV cores (kernels.py:195-225) applied to a frame batch. */
int pk_dense_matmat(pk_dense* dense, int32_t frames, const void* x_dev, void* y_dev, void* stream);
int pk_dense_rmatmat(pk_dense* dense, int32_t frames, const void* y_dev, void* g_dev, void* stream);

/* Dense K of a geometry plan built on the device (build_time_matrix, forward.py:167-194):
 * fp64 entries bit-identical to the reference's (the plan's fp64 delays), PK_F32 rounded. */
int pk_dense_from_plan(pk_dense* op, const pk_plan* plan, void* stream);
int pk_dense_matvec(pk_dense* op, const void* x_dev, int32_t x_complex, void* y_dev, void* stream);
int pk_dense_adjoint(pk_dense* op, const void* y_dev, int32_t y_complex, void* out_dev, double scale,
                     void* stream);
int pk_dense_reconstruct(pk_dense* op, int32_t nx, int32_t ny, const pk_solver_params* params,
                         const void* y_dev, void* x_out_dev, double* history_dev, int32_t* status_dev,
                         void* stream);

const char* pk_last_error(void);
int pk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PACTGPU_H */
