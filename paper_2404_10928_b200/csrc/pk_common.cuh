// pk_common.cuh -- shared device helpers, the plan object and device state.
//
// Naming follows the reference's domain (pactkit, arXiv 2404.10928): pixels,
// sensors, samples, traces, delays.  The "table" is the per-sensor residual
// trace laid out for the back-projector's two-sample interpolation (one
// 8-byte load per sensor-pixel interaction).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "pactgpu.h"

namespace pk {

// ---------------------------------------------------------------------------
// constants of the fp32 delay / fixed-point tricks
constexpr float kTwo23 = 8388608.0f;     // 2^23: floor via round-down add
constexpr uint32_t kTwo23Bits = 0x4B000000u;
constexpr float kMagic = 12582912.0f;    // 1.5 * 2^23: round-to-int via add
constexpr int32_t kMagicBits = 0x4B400000;

constexpr int kThreads = 256;  // every kernel uses 8 warps
constexpr int kBpTile = 32;    // back-projector pixel tile (32 x 32, 4 pixels/thread)
constexpr int kDivergenceStreak = 5;  // recon.py:42-43

// ---------------------------------------------------------------------------
// device state of one solve.  A plan reconstructs NF frames that share the geometry
// (NF = 1 single frame; NF = 2 or 4 batched, fp32): the delay of every sensor-pixel pair is
// evaluated once and applied to all NF frames.  Per-frame solver state lives in fr[].
constexpr int kMaxFrames = 4;

struct FrameState {
    double maxabs;     // max |x'| of the new iterate (update kernel)
    double l1sum;      // sum |x'|
    double scale64;    // fixed-point scale of the projector (2^bits / maxabs)
    double f_prev;     // objective of the last accepted iterate
    float scale32;
    int32_t nonfinite; // any non-finite x'
    int32_t accepted;  // iterations accepted (== iterations_run)
    int32_t stopped;
    int32_t stopped_by;
    int32_t grow;
    uint32_t mxw;      // max |x'| of the symmetric epilogue's CTAs as float bits (atomicMax of
                       //   non-negative floats; reset by the residual kernel and init)
};

struct DevState {
    int32_t iter;        // iterations attempted so far (shared by the frames)
    int32_t all_stopped; // every frame stopped (or iteration cap): kernels early-exit
    int32_t epoch;       // solves started on this plan (init_kernel): launch ids of the fused update
    int32_t pad1;
    // last-block counters (reset by the last block itself)
    uint32_t cnt_bp, cnt_fp, cnt_fin, cnt_misc;
    double sums[4];      // scalars of the sharded / standalone entry points
    FrameState fr[kMaxFrames];
};

// device copy of the solver parameters (read by the graph's kernels)
struct DevParams {
    double alpha[kMaxFrames], beta[kMaxFrames], step[kMaxFrames];
    double eta_alpha[kMaxFrames];  // step * alpha (soft-threshold level)
    double eps, tolerance;
    int32_t iterations, nonneg;
};

// I/O pointers of pk_reconstruct, read from device memory so that one captured graph
// serves any caller buffers.  Frame-major: y [NF][M*Q], x_out [NF][P],
// hist [NF][4][iterations], status [NF][2].
struct DevIo {
    const void* y;
    void* x_out;
    double* hist;
    int32_t* status;
};

// ---------------------------------------------------------------------------
// small PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

__device__ __forceinline__ void red_smem_s32(uint32_t addr, int32_t v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(v));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// 1-D bulk reduction shared -> global (TMA engine): dst[i] += src[i] as 32-bit integers,
// performed at L2 (order independent); bytes and both addresses multiples of 16.  Tracked by
// the issuing thread's bulk groups.
__device__ __forceinline__ void bulk_reduce_add_u32(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u32 [%0], [%1], %2;" ::"l"(dst),
                 "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the shared-memory sources of this thread's bulk groups may be overwritten
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// this thread's bulk groups are complete (their global writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// generic-proxy shared-memory writes made visible to the async proxy (TMA) before a barrier
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// programmatic dependent launch: a kernel launched with programmatic stream serialization
// may start while its predecessor drains; it must wait before touching the predecessor's
// output.  Both are no-ops for kernels launched without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------
// deterministic block reductions (fixed shuffle tree + fixed warp order)
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// LDGSTS: asynchronous 4- / 8-byte global -> shared copy (no register staging)
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gmem_src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src),
                 "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// sum over the block (NT threads, 256 by default); result valid in every thread
template <typename T, int NT = kThreads>
__device__ __forceinline__ T block_sum(T v, T* red) {  // NT = block size (red: NT / 32 slots)
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    T s = red[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) s += red[w];
    return s;
}
// four sums in one pass (one pair of barriers); red: 4 * NT / 32 slots
template <int NT = kThreads>
__device__ __forceinline__ void block_sum4(double (&v)[4], double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = warp_sum(v[q]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 4; ++q) red[q * (NT / 32) + warp] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        double s = red[q * (NT / 32)];
#pragma unroll
        for (int w = 1; w < NT / 32; ++w) s += red[q * (NT / 32) + w];
        v[q] = s;
    }
}
template <typename T, int NT = kThreads>
__device__ __forceinline__ T block_max(T v, T* red) {
    v = warp_max(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    T s = red[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) s = fmax(s, red[w]);
    return s;
}

// "last block done" detection; every thread gets the answer.  The counter is reset
// by the last block so the kernel can be relaunched (and graph-replayed).
__device__ __forceinline__ bool last_block(uint32_t* counter, uint32_t total, int* flag_smem) {
    // One gpu-scope fence per CTA, by the thread that takes the ticket (the grid-sync pattern
    // of cooperative groups): bar.sync orders the CTA's writes before thread 0's fence, which
    // is cumulative; the last CTA's thread 0 fences again before the barrier that releases
    // its readers.  A fence in every thread (MEMBAR.SC per warp) cost ~15 % of the residual
    // kernel's stall samples.
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        uint32_t prev = atomicAdd(counter, 1u);
        const int last = (prev == total - 1) ? 1 : 0;
        *flag_smem = last;
        if (last) {
            atomicExch(counter, 0u);
            __threadfence();
        }
    }
    __syncthreads();
    return *flag_smem != 0;
}

// hypot as glibc computes it (the reference's np.hypot, forward.py:157-160): one rounded
// sqrt, then Borges' correction step -- the non-FMA kernel of glibc's e_hypot.c, which
// matched libm's hypot bit for bit on 2e7 random pairs in this image (glibc 2.39).
// Explicit _rn intrinsics keep nvcc from contracting anything into FMA.
__device__ __forceinline__ double hypot_libm(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x, ay = x < y ? x : y;
    double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    double t1, t2;
    if (h <= __dmul_rn(2.0, ay)) {
        const double delta = __dsub_rn(h, ay);
        t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
        t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
    } else {
        const double delta = __dsub_rn(h, ax);
        t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
        t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
    }
    return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

// fp64 delay in samples exactly as forward.py:157-182 evaluates it: d = hypot(px - sx,
// py - sy); u = d / (c*dt).  s0 = floor(u) and frac = u - s0 are then bit-exact.
__device__ __forceinline__ double delay_f64(double px, double py, double sx, double sy,
                                            double cdt) {
    return __ddiv_rn(hypot_libm(__dsub_rn(px, sx), __dsub_rn(py, sy)), cdt);
}

}  // namespace pk

// ---------------------------------------------------------------------------
// the plan (opaque to C callers)
struct pk_plan {
    int device = 0, dtype = PK_F32;
    int nf = 1;  // frames per plan (shared geometry)
    int nx = 0, ny = 0, P = 0, Mall = 0, m0 = 0, M = 0, Q = 0;
    double c = 0, dt = 0, cdt = 0, w = 0;
    int may_truncate = 0;
    double min_delay = 0, max_delay = 0;  // in samples, host-computed bounds

    // local sensors: gid[l] = ring index of local sensor l (m0 + l, or the sensor list);
    // loc[ring index] = local index or -1 (device copies for the symmetric kernels)
    std::vector<int> gid_h;
    int* gid = nullptr;
    int* loc = nullptr;
    int listed = 0;  // the plan was made from a sensor list

    // geometry on the device
    float *pxs = nullptr, *pys = nullptr, *sxs = nullptr, *sys = nullptr;  // scaled by 1/cdt
    double *px = nullptr, *py = nullptr, *sx = nullptr, *sy = nullptr;    // original fp64

    // residual pair table [M][TS] (float2 / double2) and fixed-point accumulator [M][Q]
    int TS = 0;
    void* table = nullptr;
    long long* acc = nullptr;

    // iterates and scratch
    void* xbuf[2] = {nullptr, nullptr};
    void* ydev = nullptr;        // device copy of y for pk_reconstruct_host
    double* y64 = nullptr;       // fp64 staging of y (host API)
    double* x64 = nullptr;       // fp64 staging of the image (host API)
    void* xout_dev = nullptr;    // image in plan dtype (host API)
    double* hist_dev = nullptr;  // history for the host API
    int hist_cap = 0;
    int32_t* status_dev = nullptr;
    double* part_bp = nullptr;   // [bp blocks * 4]
    float* part_mx = nullptr;    // [symmetric epilogue CTAs] max |x'| partials (deferred stats)
    double* part_l1 = nullptr;   // [residual CTAs][2] sum |x'|, non-finite (deferred stats)
    double* part_tv = nullptr;   // [fp tiles]
    double* part_r = nullptr;    // [M]
    double* part_misc = nullptr; // [generic blocks * 4]
    pk::DevState* state = nullptr;
    pk::DevParams* params = nullptr;
    pk::DevIo* io = nullptr;

    // back-projector tiling
    int bp_tiles_x = 0, bp_tiles_y = 0, bp_L = 0, bp_CS = 0, bp_nbuf = 0, bp_smem = 0;
    int bp_split = 1, bp_ms = 0;
    int bp_atrick = 0;  // fp32 pair-table layout {r[s-1] - s*D, D}
    // D4-symmetric back-projector (bp_sym_f32_kernel + bp_sym_epi_kernel)
    int sym = 0, sym_ntiles = 0, sym_L = 0, sym_nbuf = 0, sym_smem = 0, sym_grid = 0, sym_slots = 0;
    int sym_iw = 0;  // compile-time image-window stride (slots), 0 = runtime
    int sym_nch = 0;     // chunks (of kSymCS base sensors) per tile
    int sym_wdiag = 24;  // cut weight of a diagonal chunk (off-diagonal 32); < 0: pinned (env)
    int sym_slots_cap = 0;  // partial slots allocated (the largest candidate partition's)
    int sym_lanemap = 1;
    int sym_fuse = 0;     // update fused into the back-projector's tail (solver mode, opt-in)
    int sym_epik = 0;     // solver epilogue strips per CTA (deferred stats): 0 = default (2), 1, 2, 4
    int *sym_tiles = nullptr, *sym_chunks = nullptr, *sym_cta_chunk0 = nullptr,
        *sym_cta_slot0 = nullptr, *sym_tile_slot0 = nullptr;
    float* sym_part = nullptr;  // [slots][8][4][kThreads] partial sums
    std::vector<int> sym_h[5];  // host copies: tiles, chunks, cta_chunk0, cta_slot0, tile_slot0
    // rotation-symmetric projector (fp_sym_f32_kernel)
    int fsym = 0, fsym_T = 0, fsym_qt = 0, fsym_L = 0, fsym_smem = 0, fsym_groups = 0;
    int fsym_nw = 0;      // warps per CTA (16: two CTAs per SM, 32: one)
    int fsym_ngr = 4;     // images per staging round of the bulk reductions
    int fsym_grid = 0;    // persistent CTAs (every one resident)
    int fsym_nseg = 0;    // segments (window sets) per projection
    int fsym_hs = 0;      // rows per segment at most
    int fsym_acc_ld = 0;  // accumulator row length (words)
    float fsym_hx = 0.f;  // pixel pitch in samples
    float* fsym_xr = nullptr;     // [(n/2)^2][4] x' rotation-packed by the epilogue
    int32_t* fsym_acc = nullptr;  // [M][acc_ld] int32 trace accumulator (windows reduce-added)
    int* fsym_trace = nullptr;    // [groups * 32][4] local trace of (base sensor, image)
    uint16_t* fsym_bias = nullptr;  // [M][acc_ld] biased words per accumulator position (u16)
    int4* fsym_segs = nullptr;    // [segments] {group, strip, first row, end row}
    int* fsym_cta_seg0 = nullptr; // [grid + 1]
    int* fsym_rec = nullptr;      // [frames] segment that records the frame's scale
    std::vector<int4> fsym_segs_h;
    std::vector<int> fsym_rec_h;
    std::vector<int> fsym_cta_seg0_h;
    int fin_chunks = 1;  // residual kernel: sample chunks per sensor
    float* bp_gpart = nullptr;
    uint32_t* bp_tile_cnt = nullptr;
    uint32_t* sym_sync = nullptr;  // [3][ntiles] fused-update arrival / unit / publication words
    long long sym_spin_ns = 20000;
    // projector tiling
    int fp_T = 0, fp_tiles_x = 0, fp_tiles_y = 0, fp_groups = 0, fp_L = 0, fp_bits = 0,
        fp_smem = 0;
    int misc_blocks = 0;
    void* freq_part = nullptr;  // frequency-domain forward partials (grown on first use)
    size_t freq_part_bytes = 0;

    // peer exchange of the sensor-sharded gradient (pk_peer_*): the local block holds
    // int flags[PK_PEER_MAX] (written by the peers), the barrier epoch, and T grad[2][P]
    unsigned char* peer_block = nullptr;
    int peer_world = 0, peer_rank = -1;
    void** peer_grad_dev = nullptr;     // device [world]: grad[0] of every rank (local or mapped)
    int** peer_flags_dev = nullptr;     // device [world]: flag array of every rank
    std::vector<void*> peer_opened;     // IPC mappings to close on destroy

    // graph cache of pk_reconstruct
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    cudaStream_t cap_stream = nullptr;
    cudaEvent_t bp_mid_event = nullptr;  // pk_profile_stages: recorded between K1s and its epilogue
    int graph_iters = -1;
    pk::DevParams params_host{};  // last uploaded solver parameters
    int params_valid = 0;

    int64_t device_bytes = 0;
};
