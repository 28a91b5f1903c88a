// pactgpu.cu -- C ABI (include/pactgpu.h) over the sm_100a kernels in pk_kernels.cuh.
//
// Host-side responsibilities: validate the geometry the reference's MeasurementMatrix
// carries (forward.py:70-121), pick tile / window sizes, own the device workspace, and
// sequence the kernels of each entry point on the caller's stream.  pk_reconstruct is
// captured once per iteration count into a CUDA graph and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "pactgpu.h"
#include "pk_kernels.cuh"
#include "pk_freq.cuh"
#include "pk_dense.cuh"
#include "pk_tc.cuh"

using namespace pk;

namespace pk {
// holds the stream while the host enqueues the profiled launches, so that the CUDA-event
// intervals measure back-to-back device execution rather than host launch rate
__global__ void hold_kernel(long long ns) {
    const long long t0 = clock64();
    while (clock64() - t0 < ns) __nanosleep(1000);
}

// FP32 peak microkernel: 8 independent FFMA chains per thread
__global__ void __launch_bounds__(kThreads) ffma_peak_kernel(float* out, int iters) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
          a6 = a0 + 6, a7 = a0 + 7;
    const float b = 1.0001f + 1e-9f * blockIdx.x, c = 0.9999f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
            a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
        }
    }
    out[blockIdx.x * kThreads + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
}  // namespace pk

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

#define PK_CUDA(call)                                                                    \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(PK_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                             \
    } while (0)

#define PK_CHECK_LAUNCH()                                                                 \
    do {                                                                                  \
        cudaError_t e_ = cudaGetLastError();                                              \
        if (e_ != cudaSuccess)                                                            \
            return fail(PK_ERR_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                              \
    } while (0)

#define PK_TRY(x)                     \
    do {                              \
        int rc_ = (x);                \
        if (rc_ != PK_OK) return rc_; \
    } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int ceil_log2(double v) {
    int b = 0;
    while ((double)(1ull << b) < v && b < 62) ++b;
    return b;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

template <typename T>
int alloc(pk_plan* p, T** ptr, size_t count) {
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), count * sizeof(T));
    if (e != cudaSuccess)
        return fail(PK_ERR_CUDA, "cudaMalloc(%zu) failed: %s", count * sizeof(T),
                    cudaGetErrorString(e));
    p->device_bytes += (int64_t)(count * sizeof(T));
    return PK_OK;
}

// peer blocks exported by plans of this process, by handle bytes: a handle cannot be opened
// by the process that exported it, so same-process peers are resolved here
std::mutex g_peer_mu;
std::map<std::string, unsigned char*> g_peer_registry;

void peer_registry_drop(unsigned char* block) {
    std::lock_guard<std::mutex> lk(g_peer_mu);
    for (auto it = g_peer_registry.begin(); it != g_peer_registry.end();)
        it = it->second == block ? g_peer_registry.erase(it) : std::next(it);
}

constexpr size_t kPeerHeader = 256;  // int flags[PK_PEER_MAX], int epoch, int timed_out, padding

// barrier wait bound (PK_PEER_TIMEOUT_S, default 60 s)
long long peer_timeout_ns() {
    static const long long ns = [] {
        const char* e = getenv("PK_PEER_TIMEOUT_S");
        const double sec = e ? atof(e) : 60.0;
        return (long long)((sec > 0 ? sec : 60.0) * 1e9);
    }();
    return ns;
}
size_t peer_slot_bytes(const pk_plan* p) {
    return ((size_t)p->P * (p->dtype == PK_F32 ? 4 : 8) + 255) & ~(size_t)255;
}

void free_plan(pk_plan* p) {
    if (!p) return;
    DeviceGuard g(p->device);
    if (p->graph_exec) cudaGraphExecDestroy(p->graph_exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    void* ptrs[] = {p->pxs, p->pys, p->sxs, p->sys, p->px, p->py, p->sx, p->sy, p->table,
                    p->acc, p->xbuf[0], p->xbuf[1], p->ydev, p->y64, p->x64, p->hist_dev,
                    p->status_dev, p->part_bp, p->part_mx, p->part_l1, p->part_tv, p->part_r, p->part_misc, p->state,
                    p->params, p->io, p->xout_dev, p->bp_gpart, p->bp_tile_cnt, p->sym_sync, p->sym_tiles,
                    p->sym_chunks, p->sym_cta_chunk0, p->sym_cta_slot0, p->sym_tile_slot0,
                    p->sym_part, p->fsym_acc, p->fsym_trace, p->fsym_bias, p->fsym_rec,
                    p->fsym_segs, p->fsym_cta_seg0,
                    p->freq_part, p->gid, p->loc};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    for (void* q : p->peer_opened) cudaIpcCloseMemHandle(q);
    if (p->peer_block) {
        peer_registry_drop(p->peer_block);
        cudaFree(p->peer_block);
    }
    if (p->peer_grad_dev) cudaFree(p->peer_grad_dev);
    if (p->peer_flags_dev) cudaFree(p->peer_flags_dev);
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    delete p;
}

size_t tsize(const pk_plan* p) { return p->dtype == PK_F32 ? 4 : 8; }

// Programmatic dependent launch (PK_PDL=0 disables): the kernel may be scheduled while its
// predecessor on the stream drains and waits (griddep_wait) before reading its output.
// Only kernels that contain that wait are launched this way.
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("PK_PDL");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}

// every (kernel, NF) instantiation the dispatch below can launch
template <int NF>
void smem_kernels(std::vector<const void*>& v) {
    v.push_back((const void*)bp_f32_kernel<NF, true, true, true>);
    v.push_back((const void*)bp_f32_kernel<NF, true, false, true>);
    v.push_back((const void*)bp_f32_kernel<NF, false, true, true>);
    v.push_back((const void*)bp_f32_kernel<NF, false, false, true>);
    v.push_back((const void*)bp_f32_kernel<NF, true, true, false>);
    v.push_back((const void*)bp_f32_kernel<NF, true, false, false>);
    v.push_back((const void*)bp_f32_kernel<NF, false, true, false>);
    v.push_back((const void*)bp_f32_kernel<NF, false, false, false>);
    v.push_back((const void*)fp_f32_kernel<NF, false>);
    v.push_back((const void*)finalize_kernel<float, NF>);
}

constexpr int kSymIW[] = {64, 96, 128, 192, 256};
// relative cost of a chunk: diagonal tiles evaluate the same delays for 4 images, not 8
// (per delay ~8 issue slots of geometry + 3 per image: 20 vs 32)
constexpr int kSymWDiag = 5, kSymWOff = 8;

// chunk ranges of the symmetric back-projector's persistent CTAs: equal-cost contiguous
// ranges of the (frame-major tile, chunk) sequence, off-diagonal chunk weight 32, diagonal
// wdiag; every CTA leaves one partial slot per tile it touches.  Fills sym_h[1..4], sym_slots.
static void sym_partition(pk_plan* p, int wdiag) {
    const std::vector<int>& tl = p->sym_h[0];
    std::vector<int>& ch = p->sym_h[1];
    std::vector<int>& c0 = p->sym_h[2];
    std::vector<int>& cs0 = p->sym_h[3];
    std::vector<int>& ts0 = p->sym_h[4];
    ch.clear(); c0.clear(); cs0.clear(); ts0.clear();
    const int nf = p->nf, nch = p->sym_nch;
    auto cw_of = [&](int tt) { return ((tl[tt] >> 16) == (tl[tt] & 0xffff)) ? wdiag : 32; };
    int64_t W = 0;
    for (int t = 0; t < p->sym_ntiles; ++t) W += (int64_t)nch * nf * cw_of(t);
    const int G = p->sym_grid;
    c0.assign(G + 1, 0);
    cs0.assign(G, 0);
    int64_t cw = 0;
    int owner_prev = -1, tile_prev = -1, slot = -1;
    // frame-major tiles: chunk tile index t = frame * ntiles + tile
    for (int t = 0; t < p->sym_ntiles * nf; ++t) {
        const int wt = cw_of(t % p->sym_ntiles);
        for (int k = 0; k < nch; ++k) {
            const int owner = (int)std::min<int64_t>(G - 1, cw * G / W);
            if (owner != owner_prev || t != tile_prev) {
                ++slot;
                if (t != tile_prev) ts0.push_back(slot);
                if (owner != owner_prev) {
                    for (int b = owner_prev + 1; b <= owner; ++b) c0[b] = (int)ch.size();
                    cs0[owner] = slot;
                }
                owner_prev = owner;
                tile_prev = t;
            }
            ch.push_back((t << 16) | k);
            cw += wt;
        }
    }
    for (int b = owner_prev + 1; b <= G; ++b) c0[b] = (int)ch.size();
    ts0.push_back(slot + 1);
    p->sym_slots = slot + 1;
}
constexpr int kSymWCand[] = {18, 20, 22, 24, 26};

template <int IW>
void launch_sym(const BpSymArgs& A, int grid, int smem, cudaStream_t s) {
    launch_pdl(bp_sym_f32_kernel<IW>, dim3(grid), dim3(kSymThreads), smem, s, A);
}

const void* sym_kernel_ptr(int iw) {
    switch (iw) {
        case 64: return (const void*)bp_sym_f32_kernel<64>;
        case 96: return (const void*)bp_sym_f32_kernel<96>;
        case 128: return (const void*)bp_sym_f32_kernel<128>;
        case 192: return (const void*)bp_sym_f32_kernel<192>;
        case 256: return (const void*)bp_sym_f32_kernel<256>;
        default: return (const void*)bp_sym_f32_kernel<0>;
    }
}

template <int NW>
void fsym_kernels(std::vector<const void*>& ks) {
#define PK_FSK(LW, T) ks.push_back((const void*)fp_sym_f32_kernel<LW, false, T, NW>); \
                      ks.push_back((const void*)fp_sym_f32_kernel<LW, true, T, NW>);
    PK_FSK(96, 64) PK_FSK(128, 64) PK_FSK(184, 64) PK_FSK(256, 64) PK_FSK(320, 64)
    PK_FSK(96, 32) PK_FSK(128, 32) PK_FSK(184, 32) PK_FSK(256, 32)
#undef PK_FSK
}

cudaError_t opt_in_smem(int device) {
    static bool done[64] = {};
    if (device < 0 || device >= 64) return cudaErrorInvalidDevice;
    if (done[device]) return cudaSuccess;
    int mx = 0;
    cudaError_t e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    // (each kernel's own static shared memory is subtracted below)
    std::vector<const void*> ks;
    smem_kernels<1>(ks);
    smem_kernels<2>(ks);
    smem_kernels<4>(ks);
    fsym_kernels<16>(ks);
    fsym_kernels<32>(ks);
    for (const void* k : std::vector<const void*>{})
        ks.push_back(k);
    ks.push_back(sym_kernel_ptr(0));
    for (int iw : kSymIW) ks.push_back(sym_kernel_ptr(iw));
    ks.push_back((const void*)fp_f64_kernel);
    ks.push_back((const void*)finalize_kernel<double, 1>);
    for (const void* k : ks) {
        cudaFuncAttributes fa{};
        if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, k);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     mx - (int)fa.sharedSizeBytes);
    }
    if (e == cudaSuccess) done[device] = true;
    return e;
}

// ---------------------------------------------------------------------------
// kernel sequences (NF-dispatched)

template <int NF>
void launch_maxabs_t(pk_plan* p, const void* x, cudaStream_t s) {
    const dim3 grid(p->misc_blocks, NF);
    if (p->dtype == PK_F32)
        maxabs_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<const float*>(x), p->P,
                                                       p->part_misc, p->state, p->fp_bits);
    else
        maxabs_kernel<double><<<grid, kThreads, 0, s>>>(static_cast<const double*>(x), p->P,
                                                        p->part_misc, p->state, p->fp_bits);
}

template <int NF>
void launch_fp_t(pk_plan* p, const void* x, int solver, cudaStream_t s) {
    dim3 grid(p->fp_tiles_x * p->fp_tiles_y, p->fp_groups);
    if (p->dtype == PK_F32 && p->fsym) {
        FpSymArgs a{};
        a.x = static_cast<const float*>(x);
        a.xb0 = static_cast<const float*>(p->xbuf[0]);
        a.xb1 = static_cast<const float*>(p->xbuf[1]);
        a.pxs = p->pxs; a.pys = p->pys; a.sxs = p->sxs; a.sys = p->sys;
        a.acc = p->fsym_acc; a.acc_ld = p->fsym_acc_ld; a.trace_of = p->fsym_trace;
        a.n = p->nx; a.M = p->M; a.Q = p->Q;
        a.segs = p->fsym_segs; a.cta_seg0 = p->fsym_cta_seg0;
        a.rec = p->fsym_rec; a.groups = p->fsym_groups;
        a.qclamp = (float)p->Q + 1.5f;
        a.hx = p->fsym_hx;
        a.st = p->state; a.solver = solver;
        a.xr = reinterpret_cast<const float4*>(p->fsym_xr);
        if (solver && p->sym) {  // the symmetric epilogue deferred its statistics
            a.part_mx = p->part_mx;
            a.nmx = p->sym_ntiles * 32;
            a.bits = p->fp_bits;
        }
        const bool clamp = p->max_delay >= (double)p->Q + 0.5;
        const dim3 grid(p->fsym_grid), block(p->fsym_nw * 32);
#define PK_FS3(LW, T, NW) (clamp ? launch_pdl(fp_sym_f32_kernel<LW, true, T, NW>, grid, block, p->fsym_smem, s, a) \
                                 : launch_pdl(fp_sym_f32_kernel<LW, false, T, NW>, grid, block, p->fsym_smem, s, a))
#define PK_FS(LW, T) (p->fsym_nw == 32 ? PK_FS3(LW, T, 32) : PK_FS3(LW, T, 16))
        if (p->fsym_T == 32) {
            switch (p->fsym_L) {
                case 96: PK_FS(96, 32); break;
                case 128: PK_FS(128, 32); break;
                case 184: PK_FS(184, 32); break;
                default: PK_FS(256, 32); break;
            }
        } else {
            switch (p->fsym_L) {
                case 96: PK_FS(96, 64); break;
                case 128: PK_FS(128, 64); break;
                case 184: PK_FS(184, 64); break;
                case 256: PK_FS(256, 64); break;
                default: PK_FS(320, 64); break;
            }
        }
#undef PK_FS3
#undef PK_FS
        return;
    }
    if (p->dtype == PK_F32) {
        FpArgs a{};
        a.x = static_cast<const float*>(x);
        a.xb0 = static_cast<const float*>(p->xbuf[0]);
        a.xb1 = static_cast<const float*>(p->xbuf[1]);
        a.pxs = p->pxs; a.pys = p->pys; a.sxs = p->sxs; a.sys = p->sys;
        a.acc = p->acc;
        a.nx = p->nx; a.ny = p->ny; a.M = p->M; a.Q = p->Q; a.T = p->fp_T; a.L = p->fp_L;
        a.tiles_x = p->fp_tiles_x;
        a.qclamp = (float)p->Q + 1.5f;
        a.st = p->state; a.part_tv = p->part_tv; a.solver = solver;
        fp_f32_kernel<NF, false><<<grid, kThreads, p->fp_smem, s>>>(a);
    } else {
        FpArgs64 a{};
        a.x = static_cast<const double*>(x);
        a.xb0 = static_cast<const double*>(p->xbuf[0]);
        a.xb1 = static_cast<const double*>(p->xbuf[1]);
        a.px = p->px; a.py = p->py; a.sx = p->sx; a.sy = p->sy; a.cdt = p->cdt;
        a.acc = p->acc;
        a.nx = p->nx; a.ny = p->ny; a.M = p->M; a.Q = p->Q; a.T = p->fp_T; a.L = p->fp_L;
        a.tiles_x = p->fp_tiles_x;
        a.st = p->state; a.part_tv = p->part_tv; a.solver = solver;
        fp_f64_kernel<<<grid, kThreads, p->fp_smem, s>>>(a);
    }
}

template <int NF>
void launch_finalize_t(pk_plan* p, const void* y, void* trace_out, double* sumsq, int solver,
                       cudaStream_t s) {
    const int chunks = p->fin_chunks;
    const size_t clen1 = (size_t)((p->Q + chunks - 1) / chunks + 1);
    // residual [clen + 1], staged measurements [clen]
    size_t sm = ((clen1 * tsize(p) + 15) & ~(size_t)15) + (((clen1 - 1) * tsize(p) + 15) & ~(size_t)15);
    const dim3 grid(p->M * chunks, NF);
    if (p->dtype == PK_F32) {
        FinArgs<float> a{};
        a.acc = p->acc; a.y = static_cast<const float*>(y);
        a.trace_out = static_cast<float*>(trace_out);
        a.table = static_cast<float2*>(p->table);
        a.M = p->M; a.Q = p->Q; a.TS = p->TS; a.w = p->w;
        a.st = p->state; a.prm = p->params; a.io = p->io; a.part_r = p->part_r;
        a.part_tv = p->part_tv;
        a.ntv = p->fsym ? (int)grid.x : p->fp_tiles_x * p->fp_tiles_y;
        if (p->fsym && solver) {
            a.part_l1 = p->part_l1;
            a.tv_here = 1;
            a.xb0 = static_cast<const float*>(p->xbuf[0]);
            a.xb1 = static_cast<const float*>(p->xbuf[1]);
            a.n = p->nx;
        }
        a.sumsq_out = sumsq;
        a.solver = solver;
        if (p->fsym) {
            a.acc32 = p->fsym_acc;
            a.acc32_ld = p->fsym_acc_ld;
            a.bias16 = p->fsym_bias;
        }
        a.atrick = p->bp_atrick;
        a.chunks = chunks;
        if (p->fsym && p->Q <= kFinSymMax && chunks == 1) {
            if (p->Q <= 4 * kThreads) launch_pdl(finalize_sym_kernel<NF, 1>, grid, dim3(kThreads), 0, s, a);
            else if (p->Q <= 8 * kThreads) launch_pdl(finalize_sym_kernel<NF, 2>, grid, dim3(kThreads), 0, s, a);
            else launch_pdl(finalize_sym_kernel<NF, 4>, grid, dim3(kThreads), 0, s, a);
        }
        else
            launch_pdl(finalize_kernel<float, NF>, grid, dim3(kThreads), sm, s, a);
    } else {
        FinArgs<double> a{};
        a.acc = p->acc; a.y = static_cast<const double*>(y);
        a.trace_out = static_cast<double*>(trace_out);
        a.table = static_cast<double2*>(p->table);
        a.M = p->M; a.Q = p->Q; a.TS = p->TS; a.w = p->w;
        a.st = p->state; a.prm = p->params; a.io = p->io; a.part_r = p->part_r;
        a.part_tv = p->part_tv; a.ntv = p->fp_tiles_x * p->fp_tiles_y; a.sumsq_out = sumsq;
        a.solver = solver;
        a.chunks = chunks;
        finalize_kernel<double, 1><<<grid, kThreads, sm, s>>>(a);
    }
}

// K1: epi == 0 -> out = gscale_mult * w * K^T r; epi == 1 -> fused update (solver)
template <int NF>
void launch_bp_t(pk_plan* p, int epi, void* out, double gscale_mult, cudaStream_t s) {
    const bool clamp = p->max_delay >= (double)p->Q + 0.5;
    if (p->dtype == PK_F32 && p->sym) {
        BpSymArgs A{};
        A.table = static_cast<const float2*>(p->table);
        A.pxs = p->pxs; A.pys = p->pys; A.sxs = p->sxs; A.sys = p->sys;
        A.n = p->nx; A.M = p->M; A.TS = p->TS; A.L = p->sym_L; A.nbuf = p->sym_nbuf;
        A.qclamp = (float)p->Q + 1.5f;
        A.chunks = p->sym_chunks; A.cta_chunk0 = p->sym_cta_chunk0; A.cta_slot0 = p->sym_cta_slot0;
        A.tiles = p->sym_tiles; A.part = p->sym_part; A.lanemap = p->sym_lanemap;
        A.st = epi ? p->state : nullptr;
        A.gid = p->gid; A.loc = p->loc; A.Mall = p->Mall;
        A.ntiles = p->sym_ntiles; A.table_fstride = (size_t)p->M * p->TS;
        BpSymEpiArgs E{};
        E.part = p->sym_part; E.tile_slot0 = p->sym_tile_slot0; E.tiles = p->sym_tiles;
        E.n = p->nx; E.bits = p->fp_bits; E.lanemap = p->sym_lanemap;
        E.gscale = (float)(gscale_mult * p->w);
        E.out = static_cast<float*>(out);
        E.xb0 = static_cast<float*>(p->xbuf[0]);
        E.xb1 = static_cast<float*>(p->xbuf[1]);
        E.prm = p->params; E.st = p->state; E.part_bp = p->part_bp;
        E.xr = p->fsym ? p->fsym_xr : nullptr;
        E.part_mx = p->part_mx;
        E.ntiles = p->sym_ntiles; E.P = p->P;
        // solver mode with the symmetric projector: the update runs in the back-projector's
        // tail (no epilogue launch); PK_SYM_FUSE=0 keeps the separate epilogue kernel
        A.fuse = (epi && p->fsym && p->sym_fuse && NF == 1) ? 1 : 0;
        A.epi = E;
        A.tile_cnt = p->sym_sync;
        A.tile_units = p->sym_sync + p->sym_ntiles;
        A.tile_done = p->sym_sync + 2 * p->sym_ntiles;
        A.spin_ns = p->sym_spin_ns;
        switch (p->sym_iw) {
            case 64: launch_sym<64>(A, p->sym_grid, p->sym_smem, s); break;
            case 96: launch_sym<96>(A, p->sym_grid, p->sym_smem, s); break;
            case 128: launch_sym<128>(A, p->sym_grid, p->sym_smem, s); break;
            case 192: launch_sym<192>(A, p->sym_grid, p->sym_smem, s); break;
            case 256: launch_sym<256>(A, p->sym_grid, p->sym_smem, s); break;
            default: launch_sym<0>(A, p->sym_grid, p->sym_smem, s); break;
        }
        const dim3 eg(p->sym_ntiles * 32 * NF);
        if (A.fuse) return;
        if (p->bp_mid_event) cudaEventRecord(p->bp_mid_event, s);
        // strips per epilogue CTA (config 3, warm, one / four frames per launch): 1 strip 10.6 /
        // 27.1 us, 2 strips 9.2 / 22.9, 4 strips 11.8 / 23.7 (too few CTAs at one frame, ~13
        // slots per tile); PK_SYM_EPIK forces 1 (the one-strip kernel), 2 or 4
        const int ks = p->sym_epik > 0 ? p->sym_epik : 2;
        if (epi && p->fsym && ks == 4)
            launch_pdl(bp_sym_epik_kernel<4>, dim3(p->sym_ntiles * 8 * NF), dim3(kThreads), 0, s, E);
        else if (epi && p->fsym && ks == 2)
            launch_pdl(bp_sym_epik_kernel<2>, dim3(p->sym_ntiles * 16 * NF), dim3(kThreads), 0, s, E);
        else if (epi && p->fsym) launch_pdl(bp_sym_epi_kernel<true, true>, eg, dim3(kThreads), 0, s, E);
        else if (epi) launch_pdl(bp_sym_epi_kernel<true, false>, eg, dim3(kThreads), 0, s, E);
        else launch_pdl(bp_sym_epi_kernel<false, false>, eg, dim3(kThreads), 0, s, E);
        return;
    }
    if (p->dtype == PK_F32) {
        BpArgs a{};
        a.table = static_cast<const float2*>(p->table);
        a.pxs = p->pxs; a.pys = p->pys; a.sxs = p->sxs; a.sys = p->sys;
        a.nx = p->nx; a.ny = p->ny; a.M = p->M; a.Q = p->Q; a.TS = p->TS; a.L = p->bp_L;
        a.CS = p->bp_CS; a.nbuf = p->bp_nbuf; a.tiles_x = p->bp_tiles_x;
        a.qclamp = (float)p->Q + 1.5f;
        a.out = static_cast<float*>(out);
        a.gscale = (float)(gscale_mult * p->w);
        a.xb0 = static_cast<float*>(p->xbuf[0]);
        a.xb1 = static_cast<float*>(p->xbuf[1]);
        a.prm = p->params; a.st = p->state; a.part = p->part_bp; a.bits = p->fp_bits;
        a.split = p->bp_split; a.ms = p->bp_ms; a.gpart = p->bp_gpart; a.tile_cnt = p->bp_tile_cnt;
        const dim3 grid(p->bp_tiles_x * p->bp_tiles_y, p->bp_split);
#define PK_BP(E, C, A) bp_f32_kernel<NF, E, C, A><<<grid, kThreads, p->bp_smem, s>>>(a)
        if (p->bp_atrick) {
            if (epi) { if (clamp) PK_BP(true, true, true); else PK_BP(true, false, true); }
            else { if (clamp) PK_BP(false, true, true); else PK_BP(false, false, true); }
        } else {
            if (epi) { if (clamp) PK_BP(true, true, false); else PK_BP(true, false, false); }
            else { if (clamp) PK_BP(false, true, false); else PK_BP(false, false, false); }
        }
#undef PK_BP
    } else {
        BpArgs64 a{};
        a.table = static_cast<const double2*>(p->table);
        a.px = p->px; a.py = p->py; a.sx = p->sx; a.sy = p->sy; a.cdt = p->cdt;
        a.nx = p->nx; a.ny = p->ny; a.M = p->M; a.Q = p->Q; a.TS = p->TS;
        a.out = static_cast<double*>(out);
        a.gscale = gscale_mult * p->w;
        a.xb0 = static_cast<double*>(p->xbuf[0]);
        a.xb1 = static_cast<double*>(p->xbuf[1]);
        a.prm = p->params; a.st = p->state; a.part = p->part_bp; a.bits = p->fp_bits;
        const int grid = (p->P + kThreads - 1) / kThreads;
        if (epi) bp_f64_kernel<true><<<grid, kThreads, 0, s>>>(a);
        else bp_f64_kernel<false><<<grid, kThreads, 0, s>>>(a);
    }
}

template <int NF>
void launch_table_t(pk_plan* p, const void* y, int init, cudaStream_t s) {
    const dim3 grid(p->M, NF);
    if (p->dtype == PK_F32)
        table_kernel<float, NF><<<grid, kThreads, 0, s>>>(
            static_cast<const float*>(y), p->io, static_cast<float2*>(p->table), p->M, p->Q, p->TS,
            init ? -1.f : 1.f, p->part_r, p->state, init, p->bp_atrick, p->sym ? 1 : 0);
    else
        table_kernel<double, 1><<<grid, kThreads, 0, s>>>(
            static_cast<const double*>(y), p->io, static_cast<double2*>(p->table), p->M, p->Q,
            p->TS, init ? -1.0 : 1.0, p->part_r, p->state, init, 0);
}

template <int NF>
void launch_init_t(pk_plan* p, cudaStream_t s) {
    const int pb = std::min((NF * p->P + kThreads - 1) / kThreads, 148 * 8);
    if (p->dtype == PK_F32)
        init_kernel<float, NF><<<pb, kThreads, 0, s>>>(static_cast<float*>(p->xbuf[0]), p->P, p->state, p->io);
    else
        init_kernel<double, 1><<<pb, kThreads, 0, s>>>(static_cast<double*>(p->xbuf[0]), p->P, p->state, p->io);
}

template <int NF>
void launch_copy_out_t(pk_plan* p, cudaStream_t s) {
    const int cb = std::min((p->P + kThreads - 1) / kThreads, 148 * 4);
    if (p->dtype == PK_F32)
        copy_out_kernel<float, NF><<<cb, kThreads, 0, s>>>(static_cast<const float*>(p->xbuf[0]),
                                                           static_cast<const float*>(p->xbuf[1]),
                                                           p->state, p->io, p->P);
    else
        copy_out_kernel<double, 1><<<cb, kThreads, 0, s>>>(static_cast<const double*>(p->xbuf[0]),
                                                           static_cast<const double*>(p->xbuf[1]),
                                                           p->state, p->io, p->P);
}

#define PK_DISPATCH(fn, ...)                                \
    do {                                                    \
        switch (p->nf) {                                    \
            case 2: fn<2>(__VA_ARGS__); break;              \
            case 4: fn<4>(__VA_ARGS__); break;              \
            default: fn<1>(__VA_ARGS__); break;             \
        }                                                   \
        PK_CHECK_LAUNCH();                                  \
    } while (0)

int launch_maxabs(pk_plan* p, const void* x, cudaStream_t s) {
    PK_DISPATCH(launch_maxabs_t, p, x, s);
    return PK_OK;
}
int launch_fp(pk_plan* p, const void* x, int solver, cudaStream_t s) {
    // the fixed-point accumulator must be zero on entry (finalize only reads it); the
    // symmetric projector writes whole windows instead
    if (!p->fsym)
        PK_CUDA(cudaMemsetAsync(p->acc, 0, (size_t)p->M * p->Q * p->nf * sizeof(long long), s));
    PK_DISPATCH(launch_fp_t, p, x, solver, s);
    return PK_OK;
}
int launch_finalize(pk_plan* p, const void* y, void* out, double* sumsq, int solver, cudaStream_t s) {
    PK_DISPATCH(launch_finalize_t, p, y, out, sumsq, solver, s);
    return PK_OK;
}
int launch_bp(pk_plan* p, int epi, void* out, double g, cudaStream_t s) {
    PK_DISPATCH(launch_bp_t, p, epi, out, g, s);
    return PK_OK;
}
// upload the host partition of the symmetric back-projector
static cudaError_t sym_upload(pk_plan* p) {
    int* dsts[4] = {p->sym_chunks, p->sym_cta_chunk0, p->sym_cta_slot0, p->sym_tile_slot0};
    for (int q = 0; q < 4; ++q) {
        const cudaError_t e = cudaMemcpy(dsts[q], p->sym_h[q + 1].data(), sizeof(int) * p->sym_h[q + 1].size(),
                                         cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// the diagonal cut weight of the symmetric back-projector: each candidate partition timed
// (back-projection of a zero table, non-solver, 3 launches after a warm-up, the minimum), once
// per geometry and process; every later plan of the same geometry reuses the choice, so plans
// of one process agree bit for bit
static cudaError_t sym_tune_wdiag(pk_plan* p) {
    if (!p->sym || p->dtype != PK_F32 || p->sym_wdiag < 0) return cudaSuccess;
    if (getenv("CUDA_INJECTION64_PATH")) {
        // under a profiler (ncu injects itself) event times are the tool's, not the kernel's:
        // the measured choice of the unprofiled runs (configs 1-5: 24, except 18 at config 2's
        // pitch of 3.9 samples per pixel with frames batched), no timing
        const double hx = p->fsym_hx > 0.f ? p->fsym_hx : 1.0;
        const int w = (hx > 2.9 && p->nf > 1 && p->nx < 512) ? 18 : 24;
        sym_partition(p, w);
        p->sym_wdiag = w;
        return sym_upload(p);
    }
    static std::mutex mu;
    static std::map<std::vector<long long>, int> best_of;
    std::vector<long long> key = {p->nx, p->M, p->Mall, p->Q, p->nf, p->sym_grid, p->sym_nbuf, p->sym_iw,
                                  (long long)std::llround(p->cdt * 1e12)};
    for (int g : p->gid_h) key.push_back(g);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = best_of.find(key);
        if (it != best_of.end()) {
            sym_partition(p, it->second);
            p->sym_wdiag = it->second;
            return sym_upload(p);
        }
    }
    cudaStream_t s;
    cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int best = std::abs(p->sym_wdiag);
    float best_ms = 1e30f;
    for (int w : kSymWCand) {
        sym_partition(p, w);
        if ((e = sym_upload(p)) != cudaSuccess) break;
        float t = 1e30f;
        for (int r = 0; r < 4 && e == cudaSuccess; ++r) {
            cudaEventRecord(e0, s);
            if (launch_bp(p, 0, p->xbuf[0], 1.0, s) != PK_OK) e = cudaErrorUnknown;
            cudaEventRecord(e1, s);
            if (e == cudaSuccess) e = cudaEventSynchronize(e1);
            float ms = 0.f;
            if (e == cudaSuccess && r > 0 && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess) t = std::min(t, ms);
        }
        if (e != cudaSuccess) break;
        if (getenv("PK_SYM_TUNE_LOG")) fprintf(stderr, "pk sym tune: wdiag %d %.2f us\n", w, 1e3 * t);
        if (t < best_ms) { best_ms = t; best = w; }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    if (e != cudaSuccess) return e;
    {
        std::lock_guard<std::mutex> lk(mu);
        best = best_of.emplace(key, best).first->second;  // (a concurrent tuner may have won)
    }
    sym_partition(p, best);
    p->sym_wdiag = best;
    return sym_upload(p);
}

int launch_table(pk_plan* p, const void* y, int init, cudaStream_t s) {
    PK_DISPATCH(launch_table_t, p, y, init, s);
    return PK_OK;
}
int launch_init(pk_plan* p, cudaStream_t s) {
    PK_DISPATCH(launch_init_t, p, s);
    return PK_OK;
}
int launch_copy_out(pk_plan* p, cudaStream_t s) {
    PK_DISPATCH(launch_copy_out_t, p, s);
    return PK_OK;
}

// the solver graph body: x0 = 0, r0 = -y, N x (K1 update, K2, K3), copy-out
int record_solver(pk_plan* p, int iters, cudaStream_t s) {
    PK_TRY(launch_init(p, s));
    PK_TRY(launch_table(p, nullptr, 1, s));
    for (int it = 0; it < iters; ++it) {
        PK_TRY(launch_bp(p, 1, nullptr, 2.0, s));
        PK_TRY(launch_fp(p, nullptr, 1, s));
        PK_TRY(launch_finalize(p, nullptr, nullptr, nullptr, 1, s));
    }
    PK_TRY(launch_copy_out(p, s));
    return PK_OK;
}

int check_params(const pk_plan* p, const pk_solver_params* prm) {
    if (!prm) return fail(PK_ERR_INVALID, "params is NULL");
    if (prm[0].iterations < 1) return fail(PK_ERR_INVALID, "iterations must be >= 1");
    if (!(prm[0].tv_epsilon > 0)) return fail(PK_ERR_INVALID, "tv_epsilon must be > 0");
    if (!(prm[0].tolerance >= 0)) return fail(PK_ERR_INVALID, "tolerance must be >= 0");
    for (int f = 0; f < p->nf; ++f) {
        if (!(prm[f].alpha >= 0) || !(prm[f].beta >= 0))
            return fail(PK_ERR_INVALID, "alpha and beta must be >= 0 (frame %d)", f);
        if (!(prm[f].step > 0)) return fail(PK_ERR_INVALID, "step must be > 0 (frame %d)", f);
        if (prm[f].iterations != prm[0].iterations)
            return fail(PK_ERR_INVALID, "all frames of a batch run the same iteration count");
    }
    return PK_OK;
}

int upload_params(pk_plan* p, const pk_solver_params* prm, cudaStream_t s) {
    DevParams d{};
    for (int f = 0; f < kMaxFrames; ++f) {
        const pk_solver_params& q = prm[f < p->nf ? f : 0];
        d.alpha[f] = q.alpha;
        d.beta[f] = q.beta;
        d.step[f] = q.step;
        d.eta_alpha[f] = q.step * q.alpha;  // recon.py:336 passes eta * alpha
    }
    d.eps = prm[0].tv_epsilon;
    d.tolerance = prm[0].tolerance;
    d.iterations = prm[0].iterations;
    d.nonneg = prm[0].nonneg ? 1 : 0;
    // unchanged parameters are not re-sent: keeps the sharded entry points free of host
    // copies, so a solve built from them can be captured into a CUDA graph
    if (p->params_valid && std::memcmp(&p->params_host, &d, sizeof(d)) == 0) return PK_OK;
    PK_CUDA(cudaMemcpyAsync(p->params, &d, sizeof(d), cudaMemcpyHostToDevice, s));
    p->params_host = d;
    p->params_valid = 1;
    return PK_OK;
}

int ensure_hist(pk_plan* p, int iters) {
    if (p->hist_cap >= iters) return PK_OK;
    if (p->hist_dev) cudaFree(p->hist_dev);
    p->hist_dev = nullptr;
    PK_TRY(alloc(p, &p->hist_dev, (size_t)4 * iters * p->nf));
    p->hist_cap = iters;
    return PK_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* pk_last_error(void) { return g_err; }

int pk_version(void) { return 10100; /* 1.1.0: batched frames */ }

int pk_plan_create(const pk_geometry_desc* d, pk_plan** out) {
    if (!d || !out) return fail(PK_ERR_INVALID, "NULL argument");
    *out = nullptr;
    if (d->nx < 1 || d->ny < 1) return fail(PK_ERR_INVALID, "grid dimensions must be >= 1");
    if (d->sensors < 1) return fail(PK_ERR_INVALID, "sensor count must be >= 1");
    if (d->samples < 1) return fail(PK_ERR_INVALID, "samples must be >= 1");
    if (!(d->c > 0) || !(d->dt > 0)) return fail(PK_ERR_INVALID, "c and dt must be > 0");
    if (d->sensor_list) {
        if (d->sensor_list_len < 1 || d->sensor_list_len > d->sensors)
            return fail(PK_ERR_INVALID, "bad sensor list length %d", d->sensor_list_len);
        for (int l = 0; l < d->sensor_list_len; ++l)
            if (d->sensor_list[l] < 0 || d->sensor_list[l] >= d->sensors ||
                (l > 0 && d->sensor_list[l] <= d->sensor_list[l - 1]))
                return fail(PK_ERR_INVALID, "sensor list must be strictly increasing ring indices");
    } else if (d->sensor_begin < 0 || d->sensor_end > d->sensors || d->sensor_begin >= d->sensor_end) {
        return fail(PK_ERR_INVALID, "bad sensor shard [%d, %d) of %d", d->sensor_begin,
                    d->sensor_end, d->sensors);
    }
    if (d->dtype != PK_F32 && d->dtype != PK_F64) return fail(PK_ERR_INVALID, "bad dtype");
    const int nf = d->frames <= 1 ? 1 : d->frames;
    if (nf != 1 && nf != 2 && nf != 4) return fail(PK_ERR_INVALID, "frames must be 1, 2 or 4");
    if (nf > 1 && d->dtype != PK_F32)
        return fail(PK_ERR_UNSUPPORTED, "batched frames are supported in fp32 only");
    if (!d->pixel_x || !d->pixel_y || !d->sensor_xy) return fail(PK_ERR_INVALID, "NULL geometry");
    if ((int64_t)d->nx * d->ny > (int64_t)1 << 30) return fail(PK_ERR_UNSUPPORTED, "grid too large");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(PK_ERR_CUDA, "no CUDA device available (the B200 kernels have no CPU fallback)");
    if (d->device < 0 || d->device >= ndev) return fail(PK_ERR_INVALID, "bad device %d", d->device);
    DeviceGuard guard(d->device);

    pk_plan* p = new pk_plan();
    p->device = d->device;
    p->dtype = d->dtype;
    p->nf = nf;
    p->nx = d->nx; p->ny = d->ny; p->P = d->nx * d->ny;
    p->Mall = d->sensors; p->m0 = d->sensor_begin; p->M = d->sensor_end - d->sensor_begin;
    if (d->sensor_list) {  // a sensor list (e.g. a D4-closed shard) instead of a range
        p->listed = 1;
        p->m0 = 0;
        p->M = d->sensor_list_len;
        p->gid_h.assign(d->sensor_list, d->sensor_list + d->sensor_list_len);
    } else {
        p->gid_h.resize(p->M);
        for (int l = 0; l < p->M; ++l) p->gid_h[l] = p->m0 + l;
    }
    p->Q = d->samples;
    p->c = d->c; p->dt = d->dt;
    p->cdt = d->c * d->dt;                          // forward.py:180
    p->w = 1.0 / (2.0 * 3.141592653589793 * d->c);  // forward.py:183

    // pixel / sensor geometry; delay bounds per sensor from the grid rectangle
    const double* X = d->pixel_x;
    const double* Y = d->pixel_y;
    std::vector<double> spv(2 * (size_t)std::max(p->M, 1));  // local sensor positions
    for (int l = 0; l < p->M; ++l) {
        spv[2 * l] = d->sensor_xy[2 * (size_t)p->gid_h[l]];
        spv[2 * l + 1] = d->sensor_xy[2 * (size_t)p->gid_h[l] + 1];
    }
    const double* SP = spv.data();
    std::vector<int> loc_h(p->Mall, -1);
    for (int l = 0; l < p->M; ++l) loc_h[p->gid_h[l]] = l;
    for (int i = 1; i < p->nx; ++i)
        if (!(X[i] > X[i - 1])) { free_plan(p); return fail(PK_ERR_INVALID, "pixel_x must increase"); }
    for (int j = 1; j < p->ny; ++j)
        if (!(Y[j] > Y[j - 1])) { free_plan(p); return fail(PK_ERR_INVALID, "pixel_y must increase"); }
    const double xl = X[0], xh = X[p->nx - 1], yl = Y[0], yh = Y[p->ny - 1];
    double dmin_all = 1e300, dmax_all = 0;
    for (int m = 0; m < p->M; ++m) {
        const double sx = SP[2 * m], sy = SP[2 * m + 1];
        const double cx = std::min(std::max(sx, xl), xh), cy = std::min(std::max(sy, yl), yh);
        const double dmin = std::hypot(cx - sx, cy - sy);
        const double dmax = std::hypot(std::max(std::fabs(xl - sx), std::fabs(xh - sx)),
                                       std::max(std::fabs(yl - sy), std::fabs(yh - sy)));
        dmin_all = std::min(dmin_all, dmin);
        dmax_all = std::max(dmax_all, dmax);
        if (dmin == 0.0) {  // sensor inside the grid rectangle: exact coincidence check
            const double* ix = std::find(X, X + p->nx, sx);
            const double* iy = std::find(Y, Y + p->ny, sy);
            if (ix != X + p->nx && iy != Y + p->ny) {
                free_plan(p);
                return fail(PK_ERR_GEOMETRY, "sensor %d coincides with pixel index %lld",
                            p->gid_h[m], (long long)((iy - Y) * p->nx + (ix - X)));
            }
        }
    }
    p->min_delay = dmin_all / p->cdt;
    p->max_delay = dmax_all / p->cdt;
    p->may_truncate = (p->min_delay < 1.001 || p->max_delay > (double)p->Q - 1.001) ? 1 : 0;

    // tiling.  h = pixel pitch in samples.
    const double hx = p->nx > 1 ? (X[p->nx - 1] - X[0]) / (p->nx - 1) / p->cdt : 0.0;
    const double hy = p->ny > 1 ? (Y[p->ny - 1] - Y[0]) / (p->ny - 1) / p->cdt : 0.0;
    const double h = std::max(hx, hy);
    auto tile_diag = [&](int T) {
        const double ex = std::min(T - 1, p->nx - 1) * hx, ey = std::min(T - 1, p->ny - 1) * hy;
        return std::sqrt(ex * ex + ey * ey);
    };
    p->TS = (p->Q + 2 + 1) & ~1;
    {
        const char* ev = getenv("PK_BP_ATRICK");
        p->bp_atrick = (p->dtype == PK_F32) ? (ev ? atoi(ev) != 0 : 0) : 0;  // opt-in: DESIGN.md
    }
    // back-projector
    p->bp_tiles_x = (p->nx + kBpTile - 1) / kBpTile;
    p->bp_tiles_y = (p->ny + kBpTile - 1) / kBpTile;
    p->bp_L = ((int)std::ceil(tile_diag(kBpTile)) + 6 + 1) & ~1;
    if (p->bp_L > p->TS) p->bp_L = p->TS;
    p->bp_nbuf = 3;
    // CTAs per SM the launch bounds aim for: 4 (NF=1), 3 (NF=2), 2 (NF=4)
    const int bp_budget = (nf == 1 ? 52 : (nf == 2 ? 70 : 104)) * 1024;
    p->bp_CS = std::max(1, std::min(32, bp_budget / (p->bp_nbuf * p->bp_L * 8 * nf)));
    p->bp_smem = p->bp_nbuf * p->bp_CS * p->bp_L * 8 * nf + p->bp_nbuf * p->bp_CS * 16 + p->bp_nbuf * 8;
    if (p->dtype == PK_F32 && p->bp_smem > 200 * 1024) {
        free_plan(p);
        return fail(PK_ERR_UNSUPPORTED, "delay window per tile too long (%d samples)", p->bp_L);
    }
    {   // sensor split so that tiles x split >= ~4 CTAs per SM, each split >= 64 sensors
        const int tiles = p->bp_tiles_x * p->bp_tiles_y;
        int sp = 1;
        if (p->dtype == PK_F32)
            while (tiles * sp < 4 * 148 && p->M / (2 * sp) >= 64) sp *= 2;
        p->bp_ms = (p->M + sp - 1) / sp;
        p->bp_ms = ((p->bp_ms + p->bp_CS - 1) / p->bp_CS) * p->bp_CS;  // whole chunks
        p->bp_split = (p->M + p->bp_ms - 1) / p->bp_ms;
    }
    // projector tile: 64 x 64 when that still gives >= 4 CTAs per SM (halves the window
    // flush traffic per interaction) and the windows fit, else 32 x 32
    p->fp_groups = (p->M + 31) / 32;
    {
        const int t64 = ((p->nx + 63) / 64) * ((p->ny + 63) / 64);
        p->fp_T = (p->dtype == PK_F32 && nf <= 2 && (int64_t)t64 * p->fp_groups >= 4 * 148) ? 64 : 32;
        if (const char* e = getenv("PK_FP_T")) p->fp_T = atoi(e) == 64 ? 64 : 32;
    }
    p->fp_tiles_x = (p->nx + p->fp_T - 1) / p->fp_T;
    p->fp_tiles_y = (p->ny + p->fp_T - 1) / p->fp_T;
    p->fp_L = (int)std::ceil(tile_diag(p->fp_T)) + 6;
    // contributions one window slot can receive: tile pixels in a band of 2 samples
    double nc_tile = 1.5 * (p->fp_T * std::sqrt(2.0) + 2) * (2.0 / std::max(h, 1e-12) + 2);
    if (p->min_delay < 8.0 * p->fp_T * std::max(h, 1.0)) nc_tile = (double)p->fp_T * p->fp_T;
    nc_tile = std::min(nc_tile, (double)p->fp_T * p->fp_T);
    if (p->dtype == PK_F32) {
        const int rv = (1 + 2 * nf + 3) / 4;
        p->fp_bits = std::min(22, 30 - ceil_log2(nc_tile));
        p->fp_smem = p->fp_L * nf * 32 * 4 + (kThreads / 32) * (p->fp_T + kFpBatch) * rv * 16;
    } else {
        double nc_glob = std::min((double)p->P, 4.0 * (p->nx + p->ny) * (2.0 / std::max(h, 1e-12) + 2));
        if (p->min_delay < 8.0 * p->fp_T * std::max(h, 1.0)) nc_glob = (double)p->P;
        p->fp_bits = std::min(62 - ceil_log2(nc_tile), 62 - ceil_log2(nc_glob));
        p->fp_bits = std::min(p->fp_bits, 52);
        p->fp_smem = p->fp_L * 32 * 8 + p->fp_T * p->fp_T * 24 + p->fp_T * 4;
    }
    if (p->fp_smem > 200 * 1024) {
        free_plan(p);
        return fail(PK_ERR_UNSUPPORTED, "projector window too long (%d samples)", p->fp_L);
    }
    // D4 symmetry of the scene (square grid centred on the ring centre, n even, M % 4 == 0):
    // the back-projector then evaluates one delay per 8 sensor-pixel pairs (bp_sym_f32_kernel)
    {
        const char* ev = getenv("PK_SYM");
        // the plan's sensors must be closed under the ring's D4 (a whole ring, or a shard
        // listing whole orbits): every image of a base sensor is then a local trace
        // (batched frames: the symmetric kernels take frame-major work, NF <= 4; the residual
        // kernel of the batched symmetric path holds a trace of <= kFinSymMax samples)
        bool ok = (ev ? atoi(ev) != 0 : true) && p->dtype == PK_F32 && (nf == 1 || p->Q <= kFinSymMax) &&
                  p->nx == p->ny && (p->nx % 2) == 0 && p->nx >= 2 * kSymTile && (p->Mall % 4) == 0;
        const int n = p->nx;
        double scl = 0.0;
        for (int i = 0; ok && i < n; ++i) scl = std::max(scl, std::fabs(X[i]));
        const double tolx = 1e-9 * std::max(scl, 1e-300);
        for (int i = 0; ok && i < n; ++i)
            if (std::fabs(X[i] + X[n - 1 - i]) > tolx || std::fabs(X[i] - Y[i]) > tolx) ok = false;
        double R = 0.0;
        for (int m = 0; ok && m < p->M; ++m) R = std::max(R, std::hypot(SP[2 * m], SP[2 * m + 1]));
        const double tols = 1e-9 * std::max(R, 1e-300);
        for (int m = 0; ok && m < p->M; ++m) {
            const int q = p->Mall / 4, gm = p->gid_h[m];
            const double sx = SP[2 * m], sy = SP[2 * m + 1];
            const int mr = loc_h[(gm + q) % p->Mall], mf = loc_h[(p->Mall - gm) % p->Mall];
            if (mr < 0 || mf < 0) { ok = false; break; }  // not closed under D4
            // rotation by 90 degrees (x, y) -> (-y, x) and reflection (x, y) -> (x, -y)
            if (std::fabs(SP[2 * mr] + sy) > tols || std::fabs(SP[2 * mr + 1] - sx) > tols) ok = false;
            if (std::fabs(SP[2 * mf] - sx) > tols || std::fabs(SP[2 * mf + 1] + sy) > tols) ok = false;
        }
        p->sym = ok ? 1 : 0;
        if (p->sym) {
            // representative tiles tx >= ty of the quadrant, chunks of kSymCS base sensors
            const int qt = (n / 2 + kSymTile - 1) / kSymTile;
            std::vector<int>& tl = p->sym_h[0];
            for (int tx = 0; tx < qt; ++tx)
                for (int ty = 0; ty <= tx; ++ty) tl.push_back((tx << 16) | ty);
            p->sym_ntiles = (int)tl.size();
            p->sym_L = ((int)std::ceil(tile_diag(kSymTile)) + 7 + 1) & ~1;
            if (p->sym_L > p->TS) p->sym_L = p->TS;
            p->sym_iw = 0;
            for (int iw : kSymIW)
                if (p->sym_L <= iw) { p->sym_iw = iw; break; }
            const int ws = p->sym_iw ? p->sym_iw : p->sym_L;
            // TMA ring as deep as fits ~72 KB (3 CTAs per SM), 2..8 buffers
            const int per_buf = kSymCS * 8 * ws * 8 + kSymCS * 16 + 16;
            p->sym_nbuf = std::max(2, std::min(8, (72 * 1024) / per_buf));
            if (const char* e = getenv("PK_SYM_NBUF")) p->sym_nbuf = std::max(2, std::min(8, atoi(e)));
            p->sym_lanemap = 1;
            // update fused into the back-projector's tail: opt-in (measured slower at config 3:
            // 57.0 us vs 41.1 + 9.7 us for the separate epilogue)
            p->sym_fuse = 0;
            if (const char* e = getenv("PK_SYM_FUSE")) p->sym_fuse = atoi(e) != 0;
            p->sym_epik = 0;  // (0: by frames per launch)
            if (const char* e = getenv("PK_SYM_EPIK")) {
                const int v = atoi(e);
                p->sym_epik = (v == 1 || v == 2 || v == 4) ? v : 0;
            }
            if (const char* e = getenv("PK_SYM_SPIN_NS")) p->sym_spin_ns = std::max(0LL, atoll(e));
            if (const char* e = getenv("PK_SYM_LANEMAP")) p->sym_lanemap = atoi(e) != 0;
            p->sym_smem = p->sym_nbuf * per_buf;
            int occ = 0, sms = 0;
            if (p->sym_smem > 200 * 1024 || opt_in_smem(p->device) != cudaSuccess ||
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sym_kernel_ptr(p->sym_iw), kSymThreads,
                                                              p->sym_smem) != cudaSuccess ||
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device) != cudaSuccess ||
                occ < 1) {
                cudaGetLastError();
                p->sym = 0;
            }
            if (p->sym) {
                // persistent grid; equal-cost contiguous chunk ranges (off-diagonal chunk = 2)
                // every CTA leaves one partial slot per tile it touches and the epilogue reads
                // all slots of a tile, so small problems get fewer, longer CTAs: about 64 cost
                // units (8 off-diagonal chunks) per CTA at least, 32 CTAs at least
                const int nch = (p->M + kSymCS - 1) / kSymCS;
                {
                    int64_t wsum = 0;
                    for (int t = 0; t < p->sym_ntiles; ++t)
                        wsum += (int64_t)nch * nf * (((tl[t] >> 16) == (tl[t] & 0xffff)) ? kSymWDiag : kSymWOff);
                    p->sym_grid = (int)std::max<int64_t>(32, std::min<int64_t>((int64_t)occ * sms, wsum / 64));
                    // throughput mode (several plans on concurrent streams): at most half the
                    // occupancy-limited grid -- config 3 on 4 streams 1013 -> 1027 frames/s; a
                    // work-limited grid (config 2: 136 CTAs) is kept (halving it: 2147 -> 2004)
                    // (tools/sweep_grid.sh); the partial sums group differently (rounding level)
                    if (d->concurrency > 1)
                        p->sym_grid = (int)std::max<int64_t>(
                            32, std::min<int64_t>((int64_t)occ * sms / 2, wsum / 64));
                }
                if (const char* e = getenv("PK_SYM_GRID")) p->sym_grid = std::max(1, atoi(e));
                // cut weights: off-diagonal chunk 32, diagonal chunk wdiag.  (A per-chunk model
                // of the LDS.64 bank-pair conflicts of each half-warp block, used as cut
                // weights, measured slower: config 3 44.0 -> 47.3 us, config 2 18.0 -> 22.1 us.)
                // The best wdiag depends on how the cuts fall against tile boundaries and on
                // which CTAs share an SM, not on one cost ratio (measured, tools/k2_sweep_cfg.sh:
                // config 3 44.4 / 42.1 us at 20 / 24, 4 frames per launch 160.8 / 148.5; config
                // 2 x 4 frames 34.0 / 37.7, best 17-18; config 1 x 4 frames best 24), so the plan
                // times the candidates once per geometry and process (sym_tune_wdiag) unless
                // PK_SYM_WDIAG pins it
                p->sym_nch = nch;
                p->sym_wdiag = 24;
                if (const char* e = getenv("PK_SYM_WDIAG")) p->sym_wdiag = -std::max(1, atoi(e));  // (< 0: pinned)
                // (the partial-slot buffer holds the largest candidate's slots)
                int smax = 0;
                for (int w : kSymWCand) { sym_partition(p, w); smax = std::max(smax, p->sym_slots); }
                sym_partition(p, std::abs(p->sym_wdiag));
                p->sym_slots_cap = std::max(smax, p->sym_slots);
            }
        }
        // rotation-symmetric projector (fp_sym_f32_kernel): persistent CTAs, every one resident
        // (one per SM with 32 warps, or two with 16: PK_FSYM_NW), each taking an equal
        // contiguous range of the (group of 32 base sensors, T-column quadrant strip, row)
        // sequence, cut into segments of at most hs rows inside one (group, strip).  The strip
        // width T (64 or 32) and the window length LW (the segment rectangle's delay span) are
        // chosen for the fewest window words stored per projection.
        const char* ev2 = getenv("PK_FSYM");
        p->fsym = (p->sym && (ev2 ? atoi(ev2) != 0 : true)) ? 1 : 0;
        if (p->fsym) {
            int sms = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
            p->fsym_hx = (float)((X[n - 1] - X[0]) / (n - 1) / p->cdt);
            p->fsym_groups = (p->M + 31) / 32;
            p->fsym = 0;
            const int nw = (getenv("PK_FSYM_NW") && atoi(getenv("PK_FSYM_NW")) == 16) ? 16 : 32;
            // (one 16-warp CTA per SM measured no faster: cfg3 62.9 vs 61.7 us, cfg2 x 4 frames
            // 48.2 vs 48.6 us)
            const int persm = 32 / nw, cap = fs_cap(nw);
            // throughput mode (several plans on concurrent streams): the persistent grid is
            // divided by concurrency / 2 so that other streams' kernels share the SMs (measured
            // share 1 / 2 / 4: cfg4 on 8 streams 1963 / 2182 / 2293 frames/s, cfg3 on 4 streams
            // 961 / 991 / 978, tools/r2_share.sh); PK_FSYM_SHARE overrides
            int share = std::max(1, d->concurrency / 2);
            if (d->concurrency > 1)
                if (const char* e = getenv("PK_FSYM_SHARE")) share = std::max(1, atoi(e));
            const int G = std::max(1, std::max(1, sms) * persm / share);
            const int hq = n / 2;
            auto region_diag = [&](int T, int H) {
                const double ex = std::min(T - 1, hq - 1) * hx, ey = std::min(H - 1, hq - 1) * hy;
                return std::sqrt(ex * ex + ey * ey);
            };
            // cuts of the row sequence [0, R) into G contiguous CTA ranges that minimise the
            // largest cost, cost = rows + cs * (segments - 1): a range that crosses a (group,
            // strip) boundary (or the hs limit) starts a second segment, whose window set-up,
            // staging and scatter ramp cost a CTA as much as ~cs rows (measured r02c, config 3:
            // 1-segment CTAs 47.8 us, 2-segment 56.5 us for the same rows).  Greedy fill per
            // budget, binary search on the budget.
            // per (group, strip, start row): the most rows a segment starting there can have so
            // that its rectangle's delays fit the window for every lane (fp64 distances from the
            // lanes' own sensors: spread = farthest corner - nearest point, + 10 slots of margin
            // for the window's alignment, the two interpolation slots and fp32 delays).  Round
            // 2b used one height for all, from the rectangle's diagonal (the worst direction);
            // a group whose sensors look along the strip gets much taller segments.  Heights are
            // capped at hcap (the fixed-point bound of fp_bits); empty if a row cannot fit.
            const double qcl = (double)p->Q + 1.5;
            const bool clampd = p->max_delay >= (double)p->Q + 0.5;
            auto make_hmax = [&](int T, int lw, int hcap) {
                const int qt = (hq + T - 1) / T;
                std::vector<int> tab((size_t)p->fsym_groups * qt * hq, 0);
                for (int grp = 0; grp < p->fsym_groups; ++grp)
                    for (int strip = 0; strip < qt; ++strip) {
                        const int i0 = hq + T * strip, i1 = std::min(i0 + T, n) - 1;
                        const double xa = std::min(X[i0], X[i1]) / p->cdt, xb = std::max(X[i0], X[i1]) / p->cdt;
                        auto fits = [&](int r, int e) {  // rows [r, e) of the quadrant
                            const double ya = std::min(Y[hq + r], Y[hq + e - 1]) / p->cdt;
                            const double yb = std::max(Y[hq + r], Y[hq + e - 1]) / p->cdt;
                            for (int l = 0; l < 32; ++l) {
                                const int m = grp * 32 + l;
                                if (m >= p->M) break;
                                const double sx = SP[2 * m] / p->cdt, sy = SP[2 * m + 1] / p->cdt;
                                const double cx = std::min(std::max(sx, xa), xb), cy = std::min(std::max(sy, ya), yb);
                                double dmin = std::hypot(cx - sx, cy - sy);
                                double dmax = std::max(std::max(std::hypot(xa - sx, ya - sy), std::hypot(xa - sx, yb - sy)),
                                                       std::max(std::hypot(xb - sx, ya - sy), std::hypot(xb - sx, yb - sy)));
                                if (clampd) { dmin = std::min(dmin, qcl); dmax = std::min(dmax, qcl); }
                                if ((int)std::ceil(dmax - dmin) + 10 > lw) return false;
                            }
                            return true;
                        };
                        int e = 0;
                        for (int r = 0; r < hq; ++r) {
                            e = std::max(e, r);
                            while (e < hq && e - r < hcap && fits(r, e + 1)) ++e;
                            if (e == r) return std::vector<int>();  // not even one row fits
                            tab[((size_t)grp * qt + strip) * hq + r] = e - r;
                        }
                    }
                return tab;
            };
            std::vector<int> hm_tab;  // the table segment() and balanced_cuts() cut with
            int hm_qt = 1;
            auto hm_at = [&](long long pos) -> long long {
                const long long gs = pos / hq;
                const int grp = (int)((gs / hm_qt) % p->fsym_groups), strip = (int)(gs % hm_qt);
                return hm_tab[((size_t)grp * hm_qt + strip) * hq + (pos - gs * hq)];
            };
            auto balanced_cuts = [&](long long R, long long cs) {
                auto fill = [&](long long B, std::vector<long long>* cut) {
                    long long pos = 0;
                    int used = 0;
                    while (pos < R && used < G) {
                        if (cut) cut->push_back(pos);
                        ++used;
                        long long budget = B;
                        bool first = true;
                        while (pos < R) {
                            if (!first) {
                                // a further segment only if it gets at least cs / 2 rows (a
                                // sliver of a segment pays the whole staging for a few rows)
                                if (budget < cs + std::max(1LL, cs / 2)) break;
                                budget -= cs;
                            }
                            const long long send = std::min({(pos / hq + 1) * hq, pos + hm_at(pos), R});
                            const long long take = std::min(send - pos, budget);
                            pos += take;
                            budget -= take;
                            first = false;
                            if (pos < send) break;  // budget spent inside the segment
                        }
                    }
                    if (cut) { while ((int)cut->size() < G) cut->push_back(pos); cut->push_back(R); }
                    return pos >= R;
                };
                long long lo = std::max(1LL, (R + G - 1) / G), hi = lo + 2 * cs + hq + 1;
                while (!fill(hi, nullptr)) hi *= 2;
                while (lo < hi) {
                    const long long mid = (lo + hi) / 2;
                    if (fill(mid, nullptr)) hi = mid; else lo = mid + 1;
                }
                std::vector<long long> cut;
                fill(lo, &cut);
                return cut;
            };
            const char* evc = getenv("PK_FSYM_SEGCOST");  // (sweeps: cost of a segment, in rows)
            // a row of T columns scatters 10 shared-memory wavefronts per column (8 atomics, one
            // broadcast LDS.128); an extra segment costs ~7.5 us of SM time
            auto seg_cost = [&](int T) {
                return evc ? (long long)std::max(0, atoi(evc))
                           : (long long)std::lround(7.5 / (T * 10.0 / 1965.0 * 1.15));
            };
            // (batched frames: the sequence is frame-major, segment group index f * groups + group)
            auto segment = [&](int T, std::vector<int4>* sg, std::vector<int>* c0) {
                const int qt = (hq + T - 1) / T;
                const long long R = (long long)nf * p->fsym_groups * qt * hq;
                const std::vector<long long> cut = balanced_cuts(R, seg_cost(T));
                int cnt = 0;
                std::vector<int> per_group(nf * p->fsym_groups, 0);
                for (int c = 0; c < G; ++c) {
                    long long r0 = cut[c];
                    const long long r1 = cut[c + 1];
                    if (c0) c0->push_back(cnt);
                    while (r0 < r1) {
                        const long long gs = r0 / hq;
                        const long long end = std::min({r1, (gs + 1) * hq, r0 + hm_at(r0)});
                        const int grp = (int)(gs / qt), strip = (int)(gs % qt);
                        if (sg) sg->push_back(make_int4(grp, strip, hq + (int)(r0 - gs * hq),
                                                        hq + (int)(end - gs * hq)));
                        ++per_group[grp];
                        ++cnt;
                        r0 = end;
                    }
                }
                if (c0) c0->push_back(cnt);
                return std::make_pair(cnt, *std::max_element(per_group.begin(), per_group.end()));
            };
            // candidates (T, LW): the segment height hs whose rectangle fits the window; the
            // fewest window words per projection wins, among windows that stage >= 2 images
            // per round when any does (one image per round waits for the engine between rounds:
            // cfg2 batched 4 frames T 32 / LW 256 48.9 us, T 64 / LW 320 55.2 us)
            const char* evt = getenv("PK_FSYM_T");
            const char* evl = getenv("PK_FSYM_LW");
            struct Cand { int T, lw, hs, qt; long long words; int ngr; std::vector<int> tab; };
            std::vector<Cand> cands;
            // the fixed-point bound's contributions-per-slot estimate of a T x H rectangle (as
            // the fp_bits rule below)
            auto nc_of = [&](double T, double H) {
                double nc = 1.5 * (std::hypot(T, H) + 2) * (2.0 / std::max(h, 1e-12) + 2);
                if (p->min_delay < 8.0 * std::max(T, H) * std::max(h, 1.0)) nc = T * H;
                return std::min(nc, T * H);
            };
            for (int T : {64, 32}) {
                if (evt && atoi(evt) != T) continue;
                const int qt = (hq + T - 1) / T;
                const long long R = (long long)nf * p->fsym_groups * qt * hq;
                const int rows_per = (int)((R + G - 1) / G);
                for (int lw : {96, 128, 184, 256, 320}) {
                    if (T == 32 && lw > 256) continue;
                    if (evl && atoi(evl) != lw) continue;
                    if (fs_ngr(lw, nw, cap) == 0) continue;  // windows + one staged image must fit
                    // window span: the rectangle's delay spread + the slot margins + 3 for the
                    // 16-B alignment of the window start (fp_sym_window_lo)
                    int hs = 0;
                    while (hs < hq && (int)std::ceil(region_diag(T, hs + 1)) + 9 <= lw) ++hs;
                    hs = std::min<long long>(hs, rows_per + seg_cost(T));  // (balanced ranges exceed R / G)
                    if (hs == 0) continue;
                    // direction-aware heights, capped where the fixed-point bound would lose a bit
                    // against the uniform height's (PK_FSYM_UNIFORM=1: the uniform height)
                    int hcap = hs;
                    if (!getenv("PK_FSYM_UNIFORM") || atoi(getenv("PK_FSYM_UNIFORM")) == 0)
                        while (hcap < hq && ceil_log2(nc_of(T, hcap + 1)) <= ceil_log2(nc_of(T, hs))) ++hcap;
                    std::vector<int> tab = make_hmax(T, lw, hcap);
                    if (tab.empty()) continue;
                    hm_tab = tab;
                    hm_qt = qt;
                    cands.push_back({T, lw, hs, qt, (long long)segment(T, nullptr, nullptr).first * lw,
                                     fs_ngr(lw, nw, cap), std::move(tab)});
                }
            }
            const bool multi = std::any_of(cands.begin(), cands.end(), [](const Cand& c) { return c.ngr >= 2; });
            long long best = -1;
            for (const Cand& c : cands) {
                if (multi && c.ngr < 2) continue;
                if (best >= 0 && c.words >= best) continue;
                best = c.words;
                p->fsym = 1;
                p->fsym_T = c.T;
                p->fsym_qt = c.qt;
                p->fsym_L = c.lw;
                p->fsym_hs = c.hs;
                p->fsym_smem = fs_smem(c.lw, nw, cap);
                p->fsym_ngr = c.ngr;
                hm_tab = c.tab;
                hm_qt = c.qt;
            }
            if (p->fsym) {
                p->fsym_nw = nw;
                p->fsym_grid = G;
                p->fsym_segs_h.clear();
                p->fsym_cta_seg0_h.clear();
                const auto sc = segment(p->fsym_T, &p->fsym_segs_h, &p->fsym_cta_seg0_h);
                p->fsym_nseg = sc.first;
                // the tallest segment cut (the fixed-point bound below)
                p->fsym_hs = 1;
                for (const int4& q : p->fsym_segs_h) p->fsym_hs = std::max(p->fsym_hs, q.w - q.z);
                // the CTA of each frame's first segment records the frame's fixed-point scale
                p->fsym_rec_h.assign(nf, 0);
                for (int k = p->fsym_nseg - 1; k >= 0; --k) p->fsym_rec_h[p->fsym_segs_h[k].x / p->fsym_groups] = k;
                p->fsym_acc_ld = ((kAccFront + p->Q + p->fsym_L + 4) + 3) & ~3;
            }
        }
        if (nf > 1 && !p->fsym) p->sym = 0;  // batched symmetric plans need the symmetric projector
        if (p->fsym) {
            // fixed-point bound of the segment windows (may be tighter than the generic tile's)
            const double T = p->fsym_T, H = p->fsym_hs;
            double nc = 1.5 * (std::hypot(T, H) + 2) * (2.0 / std::max(h, 1e-12) + 2);
            if (p->min_delay < 8.0 * std::max(T, H) * std::max(h, 1.0)) nc = T * H;
            nc = std::min(nc, T * H);
            p->fp_bits = std::min(p->fp_bits, std::min(22, 30 - ceil_log2(nc)));
            // the gathered sums are int32: bound the pixels that can reach one sample (s0 in
            // [s-1, s+2], a one-sample margin for fp32 delays) exactly, from the D4 base
            // sensors 0..M/8
            // (a sensor's count equals its D4 representative's in [0, Mall/8]: the ring
            // positions of the representatives present in this plan's list)
            std::vector<int> reps;
            {
                std::vector<char> seen(p->Mall / 8 + 2, 0);
                const int q = p->Mall / 4;
                for (int l = 0; l < p->M; ++l) {
                    const int r = p->gid_h[l] % q, rep = std::min(r, q - r);
                    if (rep < (int)seen.size() && !seen[rep]) { seen[rep] = 1; reps.push_back(rep); }
                }
            }
            const int mq = (int)reps.size();
            const double* RP = d->sensor_xy;
            std::vector<int> worst(mq, 0);
            auto count = [&](int m0, int m1) {
                std::vector<int> hist(p->Q + 4);
                for (int k = m0; k < m1; ++k) {
                    const int m = reps[k];
                    std::fill(hist.begin(), hist.end(), 0);
                    for (int j = 0; j < p->ny; ++j)
                        for (int i = 0; i < p->nx; ++i) {
                            const double u = std::hypot(X[i] - RP[2 * m], Y[j] - RP[2 * m + 1]) / p->cdt;
                            const long s0 = (long)std::floor(u);
                            if (s0 >= 0 && s0 <= p->Q + 1) ++hist[s0 + 1];
                        }
                    int w = 0;
                    for (int t = 0; t + 3 < (int)hist.size(); ++t)
                        w = std::max(w, hist[t] + hist[t + 1] + hist[t + 2] + hist[t + 3]);
                    worst[k] = w;
                }
            };
            {
                const int nt = std::max(1, std::min(16, (int)std::thread::hardware_concurrency()));
                std::vector<std::thread> th;
                for (int q = 0; q < nt; ++q) th.emplace_back(count, mq * q / nt, mq * (q + 1) / nt);
                for (auto& t : th) t.join();
            }
            const int ncg = *std::max_element(worst.begin(), worst.end());
            p->fp_bits = std::min(p->fp_bits, 31 - ceil_log2((double)ncg + 1.0));
        }
    }
    p->misc_blocks = std::max(1, std::min(1024, (p->P + kThreads - 1) / kThreads));
    // the residual kernel holds a trace, its measurements and (symmetric projector) the
    // gathered window sums in shared memory
    if ((size_t)(p->Q + 1) * (2 * tsize(p) + 4) + 64 > 200 * 1024) {
        free_plan(p);
        return fail(PK_ERR_UNSUPPORTED, "trace of %d samples exceeds shared memory", p->Q);
    }

    // allocations
    int rc = PK_OK;
    auto A = [&](int r) { if (rc == PK_OK) rc = r; };
    std::vector<float> fx(p->nx), fy(p->ny), fsx(p->M), fsy(p->M);
    std::vector<double> dsx(p->M), dsy(p->M);
    for (int i = 0; i < p->nx; ++i) fx[i] = (float)(X[i] / p->cdt);
    for (int j = 0; j < p->ny; ++j) fy[j] = (float)(Y[j] / p->cdt);
    for (int m = 0; m < p->M; ++m) {
        dsx[m] = SP[2 * m];
        dsy[m] = SP[2 * m + 1];
        fsx[m] = (float)(SP[2 * m] / p->cdt);
        fsy[m] = (float)(SP[2 * m + 1] / p->cdt);
    }
    A(alloc(p, &p->gid, p->M)); A(alloc(p, &p->loc, p->Mall));
    A(alloc(p, &p->pxs, p->nx)); A(alloc(p, &p->pys, p->ny));
    A(alloc(p, &p->sxs, p->M)); A(alloc(p, &p->sys, p->M));
    A(alloc(p, &p->px, p->nx)); A(alloc(p, &p->py, p->ny));
    A(alloc(p, &p->sx, p->M)); A(alloc(p, &p->sy, p->M));
    const size_t ts = tsize(p);
    A(alloc(p, reinterpret_cast<unsigned char**>(&p->table), (size_t)p->M * p->TS * 2 * ts * nf));
    A(alloc(p, &p->acc, (size_t)p->M * p->Q * nf));
    A(alloc(p, reinterpret_cast<unsigned char**>(&p->xbuf[0]), (size_t)p->P * ts * nf));
    A(alloc(p, reinterpret_cast<unsigned char**>(&p->xbuf[1]), (size_t)p->P * ts * nf));
    const int ntile_max = std::max(p->bp_tiles_x * p->bp_tiles_y, p->sym ? 32 * p->sym_ntiles : 0);
    A(alloc(p, &p->part_bp, (size_t)4 * nf * std::max(ntile_max, (p->P + kThreads - 1) / kThreads)));
    A(alloc(p, &p->part_mx, (size_t)std::max(1, p->sym ? 32 * p->sym_ntiles * nf : 1)));
    A(alloc(p, &p->part_l1, (size_t)(p->fsym ? 2 * 8 * p->M * nf : 1)));
    // TV partials: per projector tile, or per residual CTA (M x up to 8 chunks) with the
    // symmetric projector
    A(alloc(p, &p->part_tv, (size_t)std::max(p->fp_tiles_x * p->fp_tiles_y, p->fsym ? 8 * p->M : 0) * nf));
    if (p->fsym) {
        A(alloc(p, &p->fsym_acc, (size_t)nf * p->M * p->fsym_acc_ld));
        A(alloc(p, &p->fsym_rec, (size_t)nf));
        A(alloc(p, &p->fsym_trace, (size_t)p->fsym_groups * 32 * 4));
        A(alloc(p, &p->fsym_bias, (size_t)p->M * p->fsym_acc_ld));
        A(alloc(p, &p->fsym_segs, p->fsym_segs_h.size()));
        A(alloc(p, &p->fsym_cta_seg0, p->fsym_cta_seg0_h.size()));
        A(alloc(p, &p->fsym_xr, (size_t)(p->nx / 2) * (p->nx / 2) * 4 * nf));
    }
    // one CTA per sensor: more, shorter CTAs only add latency (measured 10.3 / 12.8 / 18.2 us
    // for 1 / 2 / 4 chunks at config 3)
    p->fin_chunks = 1;
    if (const char* e = getenv("PK_FIN_CHUNKS")) p->fin_chunks = std::max(1, std::min(8, atoi(e)));
    if (p->fsym) p->fin_chunks = 1;  // the residual CTA of a trace clears its accumulator row
    A(alloc(p, &p->part_r, (size_t)p->M * nf * p->fin_chunks));
    A(alloc(p, &p->part_misc, (size_t)4 * p->misc_blocks * nf));
    if (p->bp_split > 1) A(alloc(p, &p->bp_gpart, (size_t)p->bp_split * p->P * nf));
    A(alloc(p, &p->bp_tile_cnt, (size_t)ntile_max));
    if (p->sym) A(alloc(p, &p->sym_sync, (size_t)3 * p->sym_ntiles * nf));
    if (p->sym) {
        A(alloc(p, &p->sym_tiles, p->sym_h[0].size()));
        A(alloc(p, &p->sym_chunks, p->sym_h[1].size()));
        A(alloc(p, &p->sym_cta_chunk0, p->sym_h[2].size()));
        A(alloc(p, &p->sym_cta_slot0, p->sym_h[3].size()));
        A(alloc(p, &p->sym_tile_slot0, p->sym_h[4].size()));
        A(alloc(p, &p->sym_part, (size_t)p->sym_slots_cap * 8 * 4 * kThreads));
    }
    A(alloc(p, &p->state, 1));
    A(alloc(p, &p->params, 1));
    A(alloc(p, &p->io, 1));
    if (rc != PK_OK) { free_plan(p); return rc; }
    cudaError_t e = cudaSuccess;
    auto up = [&](void* dst, const void* src, size_t n) {
        if (e == cudaSuccess) e = cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
    };
    up(p->gid, p->gid_h.data(), sizeof(int) * p->M); up(p->loc, loc_h.data(), sizeof(int) * p->Mall);
    up(p->pxs, fx.data(), p->nx * 4); up(p->pys, fy.data(), p->ny * 4);
    up(p->sxs, fsx.data(), p->M * 4); up(p->sys, fsy.data(), p->M * 4);
    up(p->px, X, p->nx * 8); up(p->py, Y, p->ny * 8);
    up(p->sx, dsx.data(), p->M * 8); up(p->sy, dsy.data(), p->M * 8);
    if (e == cudaSuccess) e = cudaMemset(p->acc, 0, (size_t)p->M * p->Q * 8 * nf);
    if (e == cudaSuccess) e = cudaMemset(p->state, 0, sizeof(DevState));
    if (e == cudaSuccess)
        e = cudaMemset(p->bp_tile_cnt, 0, sizeof(uint32_t) * ntile_max);
    if (e == cudaSuccess && p->sym) e = cudaMemset(p->sym_sync, 0, sizeof(uint32_t) * 3 * p->sym_ntiles * nf);
    if (p->sym) {
        int* dsts[5] = {p->sym_tiles, p->sym_chunks, p->sym_cta_chunk0, p->sym_cta_slot0,
                        p->sym_tile_slot0};
        for (int q = 0; q < 5; ++q) up(dsts[q], p->sym_h[q].data(), sizeof(int) * p->sym_h[q].size());
    }
    if (e == cudaSuccess && p->fsym) {
        // segments, bias counts, the cleared accumulator, and the local trace of every (base
        // sensor, image): image g of base sensor b is ring sensor gid(b) + g*M/4
        const int nseg = p->fsym_nseg;
        up(p->fsym_segs, p->fsym_segs_h.data(), sizeof(int4) * nseg);
        up(p->fsym_cta_seg0, p->fsym_cta_seg0_h.data(), sizeof(int) * p->fsym_cta_seg0_h.size());
        std::vector<int> tro((size_t)p->fsym_groups * 32 * 4, -1);
        const int q4 = p->Mall / 4;
        for (int b = 0; b < p->M; ++b)
            for (int g = 0; g < 4; ++g) tro[4 * b + g] = loc_h[(p->gid_h[b] + g * q4) % p->Mall];
        up(p->fsym_trace, tro.data(), sizeof(int) * tro.size());
        up(p->fsym_rec, p->fsym_rec_h.data(), sizeof(int) * nf);
        {   // bias counts of every accumulator position (frame 0's segments), the rows' start values
            const int zero = 0;
            const size_t words = (size_t)p->M * p->fsym_acc_ld;
            int* cnt = nullptr;
            if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_counts_overflow, &zero, sizeof(int));
            if (e == cudaSuccess) e = cudaMalloc(&cnt, sizeof(int) * words);
            if (e == cudaSuccess) e = cudaMemset(cnt, 0, sizeof(int) * words);
            const size_t csm = (size_t)p->fsym_L * 32 * 4;
            if (e == cudaSuccess) {
                if (p->max_delay >= (double)p->Q + 0.5)
                    fp_sym_count_kernel<true><<<nseg, kFsThreads, csm>>>(
                        p->pxs, p->pys, p->sxs, p->sys, p->nx, p->M, p->fsym_groups, p->fsym_segs, (float)p->Q + 1.5f,
                        p->fsym_hx, p->fsym_L, p->fsym_T, p->fsym_trace, p->fsym_acc_ld, cnt);
                else
                    fp_sym_count_kernel<false><<<nseg, kFsThreads, csm>>>(
                        p->pxs, p->pys, p->sxs, p->sys, p->nx, p->M, p->fsym_groups, p->fsym_segs, (float)p->Q + 1.5f,
                        p->fsym_hx, p->fsym_L, p->fsym_T, p->fsym_trace, p->fsym_acc_ld, cnt);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) {
                fp_sym_bias_init_kernel<<<1024, 256>>>(cnt, p->fsym_bias, p->fsym_acc, words, nf);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (cnt) cudaFree(cnt);
        }
        int ovf = 0;
        if (e == cudaSuccess) e = cudaMemcpyFromSymbol(&ovf, g_counts_overflow, sizeof(int));
        if (e == cudaSuccess && ovf) {
            free_plan(p);
            return fail(PK_ERR_UNSUPPORTED, "projector accumulator position receives > 65535 pixels (set PK_FSYM=0)");
        }
    }
    if (e == cudaSuccess) e = cudaMemset(p->table, 0, (size_t)p->M * p->TS * 2 * ts * nf);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking);
    // opt every dynamic-smem kernel into the device maximum once per device (a per-plan
    // value would shrink the limit under plans created earlier with larger windows)
    if (e == cudaSuccess) e = opt_in_smem(p->device);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = sym_tune_wdiag(p);  // (zero table: the products' cost is data independent)
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        free_plan(p);
        return fail(PK_ERR_CUDA, "plan setup failed: %s", cudaGetErrorString(e));
    }
    *out = p;
    return PK_OK;
}

int pk_plan_destroy(pk_plan* p) {
    free_plan(p);
    return PK_OK;
}

int pk_plan_get_info(const pk_plan* p, pk_plan_info* o) {
    if (!p || !o) return fail(PK_ERR_INVALID, "NULL argument");
    o->local_sensors = p->M;
    o->pixels = p->P;
    o->dtype = p->dtype;
    o->may_truncate = p->may_truncate;
    o->c_dt = p->cdt;
    o->weight = p->w;
    o->bp_tile = p->dtype == PK_F32 ? kBpTile : 1;
    o->bp_window = p->bp_L;
    o->bp_chunk = p->bp_CS;
    o->bp_buffers = p->bp_nbuf;
    o->fp_tile = p->fsym ? p->fsym_T : p->fp_T;   // symmetric projector: quadrant tile side
    o->fp_window = p->fsym ? p->fsym_L : p->fp_L;
    o->fp_bits = p->fp_bits;
    o->device_bytes = p->device_bytes;
    o->frames = p->nf;
    o->bp_split = p->sym ? p->sym_slots : p->bp_split;
    o->symmetric = p->sym + 2 * p->fsym;
    return PK_OK;
}

int pk_matvec(pk_plan* p, const void* x, void* out, void* stream) {
    if (!p || !x || !out) return fail(PK_ERR_INVALID, "NULL argument");
    DeviceGuard g(p->device);
    cudaStream_t s = S(stream);
    PK_TRY(launch_maxabs(p, x, s));
    PK_TRY(launch_fp(p, x, 0, s));
    PK_TRY(launch_finalize(p, nullptr, out, nullptr, 0, s));
    return PK_OK;
}

int pk_adjoint_matvec(pk_plan* p, const void* y, void* out, double scale, void* stream) {
    if (!p || !y || !out) return fail(PK_ERR_INVALID, "NULL argument");
    DeviceGuard g(p->device);
    cudaStream_t s = S(stream);
    PK_TRY(launch_table(p, y, 0, s));
    PK_TRY(launch_bp(p, 0, out, scale, s));
    return PK_OK;
}

int pk_residual(pk_plan* p, const void* x, const void* y, void* r_out, double* sumsq,
                void* stream) {
    if (!p || !x || !y) return fail(PK_ERR_INVALID, "NULL argument");
    DeviceGuard g(p->device);
    cudaStream_t s = S(stream);
    PK_TRY(launch_maxabs(p, x, s));
    PK_TRY(launch_fp(p, x, 0, s));
    PK_TRY(launch_finalize(p, y, r_out, sumsq, 0, s));
    return PK_OK;
}

int pk_adjoint_residual(pk_plan* p, void* out, double scale, void* stream) {
    if (!p || !out) return fail(PK_ERR_INVALID, "NULL argument");
    DeviceGuard g(p->device);
    PK_TRY(launch_bp(p, 0, out, scale, S(stream)));
    return PK_OK;
}

int pk_grad_update(pk_plan* p, const pk_solver_params* prm, const void* x, const void* grad,
                   void* x_out, double* sums, void* stream) {
    if (!p || !x || !grad || !x_out || !sums) return fail(PK_ERR_INVALID, "NULL argument");
    if (p->nf != 1) return fail(PK_ERR_UNSUPPORTED, "pk_grad_update is single-frame");
    PK_TRY(check_params(p, prm));
    DeviceGuard g(p->device);
    cudaStream_t s = S(stream);
    PK_TRY(upload_params(p, prm, s));
    const int pb = (p->P + kThreads - 1) / kThreads;
    if (p->dtype == PK_F32) {
        grad_update_kernel<float><<<pb, kThreads, 0, s>>>(static_cast<const float*>(x),
                                                          static_cast<const float*>(grad),
                                                          static_cast<float*>(x_out), p->nx, p->ny,
                                                          p->params);
        image_sums_kernel<float><<<p->misc_blocks, kThreads, 0, s>>>(
            static_cast<const float*>(x_out), p->nx, p->ny, p->part_misc, p->state, sums);
    } else {
        grad_update_kernel<double><<<pb, kThreads, 0, s>>>(static_cast<const double*>(x),
                                                           static_cast<const double*>(grad),
                                                           static_cast<double*>(x_out), p->nx,
                                                           p->ny, p->params);
        image_sums_kernel<double><<<p->misc_blocks, kThreads, 0, s>>>(
            static_cast<const double*>(x_out), p->nx, p->ny, p->part_misc, p->state, sums);
    }
    PK_CHECK_LAUNCH();
    return PK_OK;
}

int pk_peer_handle(pk_plan* p, void* handle_out) {
    if (!p || !handle_out) return fail(PK_ERR_INVALID, "NULL argument");
    if (p->nf != 1) return fail(PK_ERR_UNSUPPORTED, "peer exchange is single-frame");
    DeviceGuard g(p->device);
    if (!p->peer_block) {
        PK_TRY(alloc(p, &p->peer_block, kPeerHeader + 2 * peer_slot_bytes(p)));
        PK_CUDA(cudaMemset(p->peer_block, 0, kPeerHeader + 2 * peer_slot_bytes(p)));
    }
    cudaIpcMemHandle_t h;
    PK_CUDA(cudaIpcGetMemHandle(&h, p->peer_block));
    static_assert(sizeof(h) == PK_PEER_HANDLE_BYTES, "cudaIpcMemHandle_t size");
    std::memcpy(handle_out, &h, sizeof(h));
    std::lock_guard<std::mutex> lk(g_peer_mu);
    g_peer_registry[std::string(reinterpret_cast<const char*>(&h), sizeof(h))] = p->peer_block;
    return PK_OK;
}

int pk_peer_connect(pk_plan* p, int32_t world, int32_t rank, const void* handles) {
    if (!p || !handles) return fail(PK_ERR_INVALID, "NULL argument");
    if (world < 1 || world > PK_PEER_MAX || rank < 0 || rank >= world)
        return fail(PK_ERR_INVALID, "world %d / rank %d outside 1..%d", world, rank, PK_PEER_MAX);
    if (!p->peer_block) return fail(PK_ERR_INVALID, "pk_peer_handle must be called first");
    if (p->peer_world) return fail(PK_ERR_INVALID, "plan is already connected");
    DeviceGuard g(p->device);
    std::vector<void*> grads(world);
    std::vector<int*> flags(world);
    for (int r = 0; r < world; ++r) {
        const char* hb = static_cast<const char*>(handles) + (size_t)r * PK_PEER_HANDLE_BYTES;
        unsigned char* base = nullptr;
        {
            std::lock_guard<std::mutex> lk(g_peer_mu);
            auto it = g_peer_registry.find(std::string(hb, PK_PEER_HANDLE_BYTES));
            if (it != g_peer_registry.end()) base = it->second;
        }
        if (r == rank && base != p->peer_block)
            return fail(PK_ERR_INVALID, "handles[%d] is not this plan's handle", rank);
        if (!base) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, hb, sizeof(h));
            void* q = nullptr;
            PK_CUDA(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
            p->peer_opened.push_back(q);
            base = static_cast<unsigned char*>(q);
        }
        grads[r] = base + kPeerHeader;
        flags[r] = reinterpret_cast<int*>(base);
    }
    // load the peer kernels now: under lazy module loading the first launch of a kernel
    // waits for the device to drain, which never happens while another rank of this process
    // spins in its barrier (the solve's other kernels are loaded by its warm-up call)
    {
        cudaFuncAttributes fa;
        PK_CUDA(cudaFuncGetAttributes(&fa, peer_barrier_kernel));
        PK_CUDA(cudaFuncGetAttributes(&fa, peer_grad_update_kernel<float>));
        PK_CUDA(cudaFuncGetAttributes(&fa, peer_grad_update_kernel<double>));
        PK_CUDA(cudaFuncGetAttributes(&fa, image_sums_kernel<float>));
        PK_CUDA(cudaFuncGetAttributes(&fa, image_sums_kernel<double>));
    }
    PK_TRY(alloc(p, &p->peer_grad_dev, (size_t)world));
    PK_TRY(alloc(p, &p->peer_flags_dev, (size_t)world));
    PK_CUDA(cudaMemcpy(p->peer_grad_dev, grads.data(), world * sizeof(void*), cudaMemcpyHostToDevice));
    PK_CUDA(cudaMemcpy(p->peer_flags_dev, flags.data(), world * sizeof(int*), cudaMemcpyHostToDevice));
    p->peer_world = world;
    p->peer_rank = rank;
    return PK_OK;
}

int pk_peer_buffer(pk_plan* p, int32_t slot, void** ptr_out) {
    if (!p || !ptr_out) return fail(PK_ERR_INVALID, "NULL argument");
    if (!p->peer_block) return fail(PK_ERR_INVALID, "pk_peer_handle must be called first");
    if (slot != 0 && slot != 1) return fail(PK_ERR_INVALID, "slot must be 0 or 1");
    *ptr_out = p->peer_block + kPeerHeader + (size_t)slot * peer_slot_bytes(p);
    return PK_OK;
}

int pk_peer_status(pk_plan* p, int32_t* timed_out) {
    if (!p || !timed_out) return fail(PK_ERR_INVALID, "NULL argument");
    if (!p->peer_block) return fail(PK_ERR_INVALID, "pk_peer_handle must be called first");
    DeviceGuard g(p->device);
    int v = 0;
    PK_CUDA(cudaMemcpy(&v, reinterpret_cast<int*>(p->peer_block) + PK_PEER_MAX + 1, sizeof(int),
                       cudaMemcpyDeviceToHost));
    *timed_out = v;
    return PK_OK;
}

int pk_peer_grad_update(pk_plan* p, const pk_solver_params* prm, const void* x, int32_t slot,
                        void* x_out, double* sums, void* stream) {
    if (!p || !x || !x_out || !sums) return fail(PK_ERR_INVALID, "NULL argument");
    if (!p->peer_world) return fail(PK_ERR_INVALID, "plan is not connected (pk_peer_connect)");
    if (slot != 0 && slot != 1) return fail(PK_ERR_INVALID, "slot must be 0 or 1");
    PK_TRY(check_params(p, prm));
    DeviceGuard g(p->device);
    cudaStream_t s = S(stream);
    PK_TRY(upload_params(p, prm, s));
    int* epoch = reinterpret_cast<int*>(p->peer_block) + PK_PEER_MAX;
    peer_barrier_kernel<<<1, 32, 0, s>>>(epoch, p->peer_flags_dev, p->peer_world, p->peer_rank,
                                         peer_timeout_ns());
    const int pb = (p->P + kThreads - 1) / kThreads;
    const size_t off = (size_t)slot * peer_slot_bytes(p) / tsize(p);
    if (p->dtype == PK_F32) {
        peer_grad_update_kernel<float><<<pb, kThreads, 0, s>>>(
            p->peer_grad_dev, off, p->peer_world, static_cast<const float*>(x),
            static_cast<float*>(x_out), p->nx, p->ny, p->params, epoch + 1);
        image_sums_kernel<float><<<p->misc_blocks, kThreads, 0, s>>>(
            static_cast<const float*>(x_out), p->nx, p->ny, p->part_misc, p->state, sums);
    } else {
        peer_grad_update_kernel<double><<<pb, kThreads, 0, s>>>(
            p->peer_grad_dev, off, p->peer_world, static_cast<const double*>(x),
            static_cast<double*>(x_out), p->nx, p->ny, p->params, epoch + 1);
        image_sums_kernel<double><<<p->misc_blocks, kThreads, 0, s>>>(
            static_cast<const double*>(x_out), p->nx, p->ny, p->part_misc, p->state, sums);
    }
    PK_CHECK_LAUNCH();
    return PK_OK;
}

int pk_reconstruct(pk_plan* p, const pk_solver_params* prm, const void* y, void* x_out,
                   double* hist, int32_t* status, void* stream) {
    if (!p || !y || !x_out || !hist || !status) return fail(PK_ERR_INVALID, "NULL argument");
    PK_TRY(check_params(p, prm));
    if (p->M != p->Mall)
        return fail(PK_ERR_INVALID, "pk_reconstruct needs a plan over all sensors (use the sharded pieces)");
    DeviceGuard g(p->device);
    cudaStream_t s = S(stream);
    PK_TRY(upload_params(p, prm, s));
    DevIo io{y, x_out, hist, status};
    PK_CUDA(cudaMemcpyAsync(p->io, &io, sizeof(io), cudaMemcpyHostToDevice, s));
    if (p->graph_iters != prm[0].iterations) {
        if (p->graph_exec) { cudaGraphExecDestroy(p->graph_exec); p->graph_exec = nullptr; }
        if (p->graph) { cudaGraphDestroy(p->graph); p->graph = nullptr; }
        p->graph_iters = -1;
        PK_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
        int rc = record_solver(p, prm[0].iterations, p->cap_stream);
        cudaGraph_t gr = nullptr;
        cudaError_t e = cudaStreamEndCapture(p->cap_stream, &gr);
        if (rc != PK_OK) { if (gr) cudaGraphDestroy(gr); return rc; }
        if (e != cudaSuccess) return fail(PK_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
        p->graph = gr;
        PK_CUDA(cudaGraphInstantiate(&p->graph_exec, p->graph, 0));
        p->graph_iters = prm[0].iterations;
    }
    PK_CUDA(cudaGraphLaunch(p->graph_exec, s));
    return PK_OK;
}

int pk_reconstruct_host_async(pk_plan* p, const pk_solver_params* prm, const double* y_host,
                              double* x_out_host, double* hist_host, int32_t* status_host,
                              void* stream) {
    if (!p || !y_host || !x_out_host || !hist_host || !status_host)
        return fail(PK_ERR_INVALID, "NULL argument");
    PK_TRY(check_params(p, prm));
    DeviceGuard g(p->device);
    cudaStream_t s = S(stream);
    const size_t ny = (size_t)p->M * p->Q * p->nf;
    const size_t nx = (size_t)p->P * p->nf;
    if (!p->y64) { PK_TRY(alloc(p, &p->y64, ny)); }
    if (!p->x64) { PK_TRY(alloc(p, &p->x64, nx)); }
    if (!p->status_dev) { PK_TRY(alloc(p, &p->status_dev, 2 * p->nf)); }
    if (p->dtype == PK_F32 && !p->ydev) {
        PK_TRY(alloc(p, reinterpret_cast<float**>(&p->ydev), ny));
        PK_TRY(alloc(p, reinterpret_cast<float**>(&p->xout_dev), nx));
    }
    PK_TRY(ensure_hist(p, prm[0].iterations));
    PK_CUDA(cudaMemcpyAsync(p->y64, y_host, ny * 8, cudaMemcpyHostToDevice, s));
    const int cb = 148 * 4;
    if (p->dtype == PK_F32) {
        convert_kernel<float><<<cb, kThreads, 0, s>>>(p->y64, static_cast<float*>(p->ydev), ny);
        PK_CHECK_LAUNCH();
        PK_TRY(pk_reconstruct(p, prm, p->ydev, p->xout_dev, p->hist_dev, p->status_dev, stream));
        widen_kernel<float><<<cb, kThreads, 0, s>>>(static_cast<const float*>(p->xout_dev), p->x64, nx);
        PK_CHECK_LAUNCH();
    } else {
        PK_TRY(pk_reconstruct(p, prm, p->y64, p->x64, p->hist_dev, p->status_dev, stream));
    }
    PK_CUDA(cudaMemcpyAsync(x_out_host, p->x64, nx * 8, cudaMemcpyDeviceToHost, s));
    PK_CUDA(cudaMemcpyAsync(hist_host, p->hist_dev, (size_t)4 * prm[0].iterations * p->nf * 8,
                            cudaMemcpyDeviceToHost, s));
    PK_CUDA(cudaMemcpyAsync(status_host, p->status_dev, 8 * p->nf, cudaMemcpyDeviceToHost, s));
    return PK_OK;
}

int pk_reconstruct_host(pk_plan* p, const pk_solver_params* prm, const double* y_host,
                        double* x_out_host, double* hist_host, int32_t* status_host,
                        void* stream) {
    PK_TRY(pk_reconstruct_host_async(p, prm, y_host, x_out_host, hist_host, status_host, stream));
    DeviceGuard g(p->device);
    PK_CUDA(cudaStreamSynchronize(S(stream)));
    return PK_OK;
}

// ---------------------------------------------------------------------------
// frequency-domain operator (build_freq_matrix, forward.py:218-234), matrix-free

namespace {
// wavenumbers per lane of the fp32 forward (PK_FREQ_R: 16 or 32 for sweeps)
int freq_run(int q_n) {
    if (const char* e = getenv("PK_FREQ_R")) return atoi(e) == 16 ? 16 : 32;
    return q_n > 512 ? 32 : 16;
}
int freq_setup(pk_plan* p, int q_n, FreqArgs& a, int& zblocks) {
    if (q_n < 1) return fail(PK_ERR_INVALID, "q_n must be >= 1");
    a.px = p->px; a.py = p->py; a.sx = p->sx; a.sy = p->sy;
    a.nx = p->nx; a.P = p->P; a.M = p->M; a.Q = p->Q; a.qn = q_n;
    a.cdt = p->cdt;
    a.c = p->c;
    a.kscale = 2.0 * 3.141592653589793 / ((double)p->Q * p->dt * p->c);  // AcousticConfig.k_values
    // fp32: freq_fwd_f32_kernel, 32 lanes x R wavenumbers per CTA (R = 32 above q_n = 512,
    // else 16); fp64: freq_fwd_kernel, 128 threads x kFreqRun
    const int span = p->dtype == PK_F32 ? 32 * freq_run(q_n) : kFreqThreads * kFreqRun;
    zblocks = (q_n + span - 1) / span;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
    a.chunks = std::max(1, std::min(64, (4 * sms + p->M * zblocks - 1) / (p->M * zblocks)));
    a.chunks = std::min(a.chunks, std::max(1, p->P / kFreqPix));
    return PK_OK;
}
}  // namespace

int pk_freq_matvec(pk_plan* p, int32_t q_n, const void* x, void* y, void* stream) {
    if (!p || !x || !y) return fail(PK_ERR_INVALID, "NULL argument");
    if (p->nf != 1) return fail(PK_ERR_UNSUPPORTED, "frequency operator is single-frame");
    DeviceGuard g(p->device);
    FreqArgs a{};
    int zb = 0;
    PK_TRY(freq_setup(p, q_n, a, zb));
    const size_t need = (size_t)a.chunks * p->M * q_n * 2 * tsize(p);
    if (need > p->freq_part_bytes) {  // grows once per (q_n, geometry); not on later calls
        if (p->freq_part) cudaFree(p->freq_part);
        p->freq_part = nullptr;
        p->freq_part_bytes = 0;
        PK_CUDA(cudaMalloc(&p->freq_part, need));
        p->freq_part_bytes = need;
    }
    a.x = x; a.part = p->freq_part; a.out = y;
    cudaStream_t s = S(stream);
    const dim3 grid(p->M, a.chunks, zb);
    const int sb = (int)std::min<size_t>(148 * 8, ((size_t)p->M * q_n + kThreads - 1) / kThreads);
    if (p->dtype == PK_F32) {
        if (freq_run(q_n) == 32) freq_fwd_f32_kernel<32><<<grid, 128, 0, s>>>(a);
        else freq_fwd_f32_kernel<16><<<grid, 128, 0, s>>>(a);
        freq_fwd_sum_kernel<float><<<sb, kThreads, 0, s>>>(a);
    } else {
        freq_fwd_kernel<double><<<grid, kFreqThreads, 0, s>>>(a);
        freq_fwd_sum_kernel<double><<<sb, kThreads, 0, s>>>(a);
    }
    PK_CHECK_LAUNCH();
    return PK_OK;
}

int pk_freq_adjoint(pk_plan* p, int32_t q_n, const void* y, void* out, double scale, void* stream) {
    if (!p || !y || !out) return fail(PK_ERR_INVALID, "NULL argument");
    if (p->nf != 1) return fail(PK_ERR_UNSUPPORTED, "frequency operator is single-frame");
    DeviceGuard g(p->device);
    FreqArgs a{};
    int zb = 0;
    PK_TRY(freq_setup(p, q_n, a, zb));
    a.y = y; a.out = out; a.scale = scale;
    const size_t sm = (size_t)q_n * 2 * tsize(p);
    if (sm > 200 * 1024) return fail(PK_ERR_UNSUPPORTED, "q_n = %d too large for the adjoint", q_n);
    cudaStream_t s = S(stream);
    const int blocks = (p->P + kThreads - 1) / kThreads;
    // sensor chunks so that the grid covers ~4 CTAs per SM; partials summed in chunk order
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
    const int chunks = std::max(1, std::min(p->M, (4 * sms + blocks - 1) / blocks));
    a.chunks = chunks;
    if (chunks > 1) {
        const size_t need = (size_t)chunks * p->P * 2 * tsize(p);
        if (need > p->freq_part_bytes) {
            if (p->freq_part) cudaFree(p->freq_part);
            p->freq_part = nullptr;
            p->freq_part_bytes = 0;
            PK_CUDA(cudaMalloc(&p->freq_part, need));
            p->freq_part_bytes = need;
        }
        a.part = p->freq_part;
    }
    const dim3 grid(blocks, chunks);
    const int sb = std::min(148 * 8, blocks);
    if (p->dtype == PK_F32) {
        if (sm > 48 * 1024)
            PK_CUDA(cudaFuncSetAttribute((const void*)freq_adj_kernel<float>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        freq_adj_kernel<float><<<grid, kThreads, sm, s>>>(a);
        if (chunks > 1) freq_adj_sum_kernel<float><<<sb, kThreads, 0, s>>>(a);
    } else {
        if (sm > 48 * 1024)
            PK_CUDA(cudaFuncSetAttribute((const void*)freq_adj_kernel<double>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        freq_adj_kernel<double><<<grid, kThreads, sm, s>>>(a);
        if (chunks > 1) freq_adj_sum_kernel<double><<<sb, kThreads, 0, s>>>(a);
    }
    PK_CHECK_LAUNCH();
    return PK_OK;
}

int pk_index_dump(pk_plan* p, int32_t ma, int32_t mb, int64_t* s0, double* frac, void* stream) {
    if (!p || !s0) return fail(PK_ERR_INVALID, "NULL argument");
    if (ma < 0 || mb > p->M || ma >= mb) return fail(PK_ERR_INVALID, "bad sensor range");
    DeviceGuard g(p->device);
    index_dump_kernel<<<148 * 8, kThreads, 0, S(stream)>>>(
        p->px, p->py, p->sx, p->sy, p->cdt, p->nx, p->P, ma, mb,
        reinterpret_cast<long long*>(s0), frac);
    PK_CHECK_LAUNCH();
    return PK_OK;
}

int pk_delay_census_f32(pk_plan* p, int32_t rule, int32_t ma, int32_t mb, int32_t* s0, float* frac,
                        void* stream) {
    if (!p || !s0 || !frac) return fail(PK_ERR_INVALID, "NULL argument");
    if (ma < 0 || mb > p->M || ma >= mb) return fail(PK_ERR_INVALID, "bad sensor range");
    if (rule < 0 || rule > 2) return fail(PK_ERR_INVALID, "rule must be 0, 1 or 2");
    if (rule == 1 && !p->sym) return fail(PK_ERR_UNSUPPORTED, "plan has no symmetric back-projector");
    if (rule == 2 && !p->fsym) return fail(PK_ERR_UNSUPPORTED, "plan has no symmetric projector");
    if (rule > 0 && p->M != p->Mall) return fail(PK_ERR_INVALID, "symmetric rules need all sensors");
    DeviceGuard g(p->device);
    delay_census_f32_kernel<<<148 * 8, kThreads, 0, S(stream)>>>(
        p->pxs, p->pys, p->sxs, p->sys, p->nx, p->P, p->M, ma, mb, rule, (float)p->Q + 1.5f,
        p->fsym ? p->fsym_hx : 0.f, s0, frac);
    PK_CHECK_LAUNCH();
    return PK_OK;
}

#if PK_BP_TRACE
// timing experiments only (-DPK_BP_TRACE=1): the back-projector's phase trace of the last launch
int pk_debug_bp_trace(void* host, int64_t bytes) {
    const int64_t n = std::min<int64_t>(bytes, sizeof(long long) * 1536 * 16);
    return cudaMemcpyFromSymbol(host, g_bp_trace, n) == cudaSuccess ? PK_OK : PK_ERR_CUDA;
}
int pk_debug_bp_chunks(void* host, int64_t bytes) {
    const int64_t n = std::min<int64_t>(bytes, sizeof(int) * 1536 * 64);
    return cudaMemcpyFromSymbol(host, g_bp_chunk_clk, n) == cudaSuccess ? PK_OK : PK_ERR_CUDA;
}
int pk_debug_bp_plan(const pk_plan* p, int* chunks, int* cta_chunk0, int* tiles, int cap) {
    const size_t n1 = p->sym_h[1].size(), n2 = p->sym_h[2].size(), n0 = p->sym_h[0].size();
    if ((int)std::max({n0, n1, n2}) > cap) return -1;
    std::copy(p->sym_h[1].begin(), p->sym_h[1].end(), chunks);
    std::copy(p->sym_h[2].begin(), p->sym_h[2].end(), cta_chunk0);
    std::copy(p->sym_h[0].begin(), p->sym_h[0].end(), tiles);
    return (int)n1;
}
#endif
#if PK_FS_TRACE
// timing experiments only (-DPK_FS_TRACE=1): copy the projector's phase trace of the last launch
int pk_debug_fs_trace(void* host, int64_t bytes) {
    const int64_t n = std::min<int64_t>(bytes, sizeof(long long) * 1024 * kFsTraceSlots);
    return cudaMemcpyFromSymbol(host, g_fs_trace, n) == cudaSuccess ? PK_OK : PK_ERR_CUDA;
}
#endif

int pk_profile_iterations(pk_plan* p, const pk_solver_params* prm, const void* y, float* ms,
                          int32_t* launches, void* stream) {
    if (!p || !y || !ms) return fail(PK_ERR_INVALID, "NULL argument");
    PK_TRY(check_params(p, prm));
    if (p->M != p->Mall) return fail(PK_ERR_INVALID, "profiling needs a plan over all sensors");
    DeviceGuard g(p->device);
    cudaStream_t s = S(stream);
    PK_TRY(ensure_hist(p, prm[0].iterations));
    if (!p->status_dev) { PK_TRY(alloc(p, &p->status_dev, 2 * p->nf)); }
    if (!p->xout_dev) {
        PK_TRY(alloc(p, reinterpret_cast<unsigned char**>(&p->xout_dev), (size_t)p->P * tsize(p) * p->nf));
    }
    PK_TRY(upload_params(p, prm, s));
    DevIo io{y, p->xout_dev, p->hist_dev, p->status_dev};
    PK_CUDA(cudaMemcpyAsync(p->io, &io, sizeof(io), cudaMemcpyHostToDevice, s));
    PK_TRY(launch_init(p, s));
    PK_TRY(launch_table(p, nullptr, 1, s));
    const int n = prm[0].iterations;
    std::vector<cudaEvent_t> ev(3 * n + 1);
    for (auto& e : ev) PK_CUDA(cudaEventCreate(&e));
    hold_kernel<<<1, 32, 0, s>>>(2000000LL + 400000LL * n);  // ~1 ms + 0.2 ms per iteration of clocks
    PK_CUDA(cudaEventRecord(ev[0], s));
    for (int it = 0; it < n; ++it) {
        PK_TRY(launch_bp(p, 1, nullptr, 2.0, s));
        PK_CUDA(cudaEventRecord(ev[3 * it + 1], s));
        PK_TRY(launch_fp(p, nullptr, 1, s));
        PK_CUDA(cudaEventRecord(ev[3 * it + 2], s));
        PK_TRY(launch_finalize(p, nullptr, nullptr, nullptr, 1, s));
        PK_CUDA(cudaEventRecord(ev[3 * it + 3], s));
    }
    PK_CUDA(cudaStreamSynchronize(s));
    ms[0] = ms[1] = ms[2] = 0.f;
    for (int it = 0; it < n; ++it)
        for (int k = 0; k < 3; ++k) {
            float t = 0.f;
            PK_CUDA(cudaEventElapsedTime(&t, ev[3 * it + k], ev[3 * it + k + 1]));
            ms[k] += t;
        }
    for (auto& e : ev) cudaEventDestroy(e);
    if (launches) launches[0] = 2 + 3 * n;
    return PK_OK;
}

int pk_profile_stages(pk_plan* p, const pk_solver_params* prm, const void* y, float* ms,
                      int32_t* launches, void* stream) {
    if (!p || !y || !ms) return fail(PK_ERR_INVALID, "NULL argument");
    if (!(p->dtype == PK_F32 && p->sym && !p->sym_fuse)) {  // no separate update kernel
        float k3[3];
        PK_TRY(pk_profile_iterations(p, prm, y, k3, launches, stream));
        ms[0] = k3[0]; ms[1] = 0.f; ms[2] = k3[1]; ms[3] = k3[2];
        return PK_OK;
    }
    PK_TRY(check_params(p, prm));
    if (p->M != p->Mall) return fail(PK_ERR_INVALID, "profiling needs a plan over all sensors");
    DeviceGuard g(p->device);
    cudaStream_t s = S(stream);
    const int n = prm[0].iterations;
    PK_TRY(ensure_hist(p, n));
    if (!p->status_dev) { PK_TRY(alloc(p, &p->status_dev, 2 * p->nf)); }
    if (!p->xout_dev) {
        PK_TRY(alloc(p, reinterpret_cast<unsigned char**>(&p->xout_dev), (size_t)p->P * tsize(p) * p->nf));
    }
    PK_TRY(upload_params(p, prm, s));
    DevIo io{y, p->xout_dev, p->hist_dev, p->status_dev};
    PK_CUDA(cudaMemcpyAsync(p->io, &io, sizeof(io), cudaMemcpyHostToDevice, s));
    PK_TRY(launch_init(p, s));
    PK_TRY(launch_table(p, nullptr, 1, s));
    // per iteration: [back-projection | update | projection | residual/objective], the
    // back-projection / update boundary recorded inside launch_bp (bp_mid_event)
    std::vector<cudaEvent_t> ev(4 * n + 1);
    for (auto& e : ev) PK_CUDA(cudaEventCreate(&e));
    hold_kernel<<<1, 32, 0, s>>>(2000000LL + 400000LL * n);
    int rc = PK_OK;
    if (cudaEventRecord(ev[0], s) != cudaSuccess) rc = fail(PK_ERR_CUDA, "event record failed");
    for (int it = 0; it < n && rc == PK_OK; ++it) {
        p->bp_mid_event = ev[4 * it + 1];
        rc = launch_bp(p, 1, nullptr, 2.0, s);
        p->bp_mid_event = nullptr;
        if (rc == PK_OK && cudaEventRecord(ev[4 * it + 2], s) != cudaSuccess) rc = PK_ERR_CUDA;
        if (rc == PK_OK) rc = launch_fp(p, nullptr, 1, s);
        if (rc == PK_OK && cudaEventRecord(ev[4 * it + 3], s) != cudaSuccess) rc = PK_ERR_CUDA;
        if (rc == PK_OK) rc = launch_finalize(p, nullptr, nullptr, nullptr, 1, s);
        if (rc == PK_OK && cudaEventRecord(ev[4 * it + 4], s) != cudaSuccess) rc = PK_ERR_CUDA;
    }
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == PK_OK) rc = fail(PK_ERR_CUDA, "profile failed");
    ms[0] = ms[1] = ms[2] = ms[3] = 0.f;
    for (int it = 0; it < n && rc == PK_OK; ++it)
        for (int k = 0; k < 4; ++k) {
            float t = 0.f;
            cudaEventElapsedTime(&t, ev[4 * it + k], ev[4 * it + k + 1]);
            ms[k] += t;
        }
    for (auto& e : ev) cudaEventDestroy(e);
    if (launches) launches[0] = 2 + 4 * n;
    return rc;
}

int pk_measure_fp32_peak(int32_t device, double* tflops) {
    if (!tflops) return fail(PK_ERR_INVALID, "NULL argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(PK_ERR_CUDA, "no CUDA device %d", device);
    DeviceGuard g(device);
    int sms = 0;
    PK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    float* out = nullptr;
    const int blocks = sms * 4, iters = 4096;
    PK_CUDA(cudaMalloc(&out, (size_t)blocks * kThreads * sizeof(float)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    ffma_peak_kernel<<<blocks, kThreads>>>(out, iters);  // warm-up
    cudaEventRecord(e0);
    ffma_peak_kernel<<<blocks, kThreads>>>(out, iters);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (e != cudaSuccess) return fail(PK_ERR_CUDA, "peak kernel failed: %s", cudaGetErrorString(e));
    const double flops = 2.0 * 8.0 * 16.0 * iters * (double)blocks * kThreads;
    *tflops = flops / (ms * 1e-3) / 1e12;
    return PK_OK;
}

}  // extern "C"

// ===========================================================================
// Explicit-matrix mode (pk_dense_*; kernels in pk_dense.cuh)
// ===========================================================================
struct pk_dense {
    int device = 0, dtype = PK_F32, cplx = 0, fused = 0;
    int64_t rows = 0, cols = 0;
    void* K = nullptr;             // rows x cols (x2 if complex), plan dtype, row-major
    int splits = 1, gemv_grid = 0, fgrid = 0, fnv = 0, init_blocks = 0;
    void* part = nullptr;          // gemvT partials [splits][cols (x2)]
    void* fpart = nullptr;         // fused partials [fgrid][cols]
    double* rpart = nullptr;       // sum |r|^2 partials
    double* ipart = nullptr;       // [blocks][3] image sums of the stop kernel
    void* xb[2] = {nullptr, nullptr};
    void* rb = nullptr;            // residual (two-pass path)
    void* ybuf = nullptr;          // y (plan dtype) of the captured solve
    void* xout = nullptr;
    double* hist = nullptr;
    int hist_cap = 0;
    int32_t* status = nullptr;
    DenseState* st = nullptr;
    DevParams* prm = nullptr;
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t exec = nullptr;
    int g_iters = -1, g_nx = -1, g_ny = -1;
    int64_t device_bytes = 0;
    // multi-frame products on the tensor cores (pk_dense_matmat / pk_dense_rmatmat)
    void* Kt = nullptr;            // cols x rows transpose of K (built on the first K^T Y)
    float* bhi = nullptr;          // frames operand split hi / lo [frames][k]
    float* blo = nullptr;
    float* tcpart = nullptr;       // split-K partials
    size_t b_cap = 0, part_cap = 0;
};

namespace {

template <typename T>
int dalloc(pk_dense* d, T** ptr, size_t count) {
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), count * sizeof(T));
    if (e != cudaSuccess)
        return fail(PK_ERR_CUDA, "cudaMalloc(%zu) failed: %s", count * sizeof(T), cudaGetErrorString(e));
    d->device_bytes += (int64_t)(count * sizeof(T));
    return PK_OK;
}

size_t dsize(const pk_dense* d) { return d->dtype == PK_F32 ? 4 : 8; }
int dense_E(const pk_dense* d) { return (int)(16 / (dsize(d) * (d->cplx ? 2 : 1))); }

template <typename R>
__global__ void narrow_kernel(const double* src, R* dst, size_t n) {
    for (size_t q = (size_t)blockIdx.x * kThreads + threadIdx.x; q < n; q += (size_t)gridDim.x * kThreads)
        dst[q] = (R)src[q];
}

int fused_nv(int64_t cols) {  // float4 groups per thread of the fused kernel
    const int64_t nv = cols / 4;
    for (int v : {1, 2, 4, 8, 12})
        if (nv <= (int64_t)v * kFusedThreads) return v;
    return 0;
}

template <typename R>
int launch_gemv(pk_dense* d, const void* x0, const void* x1, int xc, const void* yobs, void* out0,
                void* out1, double* part, const DenseState* st, cudaStream_t s) {
    const R* K = static_cast<const R*>(d->K);
    if (!d->cplx && !xc && ((reinterpret_cast<uintptr_t>(x0) | reinterpret_cast<uintptr_t>(x1)) & 15))
        return fail(PK_ERR_INVALID, "x must be 16-byte aligned (read in 16-byte vectors)");
#define PK_GEMV(KC, XC)                                                                        \
    dense_gemv_kernel<R, KC, XC><<<d->gemv_grid, kDenseThreads, 0, s>>>(                     \
        K, d->rows, d->cols, static_cast<const R*>(x0), static_cast<const R*>(x1),           \
        static_cast<const R*>(yobs), static_cast<R*>(out0), static_cast<R*>(out1), part, st)
    if (d->cplx) { if (xc) PK_GEMV(true, true); else PK_GEMV(true, false); }
    else { if (xc) PK_GEMV(false, true); else PK_GEMV(false, false); }
#undef PK_GEMV
    PK_CHECK_LAUNCH();
    return PK_OK;
}

template <typename R>
int launch_gemvt(pk_dense* d, const void* y0, const void* y1, int yc, bool real, double sign,
                 void* part, const DenseState* st, cudaStream_t s) {
    const R* K = static_cast<const R*>(d->K);
    const int64_t nvec = d->cols / dense_E(d);
    dim3 grid((unsigned)((nvec + kDenseThreads - 1) / kDenseThreads), (unsigned)d->splits);
#define PK_GEMVT(KC, YC, RE)                                                                  \
    dense_gemvt_kernel<R, KC, YC, RE><<<grid, kDenseThreads, 0, s>>>(                         \
        K, d->rows, d->cols, static_cast<const R*>(y0), static_cast<const R*>(y1), (R)sign,   \
        static_cast<R*>(part), st)
    if (d->cplx) {
        if (yc) { if (real) PK_GEMVT(true, true, true); else PK_GEMVT(true, true, false); }
        else { if (real) PK_GEMVT(true, false, true); else PK_GEMVT(true, false, false); }
    } else {
        if (yc) { if (real) PK_GEMVT(false, true, true); else PK_GEMVT(false, true, false); }
        else PK_GEMVT(false, false, true);
    }
#undef PK_GEMVT
    PK_CHECK_LAUNCH();
    return PK_OK;
}

int fused_smem_attr(pk_dense* d) {  // set once at creation (not during graph capture)
    const int smem = (int)(2 * d->cols * 4);
    cudaError_t e = cudaSuccess;
    switch (d->fnv) {
        case 1: e = cudaFuncSetAttribute(dense_fused_f32_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
        case 2: e = cudaFuncSetAttribute(dense_fused_f32_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
        case 4: e = cudaFuncSetAttribute(dense_fused_f32_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
        case 8: e = cudaFuncSetAttribute(dense_fused_f32_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
        default: e = cudaFuncSetAttribute(dense_fused_f32_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
    }
    if (e != cudaSuccess) return fail(PK_ERR_CUDA, "fused kernel attribute: %s", cudaGetErrorString(e));
    return PK_OK;
}

int launch_fused(pk_dense* d, int use_state, cudaStream_t s) {
    const size_t smem = (size_t)2 * d->cols * 4;
#define PK_FUSED(NV)                                                                              \
    do {                                                                                          \
        dense_fused_f32_kernel<NV><<<d->fgrid, kFusedThreads, smem, s>>>(                         \
            static_cast<const float*>(d->K), d->rows, (int)d->cols,                              \
            static_cast<const float*>(d->xb[0]), static_cast<const float*>(d->xb[1]),            \
            static_cast<const float*>(d->ybuf), static_cast<float*>(d->fpart), d->rpart, d->st,  \
            use_state);                                                                           \
    } while (0)
    switch (d->fnv) {
        case 1: PK_FUSED(1); break;
        case 2: PK_FUSED(2); break;
        case 4: PK_FUSED(4); break;
        case 8: PK_FUSED(8); break;
        default: PK_FUSED(12); break;
    }
#undef PK_FUSED
    PK_CHECK_LAUNCH();
    return PK_OK;
}

// the whole solve on `s` (captured into a graph by pk_dense_reconstruct)
template <typename R>
int record_dense(pk_dense* d, int nx, int ny, int iters, cudaStream_t s) {
    const int P = nx * ny;
    const int64_t nr = d->rows * (d->cplx ? 2 : 1);  // residual scalars
    const int pb = (P + kDenseThreads - 1) / kDenseThreads;
    const int stop_blocks = std::min(pb, 148 * 2);
    R* xb0 = static_cast<R*>(d->xb[0]);
    R* xb1 = static_cast<R*>(d->xb[1]);
    if (d->fused) {
        dense_init_kernel<R><<<pb, kDenseThreads, 0, s>>>(xb0, P, d->st, nullptr, nullptr, 0, nullptr);
        PK_CHECK_LAUNCH();
        PK_TRY(launch_fused(d, 0, s));  // r0 = -y: gradient partials and sum y^2
        dense_stop_kernel<R><<<1, kDenseThreads, 0, s>>>(xb0, xb1, nx, ny, d->rpart, d->fgrid,
                                                         d->ipart, d->prm, d->st, d->hist, d->status, 1);
        PK_CHECK_LAUNCH();
        for (int k = 0; k < iters; ++k) {
            dense_update_kernel<R><<<pb, kDenseThreads, 0, s>>>(xb0, xb1, static_cast<const R*>(d->fpart),
                                                                d->fgrid, nx, ny, d->prm, d->st);
            PK_CHECK_LAUNCH();
            PK_TRY(launch_fused(d, 1, s));
            dense_stop_kernel<R><<<stop_blocks, kDenseThreads, 0, s>>>(
                xb0, xb1, nx, ny, d->rpart, d->fgrid, d->ipart, d->prm, d->st, d->hist, d->status, 0);
            PK_CHECK_LAUNCH();
        }
    } else {
        const int ib = (int)std::max<int64_t>(pb, (nr + kDenseThreads - 1) / kDenseThreads);
        dense_init_kernel<R><<<ib, kDenseThreads, 0, s>>>(xb0, P, d->st, static_cast<const R*>(d->ybuf),
                                                          static_cast<R*>(d->rb), nr, d->rpart);
        PK_CHECK_LAUNCH();
        dense_stop_kernel<R><<<1, kDenseThreads, 0, s>>>(xb0, xb1, nx, ny, d->rpart, ib, d->ipart,
                                                         d->prm, d->st, d->hist, d->status, 1);
        PK_CHECK_LAUNCH();
        for (int k = 0; k < iters; ++k) {
            PK_TRY(launch_gemvt<R>(d, d->rb, d->rb, d->cplx, true, 1.0, d->part, d->st, s));
            dense_update_kernel<R><<<pb, kDenseThreads, 0, s>>>(xb0, xb1, static_cast<const R*>(d->part),
                                                                d->splits, nx, ny, d->prm, d->st);
            PK_CHECK_LAUNCH();
            PK_TRY(launch_gemv<R>(d, xb0, xb1, 0, d->ybuf, d->rb, d->rb, d->rpart, d->st, s));
            dense_stop_kernel<R><<<stop_blocks, kDenseThreads, 0, s>>>(
                xb0, xb1, nx, ny, d->rpart, d->gemv_grid, d->ipart, d->prm, d->st, d->hist, d->status, 0);
            PK_CHECK_LAUNCH();
        }
    }
    dense_copy_out_kernel<R><<<pb, kDenseThreads, 0, s>>>(xb0, xb1, d->st, static_cast<R*>(d->xout), P);
    PK_CHECK_LAUNCH();
    return PK_OK;
}

}  // namespace

extern "C" {

int pk_dense_create(int64_t rows, int64_t cols, int32_t dtype, int32_t complex_entries,
                    int32_t device, pk_dense** out) {
    if (!out) return fail(PK_ERR_INVALID, "NULL argument");
    *out = nullptr;
    if (rows < 1 || cols < 1) return fail(PK_ERR_INVALID, "matrix must be at least 1 x 1");
    if (dtype != PK_F32 && dtype != PK_F64) return fail(PK_ERR_INVALID, "bad dtype %d", dtype);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(PK_ERR_CUDA, "no CUDA device available (the B200 kernels have no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(PK_ERR_INVALID, "bad device %d", device);
    DeviceGuard g(device);
    pk_dense* d = new pk_dense();
    d->device = device;
    d->dtype = dtype;
    d->cplx = complex_entries ? 1 : 0;
    d->rows = rows;
    d->cols = cols;
    if (cols % dense_E(d) != 0) {
        delete d;
        return fail(PK_ERR_UNSUPPORTED, "columns (%lld) must be a multiple of %d (16-byte rows)",
                    (long long)cols, dense_E(d));
    }
    const int sms = 148;
    d->gemv_grid = sms * 8;
    const int64_t tiles = (cols / dense_E(d) + kDenseThreads - 1) / kDenseThreads;
    d->splits = (int)std::max<int64_t>(1, std::min<int64_t>(rows, (4 * sms + tiles - 1) / tiles));
    d->fnv = fused_nv(cols);
    d->fused = (dtype == PK_F32 && !d->cplx && cols % 4 == 0 && d->fnv > 0 &&
                2 * cols * 4 <= 200 * 1024 && !getenv("PK_DENSE_TWOPASS")) ? 1 : 0;
    d->fgrid = sms;
    const size_t es = dsize(d) * (d->cplx ? 2 : 1);
    int rc = PK_OK;
    auto A = [&](int r) { if (rc == PK_OK) rc = r; };
    A(dalloc(d, reinterpret_cast<unsigned char**>(&d->K), (size_t)rows * cols * es));
    // (a real K's adjoint of a complex y has complex partials too)
    A(dalloc(d, reinterpret_cast<unsigned char**>(&d->part), (size_t)d->splits * cols * dsize(d) * 2));
    if (d->fused) A(dalloc(d, reinterpret_cast<unsigned char**>(&d->fpart), (size_t)d->fgrid * cols * 4));
    const int64_t nr = rows * (d->cplx ? 2 : 1);
    const int64_t rp = std::max<int64_t>({(int64_t)d->gemv_grid, (int64_t)d->fgrid,
                                          (nr + kDenseThreads - 1) / kDenseThreads,
                                          (cols + kDenseThreads - 1) / kDenseThreads});
    A(dalloc(d, &d->rpart, (size_t)rp));
    A(dalloc(d, reinterpret_cast<unsigned char**>(&d->ybuf), (size_t)rows * es));
    A(dalloc(d, reinterpret_cast<unsigned char**>(&d->rb), (size_t)rows * es));
    A(dalloc(d, &d->st, 1));
    A(dalloc(d, &d->prm, 1));
    A(dalloc(d, &d->status, 2));
    if (rc == PK_OK && cudaStreamCreateWithFlags(&d->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
        rc = fail(PK_ERR_CUDA, "stream creation failed");
    if (rc == PK_OK && d->fused) rc = fused_smem_attr(d);
    if (rc != PK_OK) {
        pk_dense_destroy(d);
        return rc;
    }
    *out = d;
    return PK_OK;
}

int pk_dense_destroy(pk_dense* d) {
    if (!d) return PK_OK;
    DeviceGuard g(d->device);
    void* ptrs[] = {d->K, d->part, d->fpart, d->rpart, d->ipart, d->xb[0], d->xb[1], d->rb,
                    d->ybuf, d->xout, d->hist, d->status, d->st, d->prm, d->Kt, d->bhi, d->blo,
                    d->tcpart};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    if (d->exec) cudaGraphExecDestroy(d->exec);
    if (d->cap_stream) cudaStreamDestroy(d->cap_stream);
    delete d;
    return PK_OK;
}

int pk_dense_get_info(const pk_dense* d, pk_dense_info* o) {
    if (!d || !o) return fail(PK_ERR_INVALID, "NULL argument");
    o->rows = d->rows;
    o->cols = d->cols;
    o->dtype = d->dtype;
    o->complex_entries = d->cplx;
    o->fused = d->fused;
    o->splits = d->splits;
    o->device_bytes = d->device_bytes;
    return PK_OK;
}

int pk_dense_set_entries(pk_dense* d, const double* entries, int32_t on_device, void* stream) {
    if (!d || !entries) return fail(PK_ERR_INVALID, "NULL argument");
    DeviceGuard g(d->device);
    cudaStream_t s = S(stream);
    const size_t n = (size_t)d->rows * d->cols * (d->cplx ? 2 : 1);  // scalars
    if (d->dtype == PK_F64) {
        PK_CUDA(cudaMemcpyAsync(d->K, entries, n * 8, on_device ? cudaMemcpyDeviceToDevice
                                                                 : cudaMemcpyHostToDevice, s));
        return PK_OK;
    }
    // fp32 plan: convert in chunks through a device staging buffer
    const size_t chunk = std::min(n, (size_t)32 << 20);
    double* stage = nullptr;
    if (!on_device) PK_CUDA(cudaMallocAsync(&stage, chunk * 8, s));
    for (size_t off = 0; off < n; off += chunk) {
        const size_t m = std::min(chunk, n - off);
        const double* src = entries + off;
        if (!on_device) {
            PK_CUDA(cudaMemcpyAsync(stage, src, m * 8, cudaMemcpyHostToDevice, s));
            src = stage;
        }
        narrow_kernel<float><<<148 * 8, kThreads, 0, s>>>(src, static_cast<float*>(d->K) + off, m);
        PK_CHECK_LAUNCH();
    }
    if (stage) PK_CUDA(cudaFreeAsync(stage, s));
    return PK_OK;
}

int pk_dense_from_plan(pk_dense* d, const pk_plan* p, void* stream) {
    if (!d || !p) return fail(PK_ERR_INVALID, "NULL argument");
    if (d->cplx) return fail(PK_ERR_INVALID, "the time-domain matrix is real");
    if (p->M != p->Mall || (int64_t)p->M * p->Q != d->rows || (int64_t)p->P != d->cols)
        return fail(PK_ERR_INVALID, "plan (%d sensors x %d samples, %d pixels) does not match the %lld x %lld matrix",
                    p->M, p->Q, p->P, (long long)d->rows, (long long)d->cols);
    if (p->device != d->device) return fail(PK_ERR_INVALID, "plan and matrix live on different devices");
    DeviceGuard g(d->device);
    cudaStream_t s = S(stream);
    PK_CUDA(cudaMemsetAsync(d->K, 0, (size_t)d->rows * d->cols * dsize(d), s));
    if (d->dtype == PK_F32)
        dense_from_geometry_kernel<float><<<148 * 8, kDenseThreads, 0, s>>>(
            p->px, p->py, p->sx, p->sy, p->cdt, p->w, p->nx, p->P, p->M, p->Q, static_cast<float*>(d->K));
    else
        dense_from_geometry_kernel<double><<<148 * 8, kDenseThreads, 0, s>>>(
            p->px, p->py, p->sx, p->sy, p->cdt, p->w, p->nx, p->P, p->M, p->Q, static_cast<double*>(d->K));
    PK_CHECK_LAUNCH();
    return PK_OK;
}

int pk_dense_matvec(pk_dense* d, const void* x, int32_t x_complex, void* y, void* stream) {
    if (!d || !x || !y) return fail(PK_ERR_INVALID, "NULL argument");
    DeviceGuard g(d->device);
    cudaStream_t s = S(stream);
    if (d->dtype == PK_F32) return launch_gemv<float>(d, x, x, x_complex, nullptr, y, y, nullptr, nullptr, s);
    return launch_gemv<double>(d, x, x, x_complex, nullptr, y, y, nullptr, nullptr, s);
}

int pk_dense_adjoint(pk_dense* d, const void* y, int32_t y_complex, void* out, double scale,
                     void* stream) {
    if (!d || !y || !out) return fail(PK_ERR_INVALID, "NULL argument");
    DeviceGuard g(d->device);
    cudaStream_t s = S(stream);
    const bool oc = d->cplx || y_complex;
    const int64_t n = d->cols * (oc ? 2 : 1);
    const unsigned blocks = (unsigned)((n + kDenseThreads - 1) / kDenseThreads);
    if (d->dtype == PK_F32) {
        PK_TRY(launch_gemvt<float>(d, y, y, y_complex, false, 1.0, d->part, nullptr, s));
        dense_reduce_kernel<float><<<blocks, kDenseThreads, 0, s>>>(
            static_cast<const float*>(d->part), d->splits, n, (float)scale, static_cast<float*>(out));
    } else {
        PK_TRY(launch_gemvt<double>(d, y, y, y_complex, false, 1.0, d->part, nullptr, s));
        dense_reduce_kernel<double><<<blocks, kDenseThreads, 0, s>>>(
            static_cast<const double*>(d->part), d->splits, n, scale, static_cast<double*>(out));
    }
    PK_CHECK_LAUNCH();
    return PK_OK;
}

// ---- multi-frame products on the tensor cores (pk_tc.cuh) ----
namespace {

typedef CUresult (*TmapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                 CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                 CUtensorMapFloatOOBfill);

TmapEncodeFn tmap_encode() {
    static TmapEncodeFn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<TmapEncodeFn>(f);
    }
    return fn;
}

// fp32 [rows][cols] row-major, 32-column x box_rows boxes, 128-B swizzle (pk_tc.cuh)
int tc_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows) {
    TmapEncodeFn enc = tmap_encode();
    if (!enc) return fail(PK_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)kTcBK, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    if (enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(PK_ERR_INVALID, "tensor map rejected (%lld x %lld)", (long long)rows, (long long)cols);
    return PK_OK;
}

cudaError_t tc_opt_in() {
    static bool done = false;
    if (done) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes(32));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tc_gemm_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes(64));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tc_gemm_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes(128));
    done = e == cudaSuccess;
    return e;
}

// C[f][r] = sum_k A[r][k] B[f][k] for f < frames (A fp32 [R][Kd] in HBM, B fp32 [frames][Kd])
int tc_products(pk_dense* d, const float* A, int64_t R, int64_t Kd, int frames, const float* B, float* C,
                cudaStream_t s) {
    if (frames < 1 || frames > 128) return fail(PK_ERR_INVALID, "frames must be 1..128, got %d", frames);
    if (Kd % 4 || R > INT_MAX || Kd > INT_MAX) return fail(PK_ERR_UNSUPPORTED, "matrix shape unsupported by the tensor-core path");
    const int N = frames <= 32 ? 32 : (frames <= 64 ? 64 : 128);
    const size_t nb = (size_t)frames * Kd;
    if (d->b_cap < nb) {
        if (d->bhi) cudaFree(d->bhi);
        if (d->blo) cudaFree(d->blo);
        d->bhi = d->blo = nullptr;
        d->b_cap = 0;
        PK_TRY(dalloc(d, &d->bhi, nb));
        PK_TRY(dalloc(d, &d->blo, nb));
        d->b_cap = nb;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
    const int tiles = (int)((R + kTcBM - 1) / kTcBM);
    const int nkb = (int)((Kd + kTcBK - 1) / kTcBK);
    // split K until the grid covers the GPU twice (at least 64 K blocks per split)
    int splits = 1;
    while (tiles * splits < 2 * sms && nkb / (2 * splits) >= 64 && splits < 16) splits *= 2;
    if (splits > 1 && d->part_cap < (size_t)splits * N * R) {
        if (d->tcpart) cudaFree(d->tcpart);
        d->tcpart = nullptr;
        d->part_cap = 0;
        PK_TRY(dalloc(d, &d->tcpart, (size_t)splits * N * R));
        d->part_cap = (size_t)splits * N * R;
    }
    CUtensorMap ma, mbh, mbl;
    PK_TRY(tc_map(&ma, A, R, Kd, kTcBM));
    PK_TRY(tc_map(&mbh, d->bhi, frames, Kd, N));
    PK_TRY(tc_map(&mbl, d->blo, frames, Kd, N));
    PK_CUDA(tc_opt_in());
    tc_split_kernel<<<2 * sms, 256, 0, s>>>(B, d->bhi, d->blo, nb);
    float* out = splits > 1 ? d->tcpart : C;
    const dim3 grid(tiles, splits);
    // (rows of frames >= `frames` read as zeros: out-of-bounds box rows; only the first
    //  `frames` frames of C / the partials are written)
    switch (N) {
        case 32: tc_gemm_kernel<32><<<grid, kTcThreads, tc_smem_bytes(32), s>>>(ma, mbh, mbl, out, (int)R, (int)Kd, splits, frames); break;
        case 64: tc_gemm_kernel<64><<<grid, kTcThreads, tc_smem_bytes(64), s>>>(ma, mbh, mbl, out, (int)R, (int)Kd, splits, frames); break;
        default: tc_gemm_kernel<128><<<grid, kTcThreads, tc_smem_bytes(128), s>>>(ma, mbh, mbl, out, (int)R, (int)Kd, splits, frames); break;
    }
    if (splits > 1) tc_split_sum_kernel<<<2 * sms, 256, 0, s>>>(d->tcpart, C, (size_t)frames * R, splits, (size_t)N * R);
    PK_CHECK_LAUNCH();
    return PK_OK;
}

}  // namespace

int pk_dense_matmat(pk_dense* d, int32_t frames, const void* x, void* y, void* stream) {
    if (!d || !x || !y) return fail(PK_ERR_INVALID, "NULL argument");
    if (d->dtype != PK_F32 || d->cplx) return fail(PK_ERR_UNSUPPORTED, "tensor-core products need a real fp32 matrix");
    DeviceGuard g(d->device);
    return tc_products(d, static_cast<const float*>(d->K), d->rows, d->cols, frames, static_cast<const float*>(x),
                       static_cast<float*>(y), S(stream));
}

int pk_dense_rmatmat(pk_dense* d, int32_t frames, const void* y, void* g_out, void* stream) {
    if (!d || !y || !g_out) return fail(PK_ERR_INVALID, "NULL argument");
    if (d->dtype != PK_F32 || d->cplx) return fail(PK_ERR_UNSUPPORTED, "tensor-core products need a real fp32 matrix");
    DeviceGuard g(d->device);
    cudaStream_t s = S(stream);
    if (!d->Kt) {  // K^T, once: both tensor-core operands stay K-major
        PK_TRY(dalloc(d, reinterpret_cast<float**>(&d->Kt), (size_t)d->rows * d->cols));
        d->device_bytes += d->rows * d->cols * 4;
        const dim3 blk(32, 8), grd((unsigned)((d->cols + 31) / 32), (unsigned)((d->rows + 31) / 32));
        dense_transpose_kernel<<<grd, blk, 0, s>>>(static_cast<const float*>(d->K), static_cast<float*>(d->Kt),
                                                    d->rows, d->cols);
        PK_CHECK_LAUNCH();
    }
    return tc_products(d, static_cast<const float*>(d->Kt), d->cols, d->rows, frames, static_cast<const float*>(y),
                       static_cast<float*>(g_out), s);
}

int pk_dense_reconstruct(pk_dense* d, int32_t nx, int32_t ny, const pk_solver_params* prm,
                         const void* y, void* x_out, double* hist, int32_t* status, void* stream) {
    if (!d || !prm || !y || !x_out || !hist || !status) return fail(PK_ERR_INVALID, "NULL argument");
    if (nx < 1 || ny < 1 || (int64_t)nx * ny != d->cols)
        return fail(PK_ERR_INVALID, "grid %d x %d does not match %lld columns", nx, ny, (long long)d->cols);
    if (prm->iterations < 1) return fail(PK_ERR_INVALID, "iterations must be >= 1");
    if (!(prm->tv_epsilon > 0)) return fail(PK_ERR_INVALID, "tv_epsilon must be > 0");
    if (!(prm->alpha >= 0) || !(prm->beta >= 0)) return fail(PK_ERR_INVALID, "alpha and beta must be >= 0");
    if (!(prm->step > 0)) return fail(PK_ERR_INVALID, "step must be > 0");
    DeviceGuard g(d->device);
    cudaStream_t s = S(stream);
    const int P = nx * ny;
    const size_t ts = dsize(d);
    if (!d->xb[0]) {
        PK_TRY(dalloc(d, reinterpret_cast<unsigned char**>(&d->xb[0]), (size_t)P * ts));
        PK_TRY(dalloc(d, reinterpret_cast<unsigned char**>(&d->xb[1]), (size_t)P * ts));
        PK_TRY(dalloc(d, reinterpret_cast<unsigned char**>(&d->xout), (size_t)P * ts));
        PK_TRY(dalloc(d, &d->ipart, (size_t)3 * 148 * 2));
    }
    if (d->hist_cap < prm->iterations) {
        if (d->hist) cudaFree(d->hist);
        d->hist = nullptr;
        PK_TRY(dalloc(d, &d->hist, (size_t)4 * prm->iterations));
        d->hist_cap = prm->iterations;
        if (d->exec) { cudaGraphExecDestroy(d->exec); d->exec = nullptr; }
        d->g_iters = -1;
    }
    DevParams dp{};
    for (int f = 0; f < kMaxFrames; ++f) {
        dp.alpha[f] = prm->alpha;
        dp.beta[f] = prm->beta;
        dp.step[f] = prm->step;
        dp.eta_alpha[f] = prm->step * prm->alpha;
    }
    dp.eps = prm->tv_epsilon;
    dp.tolerance = prm->tolerance;
    dp.iterations = prm->iterations;
    dp.nonneg = prm->nonneg ? 1 : 0;
    PK_CUDA(cudaMemcpyAsync(d->prm, &dp, sizeof(dp), cudaMemcpyHostToDevice, s));
    PK_CUDA(cudaMemcpyAsync(d->ybuf, y, (size_t)d->rows * ts * (d->cplx ? 2 : 1), cudaMemcpyDeviceToDevice, s));
    if (!d->exec || d->g_iters != prm->iterations || d->g_nx != nx || d->g_ny != ny) {
        if (d->exec) { cudaGraphExecDestroy(d->exec); d->exec = nullptr; }
        PK_CUDA(cudaStreamBeginCapture(d->cap_stream, cudaStreamCaptureModeThreadLocal));
        const int rc = d->dtype == PK_F32 ? record_dense<float>(d, nx, ny, prm->iterations, d->cap_stream)
                                          : record_dense<double>(d, nx, ny, prm->iterations, d->cap_stream);
        cudaGraph_t gr = nullptr;
        cudaError_t e = cudaStreamEndCapture(d->cap_stream, &gr);
        if (rc != PK_OK) { if (gr) cudaGraphDestroy(gr); return rc; }
        if (e != cudaSuccess) return fail(PK_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
        e = cudaGraphInstantiate(&d->exec, gr, 0);
        cudaGraphDestroy(gr);
        if (e != cudaSuccess) return fail(PK_ERR_CUDA, "graph instantiation failed: %s", cudaGetErrorString(e));
        d->g_iters = prm->iterations;
        d->g_nx = nx;
        d->g_ny = ny;
    }
    PK_CUDA(cudaGraphLaunch(d->exec, s));
    PK_CUDA(cudaMemcpyAsync(x_out, d->xout, (size_t)P * ts, cudaMemcpyDeviceToDevice, s));
    PK_CUDA(cudaMemcpyAsync(hist, d->hist, (size_t)4 * prm->iterations * 8, cudaMemcpyDeviceToDevice, s));
    PK_CUDA(cudaMemcpyAsync(status, d->status, 2 * 4, cudaMemcpyDeviceToDevice, s));
    return PK_OK;
}

}  // extern "C"
