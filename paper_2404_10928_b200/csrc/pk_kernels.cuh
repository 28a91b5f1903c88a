// pk_kernels.cuh -- sm_100a kernels of the iterative reconstruction hot path.
//
//   K1 bp_f32 / bp_f64     back-projection K^T r (recon.py:327), optionally fused with the
//                          TV gradient, soft threshold and non-negativity (recon.py:330-338)
//   K2 fp_f32 / fp_f64     projection K x (recon.py:342) into a fixed-point accumulator
//   K3 finalize            r = K x - y, the residual pair table for the next K1, sum r^2,
//                          and (solver mode) the objective + stopping rules (recon.py:346-363)
//   misc                   table-from-trace, max|x| scale, update for sharded runs, index dump
//
// fp32 kernels are templated on NF, the number of frames that share one geometry (1, 2, 4):
// the delay of a sensor-pixel pair is evaluated once and applied to all NF frames.
// See DESIGN.md for the data layout and the per-interaction instruction budget.
#pragma once
#include <type_traits>

#include "pk_common.cuh"

namespace pk {

template <int NF>
struct Lg;
template <>
struct Lg<1> { static constexpr int v = 0; };
template <>
struct Lg<2> { static constexpr int v = 1; };
template <>
struct Lg<4> { static constexpr int v = 2; };

// soft threshold of recon.py:158-159 keeping NaN (np.maximum propagates it), then the
// optional non-negativity clamp of recon.py:337-338
template <typename T>
__device__ __forceinline__ T prox(T v, T lam, bool nonneg) {
    T mag = fabs(v) - lam;
    mag = (mag != mag) ? mag : fmax(mag, (T)0);
    T xn = (v > (T)0) ? mag : ((v < (T)0) ? -mag : (v != v ? v : (T)0));
    if (nonneg) xn = (xn != xn) ? xn : fmax(xn, (T)0);
    return xn;
}

// gradient of the eps-smoothed TV at pixel p (recon.py:178-189, same accumulation order)
template <typename T>
__device__ __forceinline__ T tv_grad_at(const T* x, size_t p, int i, int j, int nx, int ny, T e2) {
    const T x0 = x[p];
    T t = 0;
    if (i < nx - 1) { const T d = x[p + 1] - x0; t -= d / sqrt(d * d + e2); }
    if (i > 0) { const T d = x0 - x[p - 1]; t += d / sqrt(d * d + e2); }
    if (j < ny - 1) { const T d = x[p + nx] - x0; t -= d / sqrt(d * d + e2); }
    if (j > 0) { const T d = x0 - x[p - nx]; t += d / sqrt(d * d + e2); }
    return t;
}

// ===========================================================================
// K1 -- back-projector, fp32.  CTA = 32x32 pixel tile x a slice of the sensors, 256
// threads, thread owns the pixels (i0 + lx + 8k, j0 + 4*warp + ly), k = 0..3, so every
// warp instruction covers a compact 8x4 pixel footprint.  Sensors are processed in chunks
// of CS; the per-(tile, sensor) window of the residual pair table is brought into shared
// memory by the TMA engine (cp.async.bulk + mbarrier), NBUF-deep ring, refilled by the
// last warp to finish with a buffer (no CTA barrier in the loop).
//
// pair table entry s of sensor m, frame f (layout [m][s][f]): {r[s-1], r[s]-r[s-1]}
// (r[-1] = r[Q] = r[Q+1] = 0), so one interaction is
//     acc += r[s0-1] + f*(r[s0]-r[s0-1])  == (1-f) r[s0-1] + f r[s0],
// the two weights of build_time_matrix (forward.py:189-194) without the w factor.
// One LDS.64 (NF = 1) / LDS.128 (NF = 2) / 2x LDS.128 (NF = 4) per interaction.
// ===========================================================================
struct BpArgs {
    const float2* table;  // [M][TS][NF]
    const float* pxs;     // [nx] scaled pixel x
    const float* pys;     // [ny]
    const float* sxs;     // [M]
    const float* sys;     // [M]
    int nx, ny, M, Q, TS, L, CS, nbuf, tiles_x;
    float qclamp;         // Q + 1.5 (truncation clamp of the delay)
    // EPI == 0: out[f][p] = gscale * acc
    float* out;
    float gscale;
    // EPI == 1: fused update, x from xb[iter & 1] to xb[(iter+1) & 1] (each [NF][P])
    float* xb0;
    float* xb1;
    const DevParams* prm;
    DevState* st;
    double* part;         // [tiles][NF][4]
    int bits;             // projector fixed-point bits (scale = 2^bits / max|x'|)
    // sensor split: CTA (tile, s) sums sensors [s*ms, min(M, (s+1)*ms)); the last CTA of a
    // tile to finish adds the S partials in split order (deterministic) and runs the epilogue
    int split, ms;
    float* gpart;         // [split][NF][P]
    uint32_t* tile_cnt;   // [tiles]
};

template <int NF, bool EPI, bool CLAMP, bool ATRICK>
__global__ void __launch_bounds__(kThreads, NF == 1 ? 4 : (NF == 2 ? 3 : 2)) bp_f32_kernel(BpArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ float red_f[kThreads / 32];
    __shared__ double red_d[kThreads / 32];
    __shared__ int last_flag;
    __shared__ uint32_t done_cnt[8];  // per-buffer count of warps finished with it
    constexpr int LG = Lg<NF>::v;

    int iter = 0;
    if (EPI) {
        if (a.st->all_stopped) return;
        iter = a.st->iter;
    }
    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int i0 = tx * kBpTile, j0 = ty * kBpTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = lane & 7, ly = lane >> 3;
    const int j = j0 + warp * 4 + ly;
    const int mbase = blockIdx.y * a.ms;
    const int mcount = min(a.ms, a.M - mbase);
    const size_t P = (size_t)a.nx * a.ny;

    // two independent accumulator chains per pixel and frame (FFMA chain, FADD chain)
    float px[4], acc[4][NF], acc2[4][NF];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        px[k] = __ldg(a.pxs + min(i0 + lx + 8 * k, a.nx - 1));
#pragma unroll
        for (int f = 0; f < NF; ++f) acc[k][f] = acc2[k][f] = 0.f;
    }
    const float py = __ldg(a.pys + min(j, a.ny - 1));

    // shared layout: windows [nbuf][CS][L][NF] float2 | sconst [nbuf][CS] float4 | bars [nbuf]
    const size_t win_bytes = (size_t)a.nbuf * a.CS * a.L * 8 * NF;
    float4* sconst = reinterpret_cast<float4*>(smem + win_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + win_bytes + (size_t)a.nbuf * a.CS * 16);
    const uint32_t win_s = smem_u32(smem);
    const uint32_t bar_s = smem_u32(bars);

    // tile rectangle in scaled coordinates (for the per-sensor delay windows)
    const float X0 = __ldg(a.pxs + i0), X1 = __ldg(a.pxs + min(i0 + kBpTile - 1, a.nx - 1));
    const float Y0 = __ldg(a.pys + j0), Y1 = __ldg(a.pys + min(j0 + kBpTile - 1, a.ny - 1));

    if (threadIdx.x == 0) {
        for (int b = 0; b < a.nbuf; ++b) {
            mbar_init(bar_s + 8 * b, 1);
            done_cnt[b] = 0;
        }
        fence_barrier_init();
    }
    __syncthreads();

    const int nchunks = (mcount + a.CS - 1) / a.CS;
    // the calling warp computes the windows of a chunk and launches its bulk copies
    auto issue = [&](int c, int b) {
        const int m = mbase + c * a.CS + lane;
        const int n = min(a.CS, mcount - c * a.CS);
        if (lane < n) {
            const float sx = __ldg(a.sxs + m), sy = __ldg(a.sys + m);
            const float cx = fminf(fmaxf(sx, X0), X1), cy = fminf(fmaxf(sy, Y0), Y1);
            float dmin = sqrtf((cx - sx) * (cx - sx) + (cy - sy) * (cy - sy));
            if (CLAMP) dmin = fminf(dmin, a.qclamp);
            int lo = (int)floorf(dmin) - 1;
            lo = max(lo, 0) & ~1;
            lo = min(lo, a.TS - a.L);
            const uint32_t dst = win_s + (uint32_t)((b * a.CS + lane) * a.L) * (8u * NF);
            const uint32_t adj = dst - (8u * NF) * (uint32_t)lo - (8u * NF) * kTwo23Bits;
            sconst[b * a.CS + lane] = make_float4(sx, sy, __uint_as_float(adj), 0.f);
            __syncwarp(__activemask());
            if (lane == 0) mbar_expect_tx(bar_s + 8 * b, (uint32_t)(n * a.L * 8 * NF));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp(__activemask());
            bulk_g2s(dst, a.table + ((size_t)m * a.TS + lo) * NF, (uint32_t)(a.L * 8 * NF),
                     bar_s + 8 * b);
        }
    };
    if (warp == 0) {
        for (int c = 0; c < min(a.nbuf, nchunks); ++c) issue(c, c);
    }

    for (int c = 0; c < nchunks; ++c) {
        const int b = c % a.nbuf;
        mbar_wait(bar_s + 8 * b, (uint32_t)((c / a.nbuf) & 1));
        const int n = min(a.CS, mcount - c * a.CS);
        const float4* sc = sconst + b * a.CS;
#pragma unroll 2
        for (int s = 0; s < n; ++s) {
            const float4 q = sc[s];
            const float ey = py - q.y;
            const float ey2 = ey * ey;
            const uint32_t adj = __float_as_uint(q.z);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float ex = px[k] - q.x;
                float u = sqrt_approx(fmaf(ex, ex, ey2));
                if (CLAMP) u = fminf(u, a.qclamp);
                const float tb = __fadd_rd(u, kTwo23);      // 2^23 + floor(u)
                const uint32_t ad = adj + (__float_as_uint(tb) << (3 + LG));
                // ATRICK table {r[s-1] - s*D, D}: value = u*D + A; else value = f*D + r[s-1]
                const float w = ATRICK ? u : u - (tb - kTwo23);
                float A[NF], D[NF];
                if (NF == 1) {
                    const float2 v = lds_f2(ad);
                    A[0] = v.x; D[0] = v.y;
                } else {
#pragma unroll
                    for (int h = 0; h < NF / 2; ++h) {
                        const float4 v = lds_f4(ad + 16 * h);
                        A[2 * h] = v.x; D[2 * h] = v.y; A[2 * h + 1] = v.z; D[2 * h + 1] = v.w;
                    }
                }
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    acc[k][f] = fmaf(w, D[f], acc[k][f]);
                    acc2[k][f] += A[f];
                }
            }
        }
        // the last warp to finish with buffer b refills it (acq_rel shared counter)
        __syncwarp();
        uint32_t prev = 0;
        if (lane == 0) {
            const uint32_t addr = smem_u32(&done_cnt[b]);
            asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(prev) : "r"(addr) : "memory");
        }
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == kThreads / 32 - 1) {
            if (lane == 0) done_cnt[b] = 0;
            if (c + a.nbuf < nchunks) issue(c + a.nbuf, b);
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int f = 0; f < NF; ++f) acc[k][f] += acc2[k][f];

    if (a.split > 1) {
        // publish this split's partial sums; the tile's last CTA combines them in order
        if (j < a.ny) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = i0 + lx + 8 * k;
                if (i < a.nx)
#pragma unroll
                    for (int f = 0; f < NF; ++f)
                        a.gpart[((size_t)blockIdx.y * NF + f) * P + (size_t)j * a.nx + i] = acc[k][f];
            }
        }
        if (!last_block(a.tile_cnt + tile, a.split, &last_flag)) return;
        if (j < a.ny) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = i0 + lx + 8 * k;
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    float sum = 0.f;
                    if (i < a.nx)
                        for (int q = 0; q < a.split; ++q)
                            sum += __ldcg(a.gpart + ((size_t)q * NF + f) * P + (size_t)j * a.nx + i);
                    acc[k][f] = sum;
                }
            }
        }
    }

    if (!EPI) {
        if (j < a.ny) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = i0 + lx + 8 * k;
                if (i < a.nx)
#pragma unroll
                    for (int f = 0; f < NF; ++f)
                        a.out[f * P + (size_t)j * a.nx + i] = a.gscale * acc[k][f];
            }
        }
        return;
    }

    // ---- fused update epilogue (recon.py:327-338), per frame ----
    const float* xin = (iter & 1) ? a.xb1 : a.xb0;
    float* xout = (iter & 1) ? a.xb0 : a.xb1;
    const float eps = (float)a.prm->eps;
    const bool nonneg = a.prm->nonneg != 0;
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        const bool live = !a.st->fr[f].stopped;
        const float eta = (float)a.prm->step[f], lam = (float)a.prm->eta_alpha[f];
        const float beta = (float)a.prm->beta[f];
        const float* x = xin + f * P;
        float* xo = xout + f * P;
        float mx = 0.f, l1 = 0.f;
        int bad = 0;
        if (live && j < a.ny) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = i0 + lx + 8 * k;
                if (i >= a.nx) continue;
                const size_t p = (size_t)j * a.nx + i;
                float g = a.gscale * acc[k][f];
                if (beta > 0.f) g += beta * tv_grad_at<float>(x, p, i, j, a.nx, a.ny, eps * eps);
                const float xn = prox<float>(x[p] - eta * g, lam, nonneg);
                xo[p] = xn;
                if (!isfinite(xn)) bad = 1;
                mx = fmaxf(mx, fabsf(xn));
                l1 += fabsf(xn);
            }
        }
        mx = block_max(mx, red_f);
        const float l1b = block_sum(l1, red_f);
        const int badb = __syncthreads_or(bad);
        if (threadIdx.x == 0) {
            double* pp = a.part + 4 * ((size_t)tile * NF + f);
            pp[0] = mx;
            pp[1] = l1b;
            pp[2] = badb;
        }
    }
    if (last_block(&a.st->cnt_bp, gridDim.x, &last_flag)) {
#pragma unroll 1
        for (int f = 0; f < NF; ++f) {
            double m2 = 0.0, s2 = 0.0, b2 = 0.0;
            for (int q = threadIdx.x; q < (int)gridDim.x; q += kThreads) {
                const double* pp = a.part + 4 * ((size_t)q * NF + f);
                m2 = fmax(m2, pp[0]);
                s2 += pp[1];
                b2 += pp[2];
            }
            m2 = block_max(m2, red_d);
            s2 = block_sum(s2, red_d);
            b2 = block_sum(b2, red_d);
            if (threadIdx.x == 0 && !a.st->fr[f].stopped) {
                FrameState& fs = a.st->fr[f];
                fs.maxabs = m2;
                fs.l1sum = s2;
                fs.nonfinite = b2 > 0.0 ? 1 : 0;
                const double scl = (m2 > 0.0 && isfinite(m2)) ? ldexp(1.0, a.bits) / m2 : 0.0;
                fs.scale64 = scl;
                fs.scale32 = (float)scl;
            }
        }
    }
}

// ===========================================================================
// K1s -- back-projector, fp32, for D4-symmetric scenes (square grid centred on the ring
// centre, n even, M % 4 == 0 -- every BASELINE configuration).  The 8 elements g of the
// dihedral group map a pair (pixel p, sensor m) to (g p, g m) with the same distance, so
// one delay evaluation serves up to 8 pairs:
//   g:      0       1          2              3          4         5       6          7
//   pixel: (i,j)  (n-1-j,i)  (n-1-i,n-1-j)  (j,n-1-i)  (i,n-1-j)  (j,i)  (n-1-i,j)  (n-1-j,n-1-i)
//   sensor: m     m+M/4      m+M/2          m+3M/4     -m         M/4-m  M/2-m      3M/4-m
// Representative pixels are 32x32 tiles (tx, ty), tx >= ty, of the quadrant i, j >= n/2.
// Off-diagonal tiles (tx > ty) lie strictly below the diagonal and use all 8 images; a
// diagonal tile is closed under transposition, so all its pixels are representatives of
// the 4 rotations (g = 0..3) -- no idle lanes.  A thread owns the 4 representatives
// (i0 + lx + 8k, j0 + 4*warp + ly): every warp instruction covers an 8x4 footprint.
//
// Persistent CTAs: the (tile, chunk of kSymCS base sensors) sequence is cut host-side into
// equal-cost contiguous ranges (off-diagonal chunks cost 2, diagonal 1), one per CTA.  The
// image windows of a chunk (kSymCS x 8 windows of the pair table) are staged by the TMA
// engine (one cp.async.bulk per window) into an nbuf-deep ring; the last warp to finish a
// buffer refills it.  A CTA's partial sums of a tile go to one "slot" of part[]; the
// epilogue kernel adds a tile's slots in slot order (deterministic) and applies the update.
// Per pair: LDS.64 + FFMA + FADD, plus 1/NG of the delay (8 issue slots).
// ===========================================================================
constexpr int kSymTile = 32;
constexpr int kSymCS = 2;        // base sensors per chunk (x 8 images = 16 windows)
constexpr int kSymConsumers = 8; // consumer warps; warp 8 is the TMA producer
constexpr int kSymThreads = 32 * (kSymConsumers + 1);

// K1s epilogue: CTA (tile, image g, 8-column strip) adds the tile's partial slots (4 slot
// groups in parallel, then in order), maps the representatives to image g, and writes
// gscale * K^T r (EPI == false) or runs the fused update of recon.py:327-338 with the block
// statistics of the next projector scale.
struct BpSymEpiArgs {
    const float* part;        // [slots][8][4][kThreads]
    const int* tile_slot0;    // [ntiles + 1]
    const int* tiles;         // [ntiles]
    int n, bits, lanemap;
    float gscale;
    float* out;               // EPI == false
    float* xb0;               // EPI == true: x from xb[iter & 1] to xb[(iter + 1) & 1]
    float* xb1;
    const DevParams* prm;
    DevState* st;
    double* part_bp;          // [grid][4]
    float* xr;                // EPI == true, optional: rotation-packed copy of x' for the
                              // symmetric projector, [(n/2)^2][4] (fp_sym_f32_kernel)
    float* part_mx;           // DEFER: [grid] max |x'| per CTA (the projector reduces them)
    int ntiles;               // representative tiles per frame (units: frame-major tiles)
    int P;                    // pixels per frame (frame stride of x; x' packed: P / 4)
};

// rotation-packed index of pixel (i, j): the quadrant representative q = (qi, qj) in
// [h, n)^2 and rotation r with rot^r(q) = (i, j) (the image order of fp_sym_f32_kernel);
// returns 4 * ((qj - h) * h + (qi - h)) + r
__device__ __forceinline__ int sym_rot_index(int i, int j, int n) {
    const int h = n >> 1;
    int qi, qj, r;
    if (i >= h) {
        if (j >= h) { qi = i; qj = j; r = 0; }
        else { qi = n - 1 - j; qj = i; r = 3; }
    } else {
        if (j >= h) { qi = j; qj = n - 1 - i; r = 1; }
        else { qi = n - 1 - i; qj = n - 1 - j; r = 2; }
    }
    return 4 * ((qj - h) * h + (qi - h)) + r;
}

struct BpSymArgs {
    const float2* table;     // [M][TS] pair table
    const float* pxs;        // [n] scaled pixel x
    const float* pys;        // [n]
    const float* sxs;        // [M]
    const float* sys;        // [M]
    int n, M, TS, L, nbuf;
    int lanemap;             // 1: half-warps own 4x4 blocks of the 8x4 footprint; 0: 8x2 rows
    float qclamp;            // Q + 1.5
    const int* chunks;       // [total] (tile << 16) | chunk index within the tile
    const int* cta_chunk0;   // [grid + 1] chunk range of each CTA
    const int* cta_slot0;    // [grid] first partial slot of each CTA
    const int* tiles;        // [ntiles] (tx << 16) | ty
    float* part;             // [slots][8][4][kThreads]
    const DevState* st;      // solver mode: early exit once every frame stopped; else null
    const int* gid;          // [M] ring index of local sensor (base sensors are local)
    const int* loc;          // [Mall] local index of a ring sensor (the images of a base)
    int Mall;                // ring size (the D4 images are ring indices)
    int ntiles;              // tiles per frame: chunk tile indices are f * ntiles + tile
    size_t table_fstride;    // [frames][M][TS] pair tables: M * TS entries per frame
    // fused update (solver mode with the symmetric projector): the CTAs whose last tile is t
    // run the update of t once all of its partial slots are in (per-tile arrival counter);
    // the final arriver publishes the tile, waiting CTAs join within a bounded spin, and the 32
    // (image, 8-column strip) units of the tile are claimed one at a time
    int fuse;
    BpSymEpiArgs epi;
    uint32_t* tile_cnt;      // [ntiles] partial slots arrived (reset by the final arriver)
    uint32_t* tile_units;    // [ntiles] units claimed
    uint32_t* tile_done;     // [ntiles] launch id of the last publication
    long long spin_ns;       // how long a CTA waits for its last tile before leaving it
};

// lane -> (column, row) inside a warp's 8x4 footprint.  With lanemap 1 each half-warp
// covers a 4x4 block (delay span <= ~10 table entries at config 3), which lets the two
// half-warp phases of an LDS.64 share wavefronts more often than 8x2 rows.
__device__ __forceinline__ void sym_lane_xy(int lane, int lanemap, int& lx, int& ly) {
    if (lanemap) {
        lx = (lane & 3) | ((lane >> 4) << 2);
        ly = (lane >> 2) & 3;
    } else {
        lx = lane & 7;
        ly = lane >> 3;
    }
}

__device__ __forceinline__ void sym_pixel(int g, int i, int j, int n, int& ig, int& jg) {
    const int ri = n - 1 - i, rj = n - 1 - j;
    switch (g) {
        case 0: ig = i; jg = j; break;
        case 1: ig = rj; jg = i; break;
        case 2: ig = ri; jg = rj; break;
        case 3: ig = j; jg = ri; break;
        case 4: ig = i; jg = rj; break;
        case 5: ig = j; jg = i; break;
        case 6: ig = ri; jg = j; break;
        default: ig = rj; jg = ri; break;
    }
}

__device__ __forceinline__ int sym_sensor(int g, int m, int M) {
    const int q = M >> 2;
    int s;
    switch (g) {
        case 0: s = m; break;
        case 1: s = m + q; break;
        case 2: s = m + 2 * q; break;
        case 3: s = m + 3 * q; break;
        case 4: s = -m; break;
        case 5: s = q - m; break;
        case 6: s = 2 * q - m; break;
        default: s = 3 * q - m; break;
    }
    s %= M;
    return s < 0 ? s + M : s;
}

// one chunk: ns base sensors x 4 representatives x NG images
template <int NG, int IW>
__device__ __forceinline__ void sym_chunk(float (&acc)[4][8], const float (&px)[4], float py,
                                          const float4* sc, int ns, uint32_t img_stride,
                                          float qclamp) {
    for (int s = 0; s < ns; ++s) {
        const float4 q = sc[s];
        const float ey = py - q.y;
        const float ey2 = ey * ey;
        const uint32_t adj = __float_as_uint(q.z);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float ex = px[k] - q.x;
            const float u = fminf(sqrt_approx(fmaf(ex, ex, ey2)), qclamp);
            const float tb = __fadd_rd(u, kTwo23);  // 2^23 + floor(u)
            const float f = u - (tb - kTwo23);
            const uint32_t ad = adj + (__float_as_uint(tb) << 3);
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const float2 v = lds_f2(ad + (uint32_t)g * (IW > 0 ? (uint32_t)IW * 8u : img_stride));
                acc[k][g] += fmaf(f, v.y, v.x);  // (1-f) r[s0-1] + f r[s0]
            }
        }
    }
}

// units of the symmetric update (solver mode, deferred statistics): tile t, image g, 8-column
// strip k (unit index u = 4g + k), U units [u0, u0 + U) at once (every load of the U units in
// flight together) -- the tile's partial slots summed in slot order, mapped to image g, then
// TV gradient + prox + non-negativity (recon.py:327-338), x' written twice (image order and
// rotation-packed for the projector) and each unit's max |x'| partial.  256 threads; sync() is
// their barrier.  Shared scratch: part4 [U][3][64] float4, blk [U][256] float, red [U][8] float.
template <int U, typename Sync>
__device__ __forceinline__ void sym_epi_units(const BpSymEpiArgs& a, int t, int u0, int iter,
                                              float4* part4, float* blk, float* red, Sync sync) {
    const int tid = threadIdx.x;
    const int tp = __ldg(a.tiles + t);
    const int tx = tp >> 16, ty = tp & 0xffff;
    const int n = a.n, h = n >> 1;
    const int i0 = h + kSymTile * tx, j0 = h + kSymTile * ty;
    const int s0 = __ldg(a.tile_slot0 + t), s1 = __ldg(a.tile_slot0 + t + 1);
    const int sg = tid >> 6, q = tid & 63;
    int bx[U], by[U], bw[U];
    bool active[U];
#pragma unroll
    for (int v = 0; v < U; ++v) {
        const int u = u0 + v, k = u & 3, g = u >> 2;
        active[v] = u < 32 && !(tx == ty && g >= 4);
        int ia, ja, ib, jb;
        sym_pixel(g & 7, i0 + 8 * k, j0, n, ia, ja);
        sym_pixel(g & 7, i0 + 8 * k + 7, j0 + kSymTile - 1, n, ib, jb);
        bx[v] = min(ia, ib);
        by[v] = min(ja, jb);
        bw[v] = abs(ib - ia) + 1;
    }
    // the iterate and its TV neighbours are independent of the slot sums: loads first
    const float* x = (iter & 1) ? a.xb1 : a.xb0;
    float* xo = (iter & 1) ? a.xb0 : a.xb1;
    const float eta = (float)a.prm->step[0], lam = (float)a.prm->eta_alpha[0];
    const float beta = (float)a.prm->beta[0], eps = (float)a.prm->eps;
    const bool run = !a.st->fr[0].stopped;
    int pix[U];
    float xv[U], tvg[U];
#pragma unroll
    for (int v = 0; v < U; ++v) {
        const int ig = bx[v] + tid % bw[v], jg = by[v] + tid / bw[v];
        pix[v] = (run && active[v] && ig >= 0 && ig < n && jg >= 0 && jg < n) ? jg * n + ig : -1;
        xv[v] = pix[v] >= 0 ? x[pix[v]] : 0.f;
        tvg[v] = (pix[v] >= 0 && beta > 0.f) ? tv_grad_at<float>(x, pix[v], ig, jg, n, n, eps * eps) : 0.f;
    }
    float4 sum[U];
#pragma unroll
    for (int v = 0; v < U; ++v) sum[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    const size_t stride = 8 * 4 * kThreads / 4;  // float4s per slot
    for (int sb = s0 + sg; sb < s1; sb += 16) {
        float4 w4[U][4];
#pragma unroll
        for (int v = 0; v < U; ++v) {
            const int u = u0 + v;
            const float4* src = reinterpret_cast<const float4*>(a.part + (size_t)(u & 31) * kThreads) + q;
#pragma unroll
            for (int w = 0; w < 4; ++w)
                w4[v][w] = (active[v] && sb + 4 * w < s1) ? __ldcg(src + (size_t)(sb + 4 * w) * stride)
                                                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int v = 0; v < U; ++v)
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                sum[v].x += w4[v][w].x; sum[v].y += w4[v][w].y; sum[v].z += w4[v][w].z; sum[v].w += w4[v][w].w;
            }
    }
    if (sg > 0)
#pragma unroll
        for (int v = 0; v < U; ++v) part4[(v * 3 + sg - 1) * 64 + q] = sum[v];
    sync();
    if (sg == 0)
#pragma unroll
        for (int v = 0; v < U; ++v) {
            float4 sm = sum[v];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const float4 o = part4[(v * 3 + r) * 64 + q];
                sm.x += o.x; sm.y += o.y; sm.z += o.z; sm.w += o.w;
            }
            const float sv[4] = {sm.x, sm.y, sm.z, sm.w};
            const int u = u0 + v, k = u & 3, g = (u >> 2) & 7;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const int c = 4 * q + w;
                int lx, ly;
                sym_lane_xy(c & 31, a.lanemap, lx, ly);
                int ig, jg;
                sym_pixel(g, i0 + lx + 8 * k, j0 + 4 * (c >> 5) + ly, n, ig, jg);
                blk[v * 256 + (jg - by[v]) * bw[v] + (ig - bx[v])] = a.gscale * sv[w];
            }
        }
    sync();
    float mx[U];
#pragma unroll
    for (int v = 0; v < U; ++v) {
        mx[v] = 0.f;
        if (pix[v] >= 0) {
            const float xn = prox<float>(xv[v] - eta * (blk[v * 256 + tid] + beta * tvg[v]), lam, a.prm->nonneg != 0);
            xo[pix[v]] = xn;
            if (a.xr) a.xr[sym_rot_index(pix[v] % n, pix[v] / n, n)] = xn;
            mx[v] = fabsf(xn);
        }
        mx[v] = warp_max(mx[v]);
        if ((tid & 31) == 0) red[v * 8 + (tid >> 5)] = mx[v];
    }
    sync();
    if (tid < U && u0 + tid < 32) {
        float m = red[tid * 8];
#pragma unroll
        for (int w = 1; w < 8; ++w) m = fmaxf(m, red[tid * 8 + w]);
        a.part_mx[t * 32 + u0 + tid] = m;
        if (m > 0.f) atomicMax(&a.st->fr[t / a.ntiles].mxw, __float_as_uint(m));
    }
    sync();  // the scratch is reused by the next claim
}

// phase trace of the back-projector (timing experiments only: -DPK_BP_TRACE=1, tools/k1_trace.py)
#ifndef PK_BP_TRACE
#define PK_BP_TRACE 0
#endif
#if PK_BP_TRACE
__device__ long long g_bp_trace[1536][16];
__device__ int g_bp_chunk_clk[1536][64];   // consumer warp 0: clocks per chunk (first 64)
#define BP_T(i, v) do { if (threadIdx.x == 0) g_bp_trace[blockIdx.x][(i)] = (v); } while (0)
#else
#define BP_T(i, v) do { } while (0)
#endif

#ifndef PK_SYM_MINB
#define PK_SYM_MINB 3  // CTAs per SM the back-projector's registers are capped for (build knob)
#endif
template <int IW>
__global__ void __launch_bounds__(kSymThreads, PK_SYM_MINB) bp_sym_f32_kernel(BpSymArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
#if PK_BP_TRACE
    if (threadIdx.x == 0) {
        long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        g_bp_trace[blockIdx.x][0] = gt;
        g_bp_trace[blockIdx.x][1] = clock64();
    }
#endif
    griddep_wait();  // the pair table and the stop flag come from the residual kernel
    BP_T(2, clock64());
    if (a.st && a.st->all_stopped) return;
    const int c0 = a.cta_chunk0[blockIdx.x], c1 = a.cta_chunk0[blockIdx.x + 1];
    if (c0 >= c1) return;
    BP_T(3, c1 - c0);
    const int n = a.n, h = n >> 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // windows [nbuf][kSymCS][8][WS] float2 | sconst [nbuf][kSymCS] float4 | full [nbuf] | empty [nbuf]
    const int WS = IW > 0 ? IW : a.L;
    const uint32_t img_stride = (uint32_t)WS * 8u;
    const size_t win_bytes = (size_t)a.nbuf * kSymCS * 8 * img_stride;
    float4* sconst = reinterpret_cast<float4*>(smem + win_bytes);
    const uint32_t win_s = smem_u32(smem);
    const uint32_t full_s = smem_u32(smem + win_bytes + (size_t)a.nbuf * kSymCS * 16);
    const uint32_t empty_s = full_s + 8u * a.nbuf;

    if (threadIdx.x == 0) {
        for (int b = 0; b < a.nbuf; ++b) {
            mbar_init(full_s + 8 * b, 1);
            mbar_init(empty_s + 8 * b, kSymConsumers * 32);  // every consumer thread releases
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kSymConsumers) {
        // ---- producer warp: stage chunk c into buffer b once the consumers released it;
        // lane = (base sensor cs = lane >> 3, image g = lane & 7) owns one window
        const int cs = lane >> 3, g = lane & 7;
        int b = 0;
        uint32_t phase = 0;
        for (int c = c0; c < c1; ++c) {
            if (c - c0 >= a.nbuf) mbar_wait(empty_s + 8 * b, phase ^ 1u);
            const int packed = __ldg(a.chunks + c);
            const int fr = (packed >> 16) / a.ntiles;  // frame of the chunk
            const int tp = __ldg(a.tiles + (packed >> 16) - fr * a.ntiles);
            const int tx = tp >> 16, ty = tp & 0xffff;
            const int ng = (tx == ty) ? 4 : 8;
            const int i0 = h + kSymTile * tx, j0 = h + kSymTile * ty;
            const float X0 = __ldg(a.pxs + i0), X1 = __ldg(a.pxs + min(i0 + kSymTile - 1, n - 1));
            const float Y0 = __ldg(a.pys + j0), Y1 = __ldg(a.pys + min(j0 + kSymTile - 1, n - 1));
            const int m = (packed & 0xffff) * kSymCS + cs;
            const bool act = cs < kSymCS && m < a.M && g < ng;
            const int mm = min(m, a.M - 1);
            const float sx = __ldg(a.sxs + mm), sy = __ldg(a.sys + mm);
            const float cx = fminf(fmaxf(sx, X0), X1), cy = fminf(fmaxf(sy, Y0), Y1);
            const float dmin = fminf(sqrtf((cx - sx) * (cx - sx) + (cy - sy) * (cy - sy)), a.qclamp);
            int lo = (int)floorf(dmin) - 1;
            lo = min(max(lo, 0) & ~1, a.TS - a.L);
            const uint32_t dst0 =
                win_s + (uint32_t)((b * kSymCS + min(cs, kSymCS - 1)) * 8) * img_stride;
            if (cs < kSymCS && g == 0)
                sconst[b * kSymCS + cs] = make_float4(
                    sx, sy, __uint_as_float(dst0 - 8u * (uint32_t)lo - 8u * kTwo23Bits), 0.f);
            const uint32_t nact = __popc(__ballot_sync(0xffffffffu, act));
            const size_t src_row = (size_t)__ldg(a.loc + sym_sensor(g, __ldg(a.gid + mm), a.Mall)) * a.TS + lo;
            __syncwarp();
            if (lane == 0) mbar_expect_tx(full_s + 8 * b, nact * (uint32_t)(a.L * 8));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (act)
                bulk_g2s(dst0 + (uint32_t)g * img_stride, a.table + fr * a.table_fstride + src_row,
                         (uint32_t)(a.L * 8), full_s + 8 * b);
            if (++b == a.nbuf) { b = 0; phase ^= 1u; }
        }
        return;
    }

    // ---- consumer warps
    int lx, ly;
    sym_lane_xy(lane, a.lanemap, lx, ly);
    float acc[4][8];
    float px[4], py = 0.f;
    int cur = -1, slot = a.cta_slot0[blockIdx.x] - 1;
    bool diag = false;
    auto flush = [&]() {
        float* dst = a.part + (size_t)slot * 8 * 4 * kThreads + threadIdx.x;
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (g < 4 || !diag) dst[(g * 4 + k) * kThreads] = acc[k][g];
    };
    // fused update: consumer-only barrier (the producer warp has left), tiles this CTA was
    // the final arriver of
    auto cbar = []() { asm volatile("bar.sync 1, 256;" ::: "memory"); };
    __shared__ int fin_s;
    int owe0 = -1, owe1 = -1;
    auto arrive = [&](int t) {  // after the flush of tile t: count the slot in
        cbar();
        if (threadIdx.x == 0) {
            __threadfence();
            const uint32_t old = atomicAdd(a.tile_cnt + t, 1u);
            const int ns = __ldg(a.epi.tile_slot0 + t + 1) - __ldg(a.epi.tile_slot0 + t);
            fin_s = (old + 1u == (uint32_t)ns) ? 1 : 0;
        }
        cbar();
        if (fin_s) { if (owe0 < 0) owe0 = t; else owe1 = t; }
    };
    int b = 0;
    uint32_t phase = 0;
    for (int c = c0; c < c1; ++c) {
        const int packed = __ldg(a.chunks + c);
        const int t = packed >> 16;
        if (t != cur) {
            if (cur >= 0) {
                flush();
                if (a.fuse) arrive(cur);
            }
            ++slot;
            cur = t;
            const int tp = __ldg(a.tiles + t % a.ntiles);
            const int tx = tp >> 16, ty = tp & 0xffff;
            diag = tx == ty;
            const int i0 = h + kSymTile * tx, j0 = h + kSymTile * ty;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                px[k] = __ldg(a.pxs + min(i0 + lx + 8 * k, n - 1));
#pragma unroll
                for (int g = 0; g < 8; ++g) acc[k][g] = 0.f;
            }
            py = __ldg(a.pys + min(j0 + 4 * warp + ly, n - 1));
        }
        mbar_wait(full_s + 8 * b, phase);
#if PK_BP_TRACE
        if (c == c0) BP_T(4, clock64());
#endif
        const int ns = min(kSymCS, a.M - (packed & 0xffff) * kSymCS);
        const float4* sc = sconst + b * kSymCS;
#if PK_BP_TRACE
        const long long tc0 = clock64();
#endif
        if (diag) sym_chunk<4, IW>(acc, px, py, sc, ns, img_stride, a.qclamp);
        else sym_chunk<8, IW>(acc, px, py, sc, ns, img_stride, a.qclamp);
#if PK_BP_TRACE
        if (threadIdx.x == 0 && c - c0 < 64) {
            float s = 0.f;  // (a dependency on the accumulators, so the clock reads after them)
#pragma unroll
            for (int g = 0; g < 8; ++g) s += acc[0][g];
            g_bp_chunk_clk[blockIdx.x][c - c0] = (int)(clock64() - tc0) + (s == 12345.f ? 1 : 0);
        }
#endif
        // every thread releases the buffer after its own reads of it (release semantics per
        // thread: the producer's acquire then orders its refill after all of them, without
        // relying on a warp barrier before a single arrival)
        mbar_arrive(empty_s + 8 * b);
        if (++b == a.nbuf) { b = 0; phase ^= 1u; }
    }
    BP_T(5, clock64());
    griddep_launch_dependents();
    flush();
    BP_T(6, clock64());
    BP_T(7, slot - a.cta_slot0[blockIdx.x] + 1);
    if (!a.fuse) return;
    arrive(cur);
    // publish the tiles this CTA completed (counters reset for the next launch first), wait a
    // bounded time for its last tile otherwise, then claim units of those tiles
    const int iter = a.st->iter;
    const uint32_t lid = (((uint32_t)a.st->epoch << 10) | (uint32_t)(iter & 1023)) + 1u;
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2; ++q) {
            const int t = q == 0 ? owe0 : owe1;
            if (t < 0) continue;
            a.tile_cnt[t] = 0u;
            a.tile_units[t] = 0u;
            __threadfence();
            st_release_u32(a.tile_done + t, lid);
        }
        int join = (owe0 == cur || owe1 == cur) ? 1 : 0;
        if (!join) {
            long long t0, now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            for (;;) {
                if (ld_acquire_u32(a.tile_done + cur) == lid) { join = 1; break; }
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (now - t0 > a.spin_ns) break;
                __nanosleep(64);
            }
        }
        fin_s = join;
    }
    cbar();
    const int joined = fin_s;
    // scratch for the units: the (idle) TMA ring
    constexpr int kU = 4;  // units per claim
    float4* part4 = reinterpret_cast<float4*>(smem);
    float* blk = reinterpret_cast<float*>(smem + kU * 3 * 64 * 16);
    float* red = blk + kU * 256;
    __shared__ int unit_s;
    for (int q = 0; q < 3; ++q) {
        const int t = q == 0 ? owe0 : (q == 1 ? owe1 : (joined && owe0 != cur && owe1 != cur ? cur : -1));
        if (t < 0) continue;
        for (;;) {
            cbar();  // every thread has read the previous claim
            if (threadIdx.x == 0) unit_s = (int)atomicAdd(a.tile_units + t, (uint32_t)kU);
            cbar();
            const int u0 = unit_s;
            if (u0 >= 32) break;
            sym_epi_units<kU>(a.epi, t, u0, iter, part4, blk, red, cbar);
        }
    }
}

// DEFER (with the symmetric projector): no last-block reduction here -- the projector's CTAs
// reduce the max partials into the fixed-point scale and the residual kernel takes sum |x'|
// and the non-finite count with TV(x'), so no single CTA serialises the end of this kernel.
#ifndef PK_EPX
#define PK_EPX 0  // timing experiments only (tools/k2v.sh); 0 = the product
#endif
template <bool EPI, bool DEFER>
__global__ void __launch_bounds__(kThreads) bp_sym_epi_kernel(BpSymEpiArgs a) {
    __shared__ float red_f[kThreads / 32];
    __shared__ double red_d[kThreads / 32];
    __shared__ int last_flag;
    __shared__ float4 part4[3][64];            // slot-group partials 1..3
    __shared__ float blk[8 * kSymTile];        // the strip in image g, row-major (bw x bh)
    // state words issued together with the tile loads (one round trip; the stop test waits on
    // it, then the iterate loads)
    int iter = 0;
    bool all_st = false;
    if (EPI) {
        all_st = a.st->all_stopped;
        iter = a.st->iter;
    }
    // CTA = (tile, image g, strip k): the main kernel's consumer thread c holds, in slot
    // element [g][k][c], the sum for representative (i0 + 8k + lx, j0 + 4(c / 32) + ly) -- an
    // 8-column strip of the tile, 256 pixels
    const int k = blockIdx.x & 3, g = (blockIdx.x >> 2) & 7, t = blockIdx.x >> 5;  // t: frame-major
    const int fr = t / a.ntiles;
    const int tp = __ldg(a.tiles + t - fr * a.ntiles);
    const int tx = tp >> 16, ty = tp & 0xffff;
    const bool active = !(tx == ty && g >= 4);
    const int n = a.n, h = n >> 1;
    const int i0 = h + kSymTile * tx, j0 = h + kSymTile * ty;
    const int s0 = __ldg(a.tile_slot0 + t), s1 = __ldg(a.tile_slot0 + t + 1);
    const bool fr_stopped = EPI ? (bool)a.st->fr[fr].stopped : true;
    float beta_tv = 0.f, eps_tv = 0.f;
    if (EPI) { beta_tv = (float)a.prm->beta[fr]; eps_tv = (float)a.prm->eps; }
    if (all_st) return;
    // the strip's image under g is the block [bx, bx + bw) x [by, by + bh), bw * bh = 256
    int bx, by, bw;
    {
        int ia, ja, ib, jb;
        sym_pixel(g, i0 + 8 * k, j0, n, ia, ja);
        sym_pixel(g, i0 + 8 * k + 7, j0 + kSymTile - 1, n, ib, jb);
        bx = min(ia, ib);
        by = min(ja, jb);
        bw = abs(ib - ia) + 1;
    }
    // 0) one pixel per thread in image-row-major order of the strip; a pixel of the strip
    //    belongs to this CTA iff its representative is in the tile (row / column beyond the
    //    grid edge, or the reflections of a diagonal tile, are skipped).  Solver mode: its
    //    iterate value and TV gradient (final since the previous iteration) are loaded
    //    before the wait for the main kernel
    int pix;
    {
        const int ig = bx + threadIdx.x % bw, jg = by + threadIdx.x / bw;
        pix = (active && ig >= 0 && ig < n && jg >= 0 && jg < n) ? jg * n + ig : -1;
    }
    const float* x = EPI ? ((iter & 1) ? a.xb1 : a.xb0) + (size_t)fr * a.P : nullptr;
    const bool run = EPI && pix >= 0 && !fr_stopped;
    float xv = 0.f, tvg = 0.f;
    if (run) {
        xv = x[pix];
        if (beta_tv > 0.f && PK_EPX != 3) tvg = tv_grad_at<float>(x, pix, pix % n, pix / n, n, n, eps_tv * eps_tv);
    }
    // 1) slot sum: thread (sg, q) adds slots s0 + sg, s0 + sg + 4, ... of consumers 4q..4q+3
    //    (16-B loads, 8 in flight); the 4 slot groups are then added in order (deterministic)
    const int sg = threadIdx.x >> 6, q = threadIdx.x & 63;
    griddep_wait();  // partial slots of the main kernel
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    if (active && PK_EPX != 1) {
        const float4* src = reinterpret_cast<const float4*>(a.part + (size_t)(g * 4 + k) * kThreads) + q;
        const size_t stride = 8 * 4 * kThreads / 4;  // float4s per slot
        for (int sb = s0 + sg; sb < s1; sb += 32) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                v[u] = (sb + 4 * u < s1) ? __ldcg(src + (size_t)(sb + 4 * u) * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                sum.x += v[u].x; sum.y += v[u].y; sum.z += v[u].z; sum.w += v[u].w;
            }
        }
    }
    if (sg > 0) part4[sg - 1][q] = sum;
    __syncthreads();
    // 2) slot group 0 finishes the sums and scatters them into the strip (shared transpose)
    if (sg == 0) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const float4 o = part4[r][q];
            sum.x += o.x; sum.y += o.y; sum.z += o.z; sum.w += o.w;
        }
        const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = 4 * q + u;  // consumer thread of the main kernel
            int lx, ly;
            sym_lane_xy(c & 31, a.lanemap, lx, ly);
            int ig, jg;
            sym_pixel(g, i0 + lx + 8 * k, j0 + 4 * (c >> 5) + ly, n, ig, jg);
            blk[(jg - by) * bw + (ig - bx)] = a.gscale * sv[u];
        }
    }
    __syncthreads();
    // 3) the update of this thread's pixel
    const float val = blk[threadIdx.x];
    if (!EPI) {
        if (pix >= 0) a.out[(size_t)fr * a.P + pix] = val;
        return;
    }
    float* xo = ((iter & 1) ? a.xb0 : a.xb1) + (size_t)fr * a.P;
    float* xr = a.xr ? a.xr + (size_t)fr * a.P : nullptr;  // (4 * (n/2)^2 = P floats per frame)
    const float eta = (float)a.prm->step[fr], lam = (float)a.prm->eta_alpha[fr];
    const float beta = (float)a.prm->beta[fr];
    const bool nonneg = a.prm->nonneg != 0;
    float mx = 0.f, l1 = 0.f;
    int bad = 0;
    if (run) {
        const int p = pix;
        float gr = val;
        if (beta > 0.f && PK_EPX != 3) gr += beta * tvg;
        const float xn = prox<float>(xv - eta * gr, lam, nonneg);
        xo[p] = xn;
        if (xr) xr[sym_rot_index(p % n, p / n, n)] = xn;
        if (!isfinite(xn)) bad = 1;
        mx = fabsf(xn);
        l1 = fabsf(xn);
    }
    griddep_launch_dependents();
    mx = block_max(mx, red_f);
    if (DEFER) {  // sum |x'| and the non-finite count are taken by the residual kernel
        if (threadIdx.x == 0) {
            a.part_mx[blockIdx.x] = mx;
            // (NaN skipped as fmaxf over the partials does; non-finite iterates are caught by
            // the residual kernel's count)
            if (mx > 0.f) atomicMax(&a.st->fr[fr].mxw, __float_as_uint(mx));
        }
        return;
    }
    const float l1b = block_sum(l1, red_f);
    const int badb = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
        double* pp = a.part_bp + 4 * (size_t)blockIdx.x;
        pp[0] = mx;
        pp[1] = l1b;
        pp[2] = badb;
    }
    if (PK_EPX != 2 && last_block(&a.st->cnt_bp, gridDim.x, &last_flag)) {
        double m2 = 0.0, s2 = 0.0, b2 = 0.0;
        for (int q = threadIdx.x; q < (int)gridDim.x; q += kThreads) {
            const double* pp = a.part_bp + 4 * (size_t)q;
            m2 = fmax(m2, pp[0]);
            s2 += pp[1];
            b2 += pp[2];
        }
        m2 = block_max(m2, red_d);
        s2 = block_sum(s2, red_d);
        b2 = block_sum(b2, red_d);
        if (threadIdx.x == 0 && !a.st->fr[0].stopped) {
            FrameState& fs = a.st->fr[0];
            fs.maxabs = m2;
            fs.l1sum = s2;
            fs.nonfinite = b2 > 0.0 ? 1 : 0;
            const double scl = (m2 > 0.0 && isfinite(m2)) ? ldexp(1.0, a.bits) / m2 : 0.0;
            fs.scale64 = scl;
            fs.scale32 = (float)scl;
        }
    }
}

// Solver-mode epilogue with deferred statistics (the bench's path), one CTA per (tile, image
// g, block of KS strips) doing KS of bp_sym_epi_kernel<true, true>'s (tile, image, strip) CTAs:
// the strips' loads (iterate, TV gradient before the PDL wait; partial slots after it) are in
// flight together and the per-CTA fixed costs (state loads, barriers, max reduction, atomic)
// are paid once per KS strips.  Per pixel the same arithmetic and the same slot order (slot
// group sg adds slots s0 + sg, s0 + sg + 4, ... in increasing order, then the groups 0..3 in
// order), so the result is bitwise that of bp_sym_epi_kernel: the zero padding of its 8-wide
// slot batches is skipped, and adding +0.0f to a sum that starts at +0.0f is exact (such a sum
// is never -0.0f).  KS = 2 by default (config 3: 9.2 / 22.9 us at one / four frames per
// launch against 10.6 / 27.1 for one strip and 11.8 / 23.7 for four); PK_SYM_EPIK=1 restores
// the one-strip kernel (2 / 4 force KS).
template <int KS>
__global__ void __launch_bounds__(kThreads) bp_sym_epik_kernel(BpSymEpiArgs a) {
    __shared__ float red_f[kThreads / 32];
    __shared__ float4 part4[KS][3][64];        // [strip][slot group 1..3][consumer quad]
    __shared__ float blk[KS][8 * kSymTile];    // strip k0 + k in image g, row-major (bw x bh)
    // state words with the tile loads (one round trip)
    const bool all_st = a.st->all_stopped;
    const int iter = a.st->iter;
    constexpr int NB = 4 / KS;  // strip blocks per (tile, image)
    const int kb = blockIdx.x % NB, g = (blockIdx.x / NB) & 7, t = blockIdx.x / (8 * NB);  // t: frame-major
    const int k0 = kb * KS;
    const int fr = t / a.ntiles;
    const int tp = __ldg(a.tiles + t - fr * a.ntiles);
    const int s0 = __ldg(a.tile_slot0 + t), s1 = __ldg(a.tile_slot0 + t + 1);
    const bool fr_stopped = a.st->fr[fr].stopped;
    const float beta = (float)a.prm->beta[fr], eps = (float)a.prm->eps;
    const float eta = (float)a.prm->step[fr], lam = (float)a.prm->eta_alpha[fr];
    const bool nonneg = a.prm->nonneg != 0;
    const int tx = tp >> 16, ty = tp & 0xffff;
    if (all_st || (tx == ty && g >= 4)) return;  // (reflections of a diagonal tile: no pixels)
    const int n = a.n, h = n >> 1;
    const int i0 = h + kSymTile * tx, j0 = h + kSymTile * ty;
    // strip k0 + k's image under g: the block [bx, bx + bw) x [by, by + bh), bw * bh = 256
    auto strip_box = [&](int k, int& bx, int& by, int& bw) {
        int ia, ja, ib, jb;
        sym_pixel(g, i0 + 8 * (k0 + k), j0, n, ia, ja);
        sym_pixel(g, i0 + 8 * (k0 + k) + 7, j0 + kSymTile - 1, n, ib, jb);
        bx = min(ia, ib);
        by = min(ja, jb);
        bw = abs(ib - ia) + 1;
    };
    // one pixel per thread and strip (image-row-major order of the strip); iterate value and
    // TV gradient loaded before the wait (final since the previous iteration)
    const float* x = ((iter & 1) ? a.xb1 : a.xb0) + (size_t)fr * a.P;
    int pix[KS];
    float xv[KS], tvg[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) {
        int bx, by, bw;
        strip_box(k, bx, by, bw);
        const int ig = bx + threadIdx.x % bw, jg = by + threadIdx.x / bw;
        pix[k] = (!fr_stopped && ig >= 0 && ig < n && jg >= 0 && jg < n) ? jg * n + ig : -1;
        xv[k] = 0.f;
        tvg[k] = 0.f;
        if (pix[k] >= 0) {
            xv[k] = x[pix[k]];
            if (beta > 0.f) tvg[k] = tv_grad_at<float>(x, pix[k], pix[k] % n, pix[k] / n, n, n, eps * eps);
        }
    }
    // slot sums: thread (sg, q) adds slots s0 + sg, s0 + sg + 4, ... of consumers 4q..4q+3 of
    // every strip (two slots x KS strips of 16-B loads in flight per pass)
    const int sg = threadIdx.x >> 6, q = threadIdx.x & 63;
    griddep_wait();  // partial slots of the main kernel
    float4 sum[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) sum[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    {
        const float4* src = reinterpret_cast<const float4*>(a.part + (size_t)(g * 4 + k0) * kThreads) + q;
        const size_t stride = 8 * 4 * kThreads / 4;  // float4s per slot
        for (int sb = s0 + sg; sb < s1; sb += 8) {
            float4 v[2][KS];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int k = 0; k < KS; ++k)
                    v[u][k] = (sb + 4 * u < s1) ? __ldcg(src + k * (kThreads / 4) + (size_t)(sb + 4 * u) * stride)
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (sb + 4 * u >= s1) break;
#pragma unroll
                for (int k = 0; k < KS; ++k) {
                    sum[k].x += v[u][k].x; sum[k].y += v[u][k].y; sum[k].z += v[u][k].z; sum[k].w += v[u][k].w;
                }
            }
        }
    }
    if (sg > 0) {
#pragma unroll
        for (int k = 0; k < KS; ++k) part4[k][sg - 1][q] = sum[k];
    }
    __syncthreads();
    // slot group 0 finishes the sums and scatters them into the strips (shared transpose)
    if (sg == 0) {
#pragma unroll
        for (int k = 0; k < KS; ++k) {
            float4 sm = sum[k];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const float4 o = part4[k][r][q];
                sm.x += o.x; sm.y += o.y; sm.z += o.z; sm.w += o.w;
            }
            const float sv[4] = {sm.x, sm.y, sm.z, sm.w};
            int bx, by, bw;
            strip_box(k, bx, by, bw);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = 4 * q + u;  // consumer thread of the main kernel
                int lx, ly;
                sym_lane_xy(c & 31, a.lanemap, lx, ly);
                int ig, jg;
                sym_pixel(g, i0 + lx + 8 * (k0 + k), j0 + 4 * (c >> 5) + ly, n, ig, jg);
                blk[k][(jg - by) * bw + (ig - bx)] = a.gscale * sv[u];
            }
        }
    }
    __syncthreads();
    // the update of this thread's pixel of each strip (as bp_sym_epi_kernel)
    float* xo = ((iter & 1) ? a.xb0 : a.xb1) + (size_t)fr * a.P;
    float* xr = a.xr ? a.xr + (size_t)fr * a.P : nullptr;
    float mx = 0.f;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
        const int p = pix[k];
        if (p < 0) continue;
        float gr = blk[k][threadIdx.x];
        if (beta > 0.f) gr += beta * tvg[k];
        const float xn = prox<float>(xv[k] - eta * gr, lam, nonneg);
        xo[p] = xn;
        if (xr) xr[sym_rot_index(p % n, p / n, n)] = xn;
        mx = fmaxf(mx, fabsf(xn));  // (NaN skipped, as the one-strip kernel's reduction does)
    }
    griddep_launch_dependents();
    mx = block_max(mx, red_f);
    if (threadIdx.x == 0) {
        a.part_mx[blockIdx.x] = mx;
        if (mx > 0.f) atomicMax(&a.st->fr[fr].mxw, __float_as_uint(mx));
    }
}

// ===========================================================================
// K1 -- back-projector, fp64 validation mode: one pixel per thread, fp64 delay evaluated
// exactly as the reference (forward.py:157-182), table read through the L1/L2 path.
// ===========================================================================
struct BpArgs64 {
    const double2* table;
    const double *px, *py, *sx, *sy;
    double cdt;
    int nx, ny, M, Q, TS;
    double* out;
    double gscale;
    double *xb0, *xb1;
    const DevParams* prm;
    DevState* st;
    double* part;
    int bits;
};

template <bool EPI>
__global__ void __launch_bounds__(kThreads) bp_f64_kernel(BpArgs64 a) {
    __shared__ double red_d[kThreads / 32];
    __shared__ int last_flag;
    int iter = 0;
    if (EPI) {
        if (a.st->all_stopped) return;
        iter = a.st->iter;
    }
    const int p = blockIdx.x * kThreads + threadIdx.x;
    const int P = a.nx * a.ny;
    const bool valid = p < P;
    const int i = valid ? p % a.nx : 0, j = valid ? p / a.nx : 0;
    const double pxv = a.px[i], pyv = a.py[j];
    double acc = 0.0;
    if (valid) {
        for (int m = 0; m < a.M; ++m) {
            const double u = delay_f64(pxv, pyv, __ldg(a.sx + m), __ldg(a.sy + m), a.cdt);
            double fl = floor(u);
            if (fl > (double)(a.Q + 1)) fl = (double)(a.Q + 1);
            const int s0 = (int)fl;
            const double f = u - fl;
            const double2 v = __ldg(a.table + (size_t)m * a.TS + s0);
            acc += fma(f, v.y, v.x);
        }
    }
    if (!EPI) {
        if (valid) a.out[p] = a.gscale * acc;
        return;
    }
    const double* x = (iter & 1) ? a.xb1 : a.xb0;
    double* xo = (iter & 1) ? a.xb0 : a.xb1;
    double mx = 0.0, l1 = 0.0;
    int bad = 0;
    if (valid) {
        const double eps = a.prm->eps;
        double g = a.gscale * acc;
        if (a.prm->beta[0] > 0.0) g += a.prm->beta[0] * tv_grad_at<double>(x, p, i, j, a.nx, a.ny, eps * eps);
        const double xn = prox<double>(x[p] - a.prm->step[0] * g, a.prm->eta_alpha[0], a.prm->nonneg != 0);
        xo[p] = xn;
        bad = !isfinite(xn);
        mx = fabs(xn);
        l1 = fabs(xn);
    }
    mx = block_max(mx, red_d);
    const double l1b = block_sum(l1, red_d);
    const int badb = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
        double* pp = a.part + 4 * (size_t)blockIdx.x;
        pp[0] = mx;
        pp[1] = l1b;
        pp[2] = badb;
    }
    if (last_block(&a.st->cnt_bp, gridDim.x, &last_flag)) {
        double m2 = 0.0, s2 = 0.0, b2 = 0.0;
        for (int q = threadIdx.x; q < (int)gridDim.x; q += kThreads) {
            const double* pp = a.part + 4 * (size_t)q;
            m2 = fmax(m2, pp[0]);
            s2 += pp[1];
            b2 += pp[2];
        }
        m2 = block_max(m2, red_d);
        s2 = block_sum(s2, red_d);
        b2 = block_sum(b2, red_d);
        if (threadIdx.x == 0) {
            FrameState& fs = a.st->fr[0];
            fs.maxabs = m2;
            fs.l1sum = s2;
            fs.nonfinite = b2 > 0.0 ? 1 : 0;
            const double scl = (m2 > 0.0 && isfinite(m2)) ? ldexp(1.0, a.bits) / m2 : 0.0;
            fs.scale64 = scl;
            fs.scale32 = (float)scl;
        }
    }
}

// ===========================================================================
// K2 -- projector, fp32 with an exact fixed-point accumulator (deterministic).
// CTA = (T x T pixel tile, 32 consecutive sensors); lane l of every warp owns sensor
// g*32 + l, so a warp instruction is 1 pixel x 32 sensors.  Each lane scatters into its own
// sensor's windows with native 32-bit shared atomics; windows are stored slot-major
// ([slot][frame][32 lanes]) so lane l always hits bank l: conflict-free by construction.
// Contributions are integers:  xq = rint(x*scale),  a = rint(x*scale*f),  b = xq - a,
// added at trace index s0 (weight f) and s0-1 (weight 1-f) -- forward.py:189-194.
// Warps own whole image rows: a warp compacts its row's pixels that are non-zero in any
// frame (soft-threshold zeros are skipped warp-uniformly) into a private record buffer,
// pads it to a multiple of 8 with zero-weight records, and scatters 8 pixels per batch
// (8 independent chains: all arithmetic first, then the atomics).  Windows are flushed
// into the int64 trace accumulator with RED.64 (integer adds commute: deterministic).
// ===========================================================================
struct FpArgs {
    const float* x;       // [NF][P] (nullptr: solver mode, use xb[(iter+1)&1])
    const float* xb0;
    const float* xb1;
    const float* pxs;
    const float* pys;
    const float* sxs;
    const float* sys;
    long long* acc;       // [NF][M][Q]
    int nx, ny, M, Q, T, L, tiles_x;
    float qclamp;
    DevState* st;
    double* part_tv;      // solver mode: per-(tile, frame) TV(x) partials (group 0 only)
    int solver;
};

constexpr int kFpBatch = 8;

// record of one pixel: px, then {x*scale, bits(rint(x*scale) + magic)} per frame
template <int NF>
struct FpRec {
    static constexpr int kFloats = 1 + 2 * NF;
    static constexpr int kVec = (kFloats + 3) / 4;  // float4 per record
};

template <int NF, bool CLAMP>
__global__ void __launch_bounds__(kThreads, NF == 1 ? 4 : (NF == 2 ? 3 : 2)) fp_f32_kernel(FpArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ float red_f[kThreads / 32];
    constexpr int LG = Lg<NF>::v;
    constexpr int RV = FpRec<NF>::kVec;
    int iter = 0;
    if (a.solver) {
        if (a.st->all_stopped) return;
        iter = a.st->iter;
    }
    const float* x = a.x ? a.x : ((iter & 1) ? a.xb0 : a.xb1);  // bp wrote xb[(iter+1)&1]
    const size_t P = (size_t)a.nx * a.ny;
    float scale[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) scale[f] = a.st->fr[f].scale32;
    const int T = a.T;
    const int tx = blockIdx.x % a.tiles_x, ty = blockIdx.x / a.tiles_x;
    const int i0 = tx * T, j0 = ty * T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = blockIdx.y * 32 + lane;
    const bool sensor_ok = m < a.M;
    const float sx = __ldg(a.sxs + min(m, a.M - 1)), sy = __ldg(a.sys + min(m, a.M - 1));

    // shared layout: win int32 [L][NF][32] | per-warp row records float4 [8][(T+8)*RV]
    int32_t* win = reinterpret_cast<int32_t*>(smem);
    float4* rows = reinterpret_cast<float4*>(smem + (size_t)a.L * NF * 32 * 4);
    float4* rec = rows + (size_t)warp * (T + kFpBatch) * RV;

    for (int q = threadIdx.x; q < a.L * NF * 32; q += kThreads) win[q] = 0;

    // this lane's window: trace indices [lo, lo + L)
    const float X0 = __ldg(a.pxs + i0), X1 = __ldg(a.pxs + min(i0 + T - 1, a.nx - 1));
    const float Y0 = __ldg(a.pys + j0), Y1 = __ldg(a.pys + min(j0 + T - 1, a.ny - 1));
    const float cx = fminf(fmaxf(sx, X0), X1), cy = fminf(fmaxf(sy, Y0), Y1);
    float dmin = sqrtf((cx - sx) * (cx - sx) + (cy - sy) * (cy - sy));
    if (CLAMP) dmin = fminf(dmin, a.qclamp);
    const int lo = (int)floorf(dmin) - 2;
    // word address of (trace index t, frame f): win + 4*(32*(NF*(t - lo) + f) + lane)
    const uint32_t adj = smem_u32(win) + 4u * (uint32_t)lane - (128u * NF) * (uint32_t)lo -
                         (128u * NF) * kTwo23Bits;
    __syncthreads();

    float tv[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) tv[f] = 0.f;
    const bool do_tv = a.solver && blockIdx.y == 0;
    const int jend = min(T, a.ny - j0);
    // rows of this warp; the next row's pixels are loaded while the current row scatters
    float xnext[NF][2];
    auto load_row = [&](int r, float (*dst)[2]) {
#pragma unroll
        for (int f = 0; f < NF; ++f)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int ii = i0 + 32 * c + lane;
                dst[f][c] = (32 * c < T && r < jend && ii < a.nx)
                                ? x[f * P + (size_t)(j0 + r) * a.nx + ii] : 0.f;
            }
    };
    load_row(warp, xnext);
    for (int r = warp; r < jend; r += kThreads / 32) {
        const int jj = j0 + r;
        float xrow[NF][2];
#pragma unroll
        for (int f = 0; f < NF; ++f) { xrow[f][0] = xnext[f][0]; xrow[f][1] = xnext[f][1]; }
        load_row(r + kThreads / 32, xnext);
        int cnt = 0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int cc = 32 * c;
            if (cc >= T) break;
            const int ii = i0 + cc + lane;
            const bool in = ii < a.nx;
            bool nz = false;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const float xv = xrow[f][c];
                if (do_tv && in) {  // exact anisotropic TV partial, recon.py:169-170
                    const float* xf = x + f * P;
                    if (ii + 1 < a.nx) tv[f] += fabsf(xf[(size_t)jj * a.nx + ii + 1] - xv);
                    if (jj + 1 < a.ny) tv[f] += fabsf(xf[(size_t)(jj + 1) * a.nx + ii] - xv);
                }
                nz |= xv != 0.f;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, nz);
            if (nz) {
                float rv[4 * RV];
                rv[0] = __ldg(a.pxs + ii);
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    const float xs = xrow[f][c] * scale[f];
                    rv[1 + 2 * f] = xs;
                    rv[2 + 2 * f] = __int_as_float(__float_as_int(xs + kMagic));
                }
#pragma unroll
                for (int q = 1 + 2 * NF; q < 4 * RV; ++q) rv[q] = 0.f;
                float4* dst = rec + (size_t)(cnt + __popc(bal & ((1u << lane) - 1u))) * RV;
#pragma unroll
                for (int v = 0; v < RV; ++v)
                    dst[v] = make_float4(rv[4 * v], rv[4 * v + 1], rv[4 * v + 2], rv[4 * v + 3]);
            }
            cnt += __popc(bal);
        }
        if (cnt == 0) continue;  // warp-uniform
        const int cnt8 = (cnt + kFpBatch - 1) & ~(kFpBatch - 1);
        if (lane < cnt8 - cnt) {  // zero-weight padding (adds 0 at a valid window address)
            float rv[4 * RV];
            rv[0] = X0;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                rv[1 + 2 * f] = 0.f;
                rv[2 + 2 * f] = __int_as_float(kMagicBits);
            }
#pragma unroll
            for (int q = 1 + 2 * NF; q < 4 * RV; ++q) rv[q] = 0.f;
            float4* dst = rec + (size_t)(cnt + lane) * RV;
#pragma unroll
            for (int v = 0; v < RV; ++v)
                dst[v] = make_float4(rv[4 * v], rv[4 * v + 1], rv[4 * v + 2], rv[4 * v + 3]);
        }
        __syncwarp();
        if (sensor_ok) {
            const float ey = __ldg(a.pys + jj) - sy;
            const float ey2 = ey * ey;
            for (int k = 0; k < cnt8; k += kFpBatch) {
                uint32_t ad[kFpBatch];
                int32_t va[kFpBatch][NF], vb[kFpBatch][NF];
#pragma unroll
                for (int b = 0; b < kFpBatch; ++b) {
                    float rv[4 * RV];
#pragma unroll
                    for (int v = 0; v < RV; ++v) {
                        const float4 q = rec[(size_t)(k + b) * RV + v];
                        rv[4 * v] = q.x; rv[4 * v + 1] = q.y; rv[4 * v + 2] = q.z; rv[4 * v + 3] = q.w;
                    }
                    const float ex = rv[0] - sx;
                    float u = sqrt_approx(fmaf(ex, ex, ey2));
                    if (CLAMP) u = fminf(u, a.qclamp);
                    const float tb = __fadd_rd(u, kTwo23);
                    const float fr = u - (tb - kTwo23);
#pragma unroll
                    for (int f = 0; f < NF; ++f) {
                        const float fb = fmaf(rv[1 + 2 * f], fr, kMagic);
                        va[b][f] = __float_as_int(fb) - kMagicBits;                    // f   -> s0
                        vb[b][f] = __float_as_int(rv[2 + 2 * f]) - __float_as_int(fb); // 1-f -> s0-1
                    }
                    ad[b] = adj + (__float_as_uint(tb) << (7 + LG));
                }
#pragma unroll
                for (int b = 0; b < kFpBatch; ++b)
#pragma unroll
                    for (int f = 0; f < NF; ++f) {
                        red_smem_s32(ad[b] - 128u * NF + 128u * f, vb[b][f]);
                        red_smem_s32(ad[b] + 128u * f, va[b][f]);
                    }
            }
        }
        __syncwarp();  // rec is rewritten by the next row
    }
    if (do_tv) {
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const float tvb = block_sum(tv[f], red_f);
            if (threadIdx.x == 0) a.part_tv[(size_t)blockIdx.x * NF + f] = tvb;
        }
    }
    __syncthreads();

    // flush: each warp takes blocks of BS window slots, reads them row-wise (lane = sensor,
    // conflict-free), transposes them through its (now free) record buffer with a padded
    // stride, and issues the RED.64s sensor-major so that one warp instruction covers
    // 32/BS sensors x BS consecutive trace samples (BS*8-byte runs instead of 32 scattered
    // words).  Only real trace indices 0..Q-1 are flushed.
    const int cap = (T + kFpBatch) * RV * 16;  // bytes of this warp's record buffer
    const int bs = (32 * 9 * 4 <= cap) ? 8 : 4;
    int32_t* scr = reinterpret_cast<int32_t*>(rec);
    const int lanes_per_sensor = bs, sensors_per_step = 32 / bs;
    const int sub = lane % lanes_per_sensor, grp = lane / lanes_per_sensor;
    for (int k0 = warp * bs; k0 < a.L; k0 += (kThreads / 32) * bs) {
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            for (int i = 0; i < bs; ++i) {
                const int k = k0 + i;
                scr[lane * (bs + 1) + i] = (k < a.L) ? win[(k * NF + f) * 32 + lane] : 0;
            }
            __syncwarp();
            for (int r = 0; r < 32; r += sensors_per_step) {
                const int ms = r + grp;                 // sensor (lane index) of this RED
                const int lo_ms = __shfl_sync(0xffffffffu, lo, ms);
                const int v = scr[ms * (bs + 1) + sub];
                const int t = lo_ms + k0 + sub;
                const int mg = blockIdx.y * 32 + ms;
                if (v != 0 && mg < a.M && t >= 0 && t < a.Q && k0 + sub < a.L)
                    atomicAdd(reinterpret_cast<unsigned long long*>(a.acc + ((size_t)f * a.M + mg) * a.Q + t),
                              (unsigned long long)(long long)v);
            }
            __syncwarp();
        }
    }
}

// ===========================================================================
// K2s -- projector, fp32, for D4-symmetric scenes (same conditions as K1s).  The 4
// rotations r^g by 90 degrees map a pair (pixel p, sensor m) to (r^g p, m + g*M/4) with the
// same distance, so a delay evaluated for a pixel of the first quadrant (i, j >= n/2) serves
// its 4 rotation images
//   g = 0: (i, j)   1: (n-1-j, i)   2: (n-1-i, n-1-j)   3: (j, n-1-i)
// against the sensors m + g*M/4.
//
// Work = rows of (group of 32 base sensors, T-column strip of the quadrant, quadrant row),
// flattened in that order and cut host-side into one equal contiguous range per persistent
// CTA (grid = CTAs resident on the GPU, so every SM carries the same number of rows: no
// partly idle SMs).  A CTA's range is split into segments, each inside one (group, strip) and
// at most Hs rows high; per segment lane l owns base sensor m = 32*group + l and 4 windows (one
// per image sensor) of LW slots covering the delays of the segment's T x rows rectangle;
// window word (g, slot k, lane) sits at (g*LW + k)*32 + lane, so lane l always hits bank l: the
// scatter is conflict free.  Contributions are fixed-point integers: round(xs*f) at trace index
// s0 and round(xs*(1-f)) at s0-1 (xs = x*scale), added with red.shared.add.s32 as magic-biased
// float bits (the bias is pre-subtracted per slot).  At the end of a segment the CTA stores its
// windows, transposed to [g][sensor][slot], into the segment's slice of a global window array
// (no global atomics); the residual kernel gathers, for every trace sample, the windows that
// cover it (deterministic integer sums).
// Per record (1 pixel x 32 sensors x 4 images): 1 LDS.128 + ~8 delay + 8 FFMA + 8 ATOMS.
// ===========================================================================
constexpr int kFsTile = 64;      // quadrant strip width (32 where the window per pixel of a
                                 // 64 strip is larger, e.g. BASELINE config 2); rows are
                                 // 32-pixel pieces
#ifndef PK_FS_BATCH
#define PK_FS_BATCH 4
#endif
#ifndef PK_FS_UNROLL
#define PK_FS_UNROLL 2
#endif
constexpr int kFsBatch = PK_FS_BATCH;  // records per scatter batch (4: 16 independent atomic pairs)
constexpr int kFsUnroll = PK_FS_UNROLL; // scatter batches unrolled per loop iteration
constexpr int kFsThreads = 512;  // threads of the plan-setup count kernel

struct FpSymArgs {
    const float* x;          // standalone input (nullptr: solver mode, xb[(iter+1)&1])
    const float* xb0;
    const float* xb1;
    const float* pxs;
    const float* pys;
    const float* sxs;
    const float* sys;
    int32_t* acc;            // [M][acc_ld] int32 trace accumulator (row offset kAccFront);
                             //   the windows are reduce-added into it, the residual kernel
                             //   reads and clears it
    int acc_ld;
    const int* trace_of;     // [groups * 32][4] local trace of (base sensor, image), -1: none
    // (every word the scatter adds carries the magic bias kMagicBits; the accumulator rows
    // start at -count * kMagicBits per position, fp_sym_bias_kernel / the residual kernel)
    const int4* segs;        // [segments] {frame * groups + group, strip, first row, end row}
    const int* cta_seg0;     // [grid + 1] first segment of each CTA
    const int* rec;          // [frames] the segment whose CTA records the frame's scale
    int groups;              // sensor groups per frame
    int n, M, Q;
    float qclamp;
    float hx;                // pixel pitch in samples (pxs[i] ~ pxs[0] + i*hx, fp32)
    DevState* st;
    int solver;              // (TV(x') of the iterate is taken by finalize_kernel)
    const float4* xr;        // solver mode, optional: x' rotation-packed by the epilogue
    const float* part_mx;    // solver mode, optional: the epilogue's deferred max partials
    int nmx, bits;           //   (the scale is 2^bits / max, as the epilogue's last block did)
};

constexpr int kAccFront = 4;  // words before sample 0 in an accumulator row (windows may start at -4)
// shared memory of the projector: windows [4][LW][32], the transposed staging of ngr images
// [ngr][32][LW + 4] for the bulk reductions, and the per-warp records
// (cap: the dynamic shared memory one CTA may take -- 226 KB at one 32-warp CTA per SM, 112 KB
// at two 16-warp CTAs)
__host__ __device__ constexpr int fs_cap(int nw) { return (nw == 32 ? 226 : 112) * 1024; }
__host__ __device__ constexpr int fs_base_smem(int lw, int nw) { return 4 * lw * 32 * 4 + nw * (32 + kFsBatch) * 16; }
__host__ __device__ constexpr int fs_ngr(int lw, int nw, int cap) {
    return fs_base_smem(lw, nw) + 4 * 32 * (lw + 4) * 4 <= cap ? 4
         : fs_base_smem(lw, nw) + 2 * 32 * (lw + 4) * 4 <= cap ? 2
         : fs_base_smem(lw, nw) + 32 * (lw + 4) * 4 <= cap ? 1 : 0;
}
__host__ __device__ constexpr int fs_smem(int lw, int nw, int cap) {
    return fs_base_smem(lw, nw) + fs_ngr(lw, nw, cap) * 32 * (lw + 4) * 4;
}

// first trace index of the window of the quadrant rectangle [i0, i0 + T) x [j0, j1) for
// sensor (sx, sy): floor of the distance to the nearest point of the rectangle, minus 2,
// rounded down to a multiple of 4 (the bulk reductions need 16-B aligned rows)
__device__ __forceinline__ int fp_sym_window_lo(const float* pxs, const float* pys, int n, int i0,
                                                int j0, int j1, float sx, float sy, float qclamp,
                                                int tile) {
    const float X0 = __ldg(pxs + i0), X1 = __ldg(pxs + min(i0 + tile - 1, n - 1));
    const float Y0 = __ldg(pys + j0), Y1 = __ldg(pys + min(j1 - 1, n - 1));
    const float cx = fminf(fmaxf(sx, X0), X1), cy = fminf(fmaxf(sy, Y0), Y1);
    const float dmin = fminf(sqrtf((cx - sx) * (cx - sx) + (cy - sy) * (cy - sy)), qclamp);
    return ((int)floorf(dmin) - 2) & ~3;
}

// delay of column k of a 32-pixel piece (pxbs = x of the piece's first column minus the
// sensor x, in samples) for a sensor at squared row distance ey2: returns 2^23 + s0 (as float)
// and the fraction fr.  Shared by the projector and its bias-count setup kernel, so both see
// the same s0 bit for bit.
template <bool CLAMP>
__device__ __forceinline__ float fs_delay(float k, float hx, float pxbs, float ey2, float qclamp,
                                          float& fr) {
    const float ex = fmaf(k, hx, pxbs);
    float uu = sqrt_approx(fmaf(ex, ex, ey2));
    if (CLAMP) uu = fminf(uu, qclamp);
    const float tb = __fadd_rd(uu, kTwo23);
    fr = uu - (tb - kTwo23);
    return tb;
}

// plan setup: the number of biased words the projector adds at every accumulator position of
// every local trace (pixels whose delay to the trace's sensor has s0 = t or t + 1).  The
// projector adds bits(fma(xs, f, 1.5*2^23)) = round(xs*f) + bias, so an accumulator row that
// starts at -count * bias holds the exact fixed-point sum after the reductions; the residual
// kernel restores that start when it clears a row it has read.  Per segment (of frame 0: every
// frame adds the same words) the counts are histogrammed per window slot in shared memory with
// the projector's own delay code (same s0, bit for bit), then added to the 4 image traces of
// each lane's base sensor.
__device__ int g_counts_overflow;
__device__ __forceinline__ int* counts_overflow_flag() { return &g_counts_overflow; }

template <bool CLAMP>
__global__ void __launch_bounds__(kFsThreads) fp_sym_count_kernel(const float* pxs, const float* pys,
                                                                  const float* sxs, const float* sys,
                                                                  int n, int M, int groups,
                                                                  const int4* segs,
                                                                  float qclamp, float hx, int LW,
                                                                  int T, const int* trace_of,
                                                                  int acc_ld, int* counts) {
    extern __shared__ int32_t cnt[];  // [LW][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, h = n >> 1;
    const int u = blockIdx.x;
    const int4 sg = segs[u];
    if (sg.x >= groups) return;  // frames > 0 repeat frame 0's words
    const int i0 = h + T * sg.y;
    const int mm = min((sg.x % groups) * 32 + lane, M - 1);  // (segment group: f * groups + group)
    const float sx = __ldg(sxs + mm), sy = __ldg(sys + mm);
    const int lo = fp_sym_window_lo(pxs, pys, n, i0, sg.z, sg.w, sx, sy, qclamp, T);
    for (int q = threadIdx.x; q < LW * 32; q += kFsThreads) cnt[q] = 0;
    __syncthreads();
    for (int jj = sg.z + warp; jj < sg.w; jj += kFsThreads / 32) {
        const float ey = __ldg(pys + jj) - sy;
        const float ey2 = ey * ey;
        for (int c0 = i0; c0 < min(i0 + T, n); c0 += 32) {
            const float pxbs = __ldg(pxs + c0) - sx;
            const int kend = min(32, n - c0);
            for (int k = 0; k < kend; ++k) {
                float fr;
                const float tb = fs_delay<CLAMP>((float)k, hx, pxbs, ey2, qclamp, fr);
                const int slot = (int)(__float_as_uint(tb) - kTwo23Bits) - lo;
                atomicAdd(cnt + slot * 32 + lane, 1);
            }
        }
    }
    __syncthreads();
    // slot k receives the f part of pixels with s0 = lo + k and the 1-f part of those with
    // s0 = lo + k + 1, each word biased by kMagicBits
    const int b = sg.x * 32 + lane;
    const int4 tr = b < M ? __ldg(reinterpret_cast<const int4*>(trace_of) + b) : make_int4(-1, -1, -1, -1);
    for (int q = threadIdx.x; q < LW * 32; q += kFsThreads) {
        const int c = cnt[q] + (q + 32 < LW * 32 ? cnt[q + 32] : 0);
        if (c == 0 || b >= M) continue;  // (lane of q is lane: q % 32 == threadIdx.x % 32)
        const int pos = kAccFront + lo + (q >> 5);
        if (tr.x >= 0) atomicAdd(counts + (size_t)tr.x * acc_ld + pos, c);
        if (tr.y >= 0) atomicAdd(counts + (size_t)tr.y * acc_ld + pos, c);
        if (tr.z >= 0) atomicAdd(counts + (size_t)tr.z * acc_ld + pos, c);
        if (tr.w >= 0) atomicAdd(counts + (size_t)tr.w * acc_ld + pos, c);
    }
}

// plan setup: u16 bias counts of every accumulator position (checked to fit), and every
// frame's accumulator rows set to their start value -count * kMagicBits
__global__ void fp_sym_bias_init_kernel(const int* counts, uint16_t* bias, int32_t* acc, size_t words,
                                        int nf) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < words; q += (size_t)gridDim.x * blockDim.x) {
        const int c = counts[q];
        if (c > 65535) atomicMax(counts_overflow_flag(), 1);
        bias[q] = (uint16_t)min(c, 65535);
        for (int f = 0; f < nf; ++f) acc[(size_t)f * words + q] = -c * kMagicBits;
    }
}

// phase trace of the projector (timing experiments only: -DPK_FS_TRACE=1, tools/k2_trace.py):
// per CTA, clock64 stamps of its phases (slot 0: globaltimer at entry)
#ifndef PK_FS_TRACE
#define PK_FS_TRACE 0
#endif
constexpr int kFsTraceSlots = 64;
#if PK_FS_TRACE
__device__ long long g_fs_trace[1024][kFsTraceSlots];
#define FS_T(i) do { if (threadIdx.x == 0 && (i) < kFsTraceSlots) g_fs_trace[blockIdx.x][(i)] = clock64(); } while (0)
#else
#define FS_T(i) do { } while (0)
#endif

template <int LW, bool CLAMP, int T, int NW>
__global__ void __launch_bounds__(NW * 32, 32 / NW) fp_sym_f32_kernel(FpSymArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int NT = NW * 32;
    int iter = 0;
    if (a.solver) {
        if (a.st->all_stopped) return;
        iter = a.st->iter;
    }
    const int k0 = a.cta_seg0[blockIdx.x], k1 = a.cta_seg0[blockIdx.x + 1];
    if (k0 >= k1) return;
#if PK_FS_TRACE
    __shared__ long long wend_s[2];
    if (threadIdx.x == 0) {
        long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        g_fs_trace[blockIdx.x][0] = gt;
        g_fs_trace[blockIdx.x][1] = clock64();
        g_fs_trace[blockIdx.x][2] = k1 - k0;
        wend_s[0] = 0x7fffffffffffffffLL; wend_s[1] = 0;
    }
#endif
    const float* xall = a.x ? a.x : ((iter & 1) ? a.xb0 : a.xb1);  // bp wrote xb[(iter+1)&1]
    const int n = a.n, h = n >> 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // shared memory: records [NW][32 + kFsBatch] float4 | windows [4][LW][32] | staging
    // [NGR][32][LW + 4] (4 / NGR rounds per segment)
    constexpr int WW = 4 * LW * 32;  // window words
    // images per staging round (plans never launch an instantiation whose windows do not fit:
    // fs_ngr == 0), staging row stride
    constexpr int NGR = fs_ngr(LW, NW, fs_cap(NW)) > 0 ? fs_ngr(LW, NW, fs_cap(NW)) : 1, LWS = LW + 4;
    constexpr int REC = NW * (32 + kFsBatch) * 16;
    float4* rec = reinterpret_cast<float4*>(smem) + (size_t)warp * (32 + kFsBatch);
    int32_t* win = reinterpret_cast<int32_t*>(smem + REC);
    int32_t* stg0 = reinterpret_cast<int32_t*>(smem + REC + (size_t)WW * 4);
    const uint32_t win_s = smem_u32(win);
    __shared__ int piece_s[2];  // dynamic piece counter (double-buffered by segment parity)
    bool pending = false;       // this thread has bulk reductions in flight
    constexpr int P2 = T / 32;  // 32-column pieces per row

    // the 4 image values of piece q of segment (i0, j0): row j0 + q / P2, columns
    // i0 + 32 * (q % P2) + lane
    // (x, xr: the segment frame's x' and rotation-packed x', passed by value)
    // (claiming the last pieces of a segment as 8-column quarters, so the warps leave the
    // scatter together, measured no faster: the pipe stays saturated through the tail)
    auto piece_x = [&](const float* x, const float4* xr, int i0, int j0, int j1, int q, float (&v)[4]) {
        const int jj = j0 + q / P2;
        const int ii = i0 + 32 * (q % P2) + lane;
#pragma unroll
        for (int g = 0; g < 4; ++g) v[g] = 0.f;
        if (jj < j1 && ii < n && xr) {  // one coalesced 16-B load for the 4 images
            const float4 r = xr[(jj - h) * h + (ii - h)];
            v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w;
        } else if (jj < j1 && ii < n) {
            v[0] = x[jj * n + ii];
            v[1] = x[ii * n + (n - 1 - jj)];
            v[2] = x[(n - 1 - jj) * n + (n - 1 - ii)];
            v[3] = x[(n - 1 - ii) * n + jj];
        }
    };
    if (lane < kFsBatch) rec[32 + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
    float scale = 0.f;
    int cur_fr = -1;
    // the fixed-point scale of frame fr: deferred statistics (every CTA reduces the epilogue's
    // max partials of the frame; the CTA of segment rec[fr] records it for the residual kernel)
    // or the plan state.  Ends with a barrier.
    auto reduce_scale = [&](int fr, int k) {
        if (a.part_mx) {
            // the epilogue's CTAs atomicMax their max |x'| into one word per frame (equal to
            // the maximum over its partials, part_mx, which the round-2b projector reduced here)
            const float mx = __uint_as_float(__ldcg(&a.st->fr[fr].mxw));
            __syncthreads();  // (callers rely on a barrier: the windows are initialised)
            const double scl = (mx > 0.f && isfinite(mx)) ? ldexp(1.0, a.bits) / (double)mx : 0.0;
            scale = (float)scl;
            if (k == __ldg(a.rec + fr) && threadIdx.x == 0 && !a.st->fr[fr].stopped) {
                FrameState& fs = a.st->fr[fr];
                fs.maxabs = mx;
                fs.scale64 = scl;
                fs.scale32 = (float)scl;
            }
        } else {
            scale = a.st->fr[fr].scale32;
            __syncthreads();
        }
    };
    {   // windows start at zero (every staging round zeroes the words it has read, so later
        // segments find them zeroed), before the wait for the epilogue
        int4* w4 = reinterpret_cast<int4*>(win);
        for (int q = threadIdx.x; q < WW / 4; q += NT) w4[q] = make_int4(0, 0, 0, 0);
        if (threadIdx.x == 0) piece_s[k0 & 1] = NW;
    }
    griddep_wait();  // x' and its fixed-point scale come from the back-projector epilogue
    FS_T(3);
    for (int k = k0; k < k1; ++k) {
        const int4 sg = __ldg(a.segs + k);
        const int fr = sg.x / a.groups, grp = sg.x - fr * a.groups;
        if (fr != cur_fr) {  // (ends with a barrier: the windows are initialised)
            cur_fr = fr;
            reduce_scale(fr, k);
        }
        FS_T(4 + 8 * (k - k0));
        const float* x = xall + (size_t)fr * n * n;
        const float4* xr = a.x ? nullptr : a.xr + (size_t)fr * h * h;
        int32_t* acc = a.acc + (size_t)fr * a.M * a.acc_ld;
        const int i0 = h + T * sg.y, j0 = sg.z, j1 = sg.w;
        const int m = grp * 32 + lane;
        const bool sensor_ok = m < a.M;
        const int mm = min(m, a.M - 1);
        const float sx = __ldg(a.sxs + mm), sy = __ldg(a.sys + mm);
        // window: trace indices [lo, lo + LW) of this segment (fp_sym_window_lo)
        const int lo = fp_sym_window_lo(a.pxs, a.pys, n, i0, j0, j1, sx, sy, a.qclamp, T);
        // word (g, k, lane) at (g*LW + k)*32 + lane, k = t - lo for trace index t
        const uint32_t adj = win_s + 4u * (uint32_t)lane - 128u * (uint32_t)lo - 128u * kTwo23Bits;
        // the bulk reductions' destinations (trace of each image of this lane's base sensor;
        // the window start is lo), loaded while the segment scatters
        // (double-buffered by segment parity: warp 0 may start the next segment while the
        // issuing warps still read this one's)
        __shared__ int4 trv_s[2][32];
        if (warp == 0) trv_s[k & 1][lane] = sensor_ok ? __ldg(reinterpret_cast<const int4*>(a.trace_of) + m)
                                                      : make_int4(-1, -1, -1, -1);
        // pieces claimed dynamically (the first NW statically, one per warp); the 4 image
        // values of the next piece are loaded while the current one scatters
        const int npc = (j1 - j0) * P2;
        int q = warp;
        auto claim = [&]() {
            int v = 0;
            if (lane == 0) v = atomicAdd(piece_s + (k & 1), 1);
            return __shfl_sync(0xffffffffu, v, 0);
        };
        float xn[4];
        piece_x(x, xr, i0, j0, j1, q, xn);
        while (q < npc) {
            const int jj = j0 + q / P2;
            const int c0 = i0 + 32 * (q % P2);
            const bool in = c0 + lane < n;
            float xv[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) xv[g] = xn[g];
            const int qn = claim();
            piece_x(x, xr, i0, j0, j1, qn, xn);
            // dense records: lane k writes {xs0, xs1, xs2, xs3} of column c0 + k; the scatter
            // derives px from k and xq = rint(xs) from xs, so a record is one LDS.128 (the
            // record loads share the shared-memory pipe with the atomics)
            rec[lane] = in ? make_float4(xv[0] * scale, xv[1] * scale, xv[2] * scale, xv[3] * scale)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            __syncwarp();
            if (sensor_ok && c0 < n) {
                const float ey = __ldg(a.pys + jj) - sy;
                const float ey2 = ey * ey;
                // column k of the piece: x = pxs[c0] + k*hx (samples)
                const float pxbs = __ldg(a.pxs + c0) - sx;
                const int kend = min(32, n - c0);
                auto scatter = [&](auto checked) {
                    constexpr bool CHECK = decltype(checked)::value;
                    auto batch = [&](const int kk) {
                        uint32_t ad[kFsBatch];
                        int32_t va[kFsBatch][4], vb[kFsBatch][4];
#pragma unroll
                        for (int b = 0; b < kFsBatch; ++b) {
                            const float4 r0 = rec[kk + b];
                            float fr;
                            const float tb = fs_delay<CLAMP>((float)(kk + b), a.hx, pxbs, ey2, a.qclamp, fr);
                            const float xs[4] = {r0.x, r0.y, r0.z, r0.w};
                            const float omf = 1.f - fr;
                            // both halves rounded independently (the pair's mass is kept to one
                            // fixed-point unit); each word carries the magic bias, which the
                            // window pre-load removes (fp_sym_count_kernel)
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                va[b][g] = __float_as_int(fmaf(xs[g], fr, kMagic));   // f -> s0
                                vb[b][g] = __float_as_int(fmaf(xs[g], omf, kMagic));  // 1-f -> s0-1
                            }
                            ad[b] = adj + (__float_as_uint(tb) << 7);
                        }
#pragma unroll
                        for (int b = 0; b < kFsBatch; ++b)
                            if (!CHECK || kk + b < kend)  // padding columns beyond the grid add nothing
#pragma unroll
                                for (int g = 0; g < 4; ++g) {
                                    red_smem_s32(ad[b] + (uint32_t)(g * LW * 128) - 128u, vb[b][g]);
                                    red_smem_s32(ad[b] + (uint32_t)(g * LW * 128), va[b][g]);
                                }
                    };
                    if constexpr (!CHECK) {
                        // whole piece: fully unrolled, so the column index kk + b (and its float)
                        // is an immediate -- no per-record integer-to-float conversion
#pragma unroll
                        for (int kk = 0; kk < 32; kk += kFsBatch) batch(kk);
                    } else {
#pragma unroll kFsUnroll
                        for (int kk = 0; kk < kend; kk += kFsBatch) batch(kk);
                    }
                };
                if (kend == 32) scatter(std::false_type{});  // whole piece: no per-column checks
                else scatter(std::true_type{});
            }
            __syncwarp();  // rec is rewritten by the next piece
            q = qn;
        }
#if PK_FS_TRACE
        if (lane == 0) {
            const long long t = clock64();
            atomicMin((unsigned long long*)&wend_s[0], (unsigned long long)t);
            atomicMax((unsigned long long*)&wend_s[1], (unsigned long long)t);
        }
#endif
        // the staging area is rewritten below: the engine must have read the previous
        // segment's last round
        if (pending) bulk_wait_read_all();
        pending = false;
        if (k == k1 - 1) griddep_launch_dependents();
        __syncthreads();  // the segment's windows are complete
#if PK_FS_TRACE
        if (threadIdx.x == 0 && 4 + 8 * (k - k0) + 7 < kFsTraceSlots) {
            g_fs_trace[blockIdx.x][4 + 8 * (k - k0) + 1] = wend_s[0];
            g_fs_trace[blockIdx.x][4 + 8 * (k - k0) + 2] = wend_s[1];
            wend_s[0] = 0x7fffffffffffffffLL; wend_s[1] = 0;
        }
#endif
        FS_T(4 + 8 * (k - k0) + 3);

        // reduce-add the windows into the trace accumulator: per round, NGR images are
        // transposed to staging rows [image][lane][slot] (lane l's window is LW contiguous
        // words, the accumulator row segment it adds to), then thread (image, lane) issues one
        // bulk reduction of LW words (TMA engine, integer adds at L2: order independent)
        static_assert(LW % 8 == 0, "window length must be whole 32-B sectors");
        for (int g0 = 0; g0 < 4; g0 += NGR) {
            // every round stages into the staging area (a later round first waits for the
            // engine to read the earlier one), so the window rows are never staging: the
            // transposition zeroes each word it reads, and the next segment scatters into the
            // window as soon as the last round is issued
            if (g0 > 0) {
                if (pending) bulk_wait_read_all();
                pending = false;
                __syncthreads();
            }
            // thread -> (image gl, lane l, 4 slots): 4 conflict-free LDS (bank l), one STS.128
            // (row stride LW + 4 words: 8 lanes of a phase hit 8 distinct 16-B bank groups)
            constexpr int NTR = NGR * 32 * (LW / 4);  // 4-slot transposition units per round
            constexpr int TU = (NTR + NT - 1) / NT;
            {
                int4 v[TU];
#pragma unroll
                for (int u = 0; u < TU; ++u) {  // all loads first (independent), then the stores
                    const int qq = threadIdx.x + u * NT;
                    const int l = qq & 31, r = qq >> 5;
                    const int gl = r / (LW / 4), sl = (r - gl * (LW / 4)) * 4;
                    int32_t* src = win + ((g0 + gl) * LW + sl) * 32 + l;
                    if (NTR % NT == 0 || qq < NTR) {
                        v[u].x = src[0]; v[u].y = src[32]; v[u].z = src[64]; v[u].w = src[96];
                        src[0] = 0; src[32] = 0; src[64] = 0; src[96] = 0;
                    }
                }
#pragma unroll
                for (int u = 0; u < TU; ++u) {
                    const int qq = threadIdx.x + u * NT;
                    const int l = qq & 31, r = qq >> 5;
                    const int gl = r / (LW / 4), sl = (r - gl * (LW / 4)) * 4;
                    if (NTR % NT == 0 || qq < NTR) *reinterpret_cast<int4*>(stg0 + (gl * 32 + l) * LWS + sl) = v[u];
                }
            }
            if (g0 + NGR >= 4 && threadIdx.x == 0) piece_s[(k + 1) & 1] = NW;  // next segment's claims
            fence_proxy_async_smem();
            __syncthreads();
            if (g0 == 0) FS_T(4 + 8 * (k - k0) + 6);  // (transposed; the bulk issue follows)
            if (threadIdx.x < NGR * 32) {
                const int gl = threadIdx.x >> 5, l = threadIdx.x & 31;
                const int gi = g0 + gl;
                const int tr = reinterpret_cast<const int*>(trv_s[k & 1])[4 * l + gi];
                if (tr >= 0) {  // (lane l of warp gl: base sensor grp * 32 + l, window start lo)
                    bulk_reduce_add_u32(acc + (size_t)tr * a.acc_ld + kAccFront + lo,
                                        smem_u32(stg0 + (gl * 32 + l) * LWS), LW * 4);
                    bulk_commit();
                    pending = true;
                }
            }
            FS_T(4 + 8 * (k - k0) + 4 + g0 / NGR);
        }
    }
    if (pending) bulk_wait_read_all();  // the staging must outlive the engine's reads
    FS_T(kFsTraceSlots - 1);
}

// ===========================================================================
// K2 -- projector, fp64 validation mode (same structure, int64 fixed point, CAS atomics)
// ===========================================================================
struct FpArgs64 {
    const double* x;
    const double* xb0;
    const double* xb1;
    const double *px, *py, *sx, *sy;
    double cdt;
    long long* acc;
    int nx, ny, M, Q, T, L, tiles_x;
    DevState* st;
    double* part_tv;
    int solver;
};

__global__ void __launch_bounds__(kThreads) fp_f64_kernel(FpArgs64 a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double red_d[kThreads / 32];
    int iter = 0;
    if (a.solver) {
        if (a.st->all_stopped) return;
        iter = a.st->iter;
    }
    const double* x = a.x ? a.x : ((iter & 1) ? a.xb0 : a.xb1);
    const double scale = a.st->fr[0].scale64;
    const int T = a.T;
    const int tx = blockIdx.x % a.tiles_x, ty = blockIdx.x / a.tiles_x;
    const int i0 = tx * T, j0 = ty * T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = blockIdx.y * 32 + lane;
    const bool sensor_ok = m < a.M;
    const double sxv = a.sx[min(m, a.M - 1)], syv = a.sy[min(m, a.M - 1)];

    unsigned long long* win = reinterpret_cast<unsigned long long*>(smem);
    double2* rec = reinterpret_cast<double2*>(smem + (size_t)a.L * 32 * 8);  // {px, xs}
    long long* recq = reinterpret_cast<long long*>(smem + (size_t)a.L * 32 * 8 + (size_t)T * T * 16);
    int* rowcnt = reinterpret_cast<int*>(smem + (size_t)a.L * 32 * 8 + (size_t)T * T * 24);

    for (int q = threadIdx.x; q < a.L * 32; q += kThreads) win[q] = 0ull;
    double tv = 0.0;
    const bool do_tv = a.solver && blockIdx.y == 0;
    for (int r = warp; r < T; r += kThreads / 32) {
        const int jj = j0 + r;
        int base = 0;
        for (int cc = 0; cc < T; cc += 32) {
            const int ii = i0 + cc + lane;
            const bool in = ii < a.nx && jj < a.ny && (cc + lane) < T;
            const double xv = in ? x[(size_t)jj * a.nx + ii] : 0.0;
            if (do_tv && in) {
                if (ii + 1 < a.nx) tv += fabs(x[(size_t)jj * a.nx + ii + 1] - xv);
                if (jj + 1 < a.ny) tv += fabs(x[(size_t)(jj + 1) * a.nx + ii] - xv);
            }
            const bool nz = xv != 0.0;
            const uint32_t bal = __ballot_sync(0xffffffffu, nz);
            if (nz) {
                const int pos = base + __popc(bal & ((1u << lane) - 1u));
                const double xs = xv * scale;
                rec[r * T + pos] = make_double2(a.px[ii], xs);
                recq[r * T + pos] = __double2ll_rn(xs);
            }
            base += __popc(bal);
        }
        if (lane == 0) rowcnt[r] = base;
    }
    if (do_tv) {
        const double tvb = block_sum(tv, red_d);
        if (threadIdx.x == 0) a.part_tv[blockIdx.x] = tvb;
    }
    const double X0 = a.px[i0], X1 = a.px[min(i0 + T - 1, a.nx - 1)];
    const double Y0 = a.py[j0], Y1 = a.py[min(j0 + T - 1, a.ny - 1)];
    const double cx = fmin(fmax(sxv, X0), X1), cy = fmin(fmax(syv, Y0), Y1);
    double dmin = sqrt((cx - sxv) * (cx - sxv) + (cy - syv) * (cy - syv)) / a.cdt;
    dmin = fmin(dmin, (double)a.Q + 1.5);
    const int lo = (int)floor(dmin) - 2;
    __syncthreads();

    if (sensor_ok) {
        for (int r = warp; r < T; r += kThreads / 32) {
            const int cnt = rowcnt[r];
            if (cnt == 0) continue;
            const double pyv = a.py[min(j0 + r, a.ny - 1)];
            for (int k = 0; k < cnt; ++k) {
                const double2 q = rec[r * T + k];
                const long long xq = recq[r * T + k];
                const double u = delay_f64(q.x, pyv, sxv, syv, a.cdt);
                double fl = floor(u);
                if (fl > (double)(a.Q + 1)) fl = (double)(a.Q + 1);
                const int s0 = (int)fl;
                const double f = u - fl;
                const long long qa = __double2ll_rn(q.y * f);
                const long long qb = xq - qa;
                const int slot = s0 - lo;  // window slot of trace index s0
                atomicAdd(win + (size_t)(slot - 1) * 32 + lane, (unsigned long long)qb);
                atomicAdd(win + (size_t)slot * 32 + lane, (unsigned long long)qa);
            }
        }
    }
    __syncthreads();
    if (sensor_ok) {
        long long* accm = a.acc + (size_t)m * a.Q;
        for (int k = warp; k < a.L; k += kThreads / 32) {
            const long long v = (long long)win[k * 32 + lane];
            const int t = lo + k;
            if (v != 0 && t >= 0 && t < a.Q)
                atomicAdd(reinterpret_cast<unsigned long long*>(accm + t), (unsigned long long)v);
        }
    }
}

// Pair-table entry s from r[s-1] (rp) and r[s] (rc).  Plain layout {r[s-1], D}; the optional
// fp32 "A-trick" layout {r[s-1] - s*D, D} lets the back-projector use the delay u directly
// (value = fma(u, D, A)) instead of the fraction f = u - s0, saving two FADDs per pair at
// the cost of cancellation error ~ s*ulp (opt-in, PK_BP_ATRICK=1).
template <typename T>
__device__ __forceinline__ typename std::conditional<sizeof(T) == 4, float2, double2>::type
pair_entry(T rp, T rc, int s, int atrick) {
    typename std::conditional<sizeof(T) == 4, float2, double2>::type v;
    const T d = rc - rp;
    v.y = d;
    v.x = atrick ? (T)((double)rp - (double)s * (double)d) : rp;
    return v;
}

// ===========================================================================
// K3 -- residual / finalize: one CTA per (sensor, frame).  r = w*acc/scale - y, acc := 0,
// pair table, sum r^2; solver mode: the last CTA evaluates the objective and the stopping
// rules of every frame.
// ===========================================================================
// start value of 4 accumulator words from their u16 bias counts
__device__ __forceinline__ int4 bias_start4(uint2 c) {
    return make_int4(-(int)(c.x & 0xffffu) * kMagicBits, -(int)(c.x >> 16) * kMagicBits,
                     -(int)(c.y & 0xffffu) * kMagicBits, -(int)(c.y >> 16) * kMagicBits);
}

template <typename T>
struct FinArgs {
    long long* acc;      // [NF][M][Q]
    const T* y;          // [NF][M*Q]; may be null (plain projection); solver mode reads io->y
    T* trace_out;        // [NF][M*Q]; may be null
    typename std::conditional<sizeof(T) == 4, float2, double2>::type* table;  // [M][TS][NF]
    int M, Q, TS;
    double w;
    DevState* st;
    const DevParams* prm;
    const DevIo* io;
    double* part_r;      // [NF][M]
    double* part_tv;     // [tiles][NF] (written here when tv_here)
    int ntv;
    // symmetric projector mode (NF == 1): this kernel also takes TV(x') of the iterate, a
    // pixel slice per CTA, so that no projector unit carries the strided neighbour loads
    const T* xb0;
    const T* xb1;
    int n, tv_here;
    double* part_l1;     // tv_here: [grid][2] sum |x'| and non-finite count per CTA (the
                         // symmetric epilogue deferred them)
    double* sumsq_out;   // optional [NF] (pk_residual)
    int solver;
    // symmetric projector: the int32 accumulator its windows were reduce-added into (row m
    // at acc32 + m * acc32_ld + kAccFront); read and cleared here (one CTA per trace)
    int32_t* acc32;      // (nullptr: acc mode)
    int acc32_ld;
    const uint16_t* bias16;  // [M][acc32_ld] biased words per accumulator position (row start
                             //   value -count * kMagicBits, fp_sym_count_kernel)
    int atrick;
    int chunks;          // sample chunks per sensor (one CTA each)
};

// the last residual CTA: objective terms from the per-CTA partials and the stopping rules of
// every frame (recon.py:346-363); data_s / tv_s: block-shared scratch [NF]
template <typename T, int NF>
__device__ __forceinline__ void finalize_objective(const FinArgs<T>& a, int chunks, double* data_s,
                                                   double* tv_s, double* red_d) {
    __shared__ double l1_s[NF];  // (tv_here) this pass's sum |x'| and non-finite flag per frame
    __shared__ int nf_s[NF];

    if (a.tv_here) {  // symmetric projector, one pass per frame: data, TV, and the epilogue's
                      // deferred sum |x'| and non-finite count (the residual CTAs' partials are
                      // aligned: frame g's are [g * ntv, (g + 1) * ntv))
        __shared__ double red4l[4 * kThreads / 32];
        // every frame's partials loaded in one pass (one round trip, not one per frame); per
        // frame the same per-thread order and block reduction as frame by frame
        double v[NF][4];
        int stp[NF];
#pragma unroll
        for (int g = 0; g < NF; ++g) {
            v[g][0] = v[g][1] = v[g][2] = v[g][3] = 0.0;
            stp[g] = threadIdx.x == 0 ? a.st->fr[g].stopped : 1;
        }
        for (int q = threadIdx.x; q < a.ntv; q += kThreads) {
#pragma unroll
            for (int g = 0; g < NF; ++g) {
                const size_t o = (size_t)g * a.ntv + q;
                v[g][0] += a.part_r[o];
                v[g][1] += a.part_tv[o];
                v[g][2] += a.part_l1[2 * o];
                v[g][3] += a.part_l1[2 * o + 1];
            }
        }
#pragma unroll
        for (int g = 0; g < NF; ++g) {
            block_sum4(v[g], red4l);
            if (threadIdx.x == 0) {
                data_s[g] = v[g][0];
                tv_s[g] = v[g][1];
                l1_s[g] = v[g][2];
                nf_s[g] = v[g][3] > 0.0 ? 1 : 0;
                if (!stp[g]) {
                    a.st->fr[g].l1sum = v[g][2];
                    a.st->fr[g].nonfinite = v[g][3] > 0.0 ? 1 : 0;
                }
            }
        }
    } else {
#pragma unroll 1
        for (int g = 0; g < NF; ++g) {
            double d = 0.0, t = 0.0;
            for (int q = threadIdx.x; q < a.M * chunks; q += kThreads)
                d += a.part_r[(size_t)g * a.M * chunks + q];
            d = block_sum(d, red_d);
            if (a.solver) {
                for (int q = threadIdx.x; q < a.ntv; q += kThreads) t += a.part_tv[(size_t)q * NF + g];
                t = block_sum(t, red_d);
            }
            if (threadIdx.x == 0) {
                data_s[g] = d;
                tv_s[g] = t;
            }
        }
    }
    // objective and stopping rules: lane g of warp 0 takes frame g (recon.py:346-363), every
    // state / parameter word it reads loaded up front -- one round trip per launch instead of
    // a chain of dependent loads per frame behind the history stores
    if (threadIdx.x >= 32) return;
    __syncwarp();  // thread 0's shared / global writes above are visible to the warp
    if (threadIdx.x == 0 && a.sumsq_out)
        for (int g = 0; g < NF; ++g) a.sumsq_out[g] = data_s[g];
    if (!a.solver) return;
    DevState* st = a.st;
    const DevParams* prm = a.prm;
    const int it = st->iter;
    const int N = prm->iterations;
    const int g = threadIdx.x;
    int stopped_g = 1;
    if (g < NF) {
        FrameState& fs = st->fr[g];
        const FrameState f = fs;  // every field, before any store of this frame
        const double alpha = prm->alpha[g], beta = prm->beta[g], tol = prm->tolerance;
        const double l1sum = a.tv_here ? l1_s[g] : f.l1sum;
        const int nonfinite = a.tv_here ? nf_s[g] : f.nonfinite;
        int stopped = f.stopped, stopped_by = f.stopped_by, accepted = f.accepted;
        if (!stopped) {
            const double data = data_s[g];
            const double l1 = alpha * l1sum;
            const double tv = beta * tv_s[g];
            const double total = data + l1 + tv;
            if (!isfinite(total) || nonfinite) {
                stopped = 1;
                stopped_by = PK_STOP_DIVERGENCE;
            } else {
                double* h = a.io->hist + (size_t)g * 4 * N;
                h[it] = total;
                h[N + it] = data;
                h[2 * N + it] = l1;
                h[3 * N + it] = tv;
                accepted = it + 1;
                fs.accepted = accepted;
                const int grow = total > f.f_prev ? f.grow + 1 : 0;
                fs.grow = grow;
                if (grow >= kDivergenceStreak) {
                    stopped = 1;
                    stopped_by = PK_STOP_DIVERGENCE;
                } else {
                    const double rel = fabs(total - f.f_prev) / fmax(fabs(f.f_prev), 1e-300);
                    fs.f_prev = total;
                    if (tol > 0.0 && rel < tol) {
                        stopped = 1;
                        stopped_by = PK_STOP_TOLERANCE;
                    }
                }
            }
            if (stopped) {
                fs.stopped = 1;
                fs.stopped_by = stopped_by;
            }
        }
        stopped_g = stopped;
        a.io->status[2 * g] = accepted;
        a.io->status[2 * g + 1] = stopped_by;
    }
    const bool all = __all_sync(0xffffffffu, stopped_g != 0);
    if (g == 0) {
        st->iter = it + 1;
        st->all_stopped = (all || it + 1 >= N) ? 1 : 0;
    }
}

template <typename T, int NF>
#ifndef PK_FIN_MINB
#define PK_FIN_MINB 4  // <= 64 registers: 4 CTAs per SM (more registers cost occupancy: 94 regs -> +6 us)
#endif
__global__ void __launch_bounds__(kThreads, PK_FIN_MINB) finalize_kernel(FinArgs<T> a) {
    extern __shared__ __align__(128) unsigned char smem[];
    T* tr = reinterpret_cast<T*>(smem);
    __shared__ double red_d[kThreads / 32];
    __shared__ double data_s[NF], tv_s[NF];
    __shared__ int last_flag;
    if (a.solver && a.st->all_stopped) return;
    // grid (M * chunks, NF): CTA handles samples [c0, c1) of sensor m plus the one-sample
    // halo r[c0-1] its first pair-table entry needs.  The accumulator is read-only here (it
    // is cleared by a memset before the next projection), so neighbouring chunks do not race.
    const int chunks = a.chunks;
    const int m = blockIdx.x / chunks, cix = blockIdx.x % chunks, f = blockIdx.y;
    const int clen = (a.Q + chunks - 1) / chunks;
    const int c0 = cix * clen, c1 = min(a.Q, c0 + clen);
    const T* y = a.solver ? reinterpret_cast<const T*>(a.io->y) : a.y;
    const size_t MQ = (size_t)a.M * a.Q;
    long long* accm = a.acc + (size_t)f * MQ + (size_t)m * a.Q;
    const T* ym = y ? y + f * MQ + (size_t)m * a.Q : nullptr;
    T* om = a.trace_out ? a.trace_out + f * MQ + (size_t)m * a.Q : nullptr;
    int32_t* accr = a.acc32 ? a.acc32 + (size_t)m * a.acc32_ld + kAccFront : nullptr;
    // measurements staged in shared memory by LDGSTS (no registers held across the gather)
    T* ys = reinterpret_cast<T*>(smem + (((size_t)(clen + 1) * sizeof(T) + 15) & ~(size_t)15));
    if (ym) {
        for (int k = threadIdx.x; k < c1 - c0; k += kThreads) cp_async<sizeof(T)>(ys + k, ym + c0 + k);
        cp_async_commit();
    }
    griddep_wait();  // the projection's accumulator / windows and scale
    const double sc = sizeof(T) == 4 ? (double)a.st->fr[f].scale32 : a.st->fr[f].scale64;
    const double wq = sc > 0.0 ? a.w / sc : 0.0;
    // K x rounded to the working type first, then the residual in that type, so that y
    // produced by the same projection gives r == 0 exactly (recon.py:75-79 semantics)
    auto resid_y = [&](long long v, T yvv) -> T {
        const T kx = (T)((double)v * wq);
        return ym ? (T)(kx - yvv) : kx;
    };
    auto resid = [&](int s, long long v) -> T { return resid_y(v, ym ? ys[s - c0] : (T)0); };
    double tvp = 0.0, l1p = 0.0, badp = 0.0;
    auto tv_slice = [&]() {  // exact anisotropic TV of x' (recon.py:169-170), sum |x'|, non-finite
        const T* x = (a.st->iter & 1) ? a.xb0 : a.xb1;  // the back-projector wrote xb[(iter+1)&1]
        const int n = a.n, P = n * n, per = (P + gridDim.x - 1) / gridDim.x;
        const int p1 = min(P, (int)(blockIdx.x + 1) * per);
        for (int p = blockIdx.x * per + threadIdx.x; p < p1; p += kThreads) {
            const T v = x[p];
            l1p += (double)fabs(v);
            if (!isfinite(v)) badp += 1.0;
            if (p % n + 1 < n) tvp += (double)fabs(x[p + 1] - v);
            if (p + n < P) tvp += (double)fabs(x[p + n] - v);
        }
    };
    if (a.tv_here) tv_slice();
    auto sample = [&](int s) -> long long { return accr ? (long long)__ldcg(accr + s) : __ldcg(accm + s); };
    if (ym) cp_async_wait_all();
    __syncthreads();  // ys
    double ss = 0.0;
    // tr[k] holds r[c0 - 1 + k]; 4 samples per thread per step, all loads first
    if (threadIdx.x == 0) tr[0] = (c0 >= 1) ? resid_y(sample(c0 - 1), ym ? ym[c0 - 1] : (T)0) : (T)0;
    for (int s0 = c0 + 4 * threadIdx.x; s0 < c1; s0 += 4 * kThreads) {
        long long v[4];
        const bool full = s0 + 4 <= c1 && (s0 & 1) == 0;
        if (full && accr && (s0 & 3) == 0) {
            const int4 p4 = __ldcg(reinterpret_cast<const int4*>(accr + s0));
            v[0] = p4.x; v[1] = p4.y; v[2] = p4.z; v[3] = p4.w;
        } else if (full && !accr) {
            const longlong2 p0 = __ldcg(reinterpret_cast<const longlong2*>(accm + s0));
            const longlong2 p1 = __ldcg(reinterpret_cast<const longlong2*>(accm + s0 + 2));
            v[0] = p0.x; v[1] = p0.y; v[2] = p1.x; v[3] = p1.y;
        } else {
            for (int q = 0; q < 4; ++q) v[q] = (s0 + q < c1) ? sample(s0 + q) : 0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (s0 + q >= c1) break;
            const T rv = resid(s0 + q, v[q]);
            tr[s0 + q - c0 + 1] = rv;
            if (om) om[s0 + q] = rv;
            ss += (double)rv * (double)rv;
        }
    }
    __syncthreads();
    if (accr) {  // every sample of the row was read (one CTA per trace): reset it, pads included,
                 // to its start value for the next projection's reductions
        int4* row4 = reinterpret_cast<int4*>(accr - kAccFront);
        const uint2* b4 = reinterpret_cast<const uint2*>(a.bias16 + (size_t)m * a.acc32_ld);
        for (int q = threadIdx.x; q < a.acc32_ld / 4; q += kThreads) row4[q] = bias_start4(__ldg(b4 + q));
    }
    // entries e in [c0, c1) (the last chunk also writes the zero-padded tail up to TS)
    const int e1 = (cix == chunks - 1) ? a.TS : c1;
    for (int e = c0 + threadIdx.x; e < e1; e += kThreads) {
        const T rp = (e >= 1 && e - 1 < a.Q) ? tr[e - c0] : (T)0;
        const T rc = (e < a.Q) ? tr[e - c0 + 1] : (T)0;
        a.table[((size_t)m * a.TS + e) * NF + f] = pair_entry<T>(rp, rc, e, a.atrick);
    }
    griddep_launch_dependents();
    if (a.tv_here) {
        __shared__ double red4[4 * kThreads / 32];
        double v4[4] = {ss, tvp, l1p, badp};
        block_sum4(v4, red4);
        if (threadIdx.x == 0) {
            a.part_r[(size_t)f * a.M * chunks + blockIdx.x] = v4[0];
            a.part_tv[blockIdx.x] = v4[1];
            a.part_l1[2 * (size_t)blockIdx.x] = v4[2];
            a.part_l1[2 * (size_t)blockIdx.x + 1] = v4[3];
        }
    } else {
        ss = block_sum(ss, red_d);
        if (threadIdx.x == 0) a.part_r[(size_t)f * a.M * chunks + blockIdx.x] = ss;
    }
    if (!last_block(&a.st->cnt_fin, gridDim.x * gridDim.y, &last_flag)) return;
    finalize_objective<T, NF>(a, chunks, data_s, tv_s, red_d);
}

// K3 for the symmetric projector (fp32): one CTA of 256 threads per (trace, frame), every
// load issued up front -- TV(x') of the iterate (its slice) before the wait for the projection
// (final by then), then per thread groups of 4 samples: the int32 accumulator words and the
// measurements of the group and of the sample before it (so the pair-table entries of the
// group need no exchange between threads: no shared-memory staging, one barrier -- the sums'),
// r = w*acc/scale - y rounded as finalize_kernel does, the pair table, the sums; the row is
// reset to its start value after the barrier (every read of it is done).  Q <= kFinSymMax.
// G: 4-sample groups per thread (1, 2 or 4: the smallest with 4 * 256 * G >= Q; the pair-table
// entries past the groups are a short tail loop)
constexpr int kFinSymG = 4;
constexpr int kFinSymMax = 4 * kThreads * kFinSymG;  // 4096 samples
constexpr int kFinSymB = 3;  // start-value words (uint2 = 4 samples) per thread held in registers
#ifndef PK_FINSYM_MINB
#define PK_FINSYM_MINB 4  // CTAs per SM the residual kernel is compiled for (timing sweeps: 3)
#endif
template <int NF, int G>
__global__ void __launch_bounds__(kThreads, PK_FINSYM_MINB) finalize_sym_kernel(FinArgs<float> a) {
    __shared__ double red_d[kThreads / 32];
    __shared__ double red4[4 * kThreads / 32];
    __shared__ double data_s[NF], tv_s[NF];
    __shared__ int last_flag;
    // state words first (one round trip with the constant loads below; the stop test and the
    // iterate's buffer parity wait on it, the measurement / start-value loads do not)
    const bool stopped = a.solver && a.st->all_stopped;
    const int it_par = a.tv_here ? (a.st->iter & 1) : 0;
    // grid (M, frames); frame-major layouts: y [f][M][Q], accumulator [f][M][acc_ld], pair
    // table [f][M][TS], x [f][P]
    const int m = blockIdx.x, f = blockIdx.y, tid = threadIdx.x, Q = a.Q;
    const size_t fm = (size_t)f * a.M + m;
    const float* ym = a.solver ? reinterpret_cast<const float*>(a.io->y) : a.y;
    if (ym) ym += fm * Q;
    float* om = a.trace_out ? a.trace_out + fm * Q : nullptr;
    int32_t* accr = a.acc32 + fm * a.acc32_ld + kAccFront;
    // measurements (constant): loaded before the wait (G = 4: after it, with the accumulator
    // words -- 64 registers do not hold both sets across the wait)
    const bool y4ok = ym && (Q & 3) == 0;
    float4 y4[G];
    float yp[G];
    auto load_y = [&]() {
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int s0 = 4 * (tid + i * kThreads);
        y4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        yp[i] = 0.f;
        if (ym && s0 < Q) {
            if (y4ok) y4[i] = __ldg(reinterpret_cast<const float4*>(ym + s0));
            else {
                y4[i].x = __ldg(ym + s0);
                if (s0 + 1 < Q) y4[i].y = __ldg(ym + s0 + 1);
                if (s0 + 2 < Q) y4[i].z = __ldg(ym + s0 + 2);
                if (s0 + 3 < Q) y4[i].w = __ldg(ym + s0 + 3);
            }
        }
        if (ym && s0 >= 1 && s0 - 1 < Q) yp[i] = __ldg(ym + s0 - 1);
    }
    };
    // the row's start values (geometry constants): loaded with the measurements, so the row
    // reset after the sums' barrier is stores only (no further round trip at the CTA's tail)
    const int nb4 = a.acc32_ld / 4;
    const uint2* b4 = reinterpret_cast<const uint2*>(a.bias16 + (size_t)m * a.acc32_ld);
    constexpr int B = G <= 2 ? kFinSymB : 0;  // (G = 4: no registers to spare; a loop at the tail)
    uint2 bw[B > 0 ? B : 1];
    auto load_b = [&]() {
#pragma unroll
        for (int i = 0; i < B; ++i) {
            const int q = tid + i * kThreads;
            bw[i] = q < nb4 ? __ldg(b4 + q) : make_uint2(0u, 0u);
        }
    };
    if (G <= 2) { load_y(); load_b(); }
    if (stopped) return;
    double tvp = 0.0, l1p = 0.0, badp = 0.0;
    if (a.tv_here) {  // exact anisotropic TV of x' (recon.py:169-170), sum |x'|, non-finite
        const int n = a.n, P = n * n, per = (P + gridDim.x - 1) / gridDim.x;
        const float* x = (it_par ? a.xb0 : a.xb1) + (size_t)f * P;  // bp wrote xb[(iter+1)&1]
        const int p1 = min(P, (int)(blockIdx.x + 1) * per);
        // two pixels per thread per pass: their 6 loads in flight together
        for (int pb = blockIdx.x * per + tid; pb < p1; pb += 2 * kThreads) {
            float v[2], xr[2], xd[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int p = pb + u * kThreads;
                v[u] = xr[u] = xd[u] = 0.f;
                if (p < p1) {
                    v[u] = x[p];
                    if (p % n + 1 < n) xr[u] = x[p + 1];
                    if (p + n < P) xd[u] = x[p + n];
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int p = pb + u * kThreads;
                if (p >= p1) break;
                l1p += (double)fabsf(v[u]);
                if (!isfinite(v[u])) badp += 1.0;
                if (p % n + 1 < n) tvp += (double)fabsf(xr[u] - v[u]);
                if (p + n < P) tvp += (double)fabsf(xd[u] - v[u]);
            }
        }
    }
    griddep_wait();  // the projection's accumulator and scale
    if (a.solver && blockIdx.x == 0 && tid == 0) a.st->fr[f].mxw = 0u;  // (read by the projector: done)
    if (G > 2) { load_y(); load_b(); }
    int4 v4[G];
    int32_t vp[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int s0 = 4 * (tid + i * kThreads);
        v4[i] = s0 < Q ? __ldcg(reinterpret_cast<const int4*>(accr + s0)) : make_int4(0, 0, 0, 0);
        vp[i] = (s0 >= 1 && s0 - 1 < Q) ? __ldcg(accr + s0 - 1) : 0;
    }
    const double sc = (double)a.st->fr[f].scale32;
    const double wq = sc > 0.0 ? a.w / sc : 0.0;
    // K x rounded to fp32 first, then the residual (recon.py:75-79 semantics)
    auto resid = [&](int32_t v, float yv) -> float {
        const float kx = (float)((double)v * wq);
        return ym ? kx - yv : kx;
    };
    double ss = 0.0;
    float2* tab = a.table + fm * a.TS;
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int s0 = 4 * (tid + i * kThreads);
        if (s0 >= a.TS) continue;
        const int vv[4] = {v4[i].x, v4[i].y, v4[i].z, v4[i].w};
        const float yy[4] = {y4[i].x, y4[i].y, y4[i].z, y4[i].w};
        float rr[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            rr[q] = (s0 + q < Q) ? resid(vv[q], yy[q]) : 0.f;
            if (s0 + q < Q) ss += (double)rr[q] * (double)rr[q];
        }
        if (om && s0 < Q) {
            if (s0 + 4 <= Q && ((reinterpret_cast<uintptr_t>(om) & 15) == 0))
                *reinterpret_cast<float4*>(om + s0) = make_float4(rr[0], rr[1], rr[2], rr[3]);
            else
                for (int q = 0; q < 4 && s0 + q < Q; ++q) om[s0 + q] = rr[q];
        }
        // pair table entries e = s0 .. s0 + 3: {r[e-1], r[e] - r[e-1]}, zero padded beyond Q
        const float rprev = (s0 >= 1 && s0 - 1 < Q) ? resid(vp[i], yp[i]) : 0.f;
        const float2 p0 = pair_entry<float>(rprev, rr[0], s0, a.atrick);
        const float2 p1 = pair_entry<float>(rr[0], rr[1], s0 + 1, a.atrick);
        const float2 p2 = pair_entry<float>(rr[1], rr[2], s0 + 2, a.atrick);
        const float2 p3 = pair_entry<float>(rr[2], rr[3], s0 + 3, a.atrick);
        *reinterpret_cast<float4*>(tab + s0) = make_float4(p0.x, p0.y, p1.x, p1.y);  // (TS even)
        if (s0 + 2 < a.TS) *reinterpret_cast<float4*>(tab + s0 + 2) = make_float4(p2.x, p2.y, p3.x, p3.y);
        // entries past the groups (e.g. Q = 2048: e = 2048, 2049): r[e] = 0 there (Q <= 4 *
        // kThreads * G), so only e = Q = 4 * kThreads * G needs a sample -- r[Q - 1], held by
        // the thread of the last group, which writes them all (no extra load round trip)
        if (s0 + 4 == 4 * kThreads * G) {
            const float rl = (s0 + 3 < Q) ? rr[3] : 0.f;
            for (int e = s0 + 4; e < a.TS; ++e) tab[e] = pair_entry<float>(e == Q ? rl : 0.f, 0.f, e, a.atrick);
        }
    }
    griddep_launch_dependents();
    if (a.tv_here) {
        double w4[4] = {ss, tvp, l1p, badp};
        block_sum4(w4, red4);
        if (tid == 0) {
            a.part_r[fm] = w4[0];
            a.part_tv[fm] = w4[1];
            a.part_l1[2 * fm] = w4[2];
            a.part_l1[2 * fm + 1] = w4[3];
        }
    } else {
        ss = block_sum(ss, red_d);
        if (tid == 0) a.part_r[fm] = ss;
    }
    {   // (after the sums' barrier: every read of the row is done) reset the row, pads
        // included, to its start value for the next projection's reductions
        int4* row4 = reinterpret_cast<int4*>(accr - kAccFront);
#pragma unroll
        for (int i = 0; i < B; ++i) {
            const int q = tid + i * kThreads;
            if (q < nb4) row4[q] = bias_start4(bw[i]);
        }
        for (int q = tid + B * kThreads; q < nb4; q += kThreads) row4[q] = bias_start4(__ldg(b4 + q));
    }
    if (!last_block(&a.st->cnt_fin, gridDim.x * gridDim.y, &last_flag)) return;
    finalize_objective<float, NF>(a, 1, data_s, tv_s, red_d);
}

// ===========================================================================
// pair table from a trace: table[m][s][f] = {sign*y[s-1], sign*(y[s]-y[s-1])}.
// Solver init mode (sign = -1, r0 = -y): the last block writes f_prev = sum y^2 per frame.
// Grid (M, NF).
// ===========================================================================
template <typename T, int NF>
__global__ void __launch_bounds__(kThreads) table_kernel(
    const T* y_direct, const DevIo* io, typename std::conditional<sizeof(T) == 4, float2, double2>::type* table,
    int M, int Q, int TS, T sign, double* part, DevState* st, int init, int atrick, int outer = 0) {
    __shared__ double red_d[kThreads / 32];
    __shared__ int last_flag;
    const T* y = y_direct ? y_direct : reinterpret_cast<const T*>(io->y);
    const int m = blockIdx.x, f = blockIdx.y;
    const T* ym = y + (size_t)f * M * Q + (size_t)m * Q;
    double ss = 0.0;
    for (int e = threadIdx.x; e < TS; e += kThreads) {
        const T rp = (e >= 1 && e - 1 < Q) ? sign * ym[e - 1] : (T)0;
        const T rc = (e < Q) ? sign * ym[e] : (T)0;
        // interleaved [M][TS][NF] (generic kernels) or frame-major [NF][M][TS] (symmetric)
        table[outer ? ((size_t)f * M + m) * TS + e : ((size_t)m * TS + e) * NF + f] = pair_entry<T>(rp, rc, e, atrick);
        if (e < Q) ss += (double)rc * (double)rc;
    }
    if (!init) return;
    ss = block_sum(ss, red_d);
    if (threadIdx.x == 0) part[(size_t)f * M + m] = ss;
    if (!last_block(&st->cnt_misc, gridDim.x * gridDim.y, &last_flag)) return;
#pragma unroll 1
    for (int g = 0; g < NF; ++g) {
        double tot = 0.0;
        for (int q = threadIdx.x; q < M; q += kThreads) tot += part[(size_t)g * M + q];
        tot = block_sum(tot, red_d);
        if (threadIdx.x == 0) st->fr[g].f_prev = tot;
    }
}

// solver state reset + x0 = 0 (recon.py:318-320)
template <typename T, int NF>
__global__ void init_kernel(T* xb0, int P, DevState* st, const DevIo* io) {
    for (int p = blockIdx.x * kThreads + threadIdx.x; p < NF * P; p += gridDim.x * kThreads)
        xb0[p] = (T)0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->iter = 0;
        st->all_stopped = 0;
        st->epoch += 1;
        for (int g = 0; g < NF; ++g) {
            FrameState& fs = st->fr[g];
            fs.accepted = 0;
            fs.stopped = 0;
            fs.stopped_by = PK_STOP_MAX_ITERATIONS;
            fs.grow = 0;
            fs.nonfinite = 0;
            fs.mxw = 0u;
            io->status[2 * g] = 0;
            io->status[2 * g + 1] = PK_STOP_MAX_ITERATIONS;
        }
    }
}

// x_out[f] := the last accepted iterate of frame f
template <typename T, int NF>
__global__ void copy_out_kernel(const T* xb0, const T* xb1, const DevState* st, const DevIo* io,
                                int P) {
    T* dst = reinterpret_cast<T*>(io->x_out);
    for (int f = 0; f < NF; ++f) {
        const T* src = ((st->fr[f].accepted & 1) ? xb1 : xb0) + (size_t)f * P;
        for (int p = blockIdx.x * kThreads + threadIdx.x; p < P; p += gridDim.x * kThreads)
            dst[(size_t)f * P + p] = src[p];
    }
}

// max|x| per frame -> fixed-point scale of the projector (standalone products); grid (B, NF)
template <typename T>
__global__ void __launch_bounds__(kThreads) maxabs_kernel(const T* x, int P, double* part,
                                                          DevState* st, int bits) {
    __shared__ double red_d[kThreads / 32];
    __shared__ int last_flag;
    const int f = blockIdx.y;
    const T* xf = x + (size_t)f * P;
    double mx = 0.0;
    for (int p = blockIdx.x * kThreads + threadIdx.x; p < P; p += gridDim.x * kThreads)
        mx = fmax(mx, fabs((double)xf[p]));
    mx = block_max(mx, red_d);
    if (threadIdx.x == 0) part[(size_t)f * gridDim.x + blockIdx.x] = mx;
    if (!last_block(&st->cnt_misc, gridDim.x * gridDim.y, &last_flag)) return;
#pragma unroll 1
    for (int g = 0; g < (int)gridDim.y; ++g) {
        double m2 = 0.0;
        for (int q = threadIdx.x; q < (int)gridDim.x; q += kThreads)
            m2 = fmax(m2, part[(size_t)g * gridDim.x + q]);
        m2 = block_max(m2, red_d);
        if (threadIdx.x == 0) {
            FrameState& fs = st->fr[g];
            fs.maxabs = m2;
            const double sc = (m2 > 0.0 && isfinite(m2)) ? ldexp(1.0, bits) / m2 : 0.0;
            fs.scale64 = sc;
            fs.scale32 = (float)sc;
        }
    }
}

// ===========================================================================
// sharded update (recon.py:330-338 on an all-reduced gradient) and its sums (NF = 1)
// ===========================================================================
template <typename T>
__global__ void __launch_bounds__(kThreads) grad_update_kernel(const T* x, const T* grad, T* xo,
                                                               int nx, int ny,
                                                               const DevParams* prm) {
    const int p = blockIdx.x * kThreads + threadIdx.x;
    if (p >= nx * ny) return;
    const int i = p % nx, j = p / nx;
    T g = grad[p];
    const T beta = (T)prm->beta[0], eps = (T)prm->eps;
    if (beta > (T)0) g += beta * tv_grad_at<T>(x, p, i, j, nx, ny, eps * eps);
    xo[p] = prox<T>(x[p] - (T)prm->step[0] * g, (T)prm->eta_alpha[0], prm->nonneg != 0);
}

// Peer exchange (pk_peer_*).  Barrier of the world: the epoch of this rank is stored into
// every rank's flag slot [rank] with system-scope release (cumulative over the partial
// gradient written by the preceding kernel on this stream), then every peer's flag is awaited
// with acquire.  One warp; launched as its own kernel so that a waiting rank holds one CTA.
// A peer that has not arrived after timeout_ns (a dead rank) sets the timed-out word
// (epoch[1]) instead of hanging the device; the update then writes NaN (pk_peer_status).
__global__ void peer_barrier_kernel(int* epoch, int* const* flags, int world, int rank,
                                    long long timeout_ns) {
    const int t = threadIdx.x;
    int e = 0;
    if (t == 0) e = ++epoch[0];
    e = __shfl_sync(0xffffffffu, e, 0);
    if (t < world) {
        int* dst = flags[t] + rank;
        asm volatile("fence.acq_rel.sys;\n\tst.release.sys.global.s32 [%0], %1;" ::"l"(dst), "r"(e) : "memory");
        const int* src = flags[rank] + t;
        unsigned long long t0, now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        int v;
        while (true) {
            asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(src) : "memory");
            if (v >= e) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if ((long long)(now - t0) > timeout_ns) {
                atomicExch(epoch + 1, 1);
                break;
            }
            __nanosleep(200);
        }
    }
    __syncwarp();
}

// grad = sum over ranks (rank order) of slot `off` of every rank's block, fused with the
// update of grad_update_kernel.  Peer data is read with ld.global.cv (no stale L1/L2 lines).
template <typename T>
__global__ void __launch_bounds__(kThreads) peer_grad_update_kernel(void* const* grads, size_t off,
                                                                    int world, const T* x, T* xo,
                                                                    int nx, int ny,
                                                                    const DevParams* prm,
                                                                    const int* timed_out) {
    const int p = blockIdx.x * kThreads + threadIdx.x;
    if (p >= nx * ny) return;
    if (*timed_out) {
        xo[p] = (T)NAN;
        return;
    }
    const int i = p % nx, j = p / nx;
    T g = (T)0;
    for (int r = 0; r < world; ++r) g += __ldcv(static_cast<const T*>(grads[r]) + off + p);
    const T beta = (T)prm->beta[0], eps = (T)prm->eps;
    if (beta > (T)0) g += beta * tv_grad_at<T>(x, p, i, j, nx, ny, eps * eps);
    xo[p] = prox<T>(x[p] - (T)prm->step[0] * g, (T)prm->eta_alpha[0], prm->nonneg != 0);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) image_sums_kernel(const T* x, int nx, int ny,
                                                              double* part, DevState* st,
                                                              double* out) {
    __shared__ double red_d[kThreads / 32];
    __shared__ int last_flag;
    double l1 = 0.0, tv = 0.0, bad = 0.0;
    const int P = nx * ny;
    for (int p = blockIdx.x * kThreads + threadIdx.x; p < P; p += gridDim.x * kThreads) {
        const int i = p % nx, j = p / nx;
        const double v = (double)x[p];
        l1 += fabs(v);
        if (i + 1 < nx) tv += fabs((double)x[p + 1] - v);
        if (j + 1 < ny) tv += fabs((double)x[p + nx] - v);
        if (!isfinite(v)) bad += 1.0;
    }
    l1 = block_sum(l1, red_d);
    tv = block_sum(tv, red_d);
    bad = block_sum(bad, red_d);
    if (threadIdx.x == 0) {
        part[3 * blockIdx.x] = l1;
        part[3 * blockIdx.x + 1] = tv;
        part[3 * blockIdx.x + 2] = bad;
    }
    if (!last_block(&st->cnt_misc, gridDim.x, &last_flag)) return;
    double a = 0.0, b = 0.0, c = 0.0;
    for (int q = threadIdx.x; q < (int)gridDim.x; q += kThreads) {
        a += part[3 * q];
        b += part[3 * q + 1];
        c += part[3 * q + 2];
    }
    a = block_sum(a, red_d);
    b = block_sum(b, red_d);
    c = block_sum(c, red_d);
    if (threadIdx.x == 0) {
        out[0] = a;
        out[1] = b;
        out[2] = c;
    }
}

// ===========================================================================
// index dump (verification, fp64, forward.py:157-182)
// ===========================================================================
__global__ void index_dump_kernel(const double* px, const double* py, const double* sx,
                                  const double* sy, double cdt, int nx, int P, int ma, int mb,
                                  long long* s0_out, double* frac_out) {
    const size_t n = (size_t)(mb - ma) * P;
    for (size_t q = (size_t)blockIdx.x * kThreads + threadIdx.x; q < n;
         q += (size_t)gridDim.x * kThreads) {
        const int m = ma + (int)(q / P);
        const int p = (int)(q % P);
        const double u = delay_f64(px[p % nx], py[p / nx], sx[m], sy[m], cdt);
        const double fl = floor(u);
        s0_out[q] = (long long)fl;
        if (frac_out) frac_out[q] = u - fl;
    }
}

// fp32 delay census (verification): the delay s0 / frac the fp32 production kernels use for
// every pair (p, m) of local sensors [ma, mb), in layout [(m - ma)][p].  rule 0: the generic
// K1 / K2 delay (pixel and sensor coordinates scaled by 1/(c dt), bp_f32_kernel /
// fp_f32_kernel); rule 1: K1s -- the delay of the D4 representative pair (tile-level octant of
// the quadrant, bp_sym_f32_kernel / sym_chunk); rule 2: K2s -- the delay of the rotation
// representative in the quadrant, column derived from its 32-pixel piece (fs_delay).
__global__ void delay_census_f32_kernel(const float* pxs, const float* pys, const float* sxs,
                                        const float* sys, int n_x, int P, int M, int ma, int mb,
                                        int rule, float qclamp, float hx, int32_t* s0_out,
                                        float* frac_out) {
    const size_t total = (size_t)(mb - ma) * P;
    for (size_t q = (size_t)blockIdx.x * kThreads + threadIdx.x; q < total;
         q += (size_t)gridDim.x * kThreads) {
        const int m = ma + (int)(q / P);
        const int p = (int)(q % P);
        const int i = p % n_x, j = p / n_x;
        float tb, fr;
        if (rule == 0) {
            const float ex = pxs[i] - sxs[m], ey = pys[j] - sys[m];
            const float u = fminf(sqrt_approx(fmaf(ex, ex, ey * ey)), qclamp);
            tb = __fadd_rd(u, kTwo23);
            fr = u - (tb - kTwo23);
        } else if (rule == 1) {
            // the representative c (tile tx >= ty of the quadrant) and the group element g with
            // sym_pixel(g, c) = p (reflections only for off-diagonal tiles)
            const int n = n_x, h = n >> 1;
            int ci = 0, cj = 0, gg = -1;
            for (int a = 0; a < 8 && gg < 0; ++a) {
                int oi, oj;
                sym_pixel(a, i, j, n, oi, oj);  // orbit of p
                if (oi < h || oj < h) continue;
                const int tx = (oi - h) / kSymTile, ty = (oj - h) / kSymTile;
                if (tx < ty) continue;
                for (int g = 0; g < 8; ++g) {
                    if (tx == ty && g >= 4) break;
                    int ri, rj;
                    sym_pixel(g, oi, oj, n, ri, rj);
                    if (ri == i && rj == j) { ci = oi; cj = oj; gg = g; break; }
                }
            }
            const int qm = M >> 2;
            int mbase = gg < 4 ? m - gg * qm : (gg - 4) * qm - m;
            mbase %= M;
            if (mbase < 0) mbase += M;
            const float ex = pxs[ci] - sxs[mbase], ey = pys[cj] - sys[mbase];
            const float u = fminf(sqrt_approx(fmaf(ex, ex, ey * ey)), qclamp);
            tb = __fadd_rd(u, kTwo23);
            fr = u - (tb - kTwo23);
        } else {
            const int n = n_x, h = n >> 1;
            const int ri = sym_rot_index(i, j, n);
            const int r = ri & 3, qq = ri >> 2;
            const int qi = h + qq % h, qj = h + qq / h;
            int mbase = (m - r * (M >> 2)) % M;
            if (mbase < 0) mbase += M;
            const int c0 = h + 32 * ((qi - h) / 32);
            const float ey = pys[qj] - sys[mbase];
            tb = fs_delay<true>((float)(qi - c0), hx, pxs[c0] - sxs[mbase], ey * ey, qclamp, fr);
        }
        s0_out[q] = (int32_t)(__float_as_uint(tb) - kTwo23Bits);
        frac_out[q] = fr;
    }
}

// fp64 -> plan dtype conversion and back (host API)
template <typename T>
__global__ void convert_kernel(const double* src, T* dst, size_t n) {
    for (size_t q = (size_t)blockIdx.x * kThreads + threadIdx.x; q < n;
         q += (size_t)gridDim.x * kThreads)
        dst[q] = (T)src[q];
}
template <typename T>
__global__ void widen_kernel(const T* src, double* dst, size_t n) {
    for (size_t q = (size_t)blockIdx.x * kThreads + threadIdx.x; q < n;
         q += (size_t)gridDim.x * kThreads)
        dst[q] = (double)src[q];
}

}  // namespace pk
