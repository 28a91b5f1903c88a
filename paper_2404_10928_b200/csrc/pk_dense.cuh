// pk_dense.cuh -- explicit-matrix mode: a MeasurementMatrix whose
// entries are given (read_matrix / PACTMAT, forward.py:70-121, 297-330) instead of geometry.
// The reference runs every product of such a K through its numba GEMV cores
// (kernels.py:195-202 forward, 215-225 adjoint).  Here K lives in HBM in the plan dtype
// (fp32 halves the bytes) and every kernel is bound by streaming it:
//
//   dense_gemv_kernel    y = K x (- y_obs), a warp per row, 16-B loads, per-CTA sum |r|^2
//   dense_gemvt_kernel   partial K^H y over row splits, a thread per 16 B of columns
//   dense_fused_kernel   the solver's pass (real K, fp32): r = K x - y and the gradient
//                        partials K^T r from ONE read of K -- the row is held in registers
//                        between its dot product and its rank-1 accumulation, x and the
//                        CTA's gradient partial in shared memory
//   dense_update_kernel  grad = 2 sum_s partial_s (split order: deterministic), TV gradient,
//                        soft threshold, non-negativity (recon.py:327-338)
//   dense_stop_kernel    sum |x'|, TV(x'), non-finite count; the last block reduces every
//                        partial in fixed order and applies recon.py:346-363
// Complex entries (frequency-domain K) are interleaved (re, im).
#pragma once
#include <type_traits>

#include "pk_common.cuh"

namespace pk {

constexpr int kDenseThreads = 256;
constexpr int kFusedThreads = 512;

// elements (real or complex) per 16-byte load
template <typename R, bool C>
struct DVec {
    static constexpr int E = 16 / (int)(sizeof(R) * (C ? 2 : 1));
};

// 16 B of x (re-read by every row: cached, read-only path)
template <typename R>
__device__ __forceinline__ void ldx16(const R* p, R (&o)[16 / sizeof(R)]) {
    if constexpr (sizeof(R) == 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
        const double2 v = __ldg(reinterpret_cast<const double2*>(p));
        o[0] = v.x; o[1] = v.y;
    }
}

template <typename R>
__device__ __forceinline__ void ld16(const R* p, R (&o)[16 / sizeof(R)]) {
    if constexpr (sizeof(R) == 4) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(p));  // streamed once
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(p));
        o[0] = v.x; o[1] = v.y;
    }
}

// ---------------------------------------------------------------------------
// y[i] = sum_c K[i, c] x[c]  (KC: complex K; XC: complex x; output complex iff KC || XC)
// minus y_obs[i] when given; per-CTA partial of sum |y[i]|^2 into part (fp64, fixed order).
// Grid-stride over rows by warps.  cols must be a multiple of the 16-B element count.
struct DenseState;
__device__ __forceinline__ int dense_cand(const DenseState* st);

// Solver mode (st != null): x is the candidate xb[(accepted + 1) & 1] (x0 / x1) and the
// residual goes to the candidate buffer out0 / out1 likewise; standalone: x0, out0.
template <typename R, bool KC, bool XC>
__global__ void __launch_bounds__(kDenseThreads) dense_gemv_kernel(
    const R* __restrict__ K, int64_t rows, int64_t cols, const R* x0, const R* x1,
    const R* __restrict__ yobs, R* out0, R* out1, double* part, const DenseState* st) {
    constexpr bool OC = KC || XC;
    __shared__ double red[kDenseThreads / 32];
    int cand = 0;
    if (st) {
        cand = dense_cand(st);
        if (cand < 0) return;
    }
    const R* __restrict__ x = cand ? x1 : x0;
    R* __restrict__ out = cand ? out1 : out0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int E = DVec<R, KC>::E;
    constexpr int W = 16 / sizeof(R);  // scalars per 16-B load
    const int64_t nvec = cols / E;
    double ss = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * (kDenseThreads / 32) + warp; i < rows;
         i += (int64_t)gridDim.x * (kDenseThreads / 32)) {
        const R* row = K + i * cols * (KC ? 2 : 1);
        R sr = 0, si = 0;
        constexpr int U = 4;  // 16-B loads in flight per lane
        auto cols_step = [&](int64_t v0, auto nu) {
          constexpr int NU = decltype(nu)::value;
          R b[NU][W];
#pragma unroll
          for (int u = 0; u < NU; ++u) ld16(row + (v0 + 32 * u) * W, b[u]);
          // real K and x: x in the same 16-B vectors as the row (one L1 wavefront per 32
          // lanes x 16 B instead of four scalar loads at a 16-B stride)
          R xv[NU][W];
          if constexpr (!KC && !XC) {
#pragma unroll
            for (int u = 0; u < NU; ++u) ldx16(x + (v0 + 32 * u) * W, xv[u]);
          }
#pragma unroll
          for (int u = 0; u < NU; ++u) {
            const int64_t v = v0 + 32 * u;
            const R* a = b[u];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int64_t c = v * E + e;
                if constexpr (!KC && !XC) {
                    sr = fma(a[e], xv[u][e], sr);
                } else if constexpr (!KC && XC) {
                    sr = fma(a[e], __ldg(x + 2 * c), sr);
                    si = fma(a[e], __ldg(x + 2 * c + 1), si);
                } else if constexpr (KC && !XC) {
                    const R xv = __ldg(x + c);
                    sr = fma(a[2 * e], xv, sr);
                    si = fma(a[2 * e + 1], xv, si);
                } else {
                    const R xr = __ldg(x + 2 * c), xi = __ldg(x + 2 * c + 1);
                    sr = fma(a[2 * e], xr, sr);
                    sr = fma(-a[2 * e + 1], xi, sr);
                    si = fma(a[2 * e], xi, si);
                    si = fma(a[2 * e + 1], xr, si);
                }
            }
          }
        };
        int64_t v0 = lane;
        for (; v0 + 32 * (U - 1) < nvec; v0 += 32 * U) cols_step(v0, std::integral_constant<int, U>{});
        for (; v0 < nvec; v0 += 32) cols_step(v0, std::integral_constant<int, 1>{});
        sr = warp_sum(sr);
        if (OC) si = warp_sum(si);
        if (lane == 0) {
            if (yobs) {
                sr -= yobs[OC ? 2 * i : i];
                if (OC) si -= yobs[2 * i + 1];
            }
            if (out) {
                out[OC ? 2 * i : i] = sr;
                if (OC) out[2 * i + 1] = si;
            }
            ss += (double)sr * (double)sr + (OC ? (double)si * (double)si : 0.0);
        }
    }
    if (part) {
        ss = block_sum<double, kDenseThreads>(ss, red);
        if (threadIdx.x == 0) part[blockIdx.x] = ss;
    }
}

// ---------------------------------------------------------------------------
// part[s][c] = sum_{i in split s} conj(K[i, c]) y[i] (REAL: only the real part -- the
// solver's Re(K^H r), recon.py:143).  Grid (column tiles, splits); thread = 16 B of columns.
// Solver mode (st != null): y is the current residual rb[accepted & 1] (y0 / y1).
template <typename R, bool KC, bool YC, bool REAL>
__global__ void __launch_bounds__(kDenseThreads) dense_gemvt_kernel(
    const R* __restrict__ K, int64_t rows, int64_t cols, const R* y0, const R* y1, R sign,
    R* __restrict__ part, const DenseState* st) {
    int curr = 0;
    if (st) {
        const int cand = dense_cand(st);
        if (cand < 0) return;
        curr = cand ^ 1;
    }
    const R* __restrict__ y = curr ? y1 : y0;
    constexpr int E = DVec<R, KC>::E;
    constexpr int W = 16 / sizeof(R);
    constexpr bool OC = (KC || YC) && !REAL;
    const int64_t v = (int64_t)blockIdx.x * kDenseThreads + threadIdx.x;  // 16-B column group
    const int64_t nvec = cols / E;
    const int splits = gridDim.y;
    const int64_t r0 = rows * blockIdx.y / splits, r1 = rows * (blockIdx.y + 1) / splits;
    R ar[E], ai[E];
#pragma unroll
    for (int e = 0; e < E; ++e) ar[e] = ai[e] = 0;
    if (v < nvec) {
        const int64_t stride = cols * (KC ? 2 : 1);
        const R* col = K + v * W;
        constexpr int U = 8;  // rows in flight per thread
        auto rows_step = [&](int64_t i0, auto nu) {
            constexpr int NU = decltype(nu)::value;
            R a[NU][W];
#pragma unroll
            for (int u = 0; u < NU; ++u) ld16(col + (i0 + u) * stride, a[u]);
#pragma unroll
            for (int u = 0; u < NU; ++u) {
                const int64_t i = i0 + u;
                const R yr = sign * __ldg(y + (YC ? 2 * i : i));
                const R yi = YC ? sign * __ldg(y + 2 * i + 1) : (R)0;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const R kr = KC ? a[u][2 * e] : a[u][e], ki = KC ? a[u][2 * e + 1] : (R)0;
                    // conj(k) * y = (kr yr + ki yi) + i (kr yi - ki yr)
                    ar[e] = fma(kr, yr, ar[e]);
                    if (KC && YC) ar[e] = fma(ki, yi, ar[e]);
                    if (OC) {
                        if (YC) ai[e] = fma(kr, yi, ai[e]);
                        if (KC) ai[e] = fma(-ki, yr, ai[e]);
                    }
                }
            }
        };
        int64_t i0 = r0;
        for (; i0 + U <= r1; i0 += U) rows_step(i0, std::integral_constant<int, U>{});
        for (; i0 < r1; ++i0) rows_step(i0, std::integral_constant<int, 1>{});
        R* dst = part + (size_t)blockIdx.y * cols * (OC ? 2 : 1);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int64_t c = v * E + e;
            if (OC) {
                dst[2 * c] = ar[e];
                dst[2 * c + 1] = ai[e];
            } else {
                dst[c] = ar[e];
            }
        }
    }
}

// out[c] = scale * sum_s part[s][c] in split order (n scalars per split)
template <typename R>
__global__ void __launch_bounds__(kDenseThreads) dense_reduce_kernel(const R* part, int splits,
                                                                     int64_t n, R scale, R* out) {
    const int64_t c = (int64_t)blockIdx.x * kDenseThreads + threadIdx.x;
    if (c >= n) return;
    R s = 0;
    for (int q = 0; q < splits; ++q) s += part[(size_t)q * n + c];
    out[c] = scale * s;
}

// ---------------------------------------------------------------------------
// solver state of one dense solve (device)
struct DenseState {
    int32_t iter;       // iterations attempted
    int32_t accepted;   // iterations accepted (x_k lives in xb[accepted & 1])
    int32_t stopped;    // the loop is over: every kernel returns at once
    int32_t stopped_by;
    int32_t grow;
    uint32_t cnt;       // last-block counter of dense_stop_kernel
    double f_prev;
};

// candidate buffer index (accepted + 1) & 1, or -1 once the solve has stopped
__device__ __forceinline__ int dense_cand(const DenseState* st) {
    return st->stopped ? -1 : ((st->accepted + 1) & 1);
}

// ---------------------------------------------------------------------------
// Fused pass for real K: for every row i of this CTA's contiguous row range
//   r_i = K_i . x - y_i,  sumsq += r_i^2,  gacc += r_i * K_i
// K_i is loaded once (16-B streaming loads, the next row prefetched) and kept in registers
// between the dot product and the rank-1 update.  gacc ends in part[blockIdx.x][cols].
// cols % 4 == 0 and 2 * cols * 4 B of shared memory (x and gacc).
template <int NV>
__global__ void __launch_bounds__(kFusedThreads, 1) dense_fused_f32_kernel(
    const float* __restrict__ K, int64_t rows, int cols, const float* xb0, const float* xb1,
    const float* __restrict__ yobs, float* __restrict__ part, double* __restrict__ rpart,
    DenseState* st, int use_state_x) {
    extern __shared__ __align__(16) float dsm[];
    __shared__ float red[2][kFusedThreads / 32];
    if (use_state_x && st->stopped) return;
    // solver: the candidate x' = xb[(accepted + 1) & 1]; init pass (use_state_x == 0): x = xb0
    const float* x = use_state_x ? (((st->accepted + 1) & 1) ? xb1 : xb0) : xb0;
    const int nv = cols >> 2;  // float4 column groups
    float4* xs = reinterpret_cast<float4*>(dsm);
    float4* gs = xs + nv;
    for (int v = threadIdx.x; v < nv; v += kFusedThreads) {
        xs[v] = reinterpret_cast<const float4*>(x)[v];
        gs[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    const int64_t r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float4 cur[NV], nxt[NV];
    auto load = [&](int64_t i, float4 (&o)[NV]) {
        const float4* row = reinterpret_cast<const float4*>(K + i * (int64_t)cols);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int v = threadIdx.x + k * kFusedThreads;
            o[k] = (v < nv && i < r1) ? __ldcs(row + v) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    if (r0 < r1) load(r0, cur);
    double ss = 0.0;
    int b = 0;
    for (int64_t i = r0; i < r1; ++i) {
        load(i + 1, nxt);  // the next row's bytes are in flight during this row's work
        float d = 0.f;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int v = threadIdx.x + k * kFusedThreads;
            if (v < nv) {
                const float4 xv = xs[v];
                d = fmaf(cur[k].x, xv.x, d);
                d = fmaf(cur[k].y, xv.y, d);
                d = fmaf(cur[k].z, xv.z, d);
                d = fmaf(cur[k].w, xv.w, d);
            }
        }
        d = warp_sum(d);
        if (lane == 0) red[b][warp] = d;
        __syncthreads();  // (red is double-buffered: one barrier per row)
        float dot = red[b][0];
#pragma unroll
        for (int w = 1; w < kFusedThreads / 32; ++w) dot += red[b][w];
        const float r = dot - __ldg(yobs + i);
        if (threadIdx.x == 0) ss += (double)r * (double)r;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int v = threadIdx.x + k * kFusedThreads;
            if (v < nv) {
                float4 g = gs[v];
                g.x = fmaf(r, cur[k].x, g.x);
                g.y = fmaf(r, cur[k].y, g.y);
                g.z = fmaf(r, cur[k].z, g.z);
                g.w = fmaf(r, cur[k].w, g.w);
                gs[v] = g;
            }
            cur[k] = nxt[k];
        }
        b ^= 1;
    }
    __syncthreads();
    float4* dst = reinterpret_cast<float4*>(part + (size_t)blockIdx.x * cols);
    for (int v = threadIdx.x; v < nv; v += kFusedThreads) dst[v] = gs[v];
    if (threadIdx.x == 0) rpart[blockIdx.x] = ss;
}

// ---------------------------------------------------------------------------
// x' = prox(x - eta (2 sum_s part_s + beta tvgrad(x)))  into xb[(accepted + 1) & 1]
template <typename R>
__global__ void __launch_bounds__(kDenseThreads) dense_update_kernel(
    R* xb0, R* xb1, const R* __restrict__ part, int splits, int nx, int ny, const DevParams* prm,
    const DenseState* st) {
    if (st->stopped) return;
    const int p = blockIdx.x * kDenseThreads + threadIdx.x;
    const int P = nx * ny;
    if (p >= P) return;
    const R* x = (st->accepted & 1) ? xb1 : xb0;
    R* xo = (st->accepted & 1) ? xb0 : xb1;
    R g = 0;
    for (int q = 0; q < splits; ++q) g += part[(size_t)q * P + p];
    g *= (R)2;
    const R beta = (R)prm->beta[0], eps = (R)prm->eps;
    if (beta > (R)0) g += beta * tv_grad_at<R>(x, p, p % nx, p / nx, nx, ny, eps * eps);
    xo[p] = prox<R>(x[p] - (R)prm->step[0] * g, (R)prm->eta_alpha[0], prm->nonneg != 0);
}

// objective of the candidate and the stopping rules.  init: f_prev = sum r0^2 only.
template <typename R>
__global__ void __launch_bounds__(kDenseThreads) dense_stop_kernel(
    const R* xb0, const R* xb1, int nx, int ny, const double* rpart, int nr, double* ipart,
    const DevParams* prm, DenseState* st, double* hist, int32_t* status, int init) {
    __shared__ double red[kDenseThreads / 32];
    __shared__ int last_flag;
    if (st->stopped) return;
    double l1 = 0.0, tv = 0.0, bad = 0.0;
    if (!init) {
        const R* x = ((st->accepted + 1) & 1) ? xb1 : xb0;  // the candidate
        const int P = nx * ny;
        for (int p = blockIdx.x * kDenseThreads + threadIdx.x; p < P; p += gridDim.x * kDenseThreads) {
            const int i = p % nx, j = p / nx;
            const double v = (double)x[p];
            l1 += fabs(v);
            if (i + 1 < nx) tv += fabs((double)x[p + 1] - v);
            if (j + 1 < ny) tv += fabs((double)x[p + nx] - v);
            if (!isfinite(v)) bad += 1.0;
        }
        l1 = block_sum<double, kDenseThreads>(l1, red);
        tv = block_sum<double, kDenseThreads>(tv, red);
        bad = block_sum<double, kDenseThreads>(bad, red);
        if (threadIdx.x == 0) {
            ipart[3 * blockIdx.x] = l1;
            ipart[3 * blockIdx.x + 1] = tv;
            ipart[3 * blockIdx.x + 2] = bad;
        }
    }
    if (!last_block(&st->cnt, gridDim.x, &last_flag)) return;
    double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
    if (!init)
        for (int q = threadIdx.x; q < (int)gridDim.x; q += kDenseThreads) {
            a += ipart[3 * q];
            b += ipart[3 * q + 1];
            c += ipart[3 * q + 2];
        }
    for (int q = threadIdx.x; q < nr; q += kDenseThreads) d += rpart[q];
    a = block_sum<double, kDenseThreads>(a, red);
    b = block_sum<double, kDenseThreads>(b, red);
    c = block_sum<double, kDenseThreads>(c, red);
    d = block_sum<double, kDenseThreads>(d, red);
    if (threadIdx.x != 0) return;
    if (init) {
        st->f_prev = d;
        return;
    }
    const int N = prm->iterations;
    const int it = st->iter;
    const double l1v = prm->alpha[0] * a, tvv = prm->beta[0] * b;
    const double total = d + l1v + tvv;
    if (!isfinite(total) || c > 0.0) {  // recon.py:349-351: keep the previous iterate
        st->stopped = 1;
        st->stopped_by = PK_STOP_DIVERGENCE;
    } else {
        hist[it] = total;
        hist[N + it] = d;
        hist[2 * N + it] = l1v;
        hist[3 * N + it] = tvv;
        st->accepted = st->accepted + 1;
        st->grow = total > st->f_prev ? st->grow + 1 : 0;
        if (st->grow >= kDivergenceStreak) {
            st->stopped = 1;
            st->stopped_by = PK_STOP_DIVERGENCE;
        } else {
            const double rel = fabs(total - st->f_prev) / fmax(fabs(st->f_prev), 1e-300);
            st->f_prev = total;
            if (prm->tolerance > 0.0 && rel < prm->tolerance) {
                st->stopped = 1;
                st->stopped_by = PK_STOP_TOLERANCE;
            }
        }
    }
    st->iter = it + 1;
    if (st->iter >= N) st->stopped = 1;
    status[0] = st->accepted;
    status[1] = st->stopped_by;
}

// x0 = 0; two-pass path: r0 = -y (nr scalars) with per-block partials of sum r0^2
template <typename R>
__global__ void __launch_bounds__(kDenseThreads) dense_init_kernel(R* xb0, int P, DenseState* st,
                                                                   const R* y, R* r0, int64_t nr,
                                                                   double* rpart) {
    __shared__ double red[kDenseThreads / 32];
    const int64_t q = (int64_t)blockIdx.x * kDenseThreads + threadIdx.x;
    if (q < P) xb0[q] = 0;
    double ss = 0.0;
    if (r0 && q < nr) {
        const R v = -y[q];
        r0[q] = v;
        ss = (double)v * (double)v;
    }
    if (r0) {
        ss = block_sum<double, kDenseThreads>(ss, red);
        if (threadIdx.x == 0) rpart[blockIdx.x] = ss;
    }
    if (q == 0) {
        st->iter = 0;
        st->accepted = 0;
        st->stopped = 0;
        st->stopped_by = PK_STOP_MAX_ITERATIONS;
        st->grow = 0;
        st->cnt = 0;
        st->f_prev = 0.0;
    }
}

// the residual of the accepted iterate for the next gradient (two-pass path): current r
// lives in rb[accepted & 1]; dense_gemv writes the candidate's into rb[(accepted + 1) & 1]
template <typename R>
__global__ void dense_copy_out_kernel(const R* xb0, const R* xb1, const DenseState* st, R* out,
                                      int P) {
    const int p = blockIdx.x * kDenseThreads + threadIdx.x;
    if (p < P) out[p] = (st->accepted & 1) ? xb1[p] : xb0[p];
}

// build_time_matrix on the device (forward.py:167-194): K[m*Q + s0 - 1, p] = (1 - f) w when
// 1 <= s0 <= Q and K[m*Q + s0, p] = f w when 0 <= s0 <= Q - 1, with s0 / f from the fp64 delay
// evaluated exactly as the reference (delay_f64), so fp64 entries are bit-identical to the
// reference's dense K.  K must be zeroed first.
template <typename R>
__global__ void dense_from_geometry_kernel(const double* px, const double* py, const double* sx,
                                           const double* sy, double cdt, double w, int nx, int P,
                                           int M, int Q, R* K) {
    const size_t n = (size_t)M * P;
    for (size_t q = (size_t)blockIdx.x * kDenseThreads + threadIdx.x; q < n;
         q += (size_t)gridDim.x * kDenseThreads) {
        const int m = (int)(q / P), p = (int)(q % P);
        const double u = delay_f64(px[p % nx], py[p / nx], sx[m], sy[m], cdt);
        const double fl = floor(u);
        const long long s0 = (long long)fl;
        const double f = __dsub_rn(u, fl);
        if (s0 >= 1 && s0 <= Q) K[((size_t)m * Q + (size_t)(s0 - 1)) * P + p] = (R)__dmul_rn(__dsub_rn(1.0, f), w);
        if (s0 >= 0 && s0 <= Q - 1) K[((size_t)m * Q + (size_t)s0) * P + p] = (R)__dmul_rn(f, w);
    }
}

}  // namespace pk
