// pk_freq.cuh -- matrix-free frequency-domain operator.
//
// The reference builds K_f[m*q_n + (n-1), p] = i c k_n exp(-i k_n d_mp) / d_mp densely
// (forward.py:218-234, Eq. 7 of the paper), k_n = 2 pi n / (q_s dt c), n = 1..q_n.  With
// u = d / (c dt) (the delay in samples) the phase is k_n d = 2 pi n f, f = frac(u / q_s), so
//   forward  y[m, n] = i c k_n  sum_p x_p z_mp^n / d_mp,        z = exp(-2 pi i f)
//   adjoint  g_p     = sum_m (1/d_mp) sum_n (-i c k_n) y[m, n] conj(z_mp)^n
// Phases are reduced in fp64 (f and frac(n0 f)), then advanced in the working type by
// complex multiplication over short runs of n (16 in the forward, 32 in the adjoint) and
// re-anchored, so the recurrence error stays ~run length x ulp.  Distances come from the fp64
// coordinates with the reference's hypot (bit-exact u).  Sums over pixels are written as
// per-chunk partials and added in chunk order (deterministic).
#pragma once
#include "pk_common.cuh"

namespace pk {

template <typename T>
struct Cplx { using type = float2; };
template <>
struct Cplx<double> { using type = double2; };

template <typename T>
__device__ __forceinline__ void sincospi_t(T a, T* s, T* c);
template <>
__device__ __forceinline__ void sincospi_t<float>(float a, float* s, float* c) { sincospif(a, s, c); }
template <>
__device__ __forceinline__ void sincospi_t<double>(double a, double* s, double* c) { sincospi(a, s, c); }

constexpr int kFreqRun = 16;      // forward: consecutive n per thread
constexpr int kFreqThreads = 128; // forward: threads per CTA (n-blocks)
constexpr int kFreqPix = 64;      // forward: pixels staged per smem round
constexpr int kFreqAdjRun = 32;   // adjoint: Horner run length between exact phase anchors

struct FreqArgs {
    const double *px, *py, *sx, *sy;  // fp64 coordinates (plan)
    int nx, P, M, Q, qn;
    double cdt;
    int chunks;            // forward: pixel chunks (partials)
    const void* x;         // forward input [P] (plan dtype)
    void* part;            // forward partials [chunks][M][qn] complex
    const void* y;         // adjoint input [M][qn] complex
    void* out;             // forward: y [M][qn] complex; adjoint: g [P] complex
    double c, kscale;      // c and 2 pi / (q_s dt c) (k_n = n * kscale)
    double scale;          // adjoint multiplier
};

// forward, stage 1: CTA (sensor m, pixel chunk, n-range); thread t owns n = n0 .. n0+15
template <typename T>
__global__ void __launch_bounds__(kFreqThreads) freq_fwd_kernel(FreqArgs a) {
    using C = typename Cplx<T>::type;
    __shared__ T s_a[kFreqPix];       // x_p / d_mp
    __shared__ double s_f[kFreqPix];  // frac(u / Q)
    __shared__ C s_step[kFreqPix];    // exp(-2 pi i f)
    const int m = blockIdx.x, chunk = blockIdx.y;
    const int n0 = 1 + (blockIdx.z * kFreqThreads + threadIdx.x) * kFreqRun;
    const int p0 = (int)((long long)a.P * chunk / a.chunks), p1 = (int)((long long)a.P * (chunk + 1) / a.chunks);
    const double sxm = a.sx[m], sym = a.sy[m];
    const T* x = static_cast<const T*>(a.x);
    T re[kFreqRun], im[kFreqRun];
#pragma unroll
    for (int k = 0; k < kFreqRun; ++k) re[k] = im[k] = (T)0;
    for (int pb = p0; pb < p1; pb += kFreqPix) {
        __syncthreads();
        for (int q = threadIdx.x; q < kFreqPix; q += kFreqThreads) {
            const int p = pb + q;
            T av = (T)0;
            double f = 0.0;
            if (p < p1) {
                const double d = hypot_libm(__dsub_rn(a.px[p % a.nx], sxm), __dsub_rn(a.py[p / a.nx], sym));
                const double u = __ddiv_rn(d, a.cdt);
                const double v = u / a.Q;
                f = v - floor(v);
                av = (T)((double)x[p] / d);
            }
            T s, c;
            sincospi_t<T>((T)(-2.0 * f), &s, &c);
            s_a[q] = av;
            s_f[q] = f;
            s_step[q] = C{c, s};
        }
        __syncthreads();
        if (n0 > a.qn) continue;
        const int np = min(kFreqPix, p1 - pb);
        for (int q = 0; q < np; ++q) {
            const double f = s_f[q];
            const double t0 = (double)n0 * f;
            T zs, zc;
            sincospi_t<T>((T)(-2.0 * (t0 - floor(t0))), &zs, &zc);
            const C st = s_step[q];
            const T av = s_a[q];
            T wr = av * zc, wi = av * zs;  // a_p z^n0
#pragma unroll
            for (int k = 0; k < kFreqRun; ++k) {
                re[k] += wr;
                im[k] += wi;
                const T nr = wr * st.x - wi * st.y;
                wi = wr * st.y + wi * st.x;
                wr = nr;
            }
        }
    }
    C* part = static_cast<C*>(a.part) + ((size_t)chunk * a.M + m) * a.qn;
#pragma unroll
    for (int k = 0; k < kFreqRun; ++k)
        if (n0 + k <= a.qn) part[n0 + k - 1] = C{re[k], im[k]};
}

// forward, stage 1, fp32 (r02): CTA (sensor m, pixel chunk, block of 32 R wavenumbers); lane l
// owns n = n0 .. n0 + R - 1, n0 = nb + R l, and the 4 warps split each staged batch of pixels
// (their sums are added in warp order at the end: deterministic).  Per pixel the CTA stages
// a_p = x_p / d_p and the table z_p^k, k < R (z = exp(-2 pi i f_p), phase reduced in fp64);
// per (lane, pixel) one anchor w = a_p z_p^n0, then per k a complex multiply-add
// w * table[k] into independent accumulators -- 4 FFMA and one broadcast LDS.64 per
// wavenumber, no recurrence (the fp32 path of round 1 advanced z by complex multiplication
// over runs of 16: a serial chain per thread, and half the threads idle at q_n = 1024).
// Phases enter the fast sin/cos reduced to [-1/2, 1/2) turns (|error| ~ 1e-6 absolute).
template <int R>
__global__ void __launch_bounds__(128) freq_fwd_f32_kernel(FreqArgs a) {
    constexpr int NP = kFreqPix;
    __shared__ float2 s_t[NP][R];  // z_p^k
    __shared__ float s_a[NP];      // x_p / d_mp
    __shared__ double s_f[NP];     // frac(u / Q)
    __shared__ float2 s_red[3][R][32];
    const int m = blockIdx.x, chunk = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nb = 1 + blockIdx.z * 32 * R;
    const int n0 = nb + R * lane;
    const int p0 = (int)((long long)a.P * chunk / a.chunks), p1 = (int)((long long)a.P * (chunk + 1) / a.chunks);
    const double sxm = a.sx[m], sym = a.sy[m];
    const float* x = static_cast<const float*>(a.x);
    float re[R], im[R];
#pragma unroll
    for (int k = 0; k < R; ++k) re[k] = im[k] = 0.f;
    for (int pb = p0; pb < p1; pb += NP) {
        __syncthreads();
        for (int q = threadIdx.x; q < NP; q += 128) {
            const int p = pb + q;
            float av = 0.f;
            double f = 0.0;
            if (p < p1) {
                const double d = hypot_libm(__dsub_rn(a.px[p % a.nx], sxm), __dsub_rn(a.py[p / a.nx], sym));
                const double u = __ddiv_rn(d, a.cdt);
                const double v = u / a.Q;
                f = v - floor(v);
                av = (float)((double)x[p] / d);
            }
            s_a[q] = av;
            s_f[q] = f;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < NP * R; e += 128) {  // table z_q^k
            const int q = e / R, k = e - q * R;
            const double t = (double)k * s_f[q];
            const float ph = (float)(t - rint(t));  // turns in [-1/2, 1/2]
            float sn, cs;
            __sincosf(-6.283185307179586f * ph, &sn, &cs);
            s_t[q][k] = make_float2(cs, sn);
        }
        __syncthreads();
        if (n0 <= a.qn) {
            const int np = min(NP, p1 - pb);
            for (int q = warp; q < np; q += 4) {
                const double t = (double)n0 * s_f[q];
                const float ph = (float)(t - rint(t));
                float sn, cs;
                __sincosf(-6.283185307179586f * ph, &sn, &cs);
                const float av = s_a[q];
                const float wr = av * cs, wi = av * sn;  // a_p z^n0
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const float2 z = s_t[q][k];
                    re[k] = fmaf(wr, z.x, fmaf(-wi, z.y, re[k]));
                    im[k] = fmaf(wr, z.y, fmaf(wi, z.x, im[k]));
                }
            }
        }
    }
    // the 4 warps' sums, added in warp order by warp 0
    if (warp > 0)
#pragma unroll
        for (int k = 0; k < R; ++k) s_red[warp - 1][k][lane] = make_float2(re[k], im[k]);
    __syncthreads();
    if (warp > 0) return;
    float2* part = static_cast<float2*>(a.part) + ((size_t)chunk * a.M + m) * a.qn;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        float sr = re[k], si = im[k];
#pragma unroll
        for (int w = 0; w < 3; ++w) {
            const float2 o = s_red[w][k][lane];
            sr += o.x;
            si += o.y;
        }
        if (n0 + k <= a.qn) part[n0 + k - 1] = make_float2(sr, si);
    }
}

// forward, stage 2: y[m, n] = i c k_n sum_chunks part (chunk order)
template <typename T>
__global__ void __launch_bounds__(kThreads) freq_fwd_sum_kernel(FreqArgs a) {
    using C = typename Cplx<T>::type;
    const size_t total = (size_t)a.M * a.qn;
    const C* part = static_cast<const C*>(a.part);
    C* y = static_cast<C*>(a.out);
    for (size_t i = (size_t)blockIdx.x * kThreads + threadIdx.x; i < total; i += (size_t)gridDim.x * kThreads) {
        T sr = 0, si = 0;
        for (int c = 0; c < a.chunks; ++c) {
            const C v = part[(size_t)c * total + i];
            sr += v.x;
            si += v.y;
        }
        const int n = (int)(i % a.qn) + 1;
        const T w = (T)(a.c * a.kscale * n);  // c k_n
        y[i] = C{-w * si, w * sr};            // i * w * (sr + i si)
    }
}

// adjoint: thread = pixel, CTA = (pixel block, sensor chunk); per sensor, block-Horner over n
// with exact phase anchors every kFreqAdjRun wavenumbers.  b_n = -i c k_n y[m, n] * scale is
// staged in shared memory.  Per-chunk partials [chunk][P] are added in chunk order by
// freq_adj_sum_kernel (deterministic); with one chunk the kernel writes the result directly.
template <typename T>
__global__ void __launch_bounds__(kThreads) freq_adj_kernel(FreqArgs a) {
    using C = typename Cplx<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* b = reinterpret_cast<C*>(smem_raw);  // [qn]
    const int p = blockIdx.x * kThreads + threadIdx.x;
    const bool valid = p < a.P;
    const double pxv = valid ? a.px[p % a.nx] : 0.0, pyv = valid ? a.py[p / a.nx] : 0.0;
    const int m0 = (int)((long long)a.M * blockIdx.y / gridDim.y);
    const int m1 = (int)((long long)a.M * (blockIdx.y + 1) / gridDim.y);
    const C* y = static_cast<const C*>(a.y);
    T gr = 0, gi = 0;
    for (int m = m0; m < m1; ++m) {
        __syncthreads();
        for (int n = threadIdx.x; n < a.qn; n += kThreads) {
            const C v = y[(size_t)m * a.qn + n];
            const T w = (T)(a.c * a.kscale * (n + 1) * a.scale);  // c k_n * scale
            b[n] = C{w * v.y, -w * v.x};                          // -i * w * v
        }
        __syncthreads();
        if (!valid) continue;
        const double d = hypot_libm(__dsub_rn(pxv, a.sx[m]), __dsub_rn(pyv, a.sy[m]));
        const double u = __ddiv_rn(d, a.cdt);
        const double v = u / a.Q;
        const double f = v - floor(v);
        T s1, c1;
        sincospi_t<T>((T)(2.0 * f), &s1, &c1);  // z' = conj(z) = exp(+2 pi i f)
        T sr = 0, si = 0;
        if (sizeof(T) == 4 && a.qn % 2 == 0) {
            // fp32 (r02): two independent Horner chains per run, even and odd offsets in
            // w = z'^2 (h = A(w) + z' B(w)), so consecutive FMAs do not wait on each other;
            // anchors z'^nb from the fast sin/cos of a phase reduced to [-1/2, 1/2] turns
            const T s2 = 2 * s1 * c1, c2 = c1 * c1 - s1 * s1;  // w = z'^2
            for (int nb = 1; nb <= a.qn; nb += kFreqAdjRun) {
                const int ne = min(a.qn, nb + kFreqAdjRun - 1);  // (run length even: qn even)
                T ar = 0, ai = 0, br = 0, bi = 0;
                auto step = [&](int n) {  // offsets n - nb even (A), n + 1 - nb odd (B)
                    const C be = b[n - 1], bo = b[n];
                    const T tr = ar * c2 - ai * s2 + be.x;
                    ai = ar * s2 + ai * c2 + be.y;
                    ar = tr;
                    const T ur = br * c2 - bi * s2 + bo.x;
                    bi = br * s2 + bi * c2 + bo.y;
                    br = ur;
                };
                if (ne - nb + 1 == kFreqAdjRun) {
#pragma unroll
                    for (int j = kFreqAdjRun / 2 - 1; j >= 0; --j) step(nb + 2 * j);
                } else {
                    for (int n = ne - 1; n >= nb; n -= 2) step(n);
                }
                const T hr = ar + (br * c1 - bi * s1), hi = ai + (br * s1 + bi * c1);
                const double t0 = (double)nb * f;
                const float ph = (float)(t0 - rint(t0));
                float zsf, zcf;
                __sincosf(6.283185307179586f * ph, &zsf, &zcf);  // z'^nb
                const T zs = (T)zsf, zc = (T)zcf;
                sr += hr * zc - hi * zs;
                si += hr * zs + hi * zc;
            }
        } else
        for (int nb = 1; nb <= a.qn; nb += kFreqAdjRun) {
            const int ne = min(a.qn, nb + kFreqAdjRun - 1);
            // h = sum_{n=nb..ne} b_n z'^(n - nb) by Horner from the top
            T hr = 0, hi = 0;
            for (int n = ne; n >= nb; --n) {
                const C bn = b[n - 1];
                const T tr = hr * c1 - hi * s1 + bn.x;
                hi = hr * s1 + hi * c1 + bn.y;
                hr = tr;
            }
            const double t0 = (double)nb * f;
            T zs, zc;
            sincospi_t<T>((T)(2.0 * (t0 - floor(t0))), &zs, &zc);  // z'^nb
            sr += hr * zc - hi * zs;
            si += hr * zs + hi * zc;
        }
        const T inv = (T)(1.0 / d);
        gr += sr * inv;
        gi += si * inv;
    }
    if (!valid) return;
    if (gridDim.y == 1) static_cast<C*>(a.out)[p] = C{gr, gi};
    else static_cast<C*>(a.part)[(size_t)blockIdx.y * a.P + p] = C{gr, gi};
}

template <typename T>
__global__ void __launch_bounds__(kThreads) freq_adj_sum_kernel(FreqArgs a) {
    using C = typename Cplx<T>::type;
    const C* part = static_cast<const C*>(a.part);
    for (int p = blockIdx.x * kThreads + threadIdx.x; p < a.P; p += gridDim.x * kThreads) {
        T sr = 0, si = 0;
        for (int c = 0; c < a.chunks; ++c) {
            const C v = part[(size_t)c * a.P + p];
            sr += v.x;
            si += v.y;
        }
        static_cast<C*>(a.out)[p] = C{sr, si};
    }
}

}  // namespace pk
