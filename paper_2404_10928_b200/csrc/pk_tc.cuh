// pk_tc.cuh -- multi-frame explicit-matrix products on the 5th-generation tensor cores
// ("multi-frame K X becomes a GEMM, the only tensor-core case").
//
//   C[n][r] = sum_k A[r][k] * B[n][k]      r < R (rows), n < N (frames), k < Kd
//
// Both operands are K-major fp32 in HBM (A = the measurement matrix K for the forward product
// K X, or its transpose for K^T Y; B = the frames, frame-major), C is frame-major like every
// other frame buffer.  fp32 accuracy from tf32 tensor cores by the 3xTF32 split: a = a_hi +
// a_lo with a_hi = a with the low 13 mantissa bits cleared (exact in tf32) and a_lo = a - a_hi
// (exact in fp32, rounded to tf32 by the MMA: 2^-22 relative of a), and
// C += A_hi B_hi + A_hi B_lo + A_lo B_hi  (the dropped A_lo B_lo term is ~2^-22 relative).
//
// CTA = one 128-row tile of C (all N frames) over a K range (split-K for long K, partials
// reduced in split order -- deterministic); 6 warps:
//   warp 0     TMA producer: 2-D tiled loads (128-B swizzle) of A [128 x 32] and B [N x 32]
//              per stage into a kTcHi-deep ring (full / empty mbarriers)
//   warp 1     TMEM allocation, then one elected lane issues 3 x 4 tcgen05.mma.kind::tf32
//              per stage (M 128, N frames, K 8) into one of two [128 lanes x N] fp32 TMEM
//              accumulators (alternating every kTcChunk stages); tcgen05.commit releases the
//              stage and signals each finished chunk
//   warps 2-9  split each landed A tile in place (hi) and into a kTcLo-deep lo ring with the
//              same swizzled layout (position-wise, so the swizzle never needs decoding; the
//              small frames operand is split once, in HBM, and both its parts loaded by TMA);
//              add every finished TMEM chunk into fp32 registers (tcgen05.ld 32x32b: lane =
//              row, two warps per lane quarter, half the columns each); finally store C with
//              coalesced rows of consecutive r per frame
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "pk_common.cuh"

namespace pk {

#ifndef PK_TC_RAWHI
// 1: the MMAs read the raw fp32 A tile as its tf32 hi part (kind::tf32 ignores the low 13
// mantissa bits), so the split warps only write the lo part
#define PK_TC_RAWHI 1
#endif
constexpr int kTcBM = 128;      // rows per CTA (UMMA M)
constexpr int kTcBK = 32;       // fp32 per 128-B swizzle row (one TMA box row)
constexpr int kTcLo = 2;        // A lo-part ring depth
constexpr int kTcChunk = 4;     // K blocks (x 32) accumulated in TMEM before the CUDA-core sum
constexpr int kTcSplitWarps = 8;
constexpr int kTcThreads = 32 * (2 + kTcSplitWarps);

// stage of the TMA ring: A raw (split in place into A hi), B hi, B lo (split once, in HBM)
__host__ __device__ constexpr int tc_stage_bytes(int N) { return kTcBM * kTcBK * 4 + 2 * N * kTcBK * 4; }
// TMA ring depth: as deep as 227 KB allows
__host__ __device__ constexpr int tc_hi_depth(int N) {
    return (232448 - 2048 - kTcLo * kTcBM * kTcBK * 4) / tc_stage_bytes(N) < 8
               ? (232448 - 2048 - kTcLo * kTcBM * kTcBK * 4) / tc_stage_bytes(N) : 8;
}
__host__ __device__ constexpr int tc_smem_bytes(int N) {
    return 1024 /* alignment slack */ + tc_hi_depth(N) * tc_stage_bytes(N) + kTcLo * kTcBM * kTcBK * 4 +
           512 /* barriers */;
}

// K-major, 128-B swizzle shared-memory matrix descriptor (tile base 1024-B aligned): start
// address >> 4, leading byte offset 1 (unused for swizzled K-major), stride byte offset =
// 8 rows x 128 B = 1024 B (>> 4 = 64), descriptor version 1 (sm_100), layout SWIZZLE_128B (2)
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor, kind::tf32: D fp32, A/B tf32, both K-major, N >> 3, M >> 4
__host__ __device__ constexpr uint32_t tc_idesc(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTcBM >> 4) << 24);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

// 16 accumulator columns of this warp's 32 TMEM lanes (lane = row) into registers
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t u[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
          "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(u[j]);
}

// hi / lo split of the frames operand, once per product (B is small and read by every row tile)
__global__ void tc_split_kernel(const float* b, float* bhi, float* blo, size_t n) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
        const float v = b[q];
        const float h = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
        bhi[q] = h;
        blo[q] = v - h;
    }
}

// The tensor cores' fp32 accumulation drifts with the accumulation length (measured: relative
// error ~1.2e-8 x K, i.e. 2e-4 at K = 16384, tools/microbench/tc_gemm.cu), so the MMAs
// accumulate kTcChunk K blocks (128 products) in one of two TMEM buffers, and the epilogue
// warps add each finished chunk into fp32 registers (round to nearest) while the MMAs fill the
// other buffer: 1.7e-6 relative at every K measured.
template <int N>
__global__ void __launch_bounds__(kTcThreads, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                                                                const __grid_constant__ CUtensorMap map_bh,
                                                                const __grid_constant__ CUtensorMap map_bl,
                                                                float* c, int R, int Kd, int splits, int nf) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    constexpr int A_BYTES = kTcBM * kTcBK * 4, B_BYTES = N * kTcBK * 4;
    constexpr int STAGE = tc_stage_bytes(N), HI = tc_hi_depth(N);
    // TMA ring [HI] {A, B hi, B lo} | A lo ring [kTcLo]
    auto a_hi = [&](int s) { return smem + s * STAGE; };
    auto b_hi = [&](int s) { return smem + s * STAGE + A_BYTES; };
    auto b_lo = [&](int s) { return smem + s * STAGE + A_BYTES + B_BYTES; };
    auto a_lo = [&](int s) { return smem + HI * STAGE + s * A_BYTES; };
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + HI * STAGE + kTcLo * A_BYTES);
    // full[s]: TMA landed; split[s]: A hi/lo written (split warps); empty[s]: MMAs of the stage
    // done (also frees A lo stage % kTcLo); cdone[2]: a chunk accumulated in TMEM buffer b;
    // cfree[2]: the epilogue drained buffer b (split warps)
    const uint32_t full0 = smem_u32(bars), split0 = full0 + 8 * HI, empty0 = split0 + 8 * HI;
    const uint32_t cdone0 = empty0 + 8 * HI, cfree0 = cdone0 + 16;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * HI + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row0 = blockIdx.x * kTcBM;
    const int nkb = (Kd + kTcBK - 1) / kTcBK;
    const int kb0 = (int)((long long)nkb * blockIdx.y / splits), kb1 = (int)((long long)nkb * (blockIdx.y + 1) / splits);
    const int nk = kb1 - kb0, nch = (nk + kTcChunk - 1) / kTcChunk;
    // two chunk buffers of 2N columns: [0, N) = A_hi (B_hi) + A_lo B_hi, [N, 2N) = A_hi B_lo
    constexpr int TMEM_COLS = 4 * N;
    static_assert(TMEM_COLS == 128 || TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM allocation: power of 2");

    if (threadIdx.x == 0) {
        for (int s = 0; s < HI; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(split0 + 8 * s, kTcSplitWarps);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(cdone0 + 8 * b, 1);
            mbar_init(cfree0 + 8 * b, kTcSplitWarps);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // producer
            for (int i = 0; i < nk; ++i) {
                const int s = i % HI, kb = kb0 + i;
                if (i >= HI) mbar_wait(empty0 + 8 * s, ((i / HI) - 1) & 1);
                mbar_expect_tx(full0 + 8 * s, A_BYTES + 2 * B_BYTES);
                tma_load_2d(smem_u32(a_hi(s)), &map_a, kb * kTcBK, row0, full0 + 8 * s);
                tma_load_2d(smem_u32(b_hi(s)), &map_bh, kb * kTcBK, 0, full0 + 8 * s);
                tma_load_2d(smem_u32(b_lo(s)), &map_bl, kb * kTcBK, 0, full0 + 8 * s);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            constexpr uint32_t idesc = tc_idesc(N), idesc2 = tc_idesc(2 * N);
            for (int i = 0; i < nk; ++i) {
                const int s = i % HI, l = i % kTcLo, ch = i / kTcChunk, buf = ch & 1;
                if (i % kTcChunk == 0 && ch >= 2) mbar_wait(cfree0 + 8 * buf, ((ch / 2) - 1) & 1);
                mbar_wait(split0 + 8 * s, (i / HI) & 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(buf * 2 * N);
                const uint32_t ah = smem_u32(a_hi(s)), al = smem_u32(a_lo(l));
                const uint32_t bh = smem_u32(b_hi(s));
#pragma unroll
                for (int k = 0; k < kTcBK / 8; ++k) {  // K 8 tf32 = 32 B per MMA
                    const uint32_t o = 32u * k;
                    // A_hi against B_hi and B_lo in one MMA of N' = 2N (the two frame tiles are
                    // adjacent 128-B-swizzled row blocks of the stage): A_hi is read once
                    tc_mma(d, tc_desc(ah + o), tc_desc(bh + o), idesc2, (i % kTcChunk > 0 || k > 0) ? 1u : 0u);
                    tc_mma(d, tc_desc(al + o), tc_desc(bh + o), idesc, 1u);
                }
                tc_commit(empty0 + 8 * s);  // stage s and A lo stage l are free after these MMAs
                if (i % kTcChunk == kTcChunk - 1 || i == nk - 1) tc_commit(cdone0 + 8 * buf);
            }
        }
    } else {
        // split warps: split each landed A tile (hi in place, lo into the lo ring), and drain
        // every finished TMEM chunk into fp32 registers.  Two warps per TMEM lane quarter
        // (warp % 4 = rows 32 (warp % 4) ..), each drains half of the N columns.
        const int t = threadIdx.x - 64;                      // 0 .. 32 * kTcSplitWarps - 1
        const int sub = warp & 3, half = (warp - 2) >> 2;    // rows, column half
        constexpr int NH = N / 2;
        float acc[NH];
#pragma unroll
        for (int j = 0; j < NH; ++j) acc[j] = 0.f;
        auto drain = [&](int ch) {
            const int buf = ch & 1;
            mbar_wait(cdone0 + 8 * buf, (ch / 2) & 1);
            tc_fence_after();
#pragma unroll
            for (int n0 = 0; n0 < NH; n0 += 16) {
                float v[16], w[16];
                const uint32_t col = tmem + ((uint32_t)(32 * sub) << 16) + (uint32_t)(buf * 2 * N + half * NH + n0);
                tc_ld16(col, v);          // A_hi B_hi + A_lo B_hi
                tc_ld16(col + N, w);      // A_hi B_lo
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[n0 + j] += v[j] + w[j];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(cfree0 + 8 * buf);
        };
        for (int i = 0; i < nk; ++i) {
            const int s = i % HI, l = i % kTcLo;
            // A lo stage l was last read by the MMAs of stage i - kTcLo
            if (i >= kTcLo) mbar_wait(empty0 + 8 * ((i - kTcLo) % HI), ((i - kTcLo) / HI) & 1);
            mbar_wait(full0 + 8 * s, (i / HI) & 1);
            unsigned char* hi = a_hi(s);
            unsigned char* lo = a_lo(l);
#pragma unroll
            for (int o = 16 * t; o < A_BYTES; o += 16 * 32 * kTcSplitWarps) {
                const uint4 v = *reinterpret_cast<const uint4*>(hi + o);
                const uint4 h = make_uint4(v.x & 0xffffe000u, v.y & 0xffffe000u, v.z & 0xffffe000u, v.w & 0xffffe000u);
                float4 q;
                q.x = __uint_as_float(v.x) - __uint_as_float(h.x);
                q.y = __uint_as_float(v.y) - __uint_as_float(h.y);
                q.z = __uint_as_float(v.z) - __uint_as_float(h.z);
                q.w = __uint_as_float(v.w) - __uint_as_float(h.w);
#if !PK_TC_RAWHI
                *reinterpret_cast<uint4*>(hi + o) = h;
#endif
                *reinterpret_cast<float4*>(lo + o) = q;
            }
            fence_proxy_async_smem();  // generic writes -> the tensor cores' (async proxy) reads
            __syncwarp();
            if (lane == 0) mbar_arrive(split0 + 8 * s);
            // the chunk before the one this stage belongs to is complete once this chunk's
            // stages are split (its MMAs precede them): drain it
            if (i % kTcChunk == kTcChunk - 1 && i / kTcChunk >= 1) drain(i / kTcChunk - 1);
        }
        // the chunks not drained in the loop: the loop drained chunk c - 1 at the last stage of
        // every full chunk c >= 1, i.e. max(0, full chunks - 1) of them
        for (int ch = max(0, nk / kTcChunk - 1); ch < nch; ++ch) drain(ch);
        const int r = row0 + 32 * sub + lane;
        float* cout = c + (size_t)blockIdx.y * N * R;
        if (r < R)  // frames >= nf (zero rows of the padded operand) are not stored
#pragma unroll
            for (int j = 0; j < NH; ++j)
                if (half * NH + j < nf) cout[(size_t)(half * NH + j) * R + r] = acc[j];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
    }
}

// partials [splits][stride] summed in split order (deterministic) into C [0, n)
__global__ void tc_split_sum_kernel(const float* part, float* c, size_t n, int splits, size_t stride) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
        float s = part[q];
        for (int k = 1; k < splits; ++k) s += part[(size_t)k * stride + q];
        c[q] = s;
    }
}

// out [cols][rows] = in [rows][cols] (fp32), 32 x 32 tiles through shared memory
__global__ void dense_transpose_kernel(const float* in, float* out, int64_t rows, int64_t cols) {
    __shared__ float t[32][33];
    const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t r = r0 + k, c = c0 + threadIdx.x;
        if (r < rows && c < cols) t[k][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t c = c0 + k, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * rows + r] = t[threadIdx.x][k];
    }
}

}  // namespace pk
