// Which broadcast paths share the shared-memory (MIO) pipe with conflict-free ATOMS on sm_100a?
// Per iteration each warp issues 8 red.shared.add.s32 (lane -> bank lane) plus B broadcast
// loads of one kind (every lane reads the same address, warp-uniform dynamic index):
//   LDS.32 / LDS.64 / LDS.128 from shared memory, LDG.128 from global (L1 hit),
//   LDC from a __constant__ array (constant cache), SHFL.
// Reported: SM clocks per iteration per warp (4 CTAs x 8 warps per SM), so 8 ATOMS alone = the
// ATOMS cost; the increment over it is what the broadcasts add.
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float4 cbank[1024];

template <int KIND, int NB, int NA>
__global__ void k(int* out, int iters, long long* cyc, const float4* g) {
    __shared__ int s[64 * 32];
    __shared__ float4 rec[256];
    for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) s[i] = 0;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) rec[i] = make_float4(i, 1, 2, 3);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned a[8];
    for (int q = 0; q < 8; q++) a[q] = (unsigned)__cvta_generic_to_shared(s + ((lane * 37 + q * 11 + warp * 5) % 64) * 32 + lane);
    float acc = lane;
    int ia = lane;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int q = 0; q < NA; q++) asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a[q & 7]), "r"(q + 1 + ia));
#pragma unroll
        for (int b = 0; b < NB; b++) {
            const int idx = (i * NB + b + warp) & 255;  // warp-uniform
            if (KIND == 0) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(rec + idx))); acc += v; }
            if (KIND == 1) { float2 v; asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"((unsigned)__cvta_generic_to_shared(rec + idx))); acc += v.x + v.y; }
            if (KIND == 2) { float4 v; asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"((unsigned)__cvta_generic_to_shared(rec + idx))); acc += v.x + v.w; }
            if (KIND == 3) { float4 v; asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(g + idx)); acc += v.x + v.w; }
            if (KIND == 4) { const float4 v = cbank[idx]; acc += v.x + v.w; }
            if (KIND == 5) { acc += __shfl_sync(0xffffffffu, acc, (idx) & 31); }
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x] + (int)acc;
}

template <int KIND, int NB, int NA>
void run(const char* name, int* o, long long* c, const float4* g, int sms) {
    const int B = sms * 4, T = 256, it = 4000;
    static long long hc[8192];
    k<KIND, NB, NA><<<B, T>>>(o, it, c, g);
    cudaDeviceSynchronize();
    cudaMemcpy(hc, c, sizeof(long long) * B, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < B; i++) mx = hc[i] > mx ? hc[i] : mx;
    // clocks per iteration of ONE warp-slot of the SM: 32 warps per SM
    printf("%-28s %7.3f SM clk per (warp iteration)  -> %.3f clk per broadcast over ATOMS\n", name,
           mx / (it * 32.0), NB ? (mx / (it * 32.0) - NA) / NB : 0.0);
}

int main() {
    int* o;
    long long* c;
    float4* g;
    cudaMalloc(&o, 64 << 20);
    cudaMalloc(&c, 1 << 20);
    cudaMalloc(&g, 1 << 20);
    cudaMemset(g, 0, 1 << 20);
    float4 hb[1024];
    for (int i = 0; i < 1024; i++) hb[i] = make_float4(i, 1, 2, 3);
    cudaMemcpyToSymbol(cbank, hb, sizeof(hb));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 0, 8>("8 ATOMS", o, c, g, sms);
    run<0, 0, 16>("16 ATOMS", o, c, g, sms);
    run<0, 2, 8>("8 ATOMS + 2 LDS.32 bc", o, c, g, sms);
    run<1, 2, 8>("8 ATOMS + 2 LDS.64 bc", o, c, g, sms);
    run<2, 2, 8>("8 ATOMS + 2 LDS.128 bc", o, c, g, sms);
    run<2, 1, 8>("8 ATOMS + 1 LDS.128 bc", o, c, g, sms);
    run<2, 1, 16>("16 ATOMS + 1 LDS.128 bc", o, c, g, sms);
    run<3, 2, 8>("8 ATOMS + 2 LDG.128 bc", o, c, g, sms);
    run<4, 2, 8>("8 ATOMS + 2 LDC.128 bc", o, c, g, sms);
    run<4, 8, 8>("8 ATOMS + 8 LDC.128 bc", o, c, g, sms);
    run<5, 2, 8>("8 ATOMS + 2 SHFL", o, c, g, sms);
    run<2, 8, 0>("8 LDS.128 bc alone", o, c, g, sms);
    run<4, 8, 0>("8 LDC.128 bc alone", o, c, g, sms);
    run<3, 8, 0>("8 LDG.128 bc alone", o, c, g, sms);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
