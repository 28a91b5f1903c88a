// Shared-memory reduction throughput: red.shared.add.s32 vs red.shared.add.u64 (two int32
// accumulators packed in one 64-bit word), bank-clean addresses [row][lane], with and without a
// broadcast LDS.128 per 8 (resp. 4) reductions -- the projector's per-record MIO mix.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out, int iters, int mode, long long* cyc) {
    __shared__ __align__(16) unsigned long long s[64 * 32];
    for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) s[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned a32[8], a64[4];
    for (int q = 0; q < 8; q++) {
        const int row = ((lane % 16) * 9 + q) % 64;
        a32[q] = (unsigned)__cvta_generic_to_shared(reinterpret_cast<int*>(s) + (row * 32 + lane));
        if (q < 4) a64[q] = (unsigned)__cvta_generic_to_shared(s + (row * 32 + lane));
    }
    const unsigned rec = (unsigned)__cvta_generic_to_shared(s + 2000);
    float acc = 0.f;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (mode == 0) {
#pragma unroll
            for (int q = 0; q < 8; q++) asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a32[q]), "r"(q + 1));
        } else if (mode == 1) {
#pragma unroll
            for (int q = 0; q < 4; q++)
                asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(a64[q]), "l"((unsigned long long)(q + 1)));
        } else if (mode == 2) {
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(rec + 16 * (i & 7)));
            acc += v.x + v.w;
#pragma unroll
            for (int q = 0; q < 8; q++) asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a32[q]), "r"(q + 1));
        } else {
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(rec + 16 * (i & 7)));
            acc += v.x + v.w;
#pragma unroll
            for (int q = 0; q < 4; q++)
                asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(a64[q]), "l"((unsigned long long)(q + 1)));
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = (int)s[threadIdx.x] + (acc == 1.2345f);
}
int main() {
    int* o;
    long long* c;
    cudaMalloc(&o, 64 << 20);
    cudaMalloc(&c, 1 << 20);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int B = sms * 4, T = 256, it = 4000;
    static long long hc[8192];
    const char* nm[] = {"8 x red.s32", "4 x red.u64", "LDS.128 + 8 red.s32", "LDS.128 + 4 red.u64"};
    for (int m = 0; m < 4; m++) {
        k<<<B, T>>>(o, it, m, c);
        cudaDeviceSynchronize();
        cudaMemcpy(hc, c, sizeof(long long) * B, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < B; i++) mx = hc[i] > mx ? hc[i] : mx;
        // per SM: 4 CTAs x 8 warps x it records
        printf("%-22s %7.3f clk per warp-record per SM (8 int32 accumulations each)\n", nm[m], mx / (it * 4.0 * T / 32));
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
