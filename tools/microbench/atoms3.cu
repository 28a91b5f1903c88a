// Shared-memory reduction cost per warp instruction on sm_100a, by pattern:
//   rows   : lanes hit 32 different 128-B rows (bank = lane, the projector's pattern) or one row
//   active : lanes participating (predicated off lanes)
//   op     : red.shared.add.s32 / red.shared.add.f32 / plain ld+st read-modify-write
// 4 CTAs x 256 threads per SM, 8 independent reductions per iteration.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int ROWS, int ACTIVE>
__global__ void k(int* out, int iters, long long* cyc) {
    __shared__ int s[64 * 32];
    for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) s[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned a[8];
    for (int q = 0; q < 8; q++) {
        const int row = ROWS == 1 ? (q * 7 + warp) % 64 : ((lane * 37 + q * 11 + warp * 5) % 64);
        a[q] = (unsigned)__cvta_generic_to_shared(s + row * 32 + lane);
    }
    const bool on = lane < ACTIVE;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (on) {
#pragma unroll
            for (int q = 0; q < 8; q++) {
                if (OP == 0) asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a[q]), "r"(q + 1));
                else if (OP == 1) asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(a[q]), "f"(1.0f));
                else {
                    int v;
                    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a[q]));
                    asm volatile("st.shared.s32 [%0], %1;" ::"r"(a[q]), "r"(v + q));
                }
            }
        }
        __syncwarp();
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x];
}

template <int OP, int ROWS, int ACTIVE>
void run(const char* name, int* o, long long* c, int sms) {
    const int B = sms * 4, T = 256, it = 4000;
    static long long hc[8192];
    k<OP, ROWS, ACTIVE><<<B, T>>>(o, it, c);
    cudaDeviceSynchronize();
    cudaMemcpy(hc, c, sizeof(long long) * B, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < B; i++) mx = hc[i] > mx ? hc[i] : mx;
    // per SM: 4 CTAs x 8 warps x it x 8 instructions
    printf("%-34s %6.3f clk per warp instruction per SM\n", name, mx / (it * 8.0 * 4 * T / 32));
}

int main() {
    int* o;
    long long* c;
    cudaMalloc(&o, 64 << 20);
    cudaMalloc(&c, 1 << 20);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 32, 32>("red.s32  32 rows  32 lanes", o, c, sms);
    run<0, 1, 32>("red.s32   1 row   32 lanes", o, c, sms);
    run<0, 32, 16>("red.s32  32 rows  16 lanes", o, c, sms);
    run<0, 32, 8>("red.s32  32 rows   8 lanes", o, c, sms);
    run<0, 32, 1>("red.s32  32 rows   1 lane", o, c, sms);
    run<1, 32, 32>("red.f32  32 rows  32 lanes", o, c, sms);
    run<2, 32, 32>("ld+st    32 rows  32 lanes", o, c, sms);
    run<2, 32, 16>("ld+st    32 rows  16 lanes", o, c, sms);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
