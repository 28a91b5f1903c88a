// Standalone check + timing of pk_tc.cuh's 3xTF32 tcgen05 GEMM against an fp64 reference:
//   C[n][r] = sum_k A[r][k] B[n][k]
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2404_10928_b200/csrc tc_gemm.cu -o tc_gemm
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda.h>
#include "pk_tc.cuh"

using namespace pk;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return (EncodeFn)fn;
}

static CUtensorMap make_map(const float* base, int rows, int cols, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
}

__global__ void ref_kernel(const float* A, const float* B, double* C, int R, int K, int N) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x, n = blockIdx.y;
    if (r >= R) return;
    double s = 0.0;
    for (int k = 0; k < K; ++k) s += (double)A[(size_t)r * K + k] * (double)B[(size_t)n * K + k];
    C[(size_t)n * R + r] = s;
}

template <int N>
void run(int R, int K, int splits) {
    std::vector<float> hA((size_t)R * K), hB((size_t)N * K);
    srand(1);
    for (auto& v : hA) v = (float)rand() / RAND_MAX - 0.3f;
    for (auto& v : hB) v = (float)rand() / RAND_MAX;
    float *A, *B, *C, *P, *Bh, *Bl;
    double* Cr;
    cudaMalloc(&A, hA.size() * 4); cudaMalloc(&B, hB.size() * 4);
    cudaMalloc(&Bh, hB.size() * 4); cudaMalloc(&Bl, hB.size() * 4);
    cudaMalloc(&C, (size_t)N * R * 4); cudaMalloc(&P, (size_t)splits * N * R * 4);
    cudaMalloc(&Cr, (size_t)N * R * 8);
    cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap ma = make_map(A, R, K, kTcBM), mbh = make_map(Bh, N, K, N), mbl = make_map(Bl, N, K, N);
    const int smem = tc_smem_bytes(N);
    cudaFuncSetAttribute(tc_gemm_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid((R + kTcBM - 1) / kTcBM, splits);
    auto launch = [&]() {
        tc_split_kernel<<<296, 256>>>(B, Bh, Bl, (size_t)N * K);
        tc_gemm_kernel<N><<<grid, kTcThreads, smem>>>(ma, mbh, mbl, splits > 1 ? P : C, R, K, splits, N);
        if (splits > 1) tc_split_sum_kernel<<<1184, 256>>>(P, C, (size_t)N * R, splits, (size_t)N * R);
    };
    launch();
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    printf("N %d R %d K %d splits %d: %s\n", N, R, K, splits, cudaGetErrorString(e));
    if (e != cudaSuccess) exit(1);
    ref_kernel<<<dim3((R + 127) / 128, N), 128>>>(A, B, Cr, R, K, N);
    cudaDeviceSynchronize();
    std::vector<float> hC((size_t)N * R);
    std::vector<double> hR((size_t)N * R);
    cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hR.data(), Cr, hR.size() * 8, cudaMemcpyDeviceToHost);
    double num = 0, den = 0, mx = 0;
    for (size_t i = 0; i < hC.size(); ++i) {
        const double d = hC[i] - hR[i];
        num += d * d; den += hR[i] * hR[i];
        mx = fmax(mx, fabs(d) / fmax(fabs(hR[i]), 1e-30));
    }
    printf("  rel L2 %.3e  max rel %.3e   C[0]=%f ref %f\n", sqrt(num / den), mx, hC[0], hR[0]);
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0); cudaEventCreate(&t1);
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(t0);
    const int reps = 10;
    for (int w = 0; w < reps; ++w) launch();
    cudaEventRecord(t1);
    cudaEventSynchronize(t1);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    ms /= reps;
    const double bytes = (double)R * K * 4 + (double)N * K * 4 * grid.x;
    printf("  %.3f ms  %.1f TFLOP/s (3xTF32 work = 2 R N K)  A stream %.0f GB/s\n", ms,
           2.0 * R * N * K / (ms * 1e-3) / 1e12, (double)R * K * 4 / (ms * 1e-3) / 1e9);
    (void)bytes;
    cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(P); cudaFree(Cr);
}

int main() {
    run<32>(1024, 1024, 1);
    run<64>(4096, 4096, 1);
    run<64>(4096, 16384, 4);
    run<128>(16384, 16384, 1);
    run<64>(131072, 16384, 1);   // config 1 forward: K (131072 x 16384) x 64 frames
    run<64>(16384, 131072, 8);   // config 1 adjoint: K^T (16384 x 131072) x 64 frames
    return 0;
}
