// Cross-stream progress check: stream A spins on a flag that a kernel on stream B sets.
// Without preloading (argc == 1) the lazy module load of B's kernels waits for the spinning
// kernel: a deadlock under CUDA_MODULE_LOADING=LAZY (the default).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(volatile int* f, long long* out) {
    long long t0 = clock64(), n = 0;
    while (*f == 0 && n < (1ll << 31)) { __nanosleep(100); ++n; }
    *out = n;
}
__global__ void busy(float* a, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = a[i] * 2.f + 1.f;
}
__global__ void setf(int* f) { atomicExch(f, 1); }
int main(int argc, char**) {
    int* f; long long* o; float* a;
    cudaMalloc(&f, 4); cudaMalloc(&o, 8); cudaMalloc(&a, 1 << 24);
    cudaMemset(f, 0, 4);
    cudaStream_t A, B;
    cudaStreamCreateWithFlags(&A, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&B, cudaStreamNonBlocking);
    if (argc > 1) {  // force the lazy loads before anything spins
        cudaFuncAttributes at;
        cudaFuncGetAttributes(&at, busy);
        cudaFuncGetAttributes(&at, setf);
        cudaFuncGetAttributes(&at, spin);
    }
    cudaDeviceSynchronize();
    spin<<<1, 32, 0, A>>>(f, o);
    busy<<<(1 << 22) / 256, 256, 0, B>>>(a, 1 << 22);
    setf<<<1, 1, 0, B>>>(f);
    cudaError_t e = cudaStreamSynchronize(A);
    long long n = 0;
    cudaMemcpy(&n, o, 8, cudaMemcpyDeviceToHost);
    printf("spin iterations %lld (%s)\n", n, cudaGetErrorString(e));
}
