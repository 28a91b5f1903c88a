// Pipe-throughput microbenchmarks for the B200 design decisions in DESIGN.md:
// FFMA peak, MUFU.SQRT, ATOMS.ADD (32-bit int, smem), LDS.64 footprints, DFMA.
// Prints ops per SM-cycle (from clock64) and absolute rates (from cudaEvent).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void ffma_k(float* out, int iters, long long* cyc){
  float a0=threadIdx.x,a1=a0+1,a2=a0+2,a3=a0+3,a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  const float b=1.0001f, c=0.9999f;
  long long t0=clock64();
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int k=0;k<16;k++){ a0=fmaf(a0,b,c);a1=fmaf(a1,b,c);a2=fmaf(a2,b,c);a3=fmaf(a3,b,c);
      a4=fmaf(a4,b,c);a5=fmaf(a5,b,c);a6=fmaf(a6,b,c);a7=fmaf(a7,b,c);} }
  long long t1=clock64();
  if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3+a4+a5+a6+a7;
}
__global__ void dfma_k(double* out, int iters, long long* cyc){
  double a0=threadIdx.x,a1=a0+1,a2=a0+2,a3=a0+3,a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  const double b=1.0001, c=0.9999;
  long long t0=clock64();
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int k=0;k<4;k++){ a0=fma(a0,b,c);a1=fma(a1,b,c);a2=fma(a2,b,c);a3=fma(a3,b,c);
      a4=fma(a4,b,c);a5=fma(a5,b,c);a6=fma(a6,b,c);a7=fma(a7,b,c);} }
  long long t1=clock64();
  if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3+a4+a5+a6+a7;
}
__global__ void sqrt_k(float* out, int iters, long long* cyc){
  float a0=threadIdx.x+1.f,a1=a0+1,a2=a0+2,a3=a0+3,a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  long long t0=clock64();
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int k=0;k<4;k++){
#define SQ(a) asm volatile("sqrt.approx.f32 %0,%0;":"+f"(a));
      SQ(a0)SQ(a1)SQ(a2)SQ(a3)SQ(a4)SQ(a5)SQ(a6)SQ(a7)} }
  long long t1=clock64();
  if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3+a4+a5+a6+a7;
}
// mode 0: lane -> word lane (conflict-free, distinct); 1: lane/2 (2 lanes/address);
// 2: lane/4; 3: pseudo-random in a 32-word window; 4: lane*2 (2-way bank conflict)
__device__ __forceinline__ int amap(int mode, int lane, int i){
  switch(mode){case 0: return lane; case 1: return lane>>1; case 2: return lane>>2;
  case 3: return (lane*7+i*13)&31; default: return (lane*2)&63;}
}
__global__ void atoms_k(int* out, int iters, int mode, long long* cyc){
  __shared__ int s[64*32];
  if(mode>=5){ // lane l -> bank l, pseudo-random row (the projector's window pattern)
    for(int i=threadIdx.x;i<64*32;i+=blockDim.x) s[i]=0;
    __syncthreads();
    int lane=threadIdx.x&31; unsigned h=lane*2654435761u+threadIdx.x;
    long long t0=clock64();
    for(int i=0;i<iters;i++){
#pragma unroll
      for(int k=0;k<8;k++){ h=h*1664525u+1013904223u; int row=(h>>20)&63;
        int w;
        if(mode<=6) w=row*32+lane;
        else if(mode<=10) { int R=1<<(mode-6); w=((row+(lane&(R-1)))&63)*32+lane; }      // R distinct rows
        else if(mode==11) { // 1-D window, 8x4 pixel footprint, 1.93 slots/px, direction from h
          float th=(h>>8)*(6.2831853f/16777216.f); int lx=lane&7, ly=lane>>3;
          w=(int)(1.93f*(lx*__cosf(th)+ly*__sinf(th))+40.f+row); }
        else { // 1-D window, 32 lanes over 16 consecutive words (2 lanes per word, random order)
          w=row+((lane*7+k)&15); }
        asm volatile("red.shared.add.s32 [%0], %1;"::"r"((unsigned)__cvta_generic_to_shared(s+(w&2047))),"r"(k+1)); } }
    long long t1=clock64();
    __syncthreads();
    if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
    out[blockIdx.x*blockDim.x+threadIdx.x]=s[threadIdx.x];
    return;
  }
  for(int i=threadIdx.x;i<64*32;i+=blockDim.x) s[i]=0;
  __syncthreads();
  int lane=threadIdx.x&31, w=threadIdx.x>>5;
  int* base=s+(w&31)*64;
  long long t0=clock64();
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int k=0;k<8;k++){ atomicAdd(base+amap(mode,lane,k), k+1); }
  }
  long long t1=clock64();
  __syncthreads();
  if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s[threadIdx.x];
}
// LDS.64: mode 0: lane -> float2 slot lane (256B); 1: slot lane/2 (128B); 2: slot lane*5/8 (~20 slots); 3: slot (lane*7)&31 perm
// 4: slot lane&15 (both half-warps read the same 16 slots); 5: 8x4 pixel footprint at 1.93 slots/px, theta=30deg
// 6: 8x4 footprint at 1.93 slots/px along x (theta=0); 7: random within 16 slots
__global__ void lds64_k(float* out, int iters, int mode, long long* cyc){
  __shared__ float2 s[4096];
  for(int i=threadIdx.x;i<4096;i+=blockDim.x) s[i]=make_float2(i,i+1);
  __syncthreads();
  int lane=threadIdx.x&31;
  int lx=lane&7, ly=lane>>3;
  int off = mode==0? lane : mode==1? lane>>1 : mode==2? (lane*5)>>3 : mode==3? (lane*7)&31 :
            mode==4? (lane&15) : mode==5? (int)(1.93f*(lx*0.866f+ly*0.5f)) : mode==6? (int)(1.93f*lx) :
            (int)((lane*2654435761u)>>28);
  float acc=0.f, acc2=0.f;
  int o=(threadIdx.x>>5)*37;
  long long t0=clock64();
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int k=0;k<8;k++){ float2 v=s[(o+off+k*41)&4095]; acc+=v.x; acc2+=v.y; }
    o=(o+3)&1023;
  }
  long long t1=clock64();
  if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc+acc2;
}

// global reductions, coalesced: each warp adds to 32 consecutive words of a
// per-warp stripe (mode 0: s32, 1: u64, 2: plain s32 store for comparison)
__global__ void red_k(void* buf, int iters, int mode, size_t words, long long* cyc){
  int lane=threadIdx.x&31; size_t w=(blockIdx.x*(blockDim.x>>5)+(threadIdx.x>>5));
  long long t0=clock64();
  for(int i=0;i<iters;i++){
    size_t idx=((w*iters+i)*32+lane)%words;
    if(mode==0) atomicAdd((int*)buf+idx, 1);
    else if(mode==1) atomicAdd((unsigned long long*)buf+idx, 1ull);
    else ((int*)buf)[idx]=i;
  }
  long long t1=clock64();
  if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  int sms=p.multiProcessorCount; printf("device %s sms %d\n",p.name,sms);
  float* fo; double* dout; int* io; long long* cyc;
  CK(cudaMalloc(&fo, 64<<20)); CK(cudaMalloc(&dout,64<<20)); CK(cudaMalloc(&io,64<<20)); CK(cudaMalloc(&cyc, 1<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  long long hc[4096];
  auto report=[&](const char* name, int blocks, int threads, double ops_per_thread, float ms){
    cudaMemcpy(hc,cyc,sizeof(long long)*blocks,cudaMemcpyDeviceToHost);
    double mx=0; for(int i=0;i<blocks;i++) mx = hc[i]>mx?hc[i]:mx;
    double total=ops_per_thread*threads*blocks;
    int bps = blocks/sms;
    double per_sm_cyc = ops_per_thread*threads*bps/mx;
    printf("%-28s lane-ops/SM/clk(in-kernel) %7.2f   abs %.3e lane-ops/s  (%.3f ms, clk~%.0f MHz)\n",
      name, per_sm_cyc, total/(ms*1e-3), ms, mx/(ms*1e3));
  };
  int B=sms*4, T=256; float ms;
  for(int rep=0;rep<2;rep++){
  int it=4000;
  cudaEventRecord(e0); ffma_k<<<B,T>>>(fo,it,cyc); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1); report("FFMA (x2 flops)",B,T,it*128.0,ms);
  cudaEventRecord(e0); dfma_k<<<B,T>>>(dout,it/4,cyc); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1); report("DFMA",B,T,it/4*32.0,ms);
  cudaEventRecord(e0); sqrt_k<<<B,T>>>(fo,it/4,cyc); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1); report("MUFU.SQRT",B,T,it/4*32.0,ms);
  for(int m=0;m<13;m++){ char nm[64]; snprintf(nm,64,"ATOMS.ADD mode %d",m);
    cudaEventRecord(e0); atoms_k<<<B,T>>>(io,it/4,m,cyc); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); report(nm,B,T,it/4*8.0,ms);}
  for(int m=0;m<8;m++){ char nm[64]; snprintf(nm,64,"LDS.64 mode %d",m);
    cudaEventRecord(e0); lds64_k<<<B,T>>>(fo,it/2,m,cyc); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); report(nm,B,T,it/2*8.0,ms);}
  }
  void* big; CK(cudaMalloc(&big, (size_t)64<<20));
  for(int m=0;m<3;m++){ char nm[64]; snprintf(nm,64,"global RED mode %d (0 s32,1 u64,2 st)",m);
    size_t words=(size_t)(16<<20)/(m==1?8:4)*2; // 32 MB footprint, L2 resident
    cudaEventRecord(e0); red_k<<<B,T>>>(big,256,m,words,cyc); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); report(nm,B,T,256.0,ms);}
  return 0;
}
