// ATOMS (red.shared.add.s32) throughput vs address pattern, addresses precomputed.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out, int iters, int mode, long long* cyc){
  __shared__ int s[4096];
  for(int i=threadIdx.x;i<4096;i+=blockDim.x) s[i]=0;
  __syncthreads();
  int lane=threadIdx.x&31;
  unsigned a[8];
  for(int q=0;q<8;q++){
    int word;
    if(mode==0) word=lane;                                   // one row
    else if(mode<=5){ int R=1<<mode; word=((lane%R)*9+q)%64*32+lane; }  // R rows, bank=lane
    else if(mode<=8){ // lane = pixel of an 8x4 footprint, 1-D window, 1.93 slots/px
      float th=(mode-6)*0.4f+q*0.1f; int lx=lane&7, ly=lane>>3;
      word=64+(int)(1.93f*(lx*cosf(th)+ly*sinf(th))+0.37f*q); }
    else if(mode==9){ word=64+((lane*7+q)&15); }            // 16 words, 2 lanes each
    else if(mode==10){ word=64+lane/4; }                     // 8 words, 4 lanes each
    else { word=(lane*37+q*11)%64*32+lane; }                 // 32 distinct rows
    a[q]=(unsigned)__cvta_generic_to_shared(s+(word&4095));
  }
  long long t0=clock64();
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int q=0;q<8;q++) asm volatile("red.shared.add.s32 [%0], %1;"::"r"(a[q]),"r"(q+1));
  }
  long long t1=clock64();
  __syncthreads();
  if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s[threadIdx.x];
}
int main(){
  int *o; long long* c; cudaMalloc(&o,64<<20); cudaMalloc(&c,1<<20);
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  int B=sms*4,T=256,it=2000; long long hc[4096];
  const char* nm[]={"1 row","2 rows","4 rows","8 rows","16 rows","32 rows","8x4 px th0","8x4 px th.4","8x4 px th.8","16 words x2","8 words x4","32 rows b"};
  for(int m=0;m<12;m++){
    k<<<B,T>>>(o,it,m,c); cudaDeviceSynchronize();
    cudaMemcpy(hc,c,sizeof(long long)*B,cudaMemcpyDeviceToHost);
    double mx=0; for(int i=0;i<B;i++) mx=hc[i]>mx?hc[i]:mx;
    printf("%-14s %6.2f lanes/clk/SM  (%.2f clk per warp RED)\n",nm[m], it*8.0*T*4/mx, mx/(it*8.0*T*4/32));
  }
}
