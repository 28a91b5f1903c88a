// Do SHFL / LDS broadcasts compete with conflict-free ATOMS for the shared-memory pipe?
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(int* out, int iters, long long* cyc){
  __shared__ int s[4096];
  __shared__ float4 rec[64];
  for(int i=threadIdx.x;i<4096;i+=blockDim.x) s[i]=0;
  if(threadIdx.x<64) rec[threadIdx.x]=make_float4(threadIdx.x,1,2,3);
  __syncthreads();
  int lane=threadIdx.x&31;
  unsigned a[8];
  for(int q=0;q<8;q++) a[q]=(unsigned)__cvta_generic_to_shared(s+((lane*37+q*11)%64)*32+lane);
  float acc=lane; int ia=lane;
  long long t0=clock64();
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int q=0;q<8;q++){
      if(MODE==0||MODE==2||MODE==3||MODE==5) asm volatile("red.shared.add.s32 [%0], %1;"::"r"(a[q]),"r"(q+1));
      if(MODE==1||MODE==2) { acc += __shfl_sync(0xffffffffu, acc, (q+i)&31); }
      if(MODE==3||MODE==4) { float4 r=rec[(q+i)&63]; acc+=r.x+r.w; }
      if(MODE==5) { ia += __shfl_sync(0xffffffffu, ia, (q+i)&31); }
    }
  }
  long long t1=clock64();
  __syncthreads();
  if(threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s[threadIdx.x]+(int)acc+ia;
}
int main(){
  int *o; long long* c; cudaMalloc(&o,64<<20); cudaMalloc(&c,1<<20);
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  int B=sms*4,T=256,it=2000; long long hc[4096];
  const char* nm[]={"RED only","SHFL only","RED+SHFL","RED+LDS128bc","LDS128bc only","RED+SHFL(int)"};
  void (*ks[])(int*,int,long long*)={k<0>,k<1>,k<2>,k<3>,k<4>,k<5>};
  for(int m=0;m<6;m++){
    ks[m]<<<B,T>>>(o,it,c); cudaDeviceSynchronize();
    cudaMemcpy(hc,c,sizeof(long long)*B,cudaMemcpyDeviceToHost);
    double mx=0; for(int i=0;i<B;i++) mx=hc[i]>mx?hc[i]:mx;
    printf("%-16s %.3f clk per 8-op group per warp-slot (SM: %.2f warp-groups/clk)\n",nm[m], mx/(it*(double)T*4/32), it*(double)T*4/32/mx);
  }
}
