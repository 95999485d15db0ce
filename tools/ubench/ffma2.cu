// Microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) issue/throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){ u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
template<int K>
__global__ void scalar_k(float* out, float s, int iters){
  float a[K]; for(int k=0;k<K;++k) a[k]=threadIdx.x*0.001f+k;
  for(int i=0;i<iters;++i){
#pragma unroll
    for(int k=0;k<K;++k) a[k]=fmaf(a[k], s, 0.5f);
  }
  float t=0; for(int k=0;k<K;++k) t+=a[k]; out[blockIdx.x*blockDim.x+threadIdx.x]=t;
}
template<int K>
__global__ void pair_k(float* out, float s, int iters){
  u64 a[K/2]; for(int k=0;k<K/2;++k){ float x=threadIdx.x*0.001f+2*k, y=x+1; asm("mov.b64 %0, {%1,%2};" : "=l"(a[k]) : "f"(x), "f"(y)); }
  u64 ss, hh; asm("mov.b64 %0, {%1,%2};" : "=l"(ss) : "f"(s), "f"(s)); float h=0.5f; asm("mov.b64 %0, {%1,%2};" : "=l"(hh) : "f"(h), "f"(h));
  for(int i=0;i<iters;++i){
#pragma unroll
    for(int k=0;k<K/2;++k) a[k]=fma2(a[k], ss, hh);
  }
  float t=0; for(int k=0;k<K/2;++k){ float x,y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[k])); t+=x+y; } out[blockIdx.x*blockDim.x+threadIdx.x]=t;
}
int main(){
  float* out; cudaMalloc(&out, 148*8*256*4*sizeof(float));
  int iters=20000; dim3 g(148*8), b(256);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for(int rep=0;rep<2;++rep){
  cudaEventRecord(e0); scalar_k<16><<<g,b>>>(out,0.999f,iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  double fl=2.0*148*8*256*16.0*iters; printf("FFMA : %.2f ms  %.1f TFLOP/s\n", ms, fl/ms/1e9);
  cudaEventRecord(e0); pair_k<16><<<g,b>>>(out,0.999f,iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("FFMA2: %.2f ms  %.1f TFLOP/s\n", ms, fl/ms/1e9);
  }
  return 0;
}
