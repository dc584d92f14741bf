#include <cstdio>
#include <cuda_runtime.h>
#define NB 512
struct __align__(16) F4 { float x,y,z,w; };
__device__ __forceinline__ void add4_cas128(float4* p, float4 v) {
  unsigned __int128* a = reinterpret_cast<unsigned __int128*>(p);
  unsigned __int128 old = *a, assumed;
  do {
    assumed = old;
    float4 f = *reinterpret_cast<float4*>(&assumed);
    f.x += v.x; f.y += v.y; f.z += v.z; f.w += v.w;
    unsigned __int128 nv = *reinterpret_cast<unsigned __int128*>(&f);
    old = atomicCAS(a, assumed, nv);
  } while (old != assumed);
}
__device__ __forceinline__ void add2_cas64(float2* p, float2 v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(p);
  unsigned long long old = *a, assumed;
  do {
    assumed = old;
    float2 f = *reinterpret_cast<float2*>(&assumed);
    f.x += v.x; f.y += v.y;
    old = atomicCAS(a, assumed, *reinterpret_cast<unsigned long long*>(&f));
  } while (old != assumed);
}
__global__ void k_cas32(const int* __restrict__ idx, float* out, int iters){
  __shared__ float acc[NB*8];
  for(int i=threadIdx.x;i<NB*8;i+=blockDim.x) acc[i]=0;
  __syncthreads();
  int b = idx[blockIdx.x*blockDim.x+threadIdx.x] % NB;
  float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<8;k++) atomicAdd(&acc[k*NB + b], v);
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads();
  if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=acc[threadIdx.x];
}
__global__ void k_cas64(const int* __restrict__ idx, float* out, int iters){
  __shared__ float2 acc[NB*4];
  for(int i=threadIdx.x;i<NB*4;i+=blockDim.x) acc[i]=make_float2(0,0);
  __syncthreads();
  int b = idx[blockIdx.x*blockDim.x+threadIdx.x] % NB;
  float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<4;k++) add2_cas64(&acc[k*NB + b], make_float2(v,v));
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads();
  if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=acc[threadIdx.x].x;
}
__global__ void k_cas128(const int* __restrict__ idx, float* out, int iters){
  __shared__ float4 acc[NB*2];
  for(int i=threadIdx.x;i<NB*2;i+=blockDim.x) acc[i]=make_float4(0,0,0,0);
  __syncthreads();
  int b = idx[blockIdx.x*blockDim.x+threadIdx.x] % NB;
  float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<2;k++) add4_cas128(&acc[k*NB + b], make_float4(v,v,v,v));
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads();
  if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=acc[threadIdx.x].x;
}
int main(){
  const int blocks=148*4, threads=256, iters=200;
  int* idx; float* out;
  cudaMalloc(&idx, blocks*threads*4); cudaMalloc(&out, (size_t)blocks*NB*4*8);
  int* h=new int[blocks*threads]; unsigned s=1; for(int i=0;i<blocks*threads;i++){ s=s*1664525u+1013904223u; h[i]=(s>>8)%NB; }
  cudaMemcpy(idx,h,blocks*threads*4,cudaMemcpyHostToDevice);
  cudaEvent_t a,bq; cudaEventCreate(&a); cudaEventCreate(&bq);
  double nfl = (double)blocks*threads*iters*8;  // float adds
  auto run=[&](const char* name, auto kern){
    for(int w=0;w<3;w++) kern<<<blocks,threads>>>(idx,out,iters);
    cudaEventRecord(a); for(int r=0;r<5;r++) kern<<<blocks,threads>>>(idx,out,iters); cudaEventRecord(bq);
    cudaEventSynchronize(bq); float ms; cudaEventElapsedTime(&ms,a,bq); ms/=5;
    printf("%-8s %8.3f ms  %8.2f G float-adds/s  %6.3f cyc per 32 float-adds per SM\n", name, ms, nfl/ms/1e6, (ms*1e-3*1.9e9)/(nfl/32/148));
  };
  run("cas32", k_cas32); run("cas64", k_cas64); run("cas128", k_cas128);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
