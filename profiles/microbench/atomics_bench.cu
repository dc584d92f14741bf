// Microbenchmark: shared-memory scatter options on sm_100a (scratch; not product).
#include <cstdio>
#include <cuda_runtime.h>
#define NB 512
__global__ void k_cas(const int* __restrict__ idx, float* out, int iters){
  __shared__ float acc[NB*7];
  for(int i=threadIdx.x;i<NB*7;i+=blockDim.x) acc[i]=0;
  __syncthreads();
  int base = (blockIdx.x*blockDim.x+threadIdx.x);
  int b = idx[base] % NB;
  float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<6;k++) atomicAdd(&acc[b*7+k], v);
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads();
  if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=acc[threadIdx.x*7];
}
__global__ void k_int(const int* __restrict__ idx, float* out, int iters){
  __shared__ int acc[NB*7];
  for(int i=threadIdx.x;i<NB*7;i+=blockDim.x) acc[i]=0;
  __syncthreads();
  int base = (blockIdx.x*blockDim.x+threadIdx.x);
  int b = idx[base] % NB;
  int v = 1 + threadIdx.x;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<6;k++) atomicAdd(&acc[b*7+k], v);
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads();
  if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=acc[threadIdx.x*7];
}
__global__ void k_i64(const int* __restrict__ idx, float* out, int iters){
  __shared__ unsigned long long acc[NB*7];
  for(int i=threadIdx.x;i<NB*7;i+=blockDim.x) acc[i]=0;
  __syncthreads();
  int base = (blockIdx.x*blockDim.x+threadIdx.x);
  int b = idx[base] % NB;
  unsigned long long v = 1 + threadIdx.x;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<6;k++) atomicAdd(&acc[b*7+k], v);
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads();
  if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=(float)acc[threadIdx.x*7];
}
__global__ void k_lds(const int* __restrict__ idx, float* out, int iters){
  __shared__ float4 rec[NB*4];
  for(int i=threadIdx.x;i<NB*4;i+=blockDim.x) rec[i]=make_float4(i,1,2,3);
  __syncthreads();
  int base = (blockIdx.x*blockDim.x+threadIdx.x);
  int b = idx[base] % NB;
  float s=0;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<6;k++){ float4 r = rec[k*NB/2 + b]; s += r.x*r.y+r.z*r.w; }
    b = (b*1103515245u + 12345u + (int)s) % NB;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_redg(const int* __restrict__ idx, float* acc_g, int iters){
  float* acc = acc_g + (size_t)blockIdx.x*NB*7;
  int base = (blockIdx.x*blockDim.x+threadIdx.x);
  int b = idx[base] % NB;
  float v = 1.0f;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<6;k++) atomicAdd(&acc[b*7+k], v);
    b = (b*1103515245u + 12345u) % NB;
  }
}
int main(){
  const int blocks=148*4, threads=256, iters=200;
  int* idx; float* out; float* accg;
  cudaMalloc(&idx, blocks*threads*4); cudaMalloc(&out, (size_t)blocks*NB*7*4*2);
  cudaMalloc(&accg, (size_t)blocks*NB*7*4);
  int* h=new int[blocks*threads]; unsigned s=1; for(int i=0;i<blocks*threads;i++){ s=s*1664525u+1013904223u; h[i]=(s>>8)%NB; }
  cudaMemcpy(idx,h,blocks*threads*4,cudaMemcpyHostToDevice);
  cudaEvent_t a,bq; cudaEventCreate(&a); cudaEventCreate(&bq);
  double nops = (double)blocks*threads*iters*6;
  auto run=[&](const char* name, auto kern, float* o){
    for(int w=0;w<3;w++) kern<<<blocks,threads>>>(idx,o,iters);
    cudaEventRecord(a); for(int r=0;r<5;r++) kern<<<blocks,threads>>>(idx,o,iters); cudaEventRecord(bq);
    cudaEventSynchronize(bq); float ms; cudaEventElapsedTime(&ms,a,bq); ms/=5;
    printf("%-6s %8.3f ms  %8.2f Gops/s  %6.3f cyc/warp-op/SM @1.9GHz\n", name, ms, nops/ms/1e6, (ms*1e-3*1.9e9)/(nops/32/148));
  };
  run("cas", k_cas, out); run("int", k_int, out); run("i64", k_i64, out); run("lds128", k_lds, out); run("redg", k_redg, accg);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
