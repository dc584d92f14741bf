#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define NB 512
__global__ void __cluster_dims__(2,1,1) k_self(const int* __restrict__ idx, float* out, int iters){
  __shared__ float acc[NB*8];
  for(int i=threadIdx.x;i<NB*8;i+=blockDim.x) acc[i]=0;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  float* a = cl.map_shared_rank(acc, cl.block_rank());
  int b = idx[blockIdx.x*blockDim.x+threadIdx.x] % NB;
  float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<8;k++) atomicAdd(&a[k*NB + b], v);
    b = (b*1103515245u + 12345u) % NB;
  }
  cl.sync();
  if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=acc[threadIdx.x];
}
__global__ void __cluster_dims__(2,1,1) k_other(const int* __restrict__ idx, float* out, int iters){
  __shared__ float acc[NB*8];
  for(int i=threadIdx.x;i<NB*8;i+=blockDim.x) acc[i]=0;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  float* a = cl.map_shared_rank(acc, cl.block_rank() ^ 1);
  int b = idx[blockIdx.x*blockDim.x+threadIdx.x] % NB;
  float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<8;k++) atomicAdd(&a[k*NB + b], v);
    b = (b*1103515245u + 12345u) % NB;
  }
  cl.sync();
  if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=acc[threadIdx.x];
}
__global__ void k_local(const int* __restrict__ idx, float* out, int iters){
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
int main(){
  const int blocks=148*4, threads=256, iters=200;
  int* idx; float* out;
  cudaMalloc(&idx, blocks*threads*4); cudaMalloc(&out, (size_t)blocks*NB*4*8);
  int* h=new int[blocks*threads]; unsigned s=1; for(int i=0;i<blocks*threads;i++){ s=s*1664525u+1013904223u; h[i]=(s>>8)%NB; }
  cudaMemcpy(idx,h,blocks*threads*4,cudaMemcpyHostToDevice);
  cudaEvent_t a,bq; cudaEventCreate(&a); cudaEventCreate(&bq);
  double nfl = (double)blocks*threads*iters*8;
  auto run=[&](const char* name, auto kern){
    for(int w=0;w<3;w++) kern<<<blocks,threads>>>(idx,out,iters);
    cudaEventRecord(a); for(int r=0;r<5;r++) kern<<<blocks,threads>>>(idx,out,iters); cudaEventRecord(bq);
    cudaEventSynchronize(bq); float ms; cudaEventElapsedTime(&ms,a,bq); ms/=5;
    printf("%-10s %8.3f ms  %8.2f G float-adds/s  %6.3f cyc per warp-op per SM  err=%s\n", name, ms, nfl/ms/1e6, (ms*1e-3*1.9e9)/(nfl/32/148), cudaGetErrorString(cudaGetLastError()));
  };
  run("local", k_local); run("dsm_self", k_self); run("dsm_other", k_other);
  float r; cudaMemcpy(&r, out, 4, cudaMemcpyDeviceToHost); printf("check %f\n", r);
}
