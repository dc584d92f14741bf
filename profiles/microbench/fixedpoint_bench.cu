// 6-value scatter into per-CTA shared accumulators: float CAS128+CAS64 vs int64 atomics vs hi/lo int32.
#include <cstdio>
#include <cuda_runtime.h>
#define NB 512
__global__ void k_cas(const int* __restrict__ idx, float* out, int iters){
  __shared__ float4 a0[NB]; __shared__ float2 a1[NB];
  for(int i=threadIdx.x;i<NB;i+=blockDim.x){ a0[i]=make_float4(0,0,0,0); a1[i]=make_float2(0,0);} __syncthreads();
  int b = idx[blockIdx.x*blockDim.x+threadIdx.x] % NB; float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    unsigned __int128* q=reinterpret_cast<unsigned __int128*>(&a0[b]); unsigned __int128 o=*q,as;
    do{ as=o; float4 f=*reinterpret_cast<float4*>(&as); f.x+=v; f.y+=v; f.z+=v; f.w+=v; o=atomicCAS(q,as,*reinterpret_cast<unsigned __int128*>(&f)); }while(o!=as);
    unsigned long long* q2=reinterpret_cast<unsigned long long*>(&a1[b]); unsigned long long o2=*q2,a2;
    do{ a2=o2; float2 f=*reinterpret_cast<float2*>(&a2); f.x+=v; f.y+=v; o2=atomicCAS(q2,a2,*reinterpret_cast<unsigned long long*>(&f)); }while(o2!=a2);
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads(); if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=a0[threadIdx.x].x+a1[threadIdx.x].y;
}
__global__ void k_i64(const int* __restrict__ idx, float* out, int iters){
  __shared__ unsigned long long a[6*NB];
  for(int i=threadIdx.x;i<6*NB;i+=blockDim.x) a[i]=0; __syncthreads();
  int b = idx[blockIdx.x*blockDim.x+threadIdx.x] % NB; float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    long long x = __float2ll_rn(v * 1099511627776.0f);
    #pragma unroll
    for(int k=0;k<6;k++) atomicAdd(&a[k*NB+b], (unsigned long long)x);
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads(); if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=(float)a[threadIdx.x];
}
__global__ void k_hilo(const int* __restrict__ idx, float* out, int iters){
  __shared__ unsigned lo[6*NB]; __shared__ int hi[6*NB];
  for(int i=threadIdx.x;i<6*NB;i+=blockDim.x){ lo[i]=0; hi[i]=0;} __syncthreads();
  int b = idx[blockIdx.x*blockDim.x+threadIdx.x] % NB; float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    long long x = __float2ll_rn(v * 1099511627776.0f);
    unsigned xl = (unsigned)x; int xh = (int)(x >> 32);
    unsigned ol[6];
    #pragma unroll
    for(int k=0;k<6;k++) ol[k] = atomicAdd(&lo[k*NB+b], xl);
    #pragma unroll
    for(int k=0;k<6;k++) { unsigned c = (ol[k] + xl) < ol[k]; atomicAdd(&hi[k*NB+b], xh + (int)c); }
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads(); if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=(float)lo[threadIdx.x]+hi[threadIdx.x];
}
__global__ void k_i32(const int* __restrict__ idx, float* out, int iters){
  __shared__ int a[6*NB];
  for(int i=threadIdx.x;i<6*NB;i+=blockDim.x) a[i]=0; __syncthreads();
  int b = idx[blockIdx.x*blockDim.x+threadIdx.x] % NB; float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    int x = __float2int_rn(v * 1024.0f);
    #pragma unroll
    for(int k=0;k<6;k++) atomicAdd(&a[k*NB+b], x);
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads(); if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=(float)a[threadIdx.x];
}
__global__ void k_hilo6(const int* __restrict__ idx, float* out, int iters){
  __shared__ unsigned lo[6*NB]; __shared__ int hi[6*NB];
  for(int i=threadIdx.x;i<6*NB;i+=blockDim.x){ lo[i]=0; hi[i]=0;} __syncthreads();
  int b = idx[blockIdx.x*blockDim.x+threadIdx.x] % NB; float v = 1.0f + threadIdx.x*1e-3f;
  for(int it=0; it<iters; ++it){
    unsigned ol[6]; long long x[6];
    #pragma unroll
    for(int k=0;k<6;k++) { x[k] = __float2ll_rn((v + k) * 1099511627776.0f); ol[k] = atomicAdd(&lo[k*NB+b], (unsigned)x[k]); }
    #pragma unroll
    for(int k=0;k<6;k++) { unsigned c = (ol[k] + (unsigned)x[k]) < (unsigned)x[k]; atomicAdd(&hi[k*NB+b], (int)(x[k] >> 32) + (int)c); }
    b = (b*1103515245u + 12345u) % NB;
  }
  __syncthreads(); if(threadIdx.x<NB) out[blockIdx.x*NB+threadIdx.x]=(float)lo[threadIdx.x]+hi[threadIdx.x];
}
int main(){
  const int blocks=148*4, threads=256, iters=200;
  int* idx; float* out; cudaMalloc(&idx, blocks*threads*4); cudaMalloc(&out, (size_t)blocks*NB*4);
  int* h=new int[blocks*threads]; unsigned s=1; for(int i=0;i<blocks*threads;i++){ s=s*1664525u+1013904223u; h[i]=(s>>8)%NB; }
  cudaMemcpy(idx,h,blocks*threads*4,cudaMemcpyHostToDevice);
  cudaEvent_t a,bq; cudaEventCreate(&a); cudaEventCreate(&bq);
  double n = (double)blocks*threads*iters;
  auto run=[&](const char* name, auto kern){
    for(int w=0;w<3;w++) kern<<<blocks,threads>>>(idx,out,iters);
    cudaEventRecord(a); for(int r=0;r<5;r++) kern<<<blocks,threads>>>(idx,out,iters); cudaEventRecord(bq);
    cudaEventSynchronize(bq); float ms; cudaEventElapsedTime(&ms,a,bq); ms/=5;
    printf("%-8s %8.3f ms  %7.2f SM-cycles per warp 6-value scatter  err=%s\n", name, ms, (ms*1e-3*1.9e9)/(n/32/148), cudaGetErrorString(cudaGetLastError()));
  };
  run("cas", k_cas); run("i64", k_i64); run("hilo32", k_hilo); run("i32", k_i32); run("hilo6", k_hilo6);
}
