// Streaming-pattern microbenchmark for the contact loop (scratch, not product).
#include <cstdio>
#include <cuda_runtime.h>
#define W 1024
#define CW 2000
__device__ __forceinline__ float4 ldnc(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ldca(const float4* p) { return __ldg(p); }
struct f8 { float4 a, b; };
__device__ __forceinline__ f8 ld256(const float4* p) {
  f8 r;
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
    : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y), "=f"(r.b.z), "=f"(r.b.w) : "l"(p));
  return r;
}
// (1) SoA 4 streams, 1-ahead prefetch, one CTA per world
__global__ void k_soa(const float4* s0, const float4* s1, const float4* s2, const float4* s3, float* out) {
  extern __shared__ float sm[];
  const int w = blockIdx.x; const float4 *a=s0+(size_t)w*CW, *b=s1+(size_t)w*CW, *c=s2+(size_t)w*CW, *d=s3+(size_t)w*CW;
  float acc = 0; int j = threadIdx.x;
  float4 A=ldnc(a+j), B=ldnc(b+j), C=ldnc(c+j), D=ldnc(d+j);
  for (; j < CW; j += 256) {
    float4 a0=A,b0=B,c0=C,d0=D; int jn = min(j+256, CW-1);
    A=ldnc(a+jn); B=ldnc(b+jn); C=ldnc(c+jn); D=ldnc(d+jn);
    acc += a0.x + b0.y + c0.z + d0.w;
  }
  if (acc == 1234.5f) out[0] = acc + sm[threadIdx.x];
}
// (1b) SoA 4 streams, 2-ahead
__global__ void k_soa2(const float4* s0, const float4* s1, const float4* s2, const float4* s3, float* out) {
  extern __shared__ float sm[];
  const int w = blockIdx.x; const float4 *a=s0+(size_t)w*CW, *b=s1+(size_t)w*CW, *c=s2+(size_t)w*CW, *d=s3+(size_t)w*CW;
  float acc = 0; int j = threadIdx.x;
  int j1 = min(j+256, CW-1);
  float4 A=ldnc(a+j), B=ldnc(b+j), C=ldnc(c+j), D=ldnc(d+j);
  float4 A1=ldnc(a+j1), B1=ldnc(b+j1), C1=ldnc(c+j1), D1=ldnc(d+j1);
  for (; j < CW; j += 256) {
    float4 a0=A,b0=B,c0=C,d0=D; A=A1;B=B1;C=C1;D=D1; int jn = min(j+512, CW-1);
    A1=ldnc(a+jn); B1=ldnc(b+jn); C1=ldnc(c+jn); D1=ldnc(d+jn);
    acc += a0.x + b0.y + c0.z + d0.w;
  }
  if (acc == 1234.5f) out[0] = acc + sm[threadIdx.x];
}
// (3) AoS 64 B per contact, 4 x LDG.128 (L1 allocate), 1-ahead
__global__ void k_aos(const float4* s, float* out) {
  extern __shared__ float sm[];
  const float4* a = s + (size_t)blockIdx.x * CW * 4;
  float acc = 0; int j = threadIdx.x;
  float4 A=ldca(a+4*j), B=ldca(a+4*j+1), C=ldca(a+4*j+2), D=ldca(a+4*j+3);
  for (; j < CW; j += 256) {
    float4 a0=A,b0=B,c0=C,d0=D; int jn = min(j+256, CW-1);
    A=ldca(a+4*jn); B=ldca(a+4*jn+1); C=ldca(a+4*jn+2); D=ldca(a+4*jn+3);
    acc += a0.x + b0.y + c0.z + d0.w;
  }
  if (acc == 1234.5f) out[0] = acc + sm[threadIdx.x];
}
// (4) AoS with 2 x 256-bit loads, 1-ahead
__global__ void k_aos256(const float4* s, float* out) {
  extern __shared__ float sm[];
  const float4* a = s + (size_t)blockIdx.x * CW * 4;
  float acc = 0; int j = threadIdx.x;
  f8 X = ld256(a + 4*j), Y = ld256(a + 4*j + 2);
  for (; j < CW; j += 256) {
    f8 x0 = X, y0 = Y; int jn = min(j+256, CW-1);
    X = ld256(a + 4*jn); Y = ld256(a + 4*jn + 2);
    acc += x0.a.x + x0.b.y + y0.a.z + y0.b.w;
  }
  if (acc == 1234.5f) out[0] = acc + sm[threadIdx.x];
}
// (5) SoA, one CTA per 1/2 world (double the CTAs, half the loop) 

// (6) persistent: CTAs loop over worlds; flattened (world, chunk) sequence with 1-ahead prefetch
__global__ void k_persist(const float4* s0, const float4* s1, const float4* s2, const float4* s3, float* out) {
  extern __shared__ float sm[];
  float acc = 0;
  const int nchunk = (CW + 255) / 256;
  int w = blockIdx.x, ch = 0;
  auto idx = [&](int w_, int ch_) { size_t j = ch_ * 256 + threadIdx.x; if (j >= CW) j = CW - 1; return (size_t)w_ * CW + j; };
  if (w >= W) return;
  size_t i0 = idx(w, 0);
  float4 A=ldnc(s0+i0), B=ldnc(s1+i0), C=ldnc(s2+i0), D=ldnc(s3+i0);
  while (true) {
    float4 a0=A,b0=B,c0=C,d0=D;
    int nw = w, nch = ch + 1;
    if (nch == nchunk) { nch = 0; nw = w + gridDim.x; }
    if (nw < W) { size_t in = idx(nw, nch); A=ldnc(s0+in); B=ldnc(s1+in); C=ldnc(s2+in); D=ldnc(s3+in); }
    if (ch * 256 + threadIdx.x < CW) acc += a0.x + b0.y + c0.z + d0.w;
    if (nw >= W) break;
    w = nw; ch = nch;
  }
  if (acc == 1234.5f) out[0] = acc + sm[threadIdx.x];
}
// (7) flat grid-stride over the whole array
__global__ void k_flat(const float4* s0, const float4* s1, const float4* s2, const float4* s3, float* out, size_t n) {
  float acc = 0;
  for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) {
    float4 a0=ldnc(s0+i), b0=ldnc(s1+i), c0=ldnc(s2+i), d0=ldnc(s3+i);
    acc += a0.x + b0.y + c0.z + d0.w;
  }
  if (acc == 1234.5f) out[0] = acc;
}
int main() {
  size_t n = (size_t)W * CW;
  float4 *s0, *s1, *s2, *s3, *aos; float* out; float* fl;
  cudaMalloc(&s0, n*16); cudaMalloc(&s1, n*16); cudaMalloc(&s2, n*16); cudaMalloc(&s3, n*16); cudaMalloc(&aos, n*64);
  cudaMalloc(&out, 64); cudaMalloc(&fl, 512u<<20);
  cudaMemset(s0, 0, n*16); cudaMemset(s1, 0, n*16); cudaMemset(s2, 0, n*16); cudaMemset(s3, 0, n*16); cudaMemset(aos, 0, n*64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double bytes = (double)n * 64;
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    float tot = 0;
    for (int i = 0; i < 10; ++i) {
      cudaMemset(fl, 0, 512u<<20);
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms;
    }
    tot /= 10;
    printf("%-34s %8.2f us  %7.0f GB/s\n", name, tot*1e3, bytes/tot/1e6);
  };
  for (int k : {4, 8}) {
    cudaFuncSetAttribute(k_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, 53*1024);
    char nm[64];
    int smem = k == 4 ? 53*1024 : 1024;
    sprintf(nm, "persistent %d CTA/SM", k); run(nm, [&]{ k_persist<<<148*k,256,smem>>>(s0,s1,s2,s3,out); });
    sprintf(nm, "flat grid-stride %d CTA/SM", k); run(nm, [&]{ k_flat<<<148*k,256>>>(s0,s1,s2,s3,out,n); });
  }
  for (int smem : {53*1024, 1024}) {
    cudaFuncSetAttribute(k_soa, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_soa2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_aos, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_aos256, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    char nm[64];
    sprintf(nm, "soa 1-ahead smem=%dK", smem/1024); run(nm, [&]{ k_soa<<<W,256,smem>>>(s0,s1,s2,s3,out); });
    sprintf(nm, "soa 2-ahead smem=%dK", smem/1024); run(nm, [&]{ k_soa2<<<W,256,smem>>>(s0,s1,s2,s3,out); });
    sprintf(nm, "aos 4xLDG128 smem=%dK", smem/1024); run(nm, [&]{ k_aos<<<W,256,smem>>>(aos,out); });
    sprintf(nm, "aos 2xLDG256 smem=%dK", smem/1024); run(nm, [&]{ k_aos256<<<W,256,smem>>>(aos,out); });
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
