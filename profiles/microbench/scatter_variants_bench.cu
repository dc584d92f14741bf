// Warp scatter of 6 values per lane into per-CTA fixed-point accumulators with
// pile-like key structure (side a: sorted runs ~6, side b: runs ~1.5).
// V0: float Hillis-Steele run sums, tail converts + hi/lo atomics (current kernel)
// V1: per-lane fixed point, match_any + redux.sync on (hi, lo>>16, lo&0xffff), tail atomics
// V3: per-lane fixed point, every lane does hi/lo atomics (no aggregation)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define NB 512
#define NK (1 << 16)
__device__ __forceinline__ float hval(unsigned s) { return (float)((s * 2654435761u) >> 8) * (1.0f / 16777216.0f) - 0.5f; }

__device__ __forceinline__ bool seg_sum6(int key, float v[6], int lane) {
  const unsigned full = 0xffffffffu;
  const int prev = __shfl_up_sync(full, key, 1);
  const int next = __shfl_down_sync(full, key, 1);
  const bool head = lane == 0 || prev != key;
  const bool tail = lane == 31 || next != key;
  const unsigned heads = __ballot_sync(full, head);
  if (heads == full) return tail;
  const int start = 31 - __clz(heads & (full >> (31 - lane)));
  const int pos = lane - start;
  const int maxpos = (int)__reduce_max_sync(full, (unsigned)pos);
  for (int o = 1; o <= maxpos; o <<= 1) {
#pragma unroll
    for (int kk = 0; kk < 6; ++kk) {
      const float u = __shfl_up_sync(full, v[kk], o);
      if (pos >= o) v[kk] += u;
    }
  }
  return tail;
}
__device__ __forceinline__ void fx_add(unsigned* lo, int* hi, long long x) {
  const unsigned xl = (unsigned)x;
  const unsigned old = atomicAdd(lo, xl);
  atomicAdd(hi, (int)(x >> 32) + (int)((unsigned)(old + xl) < xl));
}
__device__ __forceinline__ long long f2ll_man(float f) {
  const int b = __float_as_int(f);
  const int e = ((b >> 23) & 0xff) - 150;
  const long long m = (b & 0x7f800000) ? (long long)((b & 0x7fffff) | 0x800000) : 0ll;
  const int sh = min(-e, 63);
  const long long up = m << max(e, 0);
  const long long dn = (m + ((1ll << sh) >> 1)) >> sh;
  const long long x = e >= 0 ? up : dn;
  return b < 0 ? -x : x;
}
__device__ __forceinline__ void fx_add2(unsigned* lo, int* hi, long long x) {
  atomicAdd(lo, (unsigned)x & 0xfffffu);
  atomicAdd(hi, (int)(x >> 20));
}
constexpr float S = 8589934592.0f * 64.f;  // 2^39

template <int V>
__global__ void __launch_bounds__(256, 4) k(const int* __restrict__ ka, const int* __restrict__ kb, float* out, int iters) {
  __shared__ unsigned lo[6 * NB];
  __shared__ int hi[6 * NB];
  for (int i = threadIdx.x; i < 6 * NB; i += blockDim.x) { lo[i] = 0; hi[i] = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned pos = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 32 * 7 + lane;
  for (int it = 0; it < iters; ++it) {
    pos = (pos + 32 * 8) & (NK - 1);
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int key = side ? kb[pos] : ka[pos];
      float v[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) v[q] = hval(pos * 6 + q + side);
      if (V == 0) {
        const bool tail = seg_sum6(key, v, lane) && key >= 0;
        if (tail)
#pragma unroll
          for (int q = 0; q < 6; ++q) fx_add(lo + q * NB + key, hi + q * NB + key, __float2ll_rn(v[q] * S));
      } else if (V == 1) {
        const unsigned m = __match_any_sync(0xffffffffu, key);
        const bool tail = (lane == 31 - __clz(m)) && key >= 0;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          const long long x = __float2ll_rn(v[q] * S);
          long long t;
          if (m == (1u << lane)) {
            t = x;
          } else {
            const unsigned xl = (unsigned)x;
            const int h = __reduce_add_sync(m, (int)(x >> 32));
            const unsigned a = __reduce_add_sync(m, xl >> 16);
            const unsigned b = __reduce_add_sync(m, xl & 0xffffu);
            t = ((long long)h << 32) + ((long long)a << 16) + (long long)b;
          }
          if (tail) fx_add(lo + q * NB + key, hi + q * NB + key, t);
        }
      } else if (V == 12) {
        const bool tail = seg_sum6(key, v, lane) && key >= 0;
        if (tail)
#pragma unroll
          for (int q = 0; q < 6; ++q) fx_add2(lo + q * NB + key, hi + q * NB + key, __float2ll_rn(v[q] * S));
      } else if (V == 4) {
        const bool tail = seg_sum6(key, v, lane) && key >= 0;
        if (tail)
#pragma unroll
          for (int q = 0; q < 6; ++q) fx_add(lo + q * NB + key, hi + q * NB + key, f2ll_man(v[q] * S));
      } else if (V == 5) {
        const bool tail = seg_sum6(key, v, lane) && key >= 0;
        if (tail)
#pragma unroll
          for (int q = 0; q < 6; ++q) { const long long x = __float2ll_rn(v[q] * S); lo[q * NB + key] += (unsigned)x; hi[q * NB + key] += (int)(x >> 32); }
      } else if (V == 6) {
        const bool tail = seg_sum6(key, v, lane) && key >= 0;
        if (tail)
#pragma unroll
          for (int q = 0; q < 6; ++q) atomicAdd(lo + q * NB + key, (unsigned)__float2ll_rn(v[q] * S));
      } else if (V == 7) {
        long long t = 0;
#pragma unroll
        for (int q = 0; q < 6; ++q) t += __float2ll_rn(v[q] * S);
        if (t == 12345 && key == 7) lo[0] = 1;
      } else if (V == 8) {
        const bool tail = seg_sum6(key, v, lane) && key >= 0;
        float t = 0.f;
#pragma unroll
        for (int q = 0; q < 6; ++q) t += v[q];
        if (tail && t == 12345.f) lo[0] = 1;
      } else if (V == 9) {
        float t = 0.f;
#pragma unroll
        for (int q = 0; q < 6; ++q) t += v[q];
        if (t == 12345.f && key == 7) lo[0] = 1;
      } else {
        if (key >= 0)
#pragma unroll
          for (int q = 0; q < 6; ++q) fx_add(lo + q * NB + key, hi + q * NB + key, __float2ll_rn(v[q] * S));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 6 * NB; i += blockDim.x)
    out[(size_t)blockIdx.x * 6 * NB + i] = (float)(((long long)hi[i] << 32) | lo[i]) / S;
}

// V10: lane-sequential contacts; per-lane run accumulation in registers, flush on key change
template <int K, bool BDIRECT = false>
__global__ void __launch_bounds__(256, 4) kseq(const int* __restrict__ ka, const int* __restrict__ kb, float* out, int iters) {
  __shared__ unsigned lo[6 * NB];
  __shared__ int hi[6 * NB];
  for (int i = threadIdx.x; i < 6 * NB; i += blockDim.x) { lo[i] = 0; hi[i] = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned base = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 32 * 7;
  int cka = -1, ckb = -1;
  float aa[6] = {0, 0, 0, 0, 0, 0}, ab[6] = {0, 0, 0, 0, 0, 0};
  for (int it = 0; it < iters; ++it) {
    if (it % K == 0) base = (base + 32 * K) & (NK - 1);
    const unsigned pos = (base + lane * K + it % K) & (NK - 1);
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int key = side ? kb[pos] : ka[pos];
      float* acc = side ? ab : aa;
      int& ck = side ? ckb : cka;
      if (BDIRECT && side) {
        if (key >= 0)
#pragma unroll
          for (int q = 0; q < 6; ++q) fx_add(lo + q * NB + key, hi + q * NB + key, __float2ll_rn(hval(pos * 6 + q + side) * S));
        continue;
      }
      if (key != ck) {
        if (ck >= 0)
#pragma unroll
          for (int q = 0; q < 6; ++q) fx_add(lo + q * NB + ck, hi + q * NB + ck, __float2ll_rn(acc[q] * S));
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[q] = 0.f;
        ck = key;
      }
#pragma unroll
      for (int q = 0; q < 6; ++q) acc[q] += hval(pos * 6 + q + side);
    }
  }
  if (cka >= 0) for (int q = 0; q < 6; ++q) fx_add(lo + q * NB + cka, hi + q * NB + cka, __float2ll_rn(aa[q] * S));
  if (ckb >= 0) for (int q = 0; q < 6; ++q) fx_add(lo + q * NB + ckb, hi + q * NB + ckb, __float2ll_rn(ab[q] * S));
  __syncthreads();
  for (int i = threadIdx.x; i < 6 * NB; i += blockDim.x)
    out[(size_t)blockIdx.x * 6 * NB + i] = (float)(((long long)hi[i] << 32) | lo[i]) / S;
}

int main() {
  // pile-like keys: side a sorted runs mean ~6 (10% static -1), side b runs 1-2
  std::vector<int> ha(NK), hb(NK);
  unsigned s = 7;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return s >> 8; };
  int i = 0, body = 0;
  while (i < NK) {
    int len = 1 + rnd() % 11;
    int key = (rnd() % 10 == 0) ? -1 : (body++ % NB);
    for (int j = 0; j < len && i < NK; ++j, ++i) ha[i] = key;
  }
  i = 0;
  while (i < NK) {
    int len = 1 + (rnd() % 3 == 0);
    int key = rnd() % NB;
    for (int j = 0; j < len && i < NK; ++j, ++i) hb[i] = key;
  }
  int *ka, *kb; float* out;
  const int blocks = 148 * 4, threads = 256, iters = 400;
  cudaMalloc(&ka, NK * 4); cudaMalloc(&kb, NK * 4); cudaMalloc(&out, (size_t)blocks * 6 * NB * 4);
  cudaMemcpy(ka, ha.data(), NK * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(kb, hb.data(), NK * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  double n = (double)blocks * 8 * iters;  // warp iterations (both sides)
  std::vector<float> ref;
  auto run = [&](const char* name, auto kern) {
    for (int w = 0; w < 3; w++) kern<<<blocks, threads>>>(ka, kb, out, iters);
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) kern<<<blocks, threads>>>(ka, kb, out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    std::vector<float> h((size_t)blocks * 6 * NB);
    cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost);
    double md = 0;
    if (ref.empty()) ref = h;
    else for (size_t j = 0; j < h.size(); ++j) md = fmax(md, fabs(h[j] - ref[j]));
    printf("%-6s %8.3f ms  %7.2f SM-cycles per warp iteration (2 sides)  maxdiff %.3g  %s\n", name, ms,
           (ms * 1e-3 * 1.965e9) / (n / 148), md, cudaGetErrorString(cudaGetLastError()));
  };
  run("V0", k<0>); run("V1", k<1>); run("V3", k<3>); run("base", k<9>); run("V12split", k<12>); run("V4man", k<4>); run("V5noat", k<5>); run("V6lo", k<6>); run("V7f2i", k<7>); run("V8seg", k<8>); run("seq8", kseq<8>); run("seq16", kseq<16>); run("seq8bd", kseq<8, true>);
}
