// A/B of the facet layout of S4-S5 (Eq. (7)-(9), Alg. 1 Kernel II):
// lane per contact (the product kernel's layout: each lane unrolls its
// contact's facet pairs) against the north star's lane per facet (and lane per
// facet pair) with warp-shuffle segmented sums of the facet impulses.
// 18 facets per contact (condim 6, n_t = 8, n_tor = 2, n_rol = 8: config C2b's
// cone), 2,048,000 contacts (C4's count).  Per contact the inputs are the S3
// results the kernel holds in registers (A = -k phi - kappa u_n, the channel
// velocities times kappa mu, M(phi)); the outputs are the S5 sums N, F (2), M_tor,
// M_rol (2), i.e. sum_f Lambda_f J~_f regrouped, 6 floats.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo facet_layout_bench.cu -o flb
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int NT = 8, NR = 8, PAIRS = NT / 2 + 1 + NR / 2;  // 9 symmetric pairs = 18 facets
__constant__ float2 c_dir_t[NT / 2], c_dir_r[NR / 2];

struct In { const float *A, *kt, *w1, *w2, *ator, *kr, *r1, *r2, *Mc; };
struct Out { float *N, *F1, *F2, *Mt, *R1, *R2; };

__device__ __forceinline__ void pair(float A, float a, float& Lp, float& Lm, float& d) {
  Lp = fmaxf(A + a, 0.f);
  Lm = fmaxf(A - a, 0.f);
  d = (A >= fabsf(a)) ? 2.f * a : Lp - Lm;
}

// (1) lane per contact: the product layout
__global__ void k_lane_per_contact(In in, Out out, int n) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const float A = in.A[c], kt = in.kt[c], w1 = in.w1[c], w2 = in.w2[c], at = in.ator[c];
    const float kr = in.kr[c], r1 = in.r1[c], r2 = in.r2[c], Mc = in.Mc[c];
    float N = 0.f, F1 = 0.f, F2 = 0.f, R1 = 0.f, R2 = 0.f, Mt, Lp, Lm, d;
#pragma unroll
    for (int j = 0; j < NT / 2; ++j) {
      const float2 dj = c_dir_t[j];
      pair(A, kt * fmaf(dj.x, w1, dj.y * w2), Lp, Lm, d);
      N += Lp + Lm; F1 = fmaf(d, dj.x, F1); F2 = fmaf(d, dj.y, F2);
    }
    pair(A, at, Lp, Lm, Mt);
    N += Lp + Lm;
#pragma unroll
    for (int j = 0; j < NR / 2; ++j) {
      const float2 dj = c_dir_r[j];
      pair(A, kr * fmaf(dj.x, r1, dj.y * r2), Lp, Lm, d);
      N += Lp + Lm; R1 = fmaf(d, dj.x, R1); R2 = fmaf(d, dj.y, R2);
    }
    out.N[c] = Mc * N; out.F1[c] = Mc * F1; out.F2[c] = Mc * F2;
    out.Mt[c] = Mc * Mt; out.R1[c] = Mc * R1; out.R2[c] = Mc * R2;
  }
}

// (2) lane per facet pair: 9 lanes per contact, 3 contacts per warp (27 of 32
// lanes busy); each lane evaluates its pair, then a segmented shuffle sum over
// the contact's 9 lanes (4 rounds x 6 values).
__global__ void k_lane_per_pair(In in, Out out, int n) {
  const int lane = threadIdx.x & 31, seg = lane / PAIRS, k = lane % PAIRS;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int c0 = warp * 3; c0 < n; c0 += nwarps * 3) {
    const int c = c0 + seg;
    const bool on = seg < 3 && c < n;
    float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // N, F1, F2, Mt, R1, R2
    if (on) {
      const float A = in.A[c];
      float Lp, Lm, d;
      if (k < NT / 2) {
        const float2 dj = c_dir_t[k];
        pair(A, in.kt[c] * fmaf(dj.x, in.w1[c], dj.y * in.w2[c]), Lp, Lm, d);
        v[1] = d * dj.x; v[2] = d * dj.y;
      } else if (k == NT / 2) {
        pair(A, in.ator[c], Lp, Lm, d);
        v[3] = d;
      } else {
        const float2 dj = c_dir_r[k - NT / 2 - 1];
        pair(A, in.kr[c] * fmaf(dj.x, in.r1[c], dj.y * in.r2[c]), Lp, Lm, d);
        v[4] = d * dj.x; v[5] = d * dj.y;
      }
      v[0] = Lp + Lm;
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const float u = __shfl_down_sync(0xffffffffu, v[q], o);
        if (k + o < PAIRS) v[q] += u;
      }
    }
    if (on && k == 0) {
      const float Mc = in.Mc[c];
      out.N[c] = Mc * v[0]; out.F1[c] = Mc * v[1]; out.F2[c] = Mc * v[2];
      out.Mt[c] = Mc * v[3]; out.R1[c] = Mc * v[4]; out.R2[c] = Mc * v[5];
    }
  }
}

// (3) lane per facet: 18 lanes per contact, one contact per warp (18 of 32
// lanes busy), segmented shuffle sum over 18 lanes (5 rounds x 6 values).
__global__ void k_lane_per_facet(In in, Out out, int n) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int c = warp; c < n; c += nwarps) {
    float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (lane < 2 * PAIRS) {
      const float A = in.A[c];
      const int k = lane >> 1;
      const float sg = (lane & 1) ? -1.f : 1.f;  // facet +d or -d
      float a, dx = 0.f, dy = 0.f;
      int ch;
      if (k < NT / 2) { const float2 dj = c_dir_t[k]; a = in.kt[c] * fmaf(dj.x, in.w1[c], dj.y * in.w2[c]); dx = dj.x; dy = dj.y; ch = 0; }
      else if (k == NT / 2) { a = in.ator[c]; ch = 1; }
      else { const float2 dj = c_dir_r[k - NT / 2 - 1]; a = in.kr[c] * fmaf(dj.x, in.r1[c], dj.y * in.r2[c]); dx = dj.x; dy = dj.y; ch = 2; }
      const float L = fmaxf(A + sg * a, 0.f);
      v[0] = L;
      if (ch == 0) { v[1] = sg * L * dx; v[2] = sg * L * dy; }
      else if (ch == 1) v[3] = sg * L;
      else { v[4] = sg * L * dx; v[5] = sg * L * dy; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < 6; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    if (lane == 0) {
      const float Mc = in.Mc[c];
      out.N[c] = Mc * v[0]; out.F1[c] = Mc * v[1]; out.F2[c] = Mc * v[2];
      out.Mt[c] = Mc * v[3]; out.R1[c] = Mc * v[4]; out.R2[c] = Mc * v[5];
    }
  }
}

int main() {
  const int n = 2048000;
  std::vector<float> h(9 * (size_t)n);
  srand(7);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)rand() / RAND_MAX - 0.3f;
  float* d; CK(cudaMalloc(&d, h.size() * 4));
  CK(cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  float* o; CK(cudaMalloc(&o, 3 * 6 * (size_t)n * 4));
  float2 dt[NT / 2], dr[NR / 2];
  for (int j = 0; j < NT / 2; ++j) dt[j] = make_float2(cosf(2 * M_PI * j / NT), sinf(2 * M_PI * j / NT));
  for (int j = 0; j < NR / 2; ++j) dr[j] = make_float2(cosf(2 * M_PI * j / NR), sinf(2 * M_PI * j / NR));
  CK(cudaMemcpyToSymbol(c_dir_t, dt, sizeof dt)); CK(cudaMemcpyToSymbol(c_dir_r, dr, sizeof dr));
  In in{d, d + n, d + 2 * (size_t)n, d + 3 * (size_t)n, d + 4 * (size_t)n, d + 5 * (size_t)n, d + 6 * (size_t)n,
        d + 7 * (size_t)n, d + 8 * (size_t)n};
  Out out[3];
  for (int v = 0; v < 3; ++v) {
    float* b = o + (size_t)v * 6 * n;
    out[v] = Out{b, b + n, b + 2 * (size_t)n, b + 3 * (size_t)n, b + 4 * (size_t)n, b + 5 * (size_t)n};
  }
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"lane per contact (product)", "lane per facet pair (9 lanes, shfl)", "lane per facet (18 lanes, shfl)"};
  for (int v = 0; v < 3; ++v) {
    auto launch = [&]() {
      if (v == 0) k_lane_per_contact<<<nsm * 8, 256>>>(in, out[0], n);
      else if (v == 1) k_lane_per_pair<<<nsm * 8, 256>>>(in, out[1], n);
      else k_lane_per_facet<<<nsm * 8, 256>>>(in, out[2], n);
    };
    for (int i = 0; i < 5; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < 50; ++i) launch();
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %8.2f us per 2.048M contacts x 18 facets (%.2f G facets/s)\n", names[v], ms / 50 * 1e3,
           2.048e6 * 18 / (ms / 50 * 1e-3) / 1e9);
  }
  // the three layouts agree
  std::vector<float> r(3 * 6 * (size_t)n);
  CK(cudaMemcpy(r.data(), o, r.size() * 4, cudaMemcpyDeviceToHost));
  double md = 0.0;
  for (size_t i = 0; i < 6 * (size_t)n; ++i)
    for (int v = 1; v < 3; ++v) md = fmax(md, fabs(r[i] - r[v * 6 * (size_t)n + i]) / (fabs(r[i]) + 1e-3));
  printf("max rel difference between layouts: %.2e\n", md);
  return 0;
}
