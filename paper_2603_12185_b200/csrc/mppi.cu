// mppi.cu — MPPI on the batched step (§V,
// Eq. (14)-(15); reading R27).  The rollout worlds of a
// context are P problems x N samples (world w belongs to problem w / N).
//   k_mppi_sample   U = clip(plan + eps) with eps from SplitMix64 -> Box-Muller
//                   (counter-based: element k of iteration it is a pure function
//                   of (seed, k)), thread per element
//   k_mppi_control  incremental position control: command += u_t, chain torque
//                   tau = kp (command - q) - kd qdot, thread per (world, DoF)
//   k_mppi_cost     Eq. (15) running cost c(x_t) or terminal V(x_H) of every
//                   world, accumulated into J[w], thread per world (fingertips
//                   from the chain forward kinematics)
//   k_mppi_cost_control  the running cost and the control of one rollout step in
//                   one launch (both read x_t only)
//   k_mppi_update   one CTA per problem: min over the N costs, weights
//                   exp(-(J - min)/lambda) normalised, plan = clip(sum w U)
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "chain.cuh"
#include "internal.h"

namespace cf {

namespace {

using namespace chain;

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_mppi_sample(const float* __restrict__ plan, int P, int N, int H, int Q, float sigma, float lo,
                              float hi, uint64_t seed, uint64_t iteration, float* __restrict__ U) {
  const int64_t n = (int64_t)P * N * H * Q;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int64_t hq = (int64_t)H * Q;
  const int64_t p = e / ((int64_t)N * hq);
  const int64_t th = e % hq;                                  // t * Q + j
  const uint64_t k = iteration * (uint64_t)n + (uint64_t)e;   // ((it P + p) N + i) H Q + t Q + j
  const float u1 = (float)(splitmix64(seed + 2 * k) >> 40) * (1.f / 16777216.f);
  const float u2 = (float)(splitmix64(seed + 2 * k + 1) >> 40) * (1.f / 16777216.f);
  const float eps = sigma * sqrtf(-2.f * logf(1.f - u1)) * cospif(2.f * u2);
  U[e] = fminf(fmaxf(plan[p * hq + th] + eps, lo), hi);
}

__device__ __forceinline__ void mppi_control_elem(int64_t e, const float* __restrict__ slab, int slab_stride, int qoff,
                                                  int Qp, int Q, const float* __restrict__ U, int t, int H, float kp,
                                                  float kd, float* __restrict__ command, float* __restrict__ tau) {
  const int64_t w = e / Q;
  const int j = (int)(e - w * Q);
  const float* sq = slab + (size_t)w * slab_stride + qoff;
  const float cmd = command[e] + U[(w * H + t) * Q + j];
  command[e] = cmd;
  tau[e] = kp * (cmd - sq[j]) - kd * sq[Qp + j];
}

__global__ void k_mppi_control(const float* __restrict__ slab, int slab_stride, int qoff, int Qp, int Q, int64_t W,
                               const float* __restrict__ U, int t, int H, float kp, float kd,
                               float* __restrict__ command, float* __restrict__ tau) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= W * Q) return;
  mppi_control_elem(e, slab, slab_stride, qoff, Qp, Q, U, t, H, kp, kd, command, tau);
}

__device__ __forceinline__ void mppi_cost_world(int64_t w, const MppiCostParams& C, float* __restrict__ J) {
  const int p = (int)(w / C.n_samples);
  const float* sp = C.slab + (size_t)w * C.sc.slab + C.obj;
  const size_t pb = (size_t)C.sc.Bp;
  const V3 po = v3(sp[0], sp[pb], sp[2 * pb]);
  float qw = sp[3 * pb], qx = sp[4 * pb], qy = sp[5 * pb], qz = sp[6 * pb];
  const float qn = rsqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
  const float* tq = C.target_quat + 4 * p;
  const float dq = (tq[0] * qw + tq[1] * qx + tq[2] * qy + tq[3] * qz) * qn;
  const float cq = 1.f - dq * dq;
  const V3 pt = v3(C.target_pos[3 * p], C.target_pos[3 * p + 1], C.target_pos[3 * p + 2]);
  float c;
  if (C.terminal) {
    const V3 d = sub(po, pt);
    c = C.phi1 * dot(d, d) + C.phi2 * cq;
  } else {
    c = C.w[0] * cq + C.w[1] * fabsf(po.x - pt.x) + C.w[2] * fabsf(po.y - pt.y) + C.w[3] * fabsf(po.z - pt.z);
    const int T = C.sc.T, nd = C.sc.nd;
    const float* sq = C.slab + (size_t)w * C.sc.slab + N_BODY_PLANES * C.sc.Bp;
    float ctip = 0.f, cj = 0.f;
    for (int t = 0; t < T; ++t) {
      float q[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nd) {
          q[j] = sq[t * nd + j];
          const float dj = q[j] - C.q_ref[t * nd + j];
          cj += dj * dj;
        }
      V3 a[4], o[4], d[4];
      const float* m = C.model + (size_t)t * (3 + 7 * nd);
      chain_fk(m, nd, q, a, o, d);
      const V3 tip = add(o[nd - 1], mul(m[3 + 7 * (nd - 1) + 3], d[nd - 1]));
      const V3 r = sub(po, tip);
      ctip += dot(r, r);
    }
    c += C.w[4] * ctip + C.w[5] * cj + (po.z < C.z_fallen ? C.omega_fallen : 0.f);
  }
  J[w] += c;
}

__global__ void k_mppi_cost(const __grid_constant__ MppiCostParams C, float* __restrict__ J) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= C.n_worlds) return;
  mppi_cost_world(w, C, J);
}

// Running cost and control of one rollout step in one launch (both read x_t only):
// threads [0, W) the costs, threads [W, W + W Q) the commands and torques.
__global__ void k_mppi_cost_control(const __grid_constant__ MppiCostParams C, float* __restrict__ J,
                                    const float* __restrict__ U, int t, int H, float kp, float kd,
                                    float* __restrict__ command, float* __restrict__ tau) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t W = C.n_worlds, Q = C.sc.Q;
  if (id < W) {
    mppi_cost_world(id, C, J);
  } else if (id - W < W * Q) {
    mppi_control_elem(id - W, C.slab, C.sc.slab, N_BODY_PLANES * C.sc.Bp, C.sc.Qp, (int)Q, U, t, H, kp, kd, command,
                      tau);
  }
}

// One CTA per problem (blockDim = 256): weights over the N samples, then the
// weighted plan, clipped.  A sample whose cost is not finite (a diverged
// rollout) counts as J = +inf, i.e. weight 0; when no sample of a problem has
// a finite cost the problem keeps its previous plan (weights 0).
__device__ __forceinline__ float finite_cost(float j) { return isfinite(j) ? j : INFINITY; }

__global__ void k_mppi_update(const float* __restrict__ J, const float* __restrict__ U, int N, int H, int Q,
                              float lambda, float lo, float hi, float* __restrict__ plan, float* __restrict__ weights,
                              float* __restrict__ u0) {
  extern __shared__ float sw[];  // N weights
  __shared__ float red[32];
  const int p = blockIdx.x;
  const float* Jp = J + (size_t)p * N;
  float m = INFINITY;
  for (int i = threadIdx.x; i < N; i += blockDim.x) m = fminf(m, finite_cost(Jp[i]));
  for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float jmin = red[0];
  __syncthreads();
  if (!isfinite(jmin)) {  // every rollout of this problem diverged: keep the plan
    for (int i = threadIdx.x; i < N; i += blockDim.x)
      if (weights) weights[(size_t)p * N + i] = 0.f;
    if (u0) {  // receding horizon on the kept plan: u0 = its first action, then advance it
      const int hq = H * Q;
      float* pl = plan + (size_t)p * hq;
      for (int j = threadIdx.x; j < Q; j += blockDim.x) u0[(size_t)p * Q + j] = pl[j];
      __syncthreads();
      float v[8];
      for (int e0 = 0; e0 < hq; e0 += 8 * blockDim.x) {  // in-place shift: read a block, sync, write it
        for (int k = 0; k < 8; ++k) { const int e = e0 + k * blockDim.x + threadIdx.x; v[k] = (e + Q < hq && e < hq) ? pl[e + Q] : 0.f; }
        __syncthreads();
        for (int k = 0; k < 8; ++k) { const int e = e0 + k * blockDim.x + threadIdx.x; if (e < hq) pl[e] = v[k]; }
        __syncthreads();
      }
    }
    return;
  }
  float s = 0.f;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const float ji = finite_cost(Jp[i]);
    const float wi = isfinite(ji) ? expf(-(ji - jmin) / lambda) : 0.f;
    sw[i] = wi;
    s += wi;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tot += red[k];
    red[0] = tot;
  }
  __syncthreads();
  const float inv = 1.f / red[0];
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    sw[i] *= inv;
    if (weights) weights[(size_t)p * N + i] = sw[i];
  }
  __syncthreads();
  const int hq = H * Q;
  const float* Up = U + (size_t)p * N * hq;
  for (int e = threadIdx.x; e < hq; e += blockDim.x) {
    float acc = 0.f;
    for (int i = 0; i < N; ++i) acc = fmaf(sw[i], Up[(size_t)i * hq + e], acc);
    const float a = fminf(fmaxf(acc, lo), hi);
    if (!u0) {
      plan[(size_t)p * hq + e] = a;
    } else {  // receding horizon: u0 = the first action, the plan advanced by one step
      if (e < Q) u0[(size_t)p * Q + e] = a;
      else plan[(size_t)p * hq + e - Q] = a;
      if (e >= hq - Q) plan[(size_t)p * hq + e] = 0.f;
    }
  }
}

unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

cudaError_t mppi_sample(const float* plan, int P, int N, int H, int Q, float sigma, float lo, float hi, uint64_t seed,
                        uint64_t iteration, float* U, cudaStream_t s) {
  const int64_t n = (int64_t)P * N * H * Q;
  if (n == 0) return cudaSuccess;
  k_mppi_sample<<<nblk(n), 256, 0, s>>>(plan, P, N, H, Q, sigma, lo, hi, seed, iteration, U);
  return cudaGetLastError();
}

cudaError_t mppi_control(const SceneDev& sc, const float* slab, int64_t W, const float* U, int t, int H, float kp,
                         float kd, float* command, float* tau, cudaStream_t s) {
  const int64_t n = W * sc.Q;
  if (n == 0) return cudaSuccess;
  k_mppi_control<<<nblk(n), 256, 0, s>>>(slab, sc.slab, N_BODY_PLANES * sc.Bp, sc.Qp, sc.Q, W, U, t, H, kp, kd,
                                         command, tau);
  return cudaGetLastError();
}

cudaError_t mppi_cost(const MppiCostParams& C, float* J, cudaStream_t s) {
  if (C.n_worlds == 0) return cudaSuccess;
  k_mppi_cost<<<nblk(C.n_worlds), 256, 0, s>>>(C, J);
  return cudaGetLastError();
}

cudaError_t mppi_cost_control(const MppiCostParams& C, float* J, const float* U, int t, int H, float kp, float kd,
                              float* command, float* tau, cudaStream_t s) {
  const int64_t n = C.n_worlds * (1 + C.sc.Q);
  if (n == 0) return cudaSuccess;
  k_mppi_cost_control<<<nblk(n), 256, 0, s>>>(C, J, U, t, H, kp, kd, command, tau);
  return cudaGetLastError();
}

cudaError_t mppi_update(const float* J, const float* U, int P, int N, int H, int Q, float lambda, float lo, float hi,
                        float* plan, float* weights, cudaStream_t s, float* u0) {
  if (P == 0) return cudaSuccess;
  k_mppi_update<<<P, 256, (size_t)N * sizeof(float), s>>>(J, U, N, H, Q, lambda, lo, hi, plan, weights, u0);
  return cudaGetLastError();
}

}  // namespace cf
