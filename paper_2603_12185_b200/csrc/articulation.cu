// articulation.cu — the articulated upstream of the step on the GPU (SURVEY
// §8(f) rank 2): for serial hinge chains (comfree_articulation), per world and
// chain, from the step-start joint positions and velocities in the state slab:
//   forward kinematics, joint-space inertia M(q) = armature + sum_l m_l Jv_l^T Jv_l
//   + I_l Jw_l^T Jw_l, its Cholesky factor (packed, the step's tree_L), and the
//   bias c(q, v) (Coriolis/centrifugal/gravity, Eq. (1)-(2))
//   by a Newton-Euler forward pass at zero acceleration -> tree_tau = tau - c;
// and per contact, the 6 x nd rows of a chain side (point velocity and angular
// velocity of link l at the contact point, Eq. (4)-(5)) written in
// the step's [12][n][4] jrow layout.
// One thread per (world, chain) and one per contact; everything in registers
// (nd <= 4).  HBM-bound on the slab reads and the factor / row writes.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "chain.cuh"
#include "internal.h"

namespace cf {

namespace {

using namespace chain;

// One thread per (world, chain): M, its Cholesky factor, tau - c.
__device__ __forceinline__ void chain_dynamics(int64_t id, const float* __restrict__ model, int T, int nd,
                                               const float* __restrict__ slab, int slab_stride, int qoff, int Qp,
                                               const float* __restrict__ tau_ext, float gx, float gy, float gz,
                                               float* __restrict__ L_out, float* __restrict__ tau_out,
                                               int* __restrict__ err) {
  const int64_t w = id / T;
  const int t = (int)(id - w * T);
  const float* m = model + (size_t)t * (3 + 7 * nd);
  const float* sq = slab + (size_t)w * slab_stride + qoff + t * nd;  // qpos, then qvel at + Qp
  float q[4] = {0.f, 0.f, 0.f, 0.f}, v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (j < nd) { q[j] = sq[j]; v[j] = sq[Qp + j]; }
  V3 a[4], o[4], d[4];
  chain_fk(m, nd, q, a, o, d);
  // M = armature + sum_l m_l Jv_l^T Jv_l + I_l Jw_l^T Jw_l, with
  // Jv_l[:, i] = a_i x (com_l - o_i), Jw_l[:, i] = a_i (i <= l)
  float M[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) M[i][k] = (i == k && i < nd) ? m[3 + 7 * i + 6] : 0.f;
  // bias by Newton-Euler at zero acceleration: link angular velocity w, angular
  // acceleration al, joint-origin acceleration ao; c_i = sum_l Jv_l[:, i] . F_l + Jw_l[:, i] . N_l
  float c[4] = {0.f, 0.f, 0.f, 0.f};
  V3 w3 = v3(0.f, 0.f, 0.f), al = w3, ao = w3;
  const V3 g = v3(gx, gy, gz);
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    if (l < nd) {
      const float* ml = m + 3 + 7 * l;
      const float len = ml[3], mass = ml[4], inert = ml[5];
      const V3 com = add(o[l], mul(0.5f * len, d[l]));
      V3 jv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) jv[i] = (i <= l && i < nd) ? cross(a[i], sub(com, o[i])) : v3(0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (i <= l && k <= l) M[i][k] += mass * dot(jv[i], jv[k]) + inert * dot(a[i], a[k]);
      const V3 aq = mul(v[l], a[l]);
      const V3 wl = add(w3, aq);
      const V3 all = add(al, cross(w3, aq));
      const V3 r = sub(com, o[l]);
      const V3 acom = add(add(ao, cross(all, r)), cross(wl, cross(wl, r)));
      const V3 F = mul(mass, sub(acom, g));
      const V3 N = mul(inert, all);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i <= l) c[i] += dot(jv[i], F) + dot(a[i], N);
      const V3 re = mul(2.f, r);  // joint l+1's origin: the link's far end
      ao = add(add(ao, cross(all, re)), cross(wl, cross(wl, re)));
      w3 = wl;
      al = all;
    }
  }
  // Cholesky M = L L^T (packed row-major lower triangle, L[i(i+1)/2 + j])
  float Lp[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) Lp[k] = 0.f;
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < nd) {
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        float s = M[i][j];
#pragma unroll
        for (int k = 0; k < j; ++k) s -= Lp[i * (i + 1) / 2 + k] * Lp[j * (j + 1) / 2 + k];
        if (j == i) {
          ok &= s > 0.f;
          Lp[i * (i + 1) / 2 + i] = sqrtf(fmaxf(s, 0.f));
        } else {
          Lp[i * (i + 1) / 2 + j] = s / Lp[j * (j + 1) / 2 + j];
        }
      }
    }
  }
  if (!ok) atomicOr(err, ERR_ARTICULATION);
  float* Lo = L_out + (size_t)id * 10;
#pragma unroll
  for (int k = 0; k < 10; ++k) Lo[k] = Lp[k];
  float* to = tau_out + (size_t)w * T * nd + t * nd;
  const float* te = tau_ext ? tau_ext + (size_t)w * T * nd + t * nd : nullptr;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (j < nd) to[j] = (te ? te[j] : 0.f) - c[j];
}

// One thread per contact: J rows of its chain sides (side s is chain -(2+t),
// link[2c + s] in [0, nd)) at the contact point, in the [12][n][4] layout;
// rows of free / static sides are left untouched (the step ignores them).
__device__ __forceinline__ void contact_rows(int64_t c, const float* __restrict__ model, int T, int nd,
                                             const float* __restrict__ slab, int slab_stride, int qoff,
                                             int64_t n_worlds, int64_t n, const int64_t* __restrict__ n_dev,
                                             const int32_t* __restrict__ world, const float4* __restrict__ c0,
                                             const int4* __restrict__ c3, const int32_t* __restrict__ link,
                                             float4* __restrict__ jrow, int* __restrict__ err) {
  if (n_dev && c >= *n_dev) return;
  const int4 ids = c3[c];
  const int64_t w = world[c];  // relative to the range's first world, like comfree_step
  const float4 pc = c0[c];
  const V3 p = v3(pc.x, pc.y, pc.z);
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const int id = side ? ids.y : ids.x;
    if (id >= -1) continue;
    const int t = -2 - id;
    const int l = link[2 * c + side];
    if (t >= T || l < 0 || l >= nd || w < 0 || w >= n_worlds) {
      atomicOr(err, ERR_ARTICULATION);
      continue;
    }
    const float* sq = slab + (size_t)w * slab_stride + qoff + t * nd;
    float q[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < nd) q[j] = sq[j];
    V3 a[4], o[4], d[4];
    chain_fk(model + (size_t)t * (3 + 7 * nd), nd, q, a, o, d);
    float rows[6][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool on = i <= l && i < nd;
      const V3 jl = on ? cross(a[i], sub(p, o[i])) : v3(0.f, 0.f, 0.f);
      const V3 ja = on ? a[i] : v3(0.f, 0.f, 0.f);
      rows[0][i] = jl.x; rows[1][i] = jl.y; rows[2][i] = jl.z;
      rows[3][i] = ja.x; rows[4][i] = ja.y; rows[5][i] = ja.z;
    }
#pragma unroll
    for (int r = 0; r < 6; ++r)
      jrow[(size_t)(side * 6 + r) * n + c] = make_float4(rows[r][0], rows[r][1], rows[r][2], rows[r][3]);
  }
}

// One launch: threads [0, W T) build the chains' factors and bias, threads
// [W T, W T + n) the contacts' chain rows (independent: both read q only).
__global__ void k_upstream(const float* __restrict__ model, int T, int nd, const float* __restrict__ slab,
                           int slab_stride, int qoff, int Qp, int64_t n_worlds, const float* __restrict__ tau_ext,
                           float gx, float gy, float gz, float* __restrict__ L_out, float* __restrict__ tau_out,
                           int64_t n, const int64_t* __restrict__ n_dev, const int32_t* __restrict__ world,
                           const float4* __restrict__ c0, const int4* __restrict__ c3, const int32_t* __restrict__ link,
                           float4* __restrict__ jrow, int* __restrict__ err) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = n_worlds * T;
  if (id < nt) {
    chain_dynamics(id, model, T, nd, slab, slab_stride, qoff, Qp, tau_ext, gx, gy, gz, L_out, tau_out, err);
  } else if (id - nt < n) {
    contact_rows(id - nt, model, T, nd, slab, slab_stride, qoff, n_worlds, n, n_dev, world, c0, c3, link, jrow, err);
  }
}

int blocks(int64_t n, int bs) { return (int)((n + bs - 1) / bs); }

}  // namespace

cudaError_t launch_upstream(const float* model, const SceneDev& sc, const float* slab, int64_t n_worlds,
                            const float* tau_ext, const float g[3], float* L_out, float* tau_out, int64_t n,
                            const int64_t* n_dev, const int32_t* world, const float4* c0, const int4* c3,
                            const int32_t* link, float4* jrow, int* err, cudaStream_t s) {
  const int64_t total = n_worlds * sc.T + n;
  if (total == 0) return cudaSuccess;
  k_upstream<<<blocks(total, 128), 128, 0, s>>>(model, sc.T, sc.nd, slab, sc.slab, N_BODY_PLANES * sc.Bp, sc.Qp,
                                                n_worlds, tau_ext, g[0], g[1], g[2], L_out, tau_out, n, n_dev, world,
                                                c0, c3, link, jrow, err);
  return cudaGetLastError();
}

}  // namespace cf
