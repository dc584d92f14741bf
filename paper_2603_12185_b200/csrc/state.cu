// state.cu — conversion between the public state layout (world-major AoS,
// include/comfree.h) and the library's per-world planar slab (internal.h):
// one thread per (world, body) / (world, chain DoF).
#include "internal.h"

namespace cf {

__global__ void k_public_to_slab(const float* __restrict__ pos, const float* __restrict__ quat,
                                 const float* __restrict__ vel, const float* __restrict__ omega,
                                 const float* __restrict__ qpos, const float* __restrict__ qvel,
                                 int64_t W, SceneDev sc, float* __restrict__ slab, int64_t repeat) {
  const int64_t per = (int64_t)sc.Bp + sc.Qp;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= W * per) return;
  const int64_t wd = idx / per;       // destination world
  const int64_t w = wd / repeat;      // source world (repeat > 1: broadcast)
  const int i = (int)(idx % per);
  float* S = slab + (size_t)wd * sc.slab;
  const int Bp = sc.Bp;
  if (i < Bp) {
    if (i < sc.B) {
      const size_t b = (size_t)w * sc.B + i;
      S[0 * Bp + i] = pos ? pos[3 * b] : 0.f;
      S[1 * Bp + i] = pos ? pos[3 * b + 1] : 0.f;
      S[2 * Bp + i] = pos ? pos[3 * b + 2] : 0.f;
      S[3 * Bp + i] = quat ? quat[4 * b] : 1.f;
      S[4 * Bp + i] = quat ? quat[4 * b + 1] : 0.f;
      S[5 * Bp + i] = quat ? quat[4 * b + 2] : 0.f;
      S[6 * Bp + i] = quat ? quat[4 * b + 3] : 0.f;
      S[7 * Bp + i] = vel ? vel[3 * b] : 0.f;
      S[8 * Bp + i] = vel ? vel[3 * b + 1] : 0.f;
      S[9 * Bp + i] = vel ? vel[3 * b + 2] : 0.f;
      S[10 * Bp + i] = omega ? omega[3 * b] : 0.f;
      S[11 * Bp + i] = omega ? omega[3 * b + 1] : 0.f;
      S[12 * Bp + i] = omega ? omega[3 * b + 2] : 0.f;
    } else {  // padding bodies: identity, at rest
      for (int k = 0; k < N_BODY_PLANES; ++k) S[k * Bp + i] = (k == PL_QW) ? 1.f : 0.f;
    }
  } else {
    const int j = i - Bp;
    float* qp = S + N_BODY_PLANES * Bp;
    if (j < sc.Q) {
      qp[j] = qpos ? qpos[(size_t)w * sc.Q + j] : 0.f;
      qp[sc.Qp + j] = qvel ? qvel[(size_t)w * sc.Q + j] : 0.f;
    } else {
      qp[j] = 0.f;
      qp[sc.Qp + j] = 0.f;
    }
  }
}

__global__ void k_slab_to_public(const float* __restrict__ slab, int64_t W, SceneDev sc,
                                 float* __restrict__ pos, float* __restrict__ quat, float* __restrict__ vel,
                                 float* __restrict__ omega, float* __restrict__ qpos,
                                 float* __restrict__ qvel) {
  const int64_t per = (int64_t)sc.B + sc.Q;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= W * per) return;
  const int64_t w = idx / per;
  const int i = (int)(idx % per);
  const float* S = slab + (size_t)w * sc.slab;
  const int Bp = sc.Bp;
  if (i < sc.B) {
    const size_t b = (size_t)w * sc.B + i;
    if (pos) { pos[3 * b] = S[i]; pos[3 * b + 1] = S[Bp + i]; pos[3 * b + 2] = S[2 * Bp + i]; }
    if (quat) {
      quat[4 * b] = S[3 * Bp + i]; quat[4 * b + 1] = S[4 * Bp + i];
      quat[4 * b + 2] = S[5 * Bp + i]; quat[4 * b + 3] = S[6 * Bp + i];
    }
    if (vel) { vel[3 * b] = S[7 * Bp + i]; vel[3 * b + 1] = S[8 * Bp + i]; vel[3 * b + 2] = S[9 * Bp + i]; }
    if (omega) {
      omega[3 * b] = S[10 * Bp + i]; omega[3 * b + 1] = S[11 * Bp + i]; omega[3 * b + 2] = S[12 * Bp + i];
    }
  } else {
    const int j = i - sc.B;
    const float* qp = S + N_BODY_PLANES * Bp;
    if (qpos) qpos[(size_t)w * sc.Q + j] = qp[j];
    if (qvel) qvel[(size_t)w * sc.Q + j] = qp[sc.Qp + j];
  }
}

cudaError_t launch_public_to_slab(const float* pos, const float* quat, const float* vel, const float* omega,
                                  const float* qpos, const float* qvel, int64_t W, const SceneDev& sc,
                                  float* slab, cudaStream_t s, int64_t repeat) {
  const int64_t n = W * ((int64_t)sc.Bp + sc.Qp);
  if (n == 0) return cudaSuccess;
  k_public_to_slab<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pos, quat, vel, omega, qpos, qvel, W, sc, slab,
                                                                repeat < 1 ? 1 : repeat);
  return cudaGetLastError();
}

cudaError_t launch_slab_to_public(const float* slab, int64_t W, const SceneDev& sc, float* pos, float* quat,
                                  float* vel, float* omega, float* qpos, float* qvel, cudaStream_t s) {
  const int64_t n = W * ((int64_t)sc.B + sc.Q);
  if (n == 0) return cudaSuccess;
  k_slab_to_public<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(slab, W, sc, pos, quat, vel, omega, qpos, qvel);
  return cudaGetLastError();
}

}  // namespace cf
