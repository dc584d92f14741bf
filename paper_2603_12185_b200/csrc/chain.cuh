// chain.cuh — small-vector helpers and forward kinematics of a serial hinge
// chain (comfree_articulation model layout: per chain base[3], then per joint
// axis[3], length, mass, inertia, armature), shared by the articulated
// upstream (articulation.cu) and the collision front-end (collide.cu).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace cf {
namespace chain {

struct V3 {
  float x, y, z;
};
__device__ __forceinline__ V3 v3(float x, float y, float z) { return V3{x, y, z}; }
__device__ __forceinline__ V3 add(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ V3 mul(float s, V3 a) { return v3(s * a.x, s * a.y, s * a.z); }
__device__ __forceinline__ float dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// Forward kinematics of chain t (model in `art`: per chain base[3], then per
// joint axis[3], length, mass, inertia, armature -> 3 + 7 nd floats) at q:
// world joint axes a[j], joint origins o[j], link directions d[j] (link j's +z).
__device__ __forceinline__ void chain_fk(const float* m, int nd, const float q[4], V3 a[4], V3 o[4], V3 d[4]) {
  float R[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
  V3 org = v3(m[0], m[1], m[2]);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j < nd) {
      const float* mj = m + 3 + 7 * j;
      const V3 al = v3(mj[0], mj[1], mj[2]);
      const V3 ax = v3(R[0] * al.x + R[1] * al.y + R[2] * al.z, R[3] * al.x + R[4] * al.y + R[5] * al.z,
                       R[6] * al.x + R[7] * al.y + R[8] * al.z);
      // R <- Rot(ax, q_j) R  (Rodrigues: I + s K + (1 - c) K^2)
      float s, c;
      sincosf(q[j], &s, &c);
      const float oc = 1.f - c;
      const float Q[9] = {c + oc * ax.x * ax.x, oc * ax.x * ax.y - s * ax.z, oc * ax.x * ax.z + s * ax.y,
                          oc * ax.x * ax.y + s * ax.z, c + oc * ax.y * ax.y, oc * ax.y * ax.z - s * ax.x,
                          oc * ax.x * ax.z - s * ax.y, oc * ax.y * ax.z + s * ax.x, c + oc * ax.z * ax.z};
      float N[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) N[3 * r + k] = Q[3 * r] * R[k] + Q[3 * r + 1] * R[3 + k] + Q[3 * r + 2] * R[6 + k];
#pragma unroll
      for (int k = 0; k < 9; ++k) R[k] = N[k];
      a[j] = ax;
      o[j] = org;
      d[j] = v3(R[2], R[5], R[8]);
      org = add(org, mul(mj[3], d[j]));
    }
  }
}


// Frame of link l (rotation R, row-major, and joint-l origin o) at q.
__device__ __forceinline__ void chain_link_frame(const float* m, int nd, const float q[4], int l, float R[9], V3& o) {
  float Rc[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
  V3 org = v3(m[0], m[1], m[2]);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j < nd && j <= l) {
      const float* mj = m + 3 + 7 * j;
      const V3 al = v3(mj[0], mj[1], mj[2]);
      const V3 ax = v3(Rc[0] * al.x + Rc[1] * al.y + Rc[2] * al.z, Rc[3] * al.x + Rc[4] * al.y + Rc[5] * al.z,
                       Rc[6] * al.x + Rc[7] * al.y + Rc[8] * al.z);
      float s, c;
      sincosf(q[j], &s, &c);
      const float oc = 1.f - c;
      const float Q[9] = {c + oc * ax.x * ax.x, oc * ax.x * ax.y - s * ax.z, oc * ax.x * ax.z + s * ax.y,
                          oc * ax.x * ax.y + s * ax.z, c + oc * ax.y * ax.y, oc * ax.y * ax.z - s * ax.x,
                          oc * ax.x * ax.z - s * ax.y, oc * ax.y * ax.z + s * ax.x, c + oc * ax.z * ax.z};
      float N[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) N[3 * r + k] = Q[3 * r] * Rc[k] + Q[3 * r + 1] * Rc[3 + k] + Q[3 * r + 2] * Rc[6 + k];
#pragma unroll
      for (int k = 0; k < 9; ++k) Rc[k] = N[k];
      o = org;
      org = add(org, mul(mj[3], v3(Rc[2], Rc[5], Rc[8])));
    }
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = Rc[k];
}

}  // namespace chain
}  // namespace cf
