// collide.cu — the collision front-end on the GPU:
// primitive narrowphase over a per-scene candidate pair list (the broadphase
// is the list), emitting the step's contact records directly (c0..c3 streams,
// world ids sorted, chain link ids).  Pair types: sphere-sphere, plane-sphere,
// plane-box (every corner within the margin), sphere-box / box-sphere.  Geoms
// sit on free bodies (pose from the state slab), chain links (pose from the
// forward kinematics of the articulation model) or the world.
// Conventions (R16, R25): normal from g1 to g2, phi the signed
// surface distance, contact point the midpoint of the surface points, branch-
// free tangent (Duff et al. 2017).
// Three passes, one thread per (world, pair): count, exclusive scan (CUB),
// emit at the scanned offset -> world-major, pair-ordered, deterministic.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "chain.cuh"
#include "internal.h"

namespace cf {

namespace {

using namespace chain;

enum { G_SPHERE = 0, G_BOX = 1, G_PLANE = 2 };

struct Frame {
  float R[9];
  V3 x;
};

__device__ __forceinline__ V3 rmul(const float R[9], V3 v) {
  return v3(R[0] * v.x + R[1] * v.y + R[2] * v.z, R[3] * v.x + R[4] * v.y + R[5] * v.z,
            R[6] * v.x + R[7] * v.y + R[8] * v.z);
}
__device__ __forceinline__ V3 rtmul(const float R[9], V3 v) {
  return v3(R[0] * v.x + R[3] * v.y + R[6] * v.z, R[1] * v.x + R[4] * v.y + R[7] * v.z,
            R[2] * v.x + R[5] * v.y + R[8] * v.z);
}

// World frame of geom g in world w (slab = world 0 of the range).
__device__ Frame geom_frame(const CollideParams& P, int g, int64_t w) {
  const int4 gi = P.geom[g];
  const float4 lo = P.local[g];
  const V3 loc = v3(lo.x, lo.y, lo.z);
  Frame F;
  if (gi.y >= 0) {  // free body: pose from the slab planes
    const float* sp = P.slab + (size_t)w * P.sc.slab + gi.y;
    const size_t pb = (size_t)P.sc.Bp;
    const V3 x = v3(sp[0], sp[pb], sp[2 * pb]);
    float qw = sp[3 * pb], qx = sp[4 * pb], qy = sp[5 * pb], qz = sp[6 * pb];
    const float qn = rsqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
    qw *= qn; qx *= qn; qy *= qn; qz *= qn;
    const float R[9] = {1.f - 2.f * (qy * qy + qz * qz), 2.f * (qx * qy - qw * qz), 2.f * (qx * qz + qw * qy),
                        2.f * (qx * qy + qw * qz), 1.f - 2.f * (qx * qx + qz * qz), 2.f * (qy * qz - qw * qx),
                        2.f * (qx * qz - qw * qy), 2.f * (qy * qz + qw * qx), 1.f - 2.f * (qx * qx + qy * qy)};
#pragma unroll
    for (int k = 0; k < 9; ++k) F.R[k] = R[k];
    F.x = add(x, rmul(F.R, loc));
  } else if (gi.y == -1) {  // world-fixed
#pragma unroll
    for (int k = 0; k < 9; ++k) F.R[k] = (k % 4 == 0) ? 1.f : 0.f;
    F.x = loc;
  } else {  // chain link
    const int t = -2 - gi.y, nd = P.sc.nd;
    const float* sq = P.slab + (size_t)w * P.sc.slab + N_BODY_PLANES * P.sc.Bp + t * nd;
    float q[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < nd) q[j] = sq[j];
    V3 o;
    chain_link_frame(P.model + (size_t)t * (3 + 7 * nd), nd, q, gi.z, F.R, o);
    F.x = add(o, rmul(F.R, loc));
  }
  return F;
}

__device__ __forceinline__ V3 tangent(V3 n) {
  const float s = copysignf(1.f, n.z);
  const float a = -1.f / (s + n.z);
  const float b = n.x * n.y * a;
  return v3(1.f + s * n.x * n.x * a, s * b, -s * n.x);
}

// Contacts of pair pi in world w: returns the count; with out != null writes them
// from index `base` on.
__device__ int pair_contacts(const CollideParams& P, int pi, int64_t w, int64_t base, bool emit) {
  const int2 pr = P.pairs[pi];
  const int4 g1 = P.geom[pr.x], g2 = P.geom[pr.y];
  const float margin = P.margin;
  V3 pts[8], nrm[8];
  float phis[8];
  int n = 0;
  if (g1.x == G_PLANE) {
    const float4 s1 = P.size[pr.x];
    const V3 pn = v3(s1.x, s1.y, s1.z);
    const float off = P.local[pr.x].x;
    const Frame F2 = geom_frame(P, pr.y, w);
    if (g2.x == G_SPHERE) {
      const float R = P.size[pr.y].x;
      const float phi = dot(pn, F2.x) - off - R;
      if (phi < margin) { pts[n] = sub(F2.x, mul(R + 0.5f * phi, pn)); nrm[n] = pn; phis[n] = phi; ++n; }
    } else if (g2.x == G_BOX) {
      const float4 h = P.size[pr.y];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const V3 sl = v3((k & 1) ? h.x : -h.x, (k & 2) ? h.y : -h.y, (k & 4) ? h.z : -h.z);
        const V3 corner = add(F2.x, rmul(F2.R, sl));
        const float phi = dot(pn, corner) - off;
        if (phi < margin) { pts[n] = sub(corner, mul(0.5f * phi, pn)); nrm[n] = pn; phis[n] = phi; ++n; }
      }
    }
  } else if (g1.x == G_SPHERE && g2.x == G_SPHERE) {
    const Frame F1 = geom_frame(P, pr.x, w), F2 = geom_frame(P, pr.y, w);
    const float R1 = P.size[pr.x].x, R2 = P.size[pr.y].x;
    const V3 d = sub(F2.x, F1.x);
    const float dist = sqrtf(dot(d, d));
    const V3 nn = mul(1.f / dist, d);
    const float phi = dist - R1 - R2;
    if (phi < margin) { pts[n] = add(F1.x, mul(R1 + 0.5f * phi, nn)); nrm[n] = nn; phis[n] = phi; ++n; }
  } else {  // sphere-box or box-sphere
    const bool sphere_first = g1.x == G_SPHERE;
    const int gs = sphere_first ? pr.x : pr.y, gb = sphere_first ? pr.y : pr.x;
    const Frame Fs = geom_frame(P, gs, w), Fb = geom_frame(P, gb, w);
    const float R = P.size[gs].x;
    const float4 h4 = P.size[gb];
    const float h[3] = {h4.x, h4.y, h4.z};
    const V3 cl3 = rtmul(Fb.R, sub(Fs.x, Fb.x));
    const float cl[3] = {cl3.x, cl3.y, cl3.z};
    float ql[3], nl[3] = {0.f, 0.f, 0.f}, dist;
    const bool inside = fabsf(cl[0]) <= h[0] && fabsf(cl[1]) <= h[1] && fabsf(cl[2]) <= h[2];
    if (inside) {
      int i = 0;
      float best = h[0] - fabsf(cl[0]);
#pragma unroll
      for (int k = 1; k < 3; ++k) {
        const float dk = h[k] - fabsf(cl[k]);
        if (dk < best) { best = dk; i = k; }
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) ql[k] = cl[k];
      nl[i] = cl[i] >= 0.f ? 1.f : -1.f;
      ql[i] = nl[i] * h[i];
      dist = -best;
    } else {
      float d2 = 0.f, dd[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        ql[k] = fminf(fmaxf(cl[k], -h[k]), h[k]);
        dd[k] = cl[k] - ql[k];
        d2 += dd[k] * dd[k];
      }
      dist = sqrtf(d2);
#pragma unroll
      for (int k = 0; k < 3; ++k) nl[k] = dd[k] / dist;
    }
    const float phi = dist - R;
    if (phi < margin) {
      const V3 nbox = rmul(Fb.R, v3(nl[0], nl[1], nl[2]));
      const V3 qs = add(Fb.x, rmul(Fb.R, v3(ql[0], ql[1], ql[2])));
      pts[n] = mul(0.5f, add(qs, sub(Fs.x, mul(R, nbox))));
      nrm[n] = sphere_first ? mul(-1.f, nbox) : nbox;
      phis[n] = phi;
      ++n;
    }
  }
  if (emit) {
    const int la = g1.y < -1 ? g1.z : 0, lb = g2.y < -1 ? g2.z : 0;
    for (int k = 0; k < n; ++k) {
      const int64_t c = base + k;
      const V3 t1 = tangent(nrm[k]);
      P.c0[c] = make_float4(pts[k].x, pts[k].y, pts[k].z, phis[k]);
      P.c1[c] = make_float4(nrm[k].x, nrm[k].y, nrm[k].z, P.mu_t);
      P.c2[c] = make_float4(t1.x, t1.y, t1.z, P.mu_tor);
      P.c3[c] = make_int4(g1.y, g2.y, __float_as_int(P.mu_rol), P.condim);
      P.world[c] = (int32_t)w;  // relative to the range's first world, like comfree_step
      P.link[c] = make_int2(la, lb);
    }
  }
  return n;
}

__global__ void k_collide_count(const __grid_constant__ CollideParams P, int32_t* __restrict__ counts) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= P.n_worlds * P.n_pairs) return;
  const int64_t w = id / P.n_pairs;
  counts[id] = pair_contacts(P, (int)(id - w * P.n_pairs), w, 0, false);
}

__global__ void k_collide_emit(const __grid_constant__ CollideParams P, const int32_t* __restrict__ offs,
                               int64_t capacity) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= P.n_worlds * P.n_pairs) return;
  const int64_t w = id / P.n_pairs;
  const int64_t base = offs[id];
  if (base + 8 > capacity) {  // a pair emits at most 8; only the tail can overflow
    const int n = pair_contacts(P, (int)(id - w * P.n_pairs), w, 0, false);
    if (base + n > capacity) return;
  }
  pair_contacts(P, (int)(id - w * P.n_pairs), w, base, true);
}

}  // namespace

// counts: [n_worlds * n_pairs + 1] int32 scratch, offs: same size; temp: CUB
// scratch (temp == nullptr queries *temp_bytes).  Writes the total to *total_dev.
cudaError_t collide_count_scan(const CollideParams& P, int32_t* counts, int32_t* offs, void* temp,
                               size_t* temp_bytes, cudaStream_t s) {
  const int64_t n = P.n_worlds * P.n_pairs;
  if (!temp) return cub::DeviceScan::ExclusiveSum(nullptr, *temp_bytes, counts, offs, (int)(n + 1), s);
  if (n > 0) k_collide_count<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(P, counts);
  cudaMemsetAsync(counts + n, 0, sizeof(int32_t), s);
  return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, counts, offs, (int)(n + 1), s);
}

__global__ void k_store_count(const int32_t* __restrict__ total, int64_t capacity, int64_t* __restrict__ n_dev,
                              int* __restrict__ err) {
  const int64_t t = *total;
  if (t > capacity) atomicOr(err, ERR_CONTACT_CAP);
  *n_dev = t < capacity ? t : capacity;
}

cudaError_t collide_store_count(const int32_t* total, int64_t capacity, int64_t* n_dev, int* err, cudaStream_t s) {
  k_store_count<<<1, 1, 0, s>>>(total, capacity, n_dev, err);
  return cudaGetLastError();
}

cudaError_t collide_emit(const CollideParams& P, const int32_t* offs, int64_t capacity, cudaStream_t s) {
  const int64_t n = P.n_worlds * P.n_pairs;
  if (n == 0) return cudaSuccess;
  k_collide_emit<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(P, offs, capacity);
  return cudaGetLastError();
}

}  // namespace cf
