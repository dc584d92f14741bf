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

enum { G_SPHERE = 0, G_BOX = 1, G_PLANE = 2, G_CAPSULE = 3 };
constexpr int kMaxPairContacts = 16;  // box-box vertex-face: 8 corners each way

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

// Geom frame from the frame pass (one evaluation per (world, geom) instead of
// one per candidate pair and pass).
__device__ __forceinline__ Frame load_frame(const CollideParams& P, int g, int64_t w) {
  const float4* f = P.frames + ((size_t)w * P.n_geoms + g) * 3;
  const float4 a = f[0], b = f[1], c = f[2];
  Frame F;
  F.R[0] = a.x; F.R[1] = a.y; F.R[2] = a.z;
  F.R[3] = b.x; F.R[4] = b.y; F.R[5] = b.z;
  F.R[6] = c.x; F.R[7] = c.y; F.R[8] = c.z;
  F.x = v3(a.w, b.w, c.w);
  return F;
}

__device__ __forceinline__ V3 tangent(V3 n) {
  const float s = copysignf(1.f, n.z);
  const float a = -1.f / (s + n.z);
  const float b = n.x * n.y * a;
  return v3(1.f + s * n.x * n.x * a, s * b, -s * n.x);
}

// Contact sink of one pair: EMIT = false only counts (no staging arrays: the
// count pass has no stack frame); EMIT = true stages the records for the writes.
#ifndef CF_COLLIDE_DIRECT
#define CF_COLLIDE_DIRECT 1  // emit writes each record as it is found (no local-memory staging): pile full step 205 -> 196 us
#endif
template <bool EMIT>
struct Out {
  V3 p[EMIT && !CF_COLLIDE_DIRECT ? kMaxPairContacts : 1], n[EMIT && !CF_COLLIDE_DIRECT ? kMaxPairContacts : 1];
  float phi[EMIT && !CF_COLLIDE_DIRECT ? kMaxPairContacts : 1];
  int k;
  const CollideParams* P;
  int64_t base, w;
  int b1, b2, l1, l2;
  __device__ void add(V3 pp, float ph, V3 nn);
};
__device__ __forceinline__ V3 tangent(V3 n);
template <bool EMIT>
__device__ __forceinline__ void Out<EMIT>::add(V3 pp, float ph, V3 nn) {
  if (k < kMaxPairContacts) {
    if (EMIT && CF_COLLIDE_DIRECT) {  // write the record now (no staging)
      const int64_t c = base + k;
      const V3 t1 = tangent(nn);
      P->c0[c] = make_float4(pp.x, pp.y, pp.z, ph);
      P->c1[c] = make_float4(nn.x, nn.y, nn.z, P->mu_t);
      P->c2[c] = make_float4(t1.x, t1.y, t1.z, P->mu_tor);
      P->c3[c] = make_int4(b1, b2, __float_as_int(P->mu_rol), P->condim);
      P->world[c] = (int32_t)w;
      P->link[c] = make_int2(l1, l2);
    } else if (EMIT) {
      p[k] = pp; phi[k] = ph; n[k] = nn;
    }
    ++k;
  }
}

// Capsule segment ends (end -1 first): x -+ half_len * the frame's z axis.
__device__ __forceinline__ void capsule_ends(const CollideParams& P, int g, int64_t w, V3& a, V3& b) {
  const Frame F = load_frame(P, g, w);
  const float hl = P.size[g].y;
  const V3 z = v3(F.R[2], F.R[5], F.R[8]);
  a = sub(F.x, mul(hl, z));
  b = add(F.x, mul(hl, z));
}

__device__ __forceinline__ V3 closest_on_segment(V3 a, V3 b, V3 c) {
  const V3 d = sub(b, a);
  const float t = fminf(fmaxf(dot(sub(c, a), d) / dot(d, d), 0.f), 1.f);
  return add(a, mul(t, d));
}

// Closest points of segments p1-q1 and p2-q2 (Ericson 5.1.9; parallel -> s = 0).
__device__ __forceinline__ void closest_segments(V3 p1, V3 q1, V3 p2, V3 q2, V3& c1, V3& c2) {
  const V3 d1 = sub(q1, p1), d2 = sub(q2, p2), r = sub(p1, p2);
  const float a = dot(d1, d1), e = dot(d2, d2), f = dot(d2, r), c = dot(d1, r), b = dot(d1, d2);
  const float denom = a * e - b * b;
  float s = denom > 1e-12f * a * e ? fminf(fmaxf((b * f - c * e) / denom, 0.f), 1.f) : 0.f;
  float t = (b * s + f) / e;
  if (t < 0.f) { t = 0.f; s = fminf(fmaxf(-c / a, 0.f), 1.f); }
  else if (t > 1.f) { t = 1.f; s = fminf(fmaxf((b - c) / a, 0.f), 1.f); }
  c1 = add(p1, mul(s, d1));
  c2 = add(p2, mul(t, d2));
}

template <class O>
__device__ __forceinline__ void two_spheres(V3 c1, float R1, V3 c2, float R2, float margin, O& o) {
  const V3 d = sub(c2, c1);
  const float dist = sqrtf(dot(d, d));
  const V3 nn = mul(1.f / dist, d);
  const float phi = dist - R1 - R2;
  if (phi < margin) o.add(add(c1, mul(R1 + 0.5f * phi, nn)), phi, nn);
}

// Sphere (centre c, radius R) against a box frame: phi, box-outward normal, box surface point.
__device__ __forceinline__ float sphere_box(V3 c, float R, const Frame& Fb, float4 h4, V3& nbox, V3& qs) {
  const float h[3] = {h4.x, h4.y, h4.z};
  const V3 cl3 = rtmul(Fb.R, sub(c, Fb.x));
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
  nbox = rmul(Fb.R, v3(nl[0], nl[1], nl[2]));
  qs = add(Fb.x, rmul(Fb.R, v3(ql[0], ql[1], ql[2])));
  return dist - R;
}

// Corners of box B against the faces of box A (vertex-face).
template <class O>
__device__ __forceinline__ void box_corners_on(const Frame& A, float4 hA, const Frame& Bf, float4 hB, float margin,
                                               bool flip, O& o) {
  const float ha[3] = {hA.x, hA.y, hA.z};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const V3 sl = v3((k & 1) ? hB.x : -hB.x, (k & 2) ? hB.y : -hB.y, (k & 4) ? hB.z : -hB.z);
    const V3 corner = add(Bf.x, rmul(Bf.R, sl));
    const V3 c3 = rtmul(A.R, sub(corner, A.x));
    const float cl[3] = {c3.x, c3.y, c3.z};
    float ex[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) ex[j] = fabsf(cl[j]) - ha[j];
    int i = 0;
    if (ex[1] > ex[i]) i = 1;
    if (ex[2] > ex[i]) i = 2;
    const float sd = ex[i];
    bool ok = sd < margin;
#pragma unroll
    for (int j = 0; j < 3; ++j) ok &= (j == i) || ex[j] <= 0.f;
    if (ok) {
      float nl[3] = {0.f, 0.f, 0.f};
      nl[i] = cl[i] >= 0.f ? 1.f : -1.f;
      const V3 nn = rmul(A.R, v3(nl[0], nl[1], nl[2]));
      o.add(sub(corner, mul(0.5f * sd, nn)), sd, flip ? mul(-1.f, nn) : nn);
    }
  }
}

// Contacts of pair pi in world w: returns the count; with out != null writes them
// from index `base` on.
template <bool EMIT>
__device__ int pair_contacts(const CollideParams& P, int pi, int64_t w, int64_t base) {
  constexpr bool emit = EMIT;
  const int2 pr = P.pairs[pi];
  const int4 g1 = P.geom[pr.x], g2 = P.geom[pr.y];
  const float margin = P.margin;
  Out<EMIT> o;
  o.k = 0;
  o.P = &P;
  o.base = base;
  o.w = w;
  o.b1 = g1.y;
  o.b2 = g2.y;
  o.l1 = g1.y < -1 ? g1.z : 0;
  o.l2 = g2.y < -1 ? g2.z : 0;
  const int k1 = g1.x, k2 = g2.x;
  if (k1 == G_PLANE) {
    const float4 s1 = P.size[pr.x];
    const V3 pn = v3(s1.x, s1.y, s1.z);
    const float off = P.local[pr.x].x;
    if (k2 == G_CAPSULE) {
      V3 e[2];
      capsule_ends(P, pr.y, w, e[0], e[1]);
      const float R = P.size[pr.y].x;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float phi = dot(pn, e[q]) - off - R;
        if (phi < margin) o.add(sub(e[q], mul(R + 0.5f * phi, pn)), phi, pn);
      }
    } else {
      const Frame F2 = load_frame(P, pr.y, w);
      if (k2 == G_SPHERE) {
        const float R = P.size[pr.y].x;
        const float phi = dot(pn, F2.x) - off - R;
        if (phi < margin) o.add(sub(F2.x, mul(R + 0.5f * phi, pn)), phi, pn);
      } else {  // box: every corner within the margin
        const float4 h = P.size[pr.y];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const V3 sl = v3((k & 1) ? h.x : -h.x, (k & 2) ? h.y : -h.y, (k & 4) ? h.z : -h.z);
          const V3 corner = add(F2.x, rmul(F2.R, sl));
          const float phi = dot(pn, corner) - off;
          if (phi < margin) o.add(sub(corner, mul(0.5f * phi, pn)), phi, pn);
        }
      }
    }
  } else if ((k1 == G_SPHERE || k1 == G_CAPSULE) && (k2 == G_SPHERE || k2 == G_CAPSULE)) {
    const float R1 = P.size[pr.x].x, R2 = P.size[pr.y].x;
    V3 c1, c2;
    if (k1 == G_SPHERE && k2 == G_SPHERE) {
      c1 = load_frame(P, pr.x, w).x;
      c2 = load_frame(P, pr.y, w).x;
    } else if (k1 == G_CAPSULE && k2 == G_CAPSULE) {
      V3 a1, b1, a2, b2;
      capsule_ends(P, pr.x, w, a1, b1);
      capsule_ends(P, pr.y, w, a2, b2);
      closest_segments(a1, b1, a2, b2, c1, c2);
    } else if (k1 == G_CAPSULE) {
      V3 a1, b1;
      capsule_ends(P, pr.x, w, a1, b1);
      c2 = load_frame(P, pr.y, w).x;
      c1 = closest_on_segment(a1, b1, c2);
    } else {
      V3 a2, b2;
      c1 = load_frame(P, pr.x, w).x;
      capsule_ends(P, pr.y, w, a2, b2);
      c2 = closest_on_segment(a2, b2, c1);
    }
    two_spheres(c1, R1, c2, R2, margin, o);
  } else if (k1 == G_BOX && k2 == G_BOX) {
    const Frame A = load_frame(P, pr.x, w), Bf = load_frame(P, pr.y, w);
    const float4 hA = P.size[pr.x], hB = P.size[pr.y];
    box_corners_on(A, hA, Bf, hB, margin, false, o);
    box_corners_on(Bf, hB, A, hA, margin, true, o);
  } else {  // sphere or capsule against a box
    const bool round_first = k1 != G_BOX;
    const int gr = round_first ? pr.x : pr.y, gb = round_first ? pr.y : pr.x;
    const Frame Fb = load_frame(P, gb, w);
    const float R = P.size[gr].x;
    const float4 h4 = P.size[gb];
    V3 e[2];
    int ne = 1;
    if (P.geom[gr].x == G_CAPSULE) { capsule_ends(P, gr, w, e[0], e[1]); ne = 2; }
    else e[0] = load_frame(P, gr, w).x;
    for (int q = 0; q < ne; ++q) {
      V3 nbox, qs;
      const float phi = sphere_box(e[q], R, Fb, h4, nbox, qs);
      if (phi < margin) o.add(mul(0.5f, add(qs, sub(e[q], mul(R, nbox)))), phi, round_first ? mul(-1.f, nbox) : nbox);
    }
  }
  if (emit && !CF_COLLIDE_DIRECT) {
    const int la = g1.y < -1 ? g1.z : 0, lb = g2.y < -1 ? g2.z : 0;
#pragma unroll 1
    for (int k = 0; k < o.k; ++k) {
      const int64_t c = base + k;
      const V3 t1 = tangent(o.n[k]);
      P.c0[c] = make_float4(o.p[k].x, o.p[k].y, o.p[k].z, o.phi[k]);
      P.c1[c] = make_float4(o.n[k].x, o.n[k].y, o.n[k].z, P.mu_t);
      P.c2[c] = make_float4(t1.x, t1.y, t1.z, P.mu_tor);
      P.c3[c] = make_int4(g1.y, g2.y, __float_as_int(P.mu_rol), P.condim);
      P.world[c] = (int32_t)w;  // relative to the range's first world, like comfree_step
      P.link[c] = make_int2(la, lb);
    }
  }
  return o.k;
}

__global__ void k_geom_frames(const __grid_constant__ CollideParams P) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= P.n_worlds * P.n_geoms) return;
  const int64_t w = id / P.n_geoms;
  const int g = (int)(id - w * P.n_geoms);
  const Frame F = geom_frame(P, g, w);
  float4* f = P.frames + (size_t)id * 3;
  f[0] = make_float4(F.R[0], F.R[1], F.R[2], F.x.x);
  f[1] = make_float4(F.R[3], F.R[4], F.R[5], F.x.y);
  f[2] = make_float4(F.R[6], F.R[7], F.R[8], F.x.z);
}

__global__ void k_collide_count(const __grid_constant__ CollideParams P, int32_t* __restrict__ counts) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id == P.n_worlds * P.n_pairs) counts[id] = 0;  // the scan's closing element (total = its prefix)
  if (id >= P.n_worlds * P.n_pairs) return;
  const int64_t w = id / P.n_pairs;
  counts[id] = pair_contacts<false>(P, (int)(id - w * P.n_pairs), w, 0);
}

__global__ void k_collide_emit(const __grid_constant__ CollideParams P, const int32_t* __restrict__ offs,
                               int64_t capacity, int64_t* __restrict__ n_dev, int* __restrict__ err) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n_dev && id == 0) {  // asynchronous mode: the count for the step, overflow latched
    const int64_t np = P.n_worlds * P.n_pairs;
    const int64_t t = offs[np];
    if (t > capacity) {
      atomicOr(err, ERR_CONTACT_CAP);
      // only whole pairs are emitted: the count is the offset of the first pair
      // that does not fit, i.e. the largest offs[k] <= capacity (offs is monotone)
      int64_t lo = 0, hi = np;  // offs[lo] <= capacity < offs[hi]
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (offs[mid] <= capacity) lo = mid; else hi = mid;
      }
      *n_dev = offs[lo];
    } else {
      *n_dev = t;
    }
  }
  if (id >= P.n_worlds * P.n_pairs) return;
  const int64_t w = id / P.n_pairs;
  const int64_t base = offs[id];
  if (offs[id + 1] == base) return;  // the count pass found no contact for this pair
  if (base + kMaxPairContacts > capacity) {  // only the tail can overflow
    const int n = pair_contacts<false>(P, (int)(id - w * P.n_pairs), w, 0);
    if (base + n > capacity) return;
  }
  pair_contacts<true>(P, (int)(id - w * P.n_pairs), w, base);
}

}  // namespace

// counts: [n_worlds * n_pairs + 1] int32 scratch, offs: same size; temp: CUB
// scratch (temp == nullptr queries *temp_bytes).  Writes the total to *total_dev.
cudaError_t collide_frames(const CollideParams& P, cudaStream_t s) {
  const int64_t n = P.n_worlds * P.n_geoms;
  if (n == 0) return cudaSuccess;
  k_geom_frames<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(P);
  return cudaGetLastError();
}

cudaError_t collide_count_scan(const CollideParams& P, int32_t* counts, int32_t* offs, void* temp,
                               size_t* temp_bytes, cudaStream_t s) {
  const int64_t n = P.n_worlds * P.n_pairs;
  if (!temp) return cub::DeviceScan::ExclusiveSum(nullptr, *temp_bytes, counts, offs, (int)(n + 1), s);
  k_collide_count<<<(unsigned)((n + 1 + 127) / 128), 128, 0, s>>>(P, counts);
  return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, counts, offs, (int)(n + 1), s);
}

cudaError_t collide_emit(const CollideParams& P, const int32_t* offs, int64_t capacity, int64_t* n_dev, int* err,
                         cudaStream_t s) {
  const int64_t n = P.n_worlds * P.n_pairs;
  if (n == 0 && !n_dev) return cudaSuccess;
  k_collide_emit<<<(unsigned)((n + 127) / 128 > 0 ? (n + 127) / 128 : 1), 128, 0, s>>>(P, offs, capacity, n_dev, err);
  return cudaGetLastError();
}

}  // namespace cf
