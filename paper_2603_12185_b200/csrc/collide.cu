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
#include <algorithm>
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
constexpr int kMaxPairContacts = 17;  // box-box: 8 corners each way + one edge-edge

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

// Geom frame from the world's frame array (3 float4 per geom: the rows of R
// with x in .w): the frame pass's global array, or the broadphase kernel's
// shared-memory copy.
__device__ __forceinline__ Frame load_frame(const float4* Fw, int g) {
  const float4* f = Fw + (size_t)g * 3;
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
  const float a = __fdiv_rn(-1.f, s + n.z);  // IEEE division whatever the file's -prec-div (the fused step repeats it)
  const float b = n.x * n.y * a;
  return v3(1.f + s * n.x * n.x * a, s * b, -s * n.x);
}

// Broadphase staging of one world (global, L2-resident while the world's CTA
// runs): the records found by the single narrowphase pass, in the order they
// were found: s0 = (point, phi), s1 = (normal, tag = candidate << 5 | index in
// the pair); the copy pass places them after the world's offsets are known.
struct Stage {
  float4* s0;
  float4* s1;
  int cap;
  int* count;  // shared-memory slot counter
};

// Contact sink of one pair: counts; with mode 1 (emit) writes each record as
// it is found (no local-memory staging), with mode 2 (stage) appends it to the
// world's staging area.
// The count and the emit passes must find the same contacts bit for bit (the
// emit writes exactly the slots the count reserved): either both run one
// non-inlined pair_contacts with a runtime mode, or (default) both inline it
// from a file compiled without FMA contraction (see CF_NP_INLINE).
// MODE is a compile-time constant at every call site (0 count, 1 emit, 2
// stage), so a sink carries only what its mode uses in registers.
template <int MODE>
struct Out {
  int k;
  const CollideParams* P;
  Stage S;  // by value: no pointer to a local struct (which would live in local memory)
  int64_t base, w;
  int b1, b2, l1, l2, cand;
  __device__ __forceinline__ void add(V3 pp, float ph, V3 nn);
};
__device__ __forceinline__ V3 tangent(V3 n);
template <int MODE>
__device__ __forceinline__ void Out<MODE>::add(V3 pp, float ph, V3 nn) {
  if (k < kMaxPairContacts) {
    if (MODE == 1) {  // write the record now (no staging)
      const int64_t c = base + k;
      const V3 t1 = tangent(nn);
      P->c0[c] = make_float4(pp.x, pp.y, pp.z, ph);
      P->c1[c] = make_float4(nn.x, nn.y, nn.z, P->mu_t);
      P->c2[c] = make_float4(t1.x, t1.y, t1.z, P->mu_tor);
      P->c3[c] = make_int4(b1, b2, __float_as_int(P->mu_rol), P->condim);
      P->world[c] = (int32_t)w;
      P->link[c] = make_int2(l1, l2);
    } else if (MODE == 2) {
      const int slot = atomicAdd(S.count, 1);
      if (slot < S.cap) {
        S.s0[slot] = make_float4(pp.x, pp.y, pp.z, ph);
        S.s1[slot] = make_float4(nn.x, nn.y, nn.z, __int_as_float((cand << 5) | k));
      }
    }
    ++k;
  }
}

// Per-scene geom table the narrowphase reads (global, or the broadphase
// kernel's shared-memory copy): (kind, body, link, -), size, local.
struct GeomTab {
  const int4* geom;
  const float4* size;
  const float4* local;
};

// Capsule segment ends (end -1 first): x -+ half_len * the frame's z axis.
__device__ __forceinline__ void capsule_ends(const GeomTab& T, const float4* Fw, int g, V3& a, V3& b) {
  const Frame F = load_frame(Fw, g);
  const float hl = T.size[g].y;
  const V3 z = v3(F.R[2], F.R[5], F.R[8]);
  a = sub(F.x, mul(hl, z));
  b = add(F.x, mul(hl, z));
}

#ifndef CF_NP_FASTDIV
#define CF_NP_FASTDIV 1  // one reciprocal per normal: 365 -> 331 us fused full step (IEEE divisions are subroutine calls)
#endif
// Quotients of the segment parameters (clamped to [0, 1] afterwards): the
// approximate division (2 ulp) with CF_NP_FASTDIV, IEEE division otherwise.
__device__ __forceinline__ float np_div(float x, float y) {
#if CF_NP_FASTDIV
  return __fdividef(x, y);
#else
  return x / y;
#endif
}

__device__ __forceinline__ V3 closest_on_segment(V3 a, V3 b, V3 c) {
  const V3 d = sub(b, a);
  const float t = fminf(fmaxf(np_div(dot(sub(c, a), d), dot(d, d)), 0.f), 1.f);
  return add(a, mul(t, d));
}

// Closest points of segments p1-q1 and p2-q2 (Ericson 5.1.9; parallel -> s = 0).
__device__ __forceinline__ void closest_segments(V3 p1, V3 q1, V3 p2, V3 q2, V3& c1, V3& c2) {
  const V3 d1 = sub(q1, p1), d2 = sub(q2, p2), r = sub(p1, p2);
  const float a = dot(d1, d1), e = dot(d2, d2), f = dot(d2, r), c = dot(d1, r), b = dot(d1, d2);
  const float denom = a * e - b * b;
  float s = denom > 1e-12f * a * e ? fminf(fmaxf(np_div(b * f - c * e, denom), 0.f), 1.f) : 0.f;
  float t = np_div(b * s + f, e);
  if (t < 0.f) { t = 0.f; s = fminf(fmaxf(np_div(-c, a), 0.f), 1.f); }
  else if (t > 1.f) { t = 1.f; s = fminf(fmaxf(np_div(b - c, a), 0.f), 1.f); }
  c1 = add(p1, mul(s, d1));
  c2 = add(p2, mul(t, d2));
}

template <class O>
__device__ __forceinline__ void two_spheres(V3 c1, float R1, V3 c2, float R2, float margin, O& o) {
  const V3 d = sub(c2, c1);
#if CF_NP_FASTDIV
  const float d2 = dot(d, d), idist = rsqrtf(d2), dist = d2 * idist;
  const V3 nn = mul(idist, d);
#else
  const float dist = sqrtf(dot(d, d));
  const V3 nn = mul(1.f / dist, d);
#endif
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
  if (inside) {  // per-component selects (no dynamic index: the arrays stay in registers)
    int i = 0;
    float best = h[0] - fabsf(cl[0]);
#pragma unroll
    for (int k = 1; k < 3; ++k) {
      const float dk = h[k] - fabsf(cl[k]);
      if (dk < best) { best = dk; i = k; }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      nl[k] = k == i ? (cl[k] >= 0.f ? 1.f : -1.f) : 0.f;
      ql[k] = k == i ? nl[k] * h[k] : cl[k];
    }
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
#if CF_NP_FASTDIV
    const float idist = 1.f / dist;  // one division for the three components
#pragma unroll
    for (int k = 0; k < 3; ++k) nl[k] = dd[k] * idist;
#else
#pragma unroll
    for (int k = 0; k < 3; ++k) nl[k] = dd[k] / dist;
#endif
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
    // largest excess (first of equals), by selects (no dynamic index)
    int i = 0;
    float sd = ex[0];
    if (ex[1] > sd) { i = 1; sd = ex[1]; }
    if (ex[2] > sd) { i = 2; sd = ex[2]; }
    bool ok = sd < margin;
#pragma unroll
    for (int j = 0; j < 3; ++j) ok &= (j == i) || ex[j] <= 0.f;
    if (ok) {
      float nl[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) nl[j] = j == i ? (cl[j] >= 0.f ? 1.f : -1.f) : 0.f;
      const V3 nn = rmul(A.R, v3(nl[0], nl[1], nl[2]));
      o.add(sub(corner, mul(0.5f * sd, nn)), sd, flip ? mul(-1.f, nn) : nn);
    }
  }
}

#ifndef CF_BP_SAT1
#define CF_BP_SAT1 1  // face-axis early out, corners, then the 15 axes for the edge contact: 446 vs 467 us full step (profiles/r02_broadphase.txt)
#endif
// Exact early out over the 6 face axes only (CF_BP_SAT1 variant).
__device__ __forceinline__ bool boxes_separated(const Frame& A, float4 hA4, const Frame& Bf, float4 hB4, float margin) {
  const V3 d = sub(Bf.x, A.x);
  const float hA[3] = {hA4.x, hA4.y, hA4.z}, hB[3] = {hB4.x, hB4.y, hB4.z};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const V3 L = k < 3 ? v3(A.R[k], A.R[3 + k], A.R[6 + k]) : v3(Bf.R[k - 3], Bf.R[k], Bf.R[k + 3]);
    float r = -fabsf(dot(L, d));
#pragma unroll
    for (int m = 0; m < 3; ++m)
      r += hA[m] * fabsf(L.x * A.R[m] + L.y * A.R[3 + m] + L.z * A.R[6 + m]) +
           hB[m] * fabsf(L.x * Bf.R[m] + L.y * Bf.R[3 + m] + L.z * Bf.R[6 + m]);
    if (r < -margin) return true;
  }
  return false;
}

// Box-box separating-axis test (reading R33's 15 axes: face normals of A, of
// B, then the 9 edge cross products e_A,i x e_B,j, i-major, skipped when
// |cross| <= 1e-6), overlap(L) = sum_k hA_k |L.eA_k| + hB_k |L.eB_k| - |L.d|.
// Returns false when some axis separates the boxes by more than the margin:
// then no corner is within the margin of a face either (a corner within the
// margin of a face, projected inside it, is within the margin of the box), so
// the pair has no contact at all.  Otherwise best / bi, bj / bL hold the
// first minimum overlap and its axis (bi = -1: a face axis).
struct BoxSat {
  float best;
  int bi, bj;
  V3 bL;
};
__device__ __forceinline__ bool box_sat(const Frame& A, float4 hA4, const Frame& Bf, float4 hB4, float margin,
                                        BoxSat& S) {
  const float hA[3] = {hA4.x, hA4.y, hA4.z}, hB[3] = {hB4.x, hB4.y, hB4.z};
  const V3 d = sub(Bf.x, A.x);
  V3 ea[3], eb[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ea[k] = v3(A.R[k], A.R[3 + k], A.R[6 + k]);    // column k of R: the frame's axis k
    eb[k] = v3(Bf.R[k], Bf.R[3 + k], Bf.R[6 + k]);
  }
  auto overlap = [&](V3 L) {
    float r = -fabsf(dot(L, d));
#pragma unroll
    for (int k = 0; k < 3; ++k) r += hA[k] * fabsf(dot(L, ea[k])) + hB[k] * fabsf(dot(L, eb[k]));
    return r;
  };
  S.best = INFINITY;
  S.bi = -1;
  S.bj = -1;
  S.bL = v3(0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const float ov = overlap(k < 3 ? ea[k] : eb[k - 3]);
    if (ov < -margin) return false;
    if (ov < S.best) S.best = ov;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {  // unrolled: ea / eb stay in registers
      V3 L = cross(ea[i], eb[j]);
#if CF_NP_FASTDIV
      const float l2 = dot(L, L);
      if (!(l2 > 1e-12f)) continue;  // |cross| <= 1e-6 (R33)
      L = mul(rsqrtf(l2), L);
#else
      const float nl = sqrtf(dot(L, L));
      if (!(nl > 1e-6f)) continue;
      L = mul(1.f / nl, L);
#endif
      const float ov = overlap(L);
      if (ov < -margin) return false;
      if (ov < S.best) { S.best = ov; S.bi = i; S.bj = j; S.bL = L; }
    }
  }
  return true;
}

// Box-box edge-edge contact (reading R33): when the first axis of minimum
// overlap is an edge axis and -overlap < margin, one contact at the midpoint
// of the closest points of A's edge through its support point along n and
// B's through its support point along -n (n oriented from A to B).
template <class O>
__device__ __forceinline__ void box_edge_edge(const Frame& A, float4 hA4, const Frame& Bf, float4 hB4, float margin,
                                              const BoxSat& S, O& o) {
  if (S.bi < 0 || !(-S.best < margin)) return;
  const float hA[3] = {hA4.x, hA4.y, hA4.z}, hB[3] = {hB4.x, hB4.y, hB4.z};
  const V3 d = sub(Bf.x, A.x);
  V3 ea[3], eb[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ea[k] = v3(A.R[k], A.R[3 + k], A.R[6 + k]);
    eb[k] = v3(Bf.R[k], Bf.R[3 + k], Bf.R[6 + k]);
  }
  const int bi = S.bi, bj = S.bj;
  const V3 n = dot(S.bL, d) >= 0.f ? S.bL : mul(-1.f, S.bL);
  // the edges' axes and half lengths by selects (no dynamic index)
  const V3 eai = bi == 0 ? ea[0] : (bi == 1 ? ea[1] : ea[2]), ebj = bj == 0 ? eb[0] : (bj == 1 ? eb[1] : eb[2]);
  const float hai = bi == 0 ? hA[0] : (bi == 1 ? hA[1] : hA[2]), hbj = bj == 0 ? hB[0] : (bj == 1 ? hB[1] : hB[2]);
  V3 pa = A.x, pb = Bf.x;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (k != bi) pa = add(pa, mul((dot(n, ea[k]) >= 0.f ? 1.f : -1.f) * hA[k], ea[k]));
    if (k != bj) pb = sub(pb, mul((dot(n, eb[k]) >= 0.f ? 1.f : -1.f) * hB[k], eb[k]));
  }
  V3 c1, c2;
  closest_segments(sub(pa, mul(hai, eai)), add(pa, mul(hai, eai)), sub(pb, mul(hbj, ebj)), add(pb, mul(hbj, ebj)), c1, c2);
  o.add(mul(0.5f, add(c1, c2)), -S.best, n);
}

// Contacts of the geom pair pr = (g1, g2) in world w (frames Fw): returns the
// count; EMIT writes them from record `base` on.
// CF_NP_INLINE: the count and emit specialisations inlined instead, which is
// only safe because collide.cu is compiled without FMA contraction
// (-fmad=false, build.py): every floating-point operation is then one IEEE
// operation in source order in both specialisations, so they agree bit for bit.
#ifndef CF_NP_INLINE
#define CF_NP_INLINE 1
#endif
#if CF_NP_INLINE
#define CF_NP_ATTR __forceinline__
#else
#define CF_NP_ATTR __noinline__
#endif
template <int MODE>
__device__ CF_NP_ATTR int pair_contacts_rt(const CollideParams& P, const GeomTab T, const int2 pr, const float4* Fw,
                                             int64_t w, int64_t base, const Stage S = Stage{}, int cand = 0) {
  const int4 g1 = T.geom[pr.x], g2 = T.geom[pr.y];
  const float margin = P.margin;
  Out<MODE> o;
  o.k = 0;
  o.P = &P;
  o.S = S;
  o.cand = cand;
  o.base = base;
  o.w = w;
  o.b1 = g1.y;
  o.b2 = g2.y;
  o.l1 = g1.y < -1 ? g1.z : 0;
  o.l2 = g2.y < -1 ? g2.z : 0;
  const int k1 = g1.x, k2 = g2.x;
  if (k1 == G_PLANE) {
    const float4 s1 = T.size[pr.x];
    const V3 pn = v3(s1.x, s1.y, s1.z);
    const float off = T.local[pr.x].x;
    if (k2 == G_CAPSULE) {
      V3 e[2];
      capsule_ends(T, Fw, pr.y, e[0], e[1]);
      const float R = T.size[pr.y].x;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float phi = dot(pn, e[q]) - off - R;
        if (phi < margin) o.add(sub(e[q], mul(R + 0.5f * phi, pn)), phi, pn);
      }
    } else {
      const Frame F2 = load_frame(Fw, pr.y);
      if (k2 == G_SPHERE) {
        const float R = T.size[pr.y].x;
        const float phi = dot(pn, F2.x) - off - R;
        if (phi < margin) o.add(sub(F2.x, mul(R + 0.5f * phi, pn)), phi, pn);
      } else {  // box: every corner within the margin
        const float4 h = T.size[pr.y];
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
    const float R1 = T.size[pr.x].x, R2 = T.size[pr.y].x;
    V3 c1, c2;
    if (k1 == G_SPHERE && k2 == G_SPHERE) {
      c1 = load_frame(Fw, pr.x).x;
      c2 = load_frame(Fw, pr.y).x;
    } else if (k1 == G_CAPSULE && k2 == G_CAPSULE) {
      V3 a1, b1, a2, b2;
      capsule_ends(T, Fw, pr.x, a1, b1);
      capsule_ends(T, Fw, pr.y, a2, b2);
      closest_segments(a1, b1, a2, b2, c1, c2);
    } else if (k1 == G_CAPSULE) {
      V3 a1, b1;
      capsule_ends(T, Fw, pr.x, a1, b1);
      c2 = load_frame(Fw, pr.y).x;
      c1 = closest_on_segment(a1, b1, c2);
    } else {
      V3 a2, b2;
      c1 = load_frame(Fw, pr.x).x;
      capsule_ends(T, Fw, pr.y, a2, b2);
      c2 = closest_on_segment(a2, b2, c1);
    }
    two_spheres(c1, R1, c2, R2, margin, o);
  } else if (k1 == G_BOX && k2 == G_BOX) {
    const Frame A = load_frame(Fw, pr.x), Bf = load_frame(Fw, pr.y);
    const float4 hA = T.size[pr.x], hB = T.size[pr.y];
    BoxSat S;
#if CF_BP_SAT1
    if (boxes_separated(A, hA, Bf, hB, margin)) return 0;  // no vertex-face nor edge-edge contact
    box_corners_on(A, hA, Bf, hB, margin, false, o);
    box_corners_on(Bf, hB, A, hA, margin, true, o);
    if (!box_sat(A, hA, Bf, hB, margin, S)) return o.k;
    box_edge_edge(A, hA, Bf, hB, margin, S, o);
    return o.k;
#endif
    if (!box_sat(A, hA, Bf, hB, margin, S)) return 0;  // separated beyond the margin: no contact of any kind
    box_corners_on(A, hA, Bf, hB, margin, false, o);
    box_corners_on(Bf, hB, A, hA, margin, true, o);
    box_edge_edge(A, hA, Bf, hB, margin, S, o);
  } else {  // sphere or capsule against a box
    const bool round_first = k1 != G_BOX;
    const int gr = round_first ? pr.x : pr.y, gb = round_first ? pr.y : pr.x;
    const Frame Fb = load_frame(Fw, gb);
    const float R = T.size[gr].x;
    const float4 h4 = T.size[gb];
    V3 e[3];
    int ne = 1;
    if (T.geom[gr].x == G_CAPSULE) {
      capsule_ends(T, Fw, gr, e[0], e[1]);
      ne = 2;
      // reading R34: the segment point nearest the box centre as a third sphere
      // when strictly inside the segment (a capsule lying across a box)
      const V3 d = sub(e[1], e[0]);
      const float t = np_div(dot(sub(Fb.x, e[0]), d), dot(d, d));
      e[2] = add(e[0], mul(t, d));
      if (t > 0.f && t < 1.f) ne = 3;
    } else {
      e[0] = load_frame(Fw, gr).x;
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {  // unrolled with a predicate: e[] stays in registers
      if (q < ne) {
        V3 nbox, qs;
        const float phi = sphere_box(e[q], R, Fb, h4, nbox, qs);
        if (phi < margin) o.add(mul(0.5f, add(qs, sub(e[q], mul(R, nbox)))), phi, round_first ? mul(-1.f, nbox) : nbox);
      }
    }
  }
  return o.k;
}

template <bool EMIT>
__device__ __forceinline__ int pair_contacts(const CollideParams& P, const int2 pr, const float4* Fw, int64_t w,
                                             int64_t base, const GeomTab* T = nullptr) {
  return pair_contacts_rt<EMIT ? 1 : 0>(P, T ? *T : GeomTab{P.geom, P.size, P.local}, pr, Fw, w, base);
}

// the broadphase's single pass: count and stage the records of candidate `cand`
__device__ __forceinline__ int pair_contacts_stage(const CollideParams& P, const int2 pr, const float4* Fw, int64_t w,
                                                   const GeomTab* T, const Stage S, int cand) {
  return pair_contacts_rt<2>(P, *T, pr, Fw, w, 0, S, cand);
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
  counts[id] = pair_contacts<false>(P, P.pairs[id - w * P.n_pairs], P.frames + (size_t)w * P.n_geoms * 3, w, 0);
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
  const int2 pr = P.pairs[id - w * P.n_pairs];
  const float4* Fw = P.frames + (size_t)w * P.n_geoms * 3;
  if (base + kMaxPairContacts > capacity) {  // only the tail can overflow
    const int n = pair_contacts<false>(P, pr, Fw, w, 0);
    if (base + n > capacity) return;
  }
  pair_contacts<true>(P, pr, Fw, w, base);
}

// ---------------------------------------------------------------- broadphase
// Geometry without a candidate list (reading R32): one CTA per world finds the
// world's candidate pairs and emits their contacts, in one launch:
//   1  geom frames (thread per geom) and AABBs grown by margin/2, in shared memory;
//   2  sort-and-sweep: the non-plane geoms sorted by their AABB's low end along
//      the axis of largest spread (bitonic sort), each swept forward while the
//      next low end is within its high end, the other two axes and the grown
//      bounding spheres tested (lane per sorted position, a counting and a
//      placing pass); a pair goes to the bucket of its lower geom id; plane g1 takes every geom whose
//      AABB reaches below offset + margin/2 (bucket order = geom order, by a
//      block scan); each bucket sorted -> candidates in (g1, g2) order, the
//      order reading R32 defines;
//   3  narrowphase count per candidate, block scan -> offsets in the world;
//   4  the world's base offset by a chained scan over worlds (decoupled
//      look-back on per-world status words; worlds are taken in launch order
//      from a ticket counter, so a CTA only waits on running CTAs);
//   5  narrowphase again for candidates with contacts, records written at
//      base + offset: world-major, (g1, g2)-ordered, deterministic.
// The last CTA to finish stores the device count (the offset of the first pair
// that did not fit when the capacity is exceeded) and resets the counters.
#ifndef CF_BP_THREADS
#define CF_BP_THREADS 512  // 16 warps, 2 CTAs per SM: 0.83 vs 0.91 ms collide at 256 (profiles/r02_broadphase.txt)
#endif
constexpr int kBpThreads = CF_BP_THREADS;
#ifndef CF_BP_TILE_BRANCHY
#define CF_BP_TILE_BRANCHY 2  // 2: groups of 8 loads (362 vs 365 us full step), 1: per-test predicated loads, 0: all 32 unconditional
#endif
#ifdef CF_BP_TIMELINE  // tuning diagnostic: per-world phase timestamps (globaltimer ns) into P.frames
#define BP_MARK(k)                                                                        \
  if (tid == 0) {                                                                         \
    unsigned long long t_;                                                                \
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                                 \
    reinterpret_cast<unsigned long long*>(P.frames)[w * 16 + (k)] = t_;                    \
  }
#else
#define BP_MARK(k)
#endif

#ifndef CF_BP_PUB
#define CF_BP_PUB 4
#endif
// L2 load of a record this CTA staged earlier (cache-global: not from L1)
__device__ __forceinline__ float4 ld_cg4(const float4* p) {
  float4 r;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t f2key(float f) {  // order-preserving float -> uint32
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// exclusive block scan of v over kBpThreads threads; returns the prefix, *tot the sum
__device__ __forceinline__ int block_exclusive(int v, int* tmp, int* tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = lane < kBpThreads / 32 ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    tmp[lane] = t;  // inclusive sums of the warps
  }
  __syncthreads();
  const int before = wid ? tmp[wid - 1] : 0;
  *tot = tmp[kBpThreads / 32 - 1];
  __syncthreads();
  return before + x - v;
}

// Chained-scan status words (one per world): bits 62-63 flag (1 the world's
// total is published; 2 an inclusive prefix, the virtual word before world 0),
// bit 61 "records already written" (the staging fallback), low 61 bits the value.
constexpr int kGsumShift = 8;  // worlds per group sum: 256
constexpr unsigned long long kStAgg = 1ull << 62, kStInc = 2ull << 62, kStDone = 1ull << 61,
                             kStVal = (1ull << 61) - 1;

// Sum of the totals of worlds [0, w), one warp: 32 status words per round,
// walking back to the nearest inclusive prefix; re-reads a round while a world
// before that prefix has not published its total yet.
__device__ __forceinline__ long long lookback_warp(unsigned long long* status, int64_t w, int lane) {
  const unsigned full = 0xffffffffu;
  const volatile unsigned long long* st = status;
  long long prefix = 0;
  for (int64_t j = w - 1; j >= 0;) {
    const int64_t jj = j - lane;
    const unsigned long long v = jj >= 0 ? st[jj] : kStInc;  // before world 0: an inclusive 0
    const unsigned f = (unsigned)(v >> 62);
    const unsigned inc = __ballot_sync(full, f == 2);
    const unsigned upto = inc ? ((inc & (0u - inc)) << 1) - 1u : full;  // lanes up to the nearest inclusive
    if (__ballot_sync(full, f == 0) & upto) continue;                   // a total still missing: re-read
    long long x = ((upto >> lane) & 1u) ? (long long)(v & kStVal) : 0ll;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(full, x, o);
    prefix += x;
    if (inc) break;
    j -= 32;
  }
  return prefix;
}

struct BpParams {
  int cap_c;                       // candidate capacity per world (shared memory)
  int np2;                         // power of two >= non-plane geoms
  int64_t capacity;                // output records
  unsigned long long* status;      // [n_worlds] chained-scan words (zeroed before the launch)
  int* queue;                      // [0] world ticket, [2..3] cut (int64), [4] emit ticket, [5] emit CTAs done
  int64_t* n_dev;                  // device count out (whole pairs within the capacity)
  int64_t* total;                  // all contacts of the launch (or null)
  int* err;
  float4* stage;                   // [n_worlds][4][stage_cap]: staged records (found order), placed records
  int stage_cap;                   // records per world (a world with more runs the narrowphase twice)
  unsigned long long* gsum;        // [ceil(n_worlds / 256)] totals of groups of worlds (zeroed before the launch)
  int64_t* fbase;                  // [n_worlds] or null: base offset of a world written in place (the fused step reads it)
};

__global__ void __launch_bounds__(kBpThreads, 2) k_collide_bp(const __grid_constant__ CollideParams P,
                                                              const __grid_constant__ BpParams Q) {
  extern __shared__ float4 bsm[];
  __shared__ int s_tmp[32];
  __shared__ int s_misc[8];
  const int G = P.n_geoms, tid = threadIdx.x;
  float4* Fw = bsm;                                                   // [3 G]
  float4* lo = Fw + 3 * G;                                            // [G] (.w: 1 = plane)
  float4* hi = lo + G;                                                // [G]
  uint32_t* list = reinterpret_cast<uint32_t*>(hi + G);               // [cap_c] (g1 << 16) | g2
  // list is dead until the bucket placement: it holds the sort's exchange
  // buffer and then the sweep's sorted cross-axis extents (collide_bp_min_cap)
  uint32_t* key = list + Q.cap_c;                                     // [np2]
  uint32_t* val = key + Q.np2;                                        // [np2]
  int* gbody = reinterpret_cast<int*>(val + Q.np2);                   // [G] body of each geom
  int* cnt = gbody + G;                                               // [G + 1]
  int* start = cnt + G + 1;                                           // [G + 1]
  int* ncon = start + G + 1;                                          // [cap_c]
  uint16_t* perm = reinterpret_cast<uint16_t*>(ncon + Q.cap_c);      // [cap_c] evaluation order
  if (tid == 0) s_misc[0] = atomicAdd(&Q.queue[0], 1);
  __syncthreads();
  const int64_t w = s_misc[0];
  const float hm = 0.5f * P.margin;

  BP_MARK(0);
  // 1: frames and grown AABBs
  for (int g = tid; g < G; g += kBpThreads) {
    const Frame F = geom_frame(P, g, w);
    Fw[3 * g] = make_float4(F.R[0], F.R[1], F.R[2], F.x.x);
    Fw[3 * g + 1] = make_float4(F.R[3], F.R[4], F.R[5], F.x.y);
    Fw[3 * g + 2] = make_float4(F.R[6], F.R[7], F.R[8], F.x.z);
    const int kind = P.geom[g].x;
    gbody[g] = P.geom[g].y;
    const float4 sz = P.size[g];
    V3 l = F.x, h = F.x;
    if (kind == G_SPHERE) {
      l = sub(F.x, v3(sz.x, sz.x, sz.x));
      h = add(F.x, v3(sz.x, sz.x, sz.x));
    } else if (kind == G_BOX) {
      const V3 e = v3(fabsf(F.R[0]) * sz.x + fabsf(F.R[1]) * sz.y + fabsf(F.R[2]) * sz.z,
                      fabsf(F.R[3]) * sz.x + fabsf(F.R[4]) * sz.y + fabsf(F.R[5]) * sz.z,
                      fabsf(F.R[6]) * sz.x + fabsf(F.R[7]) * sz.y + fabsf(F.R[8]) * sz.z);
      l = sub(F.x, e);
      h = add(F.x, e);
    } else if (kind == G_CAPSULE) {
      const V3 z = v3(F.R[2], F.R[5], F.R[8]);
      const V3 a = sub(F.x, mul(sz.y, z)), b = add(F.x, mul(sz.y, z));
      l = sub(v3(fminf(a.x, b.x), fminf(a.y, b.y), fminf(a.z, b.z)), v3(sz.x, sz.x, sz.x));
      h = add(v3(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fmaxf(a.z, b.z)), v3(sz.x, sz.x, sz.x));
    }
    // bounding-sphere radius about the frame origin (sphere R, box |h|,
    // capsule R + half length) grown by margin/2, with fp32 slack for the
    // AABB-centre round-off (the test must never reject a contact pair)
    const float rb = kind == G_SPHERE ? sz.x
                   : kind == G_BOX    ? sqrtf(sz.x * sz.x + sz.y * sz.y + sz.z * sz.z)
                   : kind == G_CAPSULE ? sz.x + sz.y : INFINITY;
    lo[g] = make_float4(l.x - hm, l.y - hm, l.z - hm, kind == G_PLANE ? 1.f : 0.f);
    hi[g] = make_float4(h.x + hm, h.y + hm, h.z + hm, (rb + hm) * 1.001f + 1e-6f);
  }
  for (int g = tid; g <= G; g += kBpThreads) cnt[g] = 0;
  __syncthreads();
  // sweep axis: the largest spread of the non-plane AABB centres (block reduction)
  {
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int g = tid; g < G; g += kBpThreads) {
      if (lo[g].w != 0.f) continue;
      const float c[3] = {lo[g].x + hi[g].x, lo[g].y + hi[g].y, lo[g].z + hi[g].z};
#pragma unroll
      for (int k = 0; k < 3; ++k) { mn[k] = fminf(mn[k], c[k]); mx[k] = fmaxf(mx[k], c[k]); }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      for (int o = 16; o > 0; o >>= 1) {
        mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
        mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
      }
    }
    __shared__ float red[6 * (kBpThreads / 32)];
    if ((tid & 31) == 0)
      for (int k = 0; k < 3; ++k) { red[(tid >> 5) * 6 + k] = mn[k]; red[(tid >> 5) * 6 + 3 + k] = mx[k]; }
    __syncthreads();
    if (tid == 0) {
      float a[3] = {INFINITY, INFINITY, INFINITY}, b[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int q = 0; q < kBpThreads / 32; ++q)
        for (int k = 0; k < 3; ++k) { a[k] = fminf(a[k], red[q * 6 + k]); b[k] = fmaxf(b[k], red[q * 6 + 3 + k]); }
      int ax = 0;
      for (int k = 1; k < 3; ++k)
        if (b[k] - a[k] > b[ax] - a[ax]) ax = k;
      s_misc[1] = ax;
    }
    __syncthreads();
  }
  const int ax = s_misc[1];
  BP_MARK(1);
  // 2a: bitonic sort of (low end along ax, geom) over the non-plane geoms
  for (int i = tid; i < Q.np2; i += kBpThreads) {
    const bool real = i < G && lo[i].w == 0.f;
    key[i] = real ? f2key(ax == 0 ? lo[i].x : (ax == 1 ? lo[i].y : lo[i].z)) : 0xffffffffu;
    val[i] = real ? (uint32_t)i : 0xffffffffu;
  }
  __syncthreads();
  if (Q.np2 <= kBpThreads) {
    // one element per thread (threads >= np2 idle along): the network's
    // stages with partner distance j < 32 are register shuffles, the others
    // one exchange through a double-buffered shared array
    const int n2 = Q.np2;
    uint64_t x = tid < n2 ? (((uint64_t)key[tid] << 32) | val[tid]) : ~0ull;
    uint64_t* xb = reinterpret_cast<uint64_t*>(list);  // 2 x np2 (list's storage, dead here)
    int buf = 0;
#if CF_BP_SORT_OLD
#pragma unroll 1
    for (int k = 2; k <= n2; k <<= 1) {
#pragma unroll 1
      for (int j = k >> 1; j > 0; j >>= 1) {
        uint64_t y;
        if (j >= 32) {
          if (tid < n2) xb[buf * n2 + tid] = x;
          __syncthreads();
          y = tid < n2 ? xb[buf * n2 + (tid ^ j)] : x;
          buf ^= 1;
        } else {
          y = __shfl_xor_sync(0xffffffffu, x, j);
        }
        const bool keep_min = ((tid & k) == 0) == ((tid & j) == 0);
        x = keep_min ? (x < y ? x : y) : (x < y ? y : x);
      }
    }
#else
#pragma unroll 1
    for (int k = 2; k <= n2; k <<= 1) {
      const bool up = (tid & k) == 0;
#pragma unroll 1
      for (int j = k >> 1; j >= 32; j >>= 1) {
        if (tid < n2) xb[buf * n2 + tid] = x;
        __syncthreads();
        const uint64_t y = tid < n2 ? xb[buf * n2 + (tid ^ j)] : x;
        buf ^= 1;
        const bool keep_min = up == ((tid & j) == 0);
        x = (keep_min == (y < x)) ? y : x;
      }
#pragma unroll
      for (int j = 16; j > 0; j >>= 1) {  // compile-time partner distances
        if (j < k) {
          const uint64_t y = __shfl_xor_sync(0xffffffffu, x, j);
          const bool keep_min = up == ((tid & j) == 0);
          x = (keep_min == (y < x)) ? y : x;
        }
      }
    }
#endif
    __syncthreads();
    if (tid < Q.np2) {
      key[tid] = (uint32_t)(x >> 32);
      val[tid] = (uint32_t)x;
    }
  } else {
  for (int k = 2; k <= Q.np2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < (Q.np2 >> 1); t += kBpThreads) {
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));  // lower index of the pair
        const int l = i | j;
        const bool up = (i & k) == 0;
        const uint64_t a = ((uint64_t)key[i] << 32) | val[i], b = ((uint64_t)key[l] << 32) | val[l];
        if ((a > b) == up) { key[i] = (uint32_t)(b >> 32); val[i] = (uint32_t)b; key[l] = (uint32_t)(a >> 32); val[l] = (uint32_t)a; }
      }
      __syncthreads();
    }
  }
  }
  BP_MARK(2);
  // 2b: sort-and-sweep.  The walk of sorted position i is (i, e_i], the
  // positions whose low end is within i's high end along the sweep axis (the
  // sweep axis needs no test inside it: lo_i <= lo_j <= hi_i); the walks are
  // cut into tiles of 32 tests, a thread tests a whole tile (one sorted
  // cross-axis float4 per test, unrolled) into a hit mask.  A test that
  // overlaps on the two other axes is an AABB hit, appended as the sorted
  // positions (i << 16 | j) with one list atomic per warp.  The hits are then
  // filtered by the grown bounding spheres (centre distance <= rho_i + rho_j:
  // conservative, no pair closer than the margin fails it, R32) and by the
  // owning body, counted per bucket (the lower geom id) and placed.
  auto axis_of = [&](const float4& v) { return ax == 0 ? v.x : (ax == 1 ? v.y : v.z); };
  auto plane_hit = [&](int p, int g) {  // g's grown AABB reaches below offset + margin/2
    const float4 n = P.size[p], lg = lo[g], hg = hi[g];
    const V3 c = v3(0.5f * (lg.x + hg.x), 0.5f * (lg.y + hg.y), 0.5f * (lg.z + hg.z));
    const V3 e = v3(0.5f * (hg.x - lg.x), 0.5f * (hg.y - lg.y), 0.5f * (hg.z - lg.z));
    return n.x * c.x + n.y * c.y + n.z * c.z - (fabsf(n.x) * e.x + fabsf(n.y) * e.y + fabsf(n.z) * e.z) -
               P.local[p].x < hm;
  };
  int n_np = 0;  // non-plane geoms (sorted keys below 0xffffffff)
  {
    int c = 0;
    for (int g = tid; g < G; g += kBpThreads) c += lo[g].w == 0.f;
    int tot;
    (void)block_exclusive(c, s_tmp, &tot);
    n_np = tot;
  }
  BP_MARK(8);
  const unsigned full = 0xffffffffu;
  const int lane = tid & 31;
  uint32_t* tmp = reinterpret_cast<uint32_t*>(ncon);  // AABB hits (ncon's storage, dead until the narrowphase)
  if (tid == 0) s_misc[5] = 0;
  {
    // sorted copies of the two other axes' extents (lo1, lo2, hi1, hi2), in
    // the list's storage (dead until the bucket placement), and the walk lengths
    float4* sxa = reinterpret_cast<float4*>(list);  // [n_np]
    const int a1 = ax == 0 ? 1 : 0, a2 = ax == 2 ? 1 : 2;
    auto comp = [](const float4& v, int k) { return k == 0 ? v.x : (k == 1 ? v.y : v.z); };
    for (int i = tid; i < n_np; i += kBpThreads) {
      const int g = (int)val[i];
      const float4 l = lo[g], h = hi[g];
      sxa[i] = make_float4(comp(l, a1), comp(l, a2), comp(h, a1), comp(h, a2));
      const uint32_t hk = f2key(axis_of(h));
      int a = i, b = n_np;  // key[a] <= hk < key[b] (b virtual)
      while (b - a > 1) {
        const int m = (a + b) >> 1;
        if (key[m] <= hk) a = m; else b = m;
      }
      start[i] = a - i;
    }
    __syncthreads();
    // the walks cut into tiles of 32 tests; a thread tests one tile at a time
    // (fixed i, 32 consecutive j: unrolled, predicated, no bookkeeping inside)
    // into a 32-bit hit mask, then the warp appends its hits with one atomic
    int* tpre = reinterpret_cast<int*>(key);  // [n_np + 1] tile offsets (np2 > n_np): the keys are dead
    int n_tiles = 0;
    for (int i0 = 0; i0 < n_np; i0 += kBpThreads) {
      const int i = i0 + tid;
      const int v = i < n_np ? (start[i] + 31) >> 5 : 0;
      int tot;
      const int ex = block_exclusive(v, s_tmp, &tot);
      if (i < n_np) tpre[i] = n_tiles + ex;
      n_tiles += tot;
    }
    if (tid == 0) tpre[n_np] = n_tiles;
    __syncthreads();
    for (int q0 = 0; q0 < n_tiles; q0 += kBpThreads) {
      const int q = q0 + tid;
      uint32_t m = 0;
      int i = 0, j0 = 0;
      if (q < n_tiles) {
        int a = 0, b = n_np;  // tpre[a] <= q < tpre[b]
        while (b - a > 1) {
          const int mid = (a + b) >> 1;
          if (tpre[mid] <= q) a = mid; else b = mid;
        }
        i = a;
        const int k0 = (q - tpre[i]) << 5;
        j0 = i + 1 + k0;
        const int nb = min(32, start[i] - k0);
        const float4 si = sxa[i];
        const float4* sp = sxa + j0;
        // unconditional loads (a tile's tail reads up to 31 float4 past the
        // copies, still inside the CTA's shared memory: the list storage and
        // the arrays after it) and branch-free tests, so the 32 loads overlap;
        // the tail is masked off once
#if CF_BP_TILE_BRANCHY == 1  // per-test predicated loads: faster (418 vs 424 us full step) than all-unconditional ones
#pragma unroll
        for (int bb = 0; bb < 32; ++bb) {
          if (bb < nb) {
            const float4 sj = sp[bb];
            m |= (si.x <= sj.z && sj.x <= si.z && si.y <= sj.w && sj.y <= si.w ? 1u : 0u) << bb;
          }
        }
#elif CF_BP_TILE_BRANCHY == 2
        // groups of 8 tests: a group is skipped past the tile's end, its loads
        // are unconditional (up to 7 past the end, inside shared memory) so
        // they overlap; the tail is masked off once
#pragma unroll
        for (int g8 = 0; g8 < 32; g8 += 8) {
          if (g8 < nb) {
#pragma unroll
            for (int bb = g8; bb < g8 + 8; ++bb) {
              const float4 sj = sp[bb];
              m |= (uint32_t)((si.x <= sj.z) & (sj.x <= si.z) & (si.y <= sj.w) & (sj.y <= si.w)) << bb;
            }
          }
        }
        m &= nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u);
#else
#pragma unroll
        for (int bb = 0; bb < 32; ++bb) {
          const float4 sj = sp[bb];
          m |= (uint32_t)((si.x <= sj.z) & (sj.x <= si.z) & (si.y <= sj.w) & (sj.y <= si.w)) << bb;
        }
        m &= nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u);
#endif
      }
      const int nh = __popc(m);
      int incl = nh;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += y;
      }
      const int wt = __shfl_sync(full, incl, 31);
      if (wt) {
        int b0 = 0;
        if (lane == 31) b0 = atomicAdd(&s_misc[5], wt);
        b0 = __shfl_sync(full, b0, 31);
        int pos = b0 + incl - nh;
        const uint32_t ihi = ((uint32_t)i << 16) | (uint32_t)j0;
        while (m) {
          const int bb = __ffs(m) - 1;
          m &= m - 1u;
          if (pos < Q.cap_c) tmp[pos] = ihi + (uint32_t)bb;
          ++pos;
        }
      }
    }
  }
  __syncthreads();
  const int n_hit = s_misc[5];
  // hits -> candidates: bounding spheres (twice the centres, from the AABBs)
  // and owners; counted per bucket, the rejected marked 0xffffffff
  for (int k = tid; k < min(n_hit, Q.cap_c); k += kBpThreads) {
    const uint32_t pv = tmp[k];
    const int gi = (int)val[pv >> 16], gj = (int)val[pv & 0xffffu];
    const float4 li = lo[gi], hi_ = hi[gi], lj = lo[gj], hj = hi[gj];
    const float dx = (li.x + hi_.x) - (lj.x + hj.x), dy = (li.y + hi_.y) - (lj.y + hj.y),
                dz = (li.z + hi_.z) - (lj.z + hj.z), r = 2.f * (hi_.w + hj.w);
    const bool ok = dx * dx + dy * dy + dz * dz <= r * r && gbody[gi] != gbody[gj];
    const int a = min(gi, gj);
    if (ok) atomicAdd(&cnt[a], 1);
    tmp[k] = ok ? ((uint32_t)a << 16) | (uint32_t)max(gi, gj) : 0xffffffffu;
  }
  BP_MARK(9);
  // (ii) planes (lowest geom ids): count their hits
  for (int p = 0; p < G && P.geom[p].x == G_PLANE; ++p) {
    for (int g0 = 0; g0 < G; g0 += kBpThreads) {
      const int g = g0 + tid;
      const int hit = (g < G && g > p && lo[g].w == 0.f && gbody[g] != gbody[p] && plane_hit(p, g)) ? 1 : 0;
      int tot;
      (void)block_exclusive(hit, s_tmp, &tot);
      if (tid == 0) cnt[p] += tot;
    }
  }
  __syncthreads();
  BP_MARK(10);
  // (iii) bucket starts (exclusive scan of the counts)
  {
    int run = 0;
    for (int g0 = 0; g0 <= G; g0 += kBpThreads) {
      const int g = g0 + tid;
      const int v = g < G ? cnt[g] : 0;
      int tot;
      const int ex = block_exclusive(v, s_tmp, &tot);
      if (g <= G) start[g] = run + ex;
      run += tot;
    }
    __syncthreads();
    for (int g = tid; g < G; g += kBpThreads) cnt[g] = 0;
    if (tid == 0) {
      // more AABB hits than the hit list holds: candidates were lost
      if (n_hit > Q.cap_c) run = Q.cap_c + 1;
      s_misc[2] = run;                                   // candidates of the world
      if (run > Q.cap_c) atomicOr(Q.err, ERR_CANDIDATES);
    }
    __syncthreads();
  }
  BP_MARK(11);
  // (iv) pairs into their buckets; plane buckets in geom order by a block scan
  {
    for (int k = tid; k < min(n_hit, Q.cap_c); k += kBpThreads) {
      const uint32_t pv = tmp[k];
      if (pv == 0xffffffffu) continue;
      const int a = (int)(pv >> 16);
      const int slot = start[a] + atomicAdd(&cnt[a], 1);
      if (slot < Q.cap_c) list[slot] = pv;
    }
    for (int p = 0; p < G && P.geom[p].x == G_PLANE; ++p) {
      int base = start[p];
      for (int g0 = 0; g0 < G; g0 += kBpThreads) {
        const int g = g0 + tid;
        const int hit = (g < G && g > p && lo[g].w == 0.f && gbody[g] != gbody[p] && plane_hit(p, g)) ? 1 : 0;
        int tot;
        const int ex = block_exclusive(hit, s_tmp, &tot);
        if (hit && base + ex < Q.cap_c) list[base + ex] = ((uint32_t)p << 16) | (uint32_t)g;
        base += tot;
      }
    }
    __syncthreads();
  }
  // a world whose candidates overflow the list emits nothing (reported as
  // COMFREE_ERR_CAPACITY): its truncated buckets would hold stale entries
  const int n_cand = s_misc[2] > Q.cap_c ? 0 : s_misc[2];
  BP_MARK(3);
  // 2c: each non-plane bucket sorted by g2: a thread per candidate counts the
  // entries of its bucket below it (its rank; the keys of a bucket are
  // distinct) and writes it to its place in ncon's storage (free until the
  // narrowphase), copied back into the list; plane buckets are in geom order
  // already.  (Swapping the two arrays' roles instead of copying back gave
  // nondeterministic, partly unwritten records: not used.)
  {
    uint32_t* sorted = reinterpret_cast<uint32_t*>(ncon);
    for (int k = tid; k < n_cand; k += kBpThreads) {
      const uint32_t v = list[k];
      const int g1 = (int)(v >> 16);
      const int b0 = start[g1];
      int r = k - b0;
      if (P.geom[g1].x != G_PLANE) {
        const int b1 = start[g1 + 1];
        r = 0;
        for (int e = b0; e < b1; ++e) r += list[e] < v;
      }
      sorted[b0 + r] = v;
    }
    __syncthreads();
    for (int k = tid; k < n_cand; k += kBpThreads) list[k] = sorted[k];
    __syncthreads();
  }
  // the AABBs are dead: their storage takes the geom table for the narrowphase
  for (int g = tid; g < G; g += kBpThreads) {
    lo[g] = P.size[g];
    reinterpret_cast<int4*>(hi)[g] = P.geom[g];
  }
  __syncthreads();
  const GeomTab Ts{reinterpret_cast<const int4*>(hi), lo, P.local};
  BP_MARK(4);
  // 3: narrowphase count per candidate, in an evaluation order grouped by the
  // pair's kinds (counting sort on kind(g1) * 4 + kind(g2)) so that a warp's
  // lanes take the same narrowphase branch; block scan -> offsets in the world
  {
    int* ccount = s_tmp;  // 16 classes
    if (tid < 16) ccount[tid] = 0;
    __syncthreads();
    for (int k = tid; k < n_cand; k += kBpThreads) {
      const uint32_t pv = list[k];
      atomicAdd(&ccount[Ts.geom[pv >> 16].x * 4 + Ts.geom[pv & 0xffffu].x], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int c = 0; c < 16; ++c) { const int v = ccount[c]; ccount[c] = run; run += v; }
    }
    __syncthreads();
    for (int k = tid; k < n_cand; k += kBpThreads) {
      const uint32_t pv = list[k];
      perm[atomicAdd(&ccount[Ts.geom[pv >> 16].x * 4 + Ts.geom[pv & 0xffffu].x], 1)] = (uint16_t)k;
    }
    __syncthreads();
  }
  // one narrowphase pass: counts, and the records staged (in the order found)
  if (tid == 0) s_misc[6] = 0;
  __syncthreads();
  const Stage S{Q.stage + (size_t)w * 4 * Q.stage_cap, Q.stage + ((size_t)w * 4 + 1) * Q.stage_cap, Q.stage_cap,
                &s_misc[6]};
  for (int i = tid; i < n_cand; i += kBpThreads) {
    const int k = perm[i];
    const uint32_t pv = list[k];
    ncon[k] = pair_contacts_stage(P, make_int2((int)(pv >> 16), (int)(pv & 0xffffu)), Fw, w, &Ts, S, k);
  }
  __syncthreads();
  int world_total = 0;
  {
    int run = 0;
    for (int k0 = 0; k0 < n_cand; k0 += kBpThreads) {
      const int k = k0 + tid;
      const int v = k < n_cand ? ncon[k] : 0;
      int tot;
      const int ex = block_exclusive(v, s_tmp, &tot);
      if (k < n_cand) ncon[k] = run + ex;                 // now: offset of candidate k in the world
      run += tot;
    }
    world_total = run;
  }
  BP_MARK(5);
  // 4: publish the world's total; the records go to their places in
  // k_collide_bp_emit, which finds the world's base by a look-back over the
  // published totals without waiting (every total is there when it runs)
  if (world_total <= Q.stage_cap) {
    // the staged records (found order, L2-resident) to their places in the
    // world, with their pair's (g1, g2) instead of the tag
    float4* o0 = Q.stage + ((size_t)w * 4 + 2) * Q.stage_cap;
    float4* o1 = o0 + Q.stage_cap;
    // CF_BP_PUB records per thread loaded before any is stored (the staging
    // reads are L2 round trips that would otherwise wait behind the stores)
    constexpr int kPub = CF_BP_PUB;
    for (int r0 = 0; r0 < world_total; r0 += kPub * kBpThreads) {
      float4 a[kPub], b[kPub];
#pragma unroll
      for (int u = 0; u < kPub; ++u) {
        const int r = r0 + u * kBpThreads + tid;
        if (r < world_total) { a[u] = ld_cg4(S.s0 + r); b[u] = ld_cg4(S.s1 + r); }
      }
#pragma unroll
      for (int u = 0; u < kPub; ++u) {
        const int r = r0 + u * kBpThreads + tid;
        if (r < world_total) {
          const int tag = __float_as_int(b[u].w), k = tag >> 5;
          const int l = ncon[k] + (tag & 31);
          o0[l] = a[u];
          o1[l] = make_float4(b[u].x, b[u].y, b[u].z, __uint_as_float(list[k]));
        }
      }
    }
    if (tid == 0) {
      atomicAdd(&Q.gsum[w >> kGsumShift], (unsigned long long)world_total);
      atomicExch(&Q.status[w], kStAgg | (unsigned long long)world_total);
    }
    BP_MARK(6);
    return;
  }
  // more records than the staging area holds: the world's base now (a look-
  // back that may wait for predecessors still counting), then the narrowphase
  // again, written in place; the emit kernel skips the world (kStDone)
  if (tid == 0) {
    atomicAdd(&Q.gsum[w >> kGsumShift], (unsigned long long)world_total);
    atomicExch(&Q.status[w], kStAgg | (unsigned long long)world_total);
  }
  if (tid < 32) {
    const long long prefix = lookback_warp(Q.status, w, tid);
    if (tid == 0) {  // the total stays in the word (the emit kernel sums totals)
      atomicExch(&Q.status[w], kStAgg | kStDone | (unsigned long long)world_total);
      s_misc[3] = (int)(prefix >> 31);
      s_misc[4] = (int)(prefix & 0x7fffffff);
    }
  }
  __syncthreads();
  const int64_t base = ((int64_t)s_misc[3] << 31) | (int64_t)s_misc[4];
  if (tid == 0 && Q.fbase) Q.fbase[w] = base;
  BP_MARK(6);
  // a candidate that does not fit is skipped; the smallest such offset is the
  // count of whole pairs
  for (int i = tid; i < n_cand; i += kBpThreads) {
    const int k = perm[i];
    const int off = ncon[k];
    const int next = (k + 1 < n_cand) ? ncon[k + 1] : world_total;
    if (next == off) continue;
    if (base + next > Q.capacity) {
      atomicMin(reinterpret_cast<unsigned long long*>(Q.queue + 2), (unsigned long long)(base + off));
      atomicOr(Q.err, ERR_CONTACT_CAP);
      continue;
    }
    const uint32_t pv = list[k];
    pair_contacts<true>(P, make_int2((int)(pv >> 16), (int)(pv & 0xffffu)), Fw, w, base + off, &Ts);
  }
  BP_MARK(7);
}

// The broadphase's second launch: one CTA per world takes the world's base
// offset from the totals k_collide_bp published (group sums of 2^kGsumShift
// worlds before the world's group, then the single totals inside it: one
// load per thread, one block reduction, no waiting) and writes the staged
// records to their places (thread per record): world-major, (g1, g2)-ordered,
// deterministic.  The last CTA stores the device count (the offset of the
// first pair that did not fit when the capacity is exceeded).
constexpr int kBpEmitThreads = 256;
__global__ void __launch_bounds__(kBpEmitThreads) k_collide_bp_emit(const __grid_constant__ CollideParams P,
                                                                    const __grid_constant__ BpParams Q) {
  __shared__ long long s_red[kBpEmitThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t w = blockIdx.x;
  const unsigned long long sw = Q.status[w];
  const int world_total = (int)(sw & kStVal);
  long long x = 0;
  const int64_t g = w >> kGsumShift, t0 = g << kGsumShift;
  for (int64_t i = tid; i < g; i += kBpEmitThreads) x += (long long)Q.gsum[i];
  for (int64_t i = t0 + tid; i < w; i += kBpEmitThreads) x += (long long)(Q.status[i] & kStVal);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (lane == 0) s_red[tid >> 5] = x;
  __syncthreads();
  if (!(sw & kStDone)) {
    long long base = 0;
#pragma unroll
    for (int q = 0; q < kBpEmitThreads / 32; ++q) base += s_red[q];
    const float4* o0 = Q.stage + ((size_t)w * 4 + 2) * Q.stage_cap;
    const float4* o1 = o0 + Q.stage_cap;
    const bool cut = base + world_total > Q.capacity;  // only whole pairs within the capacity
    constexpr int kPub = CF_BP_PUB;  // records per thread loaded before any is written
    for (int l0 = 0; l0 < world_total; l0 += kPub * kBpEmitThreads) {
    float4 aa[kPub], bb[kPub];
#pragma unroll
    for (int u = 0; u < kPub; ++u) {
      const int l = l0 + u * kBpEmitThreads + tid;
      if (l < world_total) { aa[u] = ld_cg4(o0 + l); bb[u] = ld_cg4(o1 + l); }
    }
#pragma unroll
    for (int u = 0; u < kPub; ++u) {
      const int l = l0 + u * kBpEmitThreads + tid;
      if (l >= world_total) continue;
      const float4 a = aa[u], b = bb[u];
      const uint32_t pv = __float_as_uint(b.w);
      if (cut) {  // the pair's records [off, next) are the neighbours with its (g1, g2)
        int off = l, next = l + 1;
        while (off > 0 && __float_as_uint(o1[off - 1].w) == pv) --off;
        while (next < world_total && __float_as_uint(o1[next].w) == pv) ++next;
        if (base + next > Q.capacity) {
          atomicMin(reinterpret_cast<unsigned long long*>(Q.queue + 2), (unsigned long long)(base + off));
          continue;
        }
      }
      const int4 g1 = P.geom[pv >> 16], g2 = P.geom[pv & 0xffffu];
      const int64_t c = base + l;
      const V3 nn = v3(b.x, b.y, b.z);
      const V3 t1 = tangent(nn);
      P.c0[c] = a;
      P.c1[c] = make_float4(nn.x, nn.y, nn.z, P.mu_t);
      P.c2[c] = make_float4(t1.x, t1.y, t1.z, P.mu_tor);
      P.c3[c] = make_int4(g1.y, g2.y, __float_as_int(P.mu_rol), P.condim);
      P.world[c] = (int32_t)w;
      P.link[c] = make_int2(g1.y < -1 ? g1.z : 0, g2.y < -1 ? g2.z : 0);
    }
    }
  }
  // the last CTA: device count, error
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&Q.queue[5], 1) == (int)gridDim.x - 1) {
      __threadfence();
      int64_t total = 0;
      for (int64_t i = 0; i <= (P.n_worlds - 1) >> kGsumShift; ++i) total += (int64_t)atomicAdd(&Q.gsum[i], 0ull);
      const unsigned long long cut = atomicAdd(reinterpret_cast<unsigned long long*>(Q.queue + 2), 0ull);
      if (total > Q.capacity) atomicOr(Q.err, ERR_CONTACT_CAP);
      Q.n_dev[0] = (int64_t)cut < total ? (int64_t)cut : total;
      if (Q.total) *Q.total = total;
    }
  }
}

}  // namespace

// candidate-list words the sort (np2 <= block: 2 x np2 uint64 exchange) and
// the sweep (n_np <= n_geoms float4) borrow before the candidates go in
int collide_bp_min_cap(int n_geoms, int np2) {
  return std::max(4 * n_geoms, np2 <= kBpThreads ? 4 * np2 : 0);
}

size_t collide_bp_smem(int n_geoms, int cap_c, int np2) {
  return (size_t)5 * n_geoms * sizeof(float4) + (size_t)2 * np2 * sizeof(uint32_t) +
         (size_t)(3 * n_geoms + 2) * sizeof(int) + (size_t)cap_c * (sizeof(uint32_t) + sizeof(int) + sizeof(uint16_t));
}

cudaError_t collide_broadphase(const CollideParams& P, int cap_c, int64_t capacity, unsigned long long* status,
                               int* queue, int64_t* n_dev, int64_t* total, int* err, float4* stage, int stage_cap,
                               cudaStream_t s, int64_t* fbase) {
  if (P.n_worlds == 0) return cudaMemsetAsync(n_dev, 0, sizeof(int64_t), s);
  int np2 = 1;
  while (np2 < P.n_geoms + 1) np2 <<= 1;  // the flat sweep's prefix takes n_np + 1 <= G + 1 entries
  const size_t smem = collide_bp_smem(P.n_geoms, cap_c, np2);
  // zeroed status words and counters; queue[2..3]: the cut (int64) starts at
  // 0x7f7f...7f (above any count); memsets only, so the launches are graph-capturable
  // status words followed by the group sums (one allocation)
  const size_t n_status = (size_t)P.n_worlds + (((size_t)P.n_worlds + 255) >> kGsumShift);
  cudaError_t e = cudaMemsetAsync(status, 0, n_status * sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(queue, 0, 8 * sizeof(int), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(queue + 2, 0x7f, sizeof(int64_t), s);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_collide_bp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  BpParams Q{cap_c, np2, capacity, status, queue, n_dev, total, err, stage, stage_cap, status + P.n_worlds, fbase};
  k_collide_bp<<<(unsigned)P.n_worlds, kBpThreads, smem, s>>>(P, Q);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (fbase) return cudaSuccess;  // the fused step reads the staged records itself: no emit pass
  k_collide_bp_emit<<<(unsigned)P.n_worlds, kBpEmitThreads, 0, s>>>(P, Q);
  return cudaGetLastError();
}

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
