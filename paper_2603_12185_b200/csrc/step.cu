// step.cu — the fused ComFree-Sim contact-resolution step (S1-S8) for sm_100a.
//
// One "world group" of WPW warps owns one world for the whole step:
//   prologue  S1  per body: smooth prediction v_s, omega_s (Eq. (2), P:91-97;
//                 Alg. 1 Kernel I), world inverse inertia
//                 R diag(I_b^-1) R^T; per chain: qd_s = qd + L^-T L^-1 (tau - c) dt.
//                 Records go to shared memory (the per-world body slab).
//   main loop     one lane per contact, contact-major SoA float4 streams read
//                 with 128-bit non-allocating loads, next contact prefetched:
//             S2  relative twist of b w.r.t. a at the contact point (Eq. (4)-(5))
//             S3  M(phi) = r/(1-r) / (tr_a + tr_b) (Eq. (12)-(13))
//             S4  every facet: Lambda_f = M (-k phi - kappa s_f)_+ with
//                 s_f = J~_f v_s (Eq. (7)-(9), sign of Eq. (9));
//                 kappa = k dt + d (K dt = k M, D dt = d M, Eq. (12) literal)
//             S5  facet impulses regrouped into the contact wrench
//                 (f_c, tau_c) = sum_f J~_f^T Lambda_f in contact space
//             S6  scatter J^T (f_c, tau_c) into per-world shared-memory
//                 accumulators (Alg. 1 Kernel III) — no global atomics
//   epilogue  S7  v+ = v_s + M^-1 p (Eq. (10), Alg. 1 Kernel IV), semi-implicit
//                 Euler with exp-map quaternion update; chains q+ = q + qd+ dt;
//                 finite check and per-world statistics.
// WPW = 8: one 256-thread CTA per world (dense piles); WPW = 1: eight worlds per
// CTA, one warp each (small worlds: hand + cube).
#include <cuda_runtime.h>
#include <math.h>

#include "internal.h"

namespace cf {

static constexpr int kWarps = 8;
static constexpr int kThreads = kWarps * 32;

struct GroupLayout {  // float offsets inside one group's shared-memory window
  int rec, quat, acc, tq, tL, tacc, red, total;
};

__host__ __device__ inline GroupLayout group_layout(const SceneDev& sc) {
  GroupLayout L;
  int o = 0;
  L.rec = o;  o += 16 * sc.Bp;   // float4 rec[4][Bp]: (v_s,im) (w_s,Ixx) (x,Iyy) (Izz,Ixy,Ixz,Iyz)
  L.quat = o; o += 4 * sc.Bp;    // float4 quat[Bp] (step-start orientation)
  L.acc = o;  o += 6 * sc.Bp;    // float acc[6][Bp]: generalized impulse p (lin, ang)
  L.tq = o;   o += 4 * sc.T;     // float4 qd_s[T]
  L.tL = o;   o += 12 * sc.T;    // float L[T][12] (10 used)
  L.tacc = o; o += 4 * sc.T;     // float p_chain[T][4]
  L.red = o;  o += 16;           // reductions
  L.total = (o + 3) & ~3;
  return L;
}

size_t step_smem_bytes(const SceneDev& sc, int wpw) {
  return (size_t)(kWarps / wpw) * group_layout(sc).total * sizeof(float);
}

template <int WPW>
__device__ __forceinline__ void group_sync(int group) {
  if (WPW == 1) {
    __syncwarp();
  } else if (WPW == kWarps) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(group + 1), "r"(WPW * 32) : "memory");
  }
}

// 128-bit streaming loads: read once, do not allocate in L1.
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float3 cross3(float3 a, float3 b) {
  return make_float3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float dot3(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

__device__ __forceinline__ int tri(int i, int j) { return i * (i + 1) / 2 + j; }

// x <- (L L^T)^-1 x for a chain of nd <= 4 DoFs (forward then backward substitution)
__device__ __forceinline__ void chol_solve(const float* L, int nd, float x[4]) {
  float y[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < nd) {
      float s = x[i];
#pragma unroll
      for (int j = 0; j < i; ++j) s -= L[tri(i, j)] * y[j];
      y[i] = s / L[tri(i, i)];
    }
  }
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    if (i < nd) {
      float s = y[i];
#pragma unroll
      for (int j = i + 1; j < 4; ++j)
        if (j < nd) s -= L[tri(j, i)] * x[j];
      x[i] = s / L[tri(i, i)];
    }
  }
}

// ||L^-1 v||^2 = v^T M^-1 v (forward substitution only)
__device__ __forceinline__ float chol_quad(const float* L, int nd, float4 v4) {
  float v[4] = {v4.x, v4.y, v4.z, v4.w};
  float y[4] = {0.f, 0.f, 0.f, 0.f};
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < nd) {
      float s = v[i];
#pragma unroll
      for (int j = 0; j < i; ++j) s -= L[tri(i, j)] * y[j];
      y[i] = s / L[tri(i, i)];
      acc += y[i] * y[i];
    }
  }
  return acc;
}

__device__ __forceinline__ float dot4(float4 a, float4 b) { return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w; }

// Eq. (13): r(|phi|) with x clamped to [0, 1] (reading R7)
__device__ __forceinline__ float impedance_r(const StepParams& P, float phi) {
  float x = fminf(fabsf(phi) * P.inv_width, 1.0f);
  float m = P.mid, g;
  if (x < m) {
    float u = x / m;
    g = m * (P.power_is_2 ? u * u : __powf(u, P.power));
  } else {
    float u = (1.0f - x) / (1.0f - m);
    g = 1.0f - (1.0f - m) * (P.power_is_2 ? u * u : __powf(u, P.power));
  }
  return P.r_min + P.r_span * g;
}

// Facets of one 2-D channel (tangential or rolling): L_j = (A + kmu (d_j . w))_+,
// accumulating N += L_j and F += L_j d_j.  NT = 4 uses the exact axis set.
template <int NT>
__device__ __forceinline__ void channel2(float A, float kmu, float w1, float w2, const float2* dir,
                                         int n, float& N, float& F1, float& F2, int& act,
                                         float* out, float Mc) {
  if (NT == 4) {
    float a1 = kmu * w1, a2 = kmu * w2;
    float L0 = fmaxf(A + a1, 0.f), L1 = fmaxf(A + a2, 0.f);
    float L2 = fmaxf(A - a1, 0.f), L3 = fmaxf(A - a2, 0.f);
    N += (L0 + L2) + (L1 + L3);
    F1 += L0 - L2;
    F2 += L1 - L3;
    act += (L0 > 0.f) + (L1 > 0.f) + (L2 > 0.f) + (L3 > 0.f);
    if (out) {
      out[0] = Mc * L0; out[1] = Mc * L1; out[2] = Mc * L2; out[3] = Mc * L3;
    }
  } else {
    for (int j = 0; j < n; ++j) {
      float2 d = dir[j];
      float L = fmaxf(fmaf(kmu, fmaf(d.x, w1, d.y * w2), A), 0.f);
      N += L;
      F1 = fmaf(L, d.x, F1);
      F2 = fmaf(L, d.y, F2);
      act += (L > 0.f);
      if (out) out[j] = Mc * L;
    }
  }
}

template <int WPW, int NT>
__global__ void __launch_bounds__(kThreads, 4) k_step(const __grid_constant__ StepParams P) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const SceneDev& sc = P.sc;
  const GroupLayout GL = group_layout(sc);
  constexpr int kGroups = kWarps / WPW;
  constexpr int kGT = WPW * 32;
  const int group = threadIdx.x / kGT;
  const int gt = threadIdx.x % kGT;
  const int64_t w = (int64_t)blockIdx.x * kGroups + group;
  if (w >= P.n_worlds) return;  // whole group leaves together

  float* G = smem + (size_t)group * GL.total;
  float4* rec = reinterpret_cast<float4*>(G + GL.rec);
  float4* quat_s = reinterpret_cast<float4*>(G + GL.quat);
  float* acc = G + GL.acc;
  float4* tq = reinterpret_cast<float4*>(G + GL.tq);
  float* tL = G + GL.tL;
  float* tacc = G + GL.tacc;
  float* red = G + GL.red;
  const int B = sc.B, Bp = sc.Bp, T = sc.T, nd = sc.nd;
  float* slab = P.slab + (size_t)w * sc.slab;
  const float dt = P.dt;

  // ---------------- S1: smooth prediction (Kernel I) ----------------
  for (int i = gt; i < B; i += kGT) {
    float3 x = make_float3(slab[0 * Bp + i], slab[1 * Bp + i], slab[2 * Bp + i]);
    float4 q = make_float4(slab[3 * Bp + i], slab[4 * Bp + i], slab[5 * Bp + i], slab[6 * Bp + i]);
    float3 v = make_float3(slab[7 * Bp + i], slab[8 * Bp + i], slab[9 * Bp + i]);
    float3 om = make_float3(slab[10 * Bp + i], slab[11 * Bp + i], slab[12 * Bp + i]);
    const float im = sc.inv_mass[i];
    const float3 ib = make_float3(sc.inv_inertia[i], sc.inv_inertia[Bp + i], sc.inv_inertia[2 * Bp + i]);
    // rotation of the normalised quaternion (reading R15)
    float qn = rsqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    float qw = q.x * qn, qx = q.y * qn, qy = q.z * qn, qz = q.w * qn;
    float R00 = 1.f - 2.f * (qy * qy + qz * qz), R01 = 2.f * (qx * qy - qw * qz), R02 = 2.f * (qx * qz + qw * qy);
    float R10 = 2.f * (qx * qy + qw * qz), R11 = 1.f - 2.f * (qx * qx + qz * qz), R12 = 2.f * (qy * qz - qw * qx);
    float R20 = 2.f * (qx * qz - qw * qy), R21 = 2.f * (qy * qz + qw * qx), R22 = 1.f - 2.f * (qx * qx + qy * qy);
    // Iw^-1 = R diag(ib) R^T
    float Ixx = R00 * R00 * ib.x + R01 * R01 * ib.y + R02 * R02 * ib.z;
    float Iyy = R10 * R10 * ib.x + R11 * R11 * ib.y + R12 * R12 * ib.z;
    float Izz = R20 * R20 * ib.x + R21 * R21 * ib.y + R22 * R22 * ib.z;
    float Ixy = R00 * R10 * ib.x + R01 * R11 * ib.y + R02 * R12 * ib.z;
    float Ixz = R00 * R20 * ib.x + R01 * R21 * ib.y + R02 * R22 * ib.z;
    float Iyz = R10 * R20 * ib.x + R11 * R21 * ib.y + R12 * R22 * ib.z;
    float3 fl = make_float3(0.f, 0.f, 0.f), ta = make_float3(0.f, 0.f, 0.f);
    if (P.f_ext) {
      const float* fe = P.f_ext + ((size_t)w * B + i) * 6;
      fl = make_float3(fe[0], fe[1], fe[2]);
      ta = make_float3(fe[3], fe[4], fe[5]);
    }
    float3 vs = v;
    if (im > 0.f) {
      vs.x += (im * fl.x + P.g[0]) * dt;
      vs.y += (im * fl.y + P.g[1]) * dt;
      vs.z += (im * fl.z + P.g[2]) * dt;
    }
    // bias c = omega x (Iw omega), Iw = R diag(1/ib) R^T on unlocked axes
    float3 wl = make_float3(R00 * om.x + R10 * om.y + R20 * om.z, R01 * om.x + R11 * om.y + R21 * om.z,
                            R02 * om.x + R12 * om.y + R22 * om.z);
    wl.x *= ib.x > 0.f ? 1.f / ib.x : 0.f;
    wl.y *= ib.y > 0.f ? 1.f / ib.y : 0.f;
    wl.z *= ib.z > 0.f ? 1.f / ib.z : 0.f;
    float3 Iwo = make_float3(R00 * wl.x + R01 * wl.y + R02 * wl.z, R10 * wl.x + R11 * wl.y + R12 * wl.z,
                             R20 * wl.x + R21 * wl.y + R22 * wl.z);
    float3 gy = cross3(om, Iwo);
    float3 rh = make_float3(ta.x - gy.x, ta.y - gy.y, ta.z - gy.z);
    float3 ws = make_float3(om.x + (Ixx * rh.x + Ixy * rh.y + Ixz * rh.z) * dt,
                            om.y + (Ixy * rh.x + Iyy * rh.y + Iyz * rh.z) * dt,
                            om.z + (Ixz * rh.x + Iyz * rh.y + Izz * rh.z) * dt);
    rec[i] = make_float4(vs.x, vs.y, vs.z, im);
    rec[Bp + i] = make_float4(ws.x, ws.y, ws.z, Ixx);
    rec[2 * Bp + i] = make_float4(x.x, x.y, x.z, Iyy);
    rec[3 * Bp + i] = make_float4(Izz, Ixy, Ixz, Iyz);
    quat_s[i] = q;
#pragma unroll
    for (int k = 0; k < 6; ++k) acc[k * Bp + i] = 0.f;
  }
  for (int t = gt; t < T; t += kGT) {
    const float* Lg = P.tree_L + ((size_t)w * T + t) * 10;
    float* Ls = tL + 12 * t;
#pragma unroll
    for (int k = 0; k < 10; ++k) Ls[k] = Lg[k];
    float x[4] = {0.f, 0.f, 0.f, 0.f}, qd[4] = {0.f, 0.f, 0.f, 0.f};
    const float* qv = slab + N_BODY_PLANES * Bp + sc.Qp + t * nd;
    const float* tau = P.tree_tau + (size_t)w * sc.Q + t * nd;
    for (int j = 0; j < nd; ++j) { x[j] = tau[j]; qd[j] = qv[j]; }
    chol_solve(Ls, nd, x);
    tq[t] = make_float4(qd[0] + x[0] * dt, qd[1] + x[1] * dt, qd[2] + x[2] * dt, qd[3] + x[3] * dt);
#pragma unroll
    for (int k = 0; k < 4; ++k) tacc[4 * t + k] = 0.f;
  }
  if (gt < 16) red[gt] = 0.f;
  group_sync<WPW>(group);

  // ---------------- S2-S6: contacts ----------------
  const int64_t cbeg = P.off[w], cend = P.off[w + 1];
  const float k = P.k, kappa = P.kappa;
  int n_active = 0;
  float max_pen = 0.f;
  int64_t c = cbeg + gt;
  float4 C0, C1, C2;
  int4 C3;
  if (c < cend) { C0 = ld_stream(P.c0 + c); C1 = ld_stream(P.c1 + c); C2 = ld_stream(P.c2 + c); C3 = ld_stream(P.c3 + c); }
  for (; c < cend; c += kGT) {
    const float4 c0 = C0, c1 = C1, c2 = C2;
    const int4 c3 = C3;
    if (c + kGT < cend) {  // prefetch the next contact of this lane
      C0 = ld_stream(P.c0 + c + kGT); C1 = ld_stream(P.c1 + c + kGT);
      C2 = ld_stream(P.c2 + c + kGT); C3 = ld_stream(P.c3 + c + kGT);
    }
    const int ida = c3.x, idb = c3.y, cd = c3.w;
    const float mu_rol = __int_as_float(c3.z);
    const float3 p = make_float3(c0.x, c0.y, c0.z);
    const float phi = c0.w;
    const float3 n = make_float3(c1.x, c1.y, c1.z);
    const float3 t1 = make_float3(c2.x, c2.y, c2.z);
    const float mu_t = c1.w, mu_tor = c2.w;
    max_pen = fmaxf(max_pen, -phi);
    bool bad = (cd != 1 && cd != 3 && cd != 4 && cd != 6);
    bad |= ida >= B || idb >= B || (ida == -1 && idb == -1);
    bad |= (ida < -1 && (-2 - ida >= T || !P.jrow)) || (idb < -1 && (-2 - idb >= T || !P.jrow));
    if (bad) {
      atomicOr(P.err, (cd != 1 && cd != 3 && cd != 4 && cd != 6) ? ERR_CONDIM : ERR_BODY_RANGE);
      continue;
    }
    // S2: relative twist b w.r.t. a and S3 traces
    float3 vrel = make_float3(0.f, 0.f, 0.f), wrel = make_float3(0.f, 0.f, 0.f);
    float tr = 0.f;
    float3 ra = make_float3(0.f, 0.f, 0.f), rb = make_float3(0.f, 0.f, 0.f);
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int id = side ? idb : ida;
      const float sg = side ? 1.f : -1.f;
      if (id >= 0) {
        const float4 r0 = rec[id], r1 = rec[Bp + id], r2 = rec[2 * Bp + id], r3 = rec[3 * Bp + id];
        const float3 r = make_float3(p.x - r2.x, p.y - r2.y, p.z - r2.z);
        const float3 wxr = cross3(make_float3(r1.x, r1.y, r1.z), r);
        vrel.x += sg * (r0.x + wxr.x); vrel.y += sg * (r0.y + wxr.y); vrel.z += sg * (r0.z + wxr.z);
        wrel.x += sg * r1.x; wrel.y += sg * r1.y; wrel.z += sg * r1.z;
        // tr(J M^-1 J^T) of the linear point Jacobian: 3 im + tr(I)|r|^2 - r^T I r
        const float Ixx = r1.w, Iyy = r2.w, Izz = r3.x, Ixy = r3.y, Ixz = r3.z, Iyz = r3.w;
        const float3 Ir = make_float3(Ixx * r.x + Ixy * r.y + Ixz * r.z, Ixy * r.x + Iyy * r.y + Iyz * r.z,
                                      Ixz * r.x + Iyz * r.y + Izz * r.z);
        tr += 3.f * r0.w + (Ixx + Iyy + Izz) * dot3(r, r) - dot3(r, Ir);
        if (side) rb = r; else ra = r;
      } else if (id < -1) {
        const int t = -2 - id;
        const float4 qd = tq[t];
        const float* Ls = tL + 12 * t;
        const float4* jr = P.jrow + (size_t)(side * 6) * P.n_contacts + c;
        float vp[3], wp[3];
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const float4 jl = ld_stream(jr + (size_t)kk * P.n_contacts);
          const float4 ja = ld_stream(jr + (size_t)(kk + 3) * P.n_contacts);
          vp[kk] = dot4(jl, qd);
          wp[kk] = dot4(ja, qd);
          tr += chol_quad(Ls, nd, jl);
        }
        vrel.x += sg * vp[0]; vrel.y += sg * vp[1]; vrel.z += sg * vp[2];
        wrel.x += sg * wp[0]; wrel.y += sg * wp[1]; wrel.z += sg * wp[2];
      }
    }
    const float3 t2 = cross3(n, t1);
    const float un = dot3(n, vrel);
    // S3: M(phi) (Eq. (12)-(13))
    const float r = impedance_r(P, phi);
    const float Mc = r / ((1.f - r) * tr);
    // S4: Lambda_f = Mc (A + kappa mu (d . w))_+,  A = -k phi - kappa u_n
    const float A = -k * phi - kappa * un;
    float N = 0.f, F1 = 0.f, F2 = 0.f, Mt = 0.f, R1 = 0.f, R2 = 0.f;
    float* out = nullptr;
    if (P.impulses) {
      const int64_t orig = P.perm ? (int64_t)P.perm[c] : c;
      const int64_t base = P.foff[orig];
      const int nf = cd == 1 ? 1 : P.n_t + (cd >= 4 ? 2 : 0) + (cd == 6 ? P.n_rol : 0);
      if (base + nf <= P.impulses_cap) out = P.impulses + base;
      else atomicOr(P.err, ERR_IMPULSE_CAP);
    }
    if (cd == 1) {
      const float L = fmaxf(A, 0.f);
      N = L;
      n_active += (L > 0.f);
      if (out) out[0] = Mc * L;
    } else {
      const float wt1 = dot3(t1, vrel), wt2 = dot3(t2, vrel);
      channel2<NT>(A, kappa * mu_t, wt1, wt2, P.dir_t, P.n_t, N, F1, F2, n_active, out, Mc);
      if (cd >= 4) {
        const float wtor = dot3(n, wrel);
        const float a = kappa * mu_tor * wtor;
        const float Lp = fmaxf(A + a, 0.f), Lm = fmaxf(A - a, 0.f);
        N += Lp + Lm;
        Mt = Lp - Lm;
        n_active += (Lp > 0.f) + (Lm > 0.f);
        if (out) { out[P.n_t] = Mc * Lp; out[P.n_t + 1] = Mc * Lm; }
      }
      if (cd == 6) {
        const float wr1 = dot3(t1, wrel), wr2 = dot3(t2, wrel);
        channel2<0>(A, kappa * mu_rol, wr1, wr2, P.dir_r, P.n_rol, N, R1, R2, n_active,
                    out ? out + P.n_t + 2 : nullptr, Mc);
      }
    }
    // S5: contact wrench on b (impulse units): f = Mc (N n - mu_t F . (t1,t2)),
    //     tau = -Mc (mu_tor Mt n + mu_rol R . (t1,t2))
    const float ft1 = -mu_t * F1, ft2 = -mu_t * F2;
    const float3 f = make_float3(Mc * (N * n.x + ft1 * t1.x + ft2 * t2.x),
                                 Mc * (N * n.y + ft1 * t1.y + ft2 * t2.y),
                                 Mc * (N * n.z + ft1 * t1.z + ft2 * t2.z));
    const float mt = -mu_tor * Mt, mr1 = -mu_rol * R1, mr2 = -mu_rol * R2;
    const float3 tau = make_float3(Mc * (mt * n.x + mr1 * t1.x + mr2 * t2.x),
                                   Mc * (mt * n.y + mr1 * t1.y + mr2 * t2.y),
                                   Mc * (mt * n.z + mr1 * t1.z + mr2 * t2.z));
    // S6: scatter J^T (f, tau): free body (f, r x f + tau), chain J_lin^T f + J_ang^T tau
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int id = side ? idb : ida;
      const float sg = side ? 1.f : -1.f;
      if (id >= 0) {
        const float3 rr = side ? rb : ra;
        const float3 m = cross3(rr, f);
        atomicAdd(&acc[0 * Bp + id], sg * f.x);
        atomicAdd(&acc[1 * Bp + id], sg * f.y);
        atomicAdd(&acc[2 * Bp + id], sg * f.z);
        atomicAdd(&acc[3 * Bp + id], sg * (m.x + tau.x));
        atomicAdd(&acc[4 * Bp + id], sg * (m.y + tau.y));
        atomicAdd(&acc[5 * Bp + id], sg * (m.z + tau.z));
      } else if (id < -1) {
        const int t = -2 - id;
        const float4* jr = P.jrow + (size_t)(side * 6) * P.n_contacts + c;
        float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const float fv[3] = {f.x, f.y, f.z}, tv[3] = {tau.x, tau.y, tau.z};
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const float4 jl = ld_stream(jr + (size_t)kk * P.n_contacts);
          const float4 ja = ld_stream(jr + (size_t)(kk + 3) * P.n_contacts);
          s4.x += jl.x * fv[kk] + ja.x * tv[kk];
          s4.y += jl.y * fv[kk] + ja.y * tv[kk];
          s4.z += jl.z * fv[kk] + ja.z * tv[kk];
          s4.w += jl.w * fv[kk] + ja.w * tv[kk];
        }
        const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
        for (int j = 0; j < nd; ++j) atomicAdd(&tacc[4 * t + j], sg * sv[j]);
      }
    }
  }
  group_sync<WPW>(group);

  // ---------------- S7: velocity correction + integration (Kernel IV) ----------------
  float ke = 0.f;
  bool nonfinite = false;
  for (int i = gt; i < B; i += kGT) {
    const float4 r0 = rec[i], r1 = rec[Bp + i], r2 = rec[2 * Bp + i], r3 = rec[3 * Bp + i];
    const float4 q = quat_s[i];
    const float im = r0.w;
    const float Ixx = r1.w, Iyy = r2.w, Izz = r3.x, Ixy = r3.y, Ixz = r3.z, Iyz = r3.w;
    const float pl0 = acc[i], pl1 = acc[Bp + i], pl2 = acc[2 * Bp + i];
    const float pa0 = acc[3 * Bp + i], pa1 = acc[4 * Bp + i], pa2 = acc[5 * Bp + i];
    const float3 v = make_float3(r0.x + im * pl0, r0.y + im * pl1, r0.z + im * pl2);
    const float3 om = make_float3(r1.x + Ixx * pa0 + Ixy * pa1 + Ixz * pa2,
                                  r1.y + Ixy * pa0 + Iyy * pa1 + Iyz * pa2,
                                  r1.z + Ixz * pa0 + Iyz * pa1 + Izz * pa2);
    const float3 x = make_float3(r2.x + v.x * dt, r2.y + v.y * dt, r2.z + v.z * dt);
    // q+ = normalize(exp(omega dt / 2) (x) q), world-frame omega
    const float3 th = make_float3(om.x * dt, om.y * dt, om.z * dt);
    const float ang = sqrtf(dot3(th, th));
    float sh, ch;
    sincosf(0.5f * ang, &sh, &ch);
    const float s = ang > 0.f ? sh / ang : 0.5f;
    const float ew = ch, ex = s * th.x, ey = s * th.y, ez = s * th.z;
    float nw = ew * q.x - ex * q.y - ey * q.z - ez * q.w;
    float nx = ew * q.y + ex * q.x + ey * q.w - ez * q.z;
    float ny = ew * q.z - ex * q.w + ey * q.x + ez * q.y;
    float nz = ew * q.w + ex * q.z - ey * q.y + ez * q.x;
    const float inv = 1.0f / sqrtf(nw * nw + nx * nx + ny * ny + nz * nz);
    nw *= inv; nx *= inv; ny *= inv; nz *= inv;
    slab[0 * Bp + i] = x.x; slab[1 * Bp + i] = x.y; slab[2 * Bp + i] = x.z;
    slab[3 * Bp + i] = nw; slab[4 * Bp + i] = nx; slab[5 * Bp + i] = ny; slab[6 * Bp + i] = nz;
    slab[7 * Bp + i] = v.x; slab[8 * Bp + i] = v.y; slab[9 * Bp + i] = v.z;
    slab[10 * Bp + i] = om.x; slab[11 * Bp + i] = om.y; slab[12 * Bp + i] = om.z;
    if (P.check_finite) {
      const float chk = x.x + x.y + x.z + v.x + v.y + v.z + om.x + om.y + om.z + nw + nx + ny + nz;
      nonfinite |= !isfinite(chk);
    }
    if (P.wstats) {
      // KE = 1/2 m v^2 + 1/2 omega^T Iw(q+) omega
      const float3 ib = make_float3(sc.inv_inertia[i], sc.inv_inertia[Bp + i], sc.inv_inertia[2 * Bp + i]);
      const float R00 = 1.f - 2.f * (ny * ny + nz * nz), R01 = 2.f * (nx * ny - nw * nz), R02 = 2.f * (nx * nz + nw * ny);
      const float R10 = 2.f * (nx * ny + nw * nz), R11 = 1.f - 2.f * (nx * nx + nz * nz), R12 = 2.f * (ny * nz - nw * nx);
      const float R20 = 2.f * (nx * nz - nw * ny), R21 = 2.f * (ny * nz + nw * nx), R22 = 1.f - 2.f * (nx * nx + ny * ny);
      const float l0 = R00 * om.x + R10 * om.y + R20 * om.z;
      const float l1 = R01 * om.x + R11 * om.y + R21 * om.z;
      const float l2 = R02 * om.x + R12 * om.y + R22 * om.z;
      ke += 0.5f * ((ib.x > 0.f ? l0 * l0 / ib.x : 0.f) + (ib.y > 0.f ? l1 * l1 / ib.y : 0.f) +
                    (ib.z > 0.f ? l2 * l2 / ib.z : 0.f));
      if (im > 0.f) ke += 0.5f * dot3(v, v) / im;
    }
  }
  for (int t = gt; t < T; t += kGT) {
    float x[4] = {tacc[4 * t], tacc[4 * t + 1], tacc[4 * t + 2], tacc[4 * t + 3]};
    const float* Ls = tL + 12 * t;
    chol_solve(Ls, nd, x);
    const float4 qs = tq[t];
    const float qsv[4] = {qs.x, qs.y, qs.z, qs.w};
    float* qp = slab + N_BODY_PLANES * Bp + t * nd;
    float* qv = slab + N_BODY_PLANES * Bp + sc.Qp + t * nd;
    float qdn[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < nd; ++j) {
      qdn[j] = qsv[j] + x[j];
      qv[j] = qdn[j];
      qp[j] = qp[j] + qdn[j] * dt;
      if (P.check_finite) nonfinite |= !isfinite(qp[j] + qdn[j]);
    }
    if (P.wstats) {  // 1/2 qd^T L L^T qd
      for (int i2 = 0; i2 < nd; ++i2) {
        float y = 0.f;
        for (int j = i2; j < nd; ++j) y += Ls[tri(j, i2)] * qdn[j];
        ke += 0.5f * y * y;
      }
    }
  }
  if (nonfinite) {
    atomicOr(P.err, ERR_NONFINITE);
    atomicMin(P.first_bad, (unsigned long long)(P.world_base + w));
  }
  if (P.wstats) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      n_active += __shfl_xor_sync(0xffffffffu, n_active, o);
      max_pen = fmaxf(max_pen, __shfl_xor_sync(0xffffffffu, max_pen, o));
      ke += __shfl_xor_sync(0xffffffffu, ke, o);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(reinterpret_cast<int*>(&red[0]), n_active);
      atomicMax(reinterpret_cast<int*>(&red[1]), __float_as_int(fmaxf(max_pen, 0.f)));
      atomicAdd(&red[2], ke);
    }
    group_sync<WPW>(group);
    if (gt == 0) {
      comfree_world_stats ws;
      ws.contacts = (int32_t)(cend - cbeg);
      ws.active_facets = *reinterpret_cast<int*>(&red[0]);
      ws.max_penetration = __int_as_float(*reinterpret_cast<int*>(&red[1]));
      ws.kinetic_energy = red[2];
      P.wstats[w] = ws;
    }
  }
}

template <int WPW>
static cudaError_t launch_wpw(const StepParams& p, cudaStream_t s) {
  const int groups = kWarps / WPW;
  const size_t smem = step_smem_bytes(p.sc, WPW);
  const unsigned grid = (unsigned)((p.n_worlds + groups - 1) / groups);
  if (grid == 0) return cudaSuccess;
  cudaError_t e;
  if (p.n_t == 4) {
    e = cudaFuncSetAttribute(k_step<WPW, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_step<WPW, 4><<<grid, kThreads, smem, s>>>(p);
  } else {
    e = cudaFuncSetAttribute(k_step<WPW, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_step<WPW, 0><<<grid, kThreads, smem, s>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_step(const StepParams& p, int wpw, cudaStream_t s) {
  switch (wpw) {
    case 1: return launch_wpw<1>(p, s);
    case 2: return launch_wpw<2>(p, s);
    case 4: return launch_wpw<4>(p, s);
    default: return launch_wpw<8>(p, s);
  }
}

}  // namespace cf
