// step_impl.cuh — the fused ComFree-Sim contact-resolution step (S1-S8), sm_100a.
//
// One "world group" of WPW warps owns one world for the whole step:
//   prologue  S1  per body: smooth prediction v_s, omega_s (Eq. (2), P:91-97;
//                 Alg. 1 Kernel I) and the world inverse inertia
//                 R diag(I_b^-1) R^T; per chain: qd_s = qd + L^-T L^-1 (tau - c) dt.
//                 Records go to shared memory (the per-world body slab).
//   main loop     one lane per contact over the contact-major SoA float4 streams
//                 (128-bit non-allocating loads, next contact prefetched):
//             S2  relative twist of b w.r.t. a at the contact point (Eq. (4)-(5))
//             S3  M(phi) = r/(1-r) / (tr_a + tr_b) (Eq. (12)-(13))
//             S4  every facet f: Lambda_f = M (-k phi - kappa s_f)_+,
//                 s_f = J~_f v_s (Eq. (7)-(9), sign of Eq. (9)),
//                 kappa = k dt + d (K dt = k M, D dt = d M; Eq. (12) literal)
//             S5  facet impulses regrouped into the contact wrench (f_c, tau_c)
//                 = sum_f J~_f^T Lambda_f in contact space; symmetric facet
//                 pairs are differenced exactly (2a when both are active)
//             S6  J^T (f_c, tau_c) scattered into per-world shared-memory
//                 accumulators (Alg. 1 Kernel III) as 64-bit fixed
//                 point with native int32 atomics (deterministic): side a sums
//                 runs of equal body ids in the warp first, side b adds directly
//                 — no global atomics
//   epilogue  S7  v+ = v_s + M^-1 p (Eq. (10), Alg. 1 Kernel IV), semi-implicit
//                 Euler with the exp-map quaternion update; chains q+ = q + qd+ dt;
//                 finite check and per-world statistics.
// WPW = 8: one 256-thread CTA per world (dense piles); WPW = 1: eight worlds per
// CTA, one warp each (hand + cube); pick_wpw (capi.cpp) chooses.  TREES / IMP
// compile the articulated sides and the optional outputs (per-facet impulses,
// per-world statistics) in or out.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <climits>
#include <cstdlib>

#include "internal.h"

namespace cf {

#ifndef CF_HI_ALWAYS
#define CF_HI_ALWAYS 1
#endif
#ifndef CF_MINB
#define CF_MINB 4
#endif
#ifndef CF_S1_UNROLL
#define CF_S1_UNROLL 1
#endif
#ifndef CF_L2AHEAD
#define CF_L2AHEAD 0  // measured slightly slower (59.7 vs 59.4 us, C4)
#endif
#ifndef CF_EARLY_C0
#define CF_EARLY_C0 0
#endif
#ifndef CF_EARLY_C3
#define CF_EARLY_C3 1
#endif
#ifndef CF_NEG_HEADS
#define CF_NEG_HEADS 1
#endif
#ifndef CF_EARLY_RANGE
#define CF_EARLY_RANGE 0  // measured: C4 neutral, C3 hand -2%, C5 mixed +2% (profiles/r01_ab_session2.txt)
#endif
static constexpr int kS1Unroll = CF_S1_UNROLL;  // S1 bodies per thread in flight (unstaged S1)
static constexpr int kWarps = 8;
static constexpr int kThreads = kWarps * 32;

struct GroupLayout {  // float offsets inside one group's shared-memory window
  int rec, accl, acch, tq, tqp, tL, tacl, tach, red, total;
};

__host__ __device__ inline GroupLayout group_layout(const SceneDev& sc) {
  GroupLayout L;
  int o = 0;
  L.rec = o;  o += 16 * sc.Bp;   // float4 rec[4][Bp]: (v_s,im) (w_s,Ixx) (x,Iyy) (Izz,Ixy,Ixz,Iyz)
  L.accl = o; o += 6 * sc.Bp;    // (uint32 lo, int32 hi)[6][Bp]: generalized impulse p (lin, ang) as
  L.acch = o; o += 6 * sc.Bp;    //   64-bit fixed point, per-body scale (S6); 12 Bp words from accl
  o = (o + 3) & ~3;
  L.tq = o;   o += 4 * sc.T;     // float4 qd_s[T]
  L.tqp = o;  o += 4 * sc.T;     // float4 q[T] (step-start chain positions, read in S1)
  L.tL = o;   o += 16 * sc.T;    // float L[T][16]: 10 packed, 4 reciprocal diagonals, scale, -
  L.tacl = o; o += 4 * sc.T;     // uint32 chain impulse lo[T][4]
  L.tach = o; o += 4 * sc.T;     // int32  chain impulse hi[T][4]
  L.red = o;  o += 48;           // reductions: counters [0, 8), contact range [12, 16), per-warp KE [16, 48)
  L.total = (o + 3) & ~3;
  return L;
}

// persistent kernel: one group layout (+ two slab staging buffers + 2 mbarriers)
__host__ __device__ inline size_t persist_smem_bytes(const SceneDev& sc, bool stage) {
  return (size_t)(group_layout(sc).total + (stage ? 2 * N_BODY_PLANES * sc.Bp : 0)) * sizeof(float) + 16;
}

template <int WPW, int CW = kWarps>
__device__ __forceinline__ void group_sync(int group) {
  if (WPW == 1) {
    __syncwarp();
  } else if (WPW == CW) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(group + 1), "r"(WPW * 32) : "memory");
  }
}

// 128-bit streaming loads: read once, do not allocate in L1 (CF_LD_HINT 2:
// 256-byte L2 fetch granularity, measured neutral: 57.25 vs 57.24 us).
#ifndef CF_LD_HINT
#define CF_LD_HINT 0
#endif
#if CF_LD_HINT == 2
#define CF_LD_Q ".L2::256B"
#else
#define CF_LD_Q ""
#endif
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate" CF_LD_Q ".v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate" CF_LD_Q ".v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float3 cross3(float3 a, float3 b) {
  return make_float3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float dot3(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ float dot4(float4 a, float4 b) { return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w; }
#ifdef CF_TIMELINE
__device__ __forceinline__ unsigned tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return (unsigned)t;
}
#define TL_MARK(k)                                                                     \
  if (P.timeline && threadIdx.x == 0) {                                                \
    unsigned* tlp = P.timeline + 8 * (size_t)blockIdx.x;                               \
    if ((k) == 0) { unsigned sm; asm volatile("mov.u32 %0, %smid;" : "=r"(sm)); tlp[0] = sm; } \
    tlp[1 + (k)] = tl_now();                                                           \
  }
#else
#define TL_MARK(k)
#endif
__device__ __forceinline__ int tri(int i, int j) { return i * (i + 1) / 2 + j; }

// x <- (L L^T)^-1 x for a chain of nd <= 4 DoFs (forward then backward
// substitution); L[10 + i] holds 1 / L(i,i), precomputed once per step.
__device__ __forceinline__ void chol_solve(const float* L, int nd, float x[4]) {
  float y[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < nd) {
      float s = x[i];
#pragma unroll
      for (int j = 0; j < i; ++j) s -= L[tri(i, j)] * y[j];
      y[i] = s * L[10 + i];
    }
  }
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    if (i < nd) {
      float s = y[i];
#pragma unroll
      for (int j = i + 1; j < 4; ++j)
        if (j < nd) s -= L[tri(j, i)] * x[j];
      x[i] = s * L[10 + i];
    }
  }
}

// ||L^-1 v||^2 = v^T M^-1 v (forward substitution only)
__device__ __forceinline__ float chol_quad(const float* L, int nd, float4 v4) {
  const float v[4] = {v4.x, v4.y, v4.z, v4.w};
  float y[4] = {0.f, 0.f, 0.f, 0.f};
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < nd) {
      float s = v[i];
#pragma unroll
      for (int j = 0; j < i; ++j) s -= L[tri(i, j)] * y[j];
      y[i] = s * L[10 + i];
      acc += y[i] * y[i];
    }
  }
  return acc;
}

// Eq. (13): r(|phi|) with x clamped to [0, 1] (reading R7); branch-free.
template <bool FAST>
__device__ __forceinline__ float impedance_r(const StepParams& P, float phi) {
  const float x = fminf(fabsf(phi) * P.inv_width, 1.0f);
  const float m = P.mid;
  const float ulo = x * P.inv_mid, uhi = (1.0f - x) * P.inv_1m_mid;
  const float plo = FAST ? ulo * ulo : __powf(ulo, P.power);   // FAST: p = 2
  const float phi_ = FAST ? uhi * uhi : __powf(uhi, P.power);
  const float g = x < m ? m * plo : 1.0f - (1.0f - m) * phi_;
  return P.r_min + P.r_span * g;
}

// One symmetric facet pair (+d, -d) of a channel: L+- = (A +- a)_+.  The pair's
// contribution to the channel's friction sum is L+ - L- = 2a exactly while both
// are active (no cancellation against A).
__device__ __forceinline__ void facet_pair(float A, float a, float& Lp, float& Lm, float& diff) {
  Lp = fmaxf(A + a, 0.f);
  Lm = fmaxf(A - a, 0.f);
  diff = (A >= fabsf(a)) ? 2.f * a : Lp - Lm;
}

// Facets of one 2-D channel (tangential or rolling), d_j and d_{j+n/2} = -d_j:
// N += sum L, F += sum L d.  NT = 4 is the exact axis set and is only used for
// the first channel (tangential): it assigns N, F instead of adding to zero.
template <int NT, bool IMP>
__device__ __forceinline__ void channel2(float A, float kmu, float w1, float w2, const float2* dir, int n,
                                         float& N, float& F1, float& F2, int& act, float* out, float Mc) {
  if (NT == 4) {
    float L0, L2, d0, L1, L3, d1;
    facet_pair(A, kmu * w1, L0, L2, d0);
    facet_pair(A, kmu * w2, L1, L3, d1);
    N = (L0 + L2) + (L1 + L3);
    F1 = d0;
    F2 = d1;
    act += (L0 > 0.f) + (L1 > 0.f) + (L2 > 0.f) + (L3 > 0.f);
    if (IMP && out) { out[0] = Mc * L0; out[1] = Mc * L1; out[2] = Mc * L2; out[3] = Mc * L3; }
  } else {
    const int h = n >> 1;
    for (int j = 0; j < h; ++j) {
      const float2 d = dir[j];
      float Lp, Lm, df;
      facet_pair(A, kmu * fmaf(d.x, w1, d.y * w2), Lp, Lm, df);
      N += Lp + Lm;
      F1 = fmaf(df, d.x, F1);
      F2 = fmaf(df, d.y, F2);
      act += (Lp > 0.f) + (Lm > 0.f);
      if (IMP && out) { out[j] = Mc * Lp; out[j + h] = Mc * Lm; }
    }
  }
}

// S6 run aggregation.  Lanes hold (body key, 6 values); runs of equal keys in
// consecutive lanes are summed (Hillis-Steele inside each run, bounded by the
// longest run of the warp) and only each run's last lane then adds to shared
// memory.  When the warp's keys are mostly distinct (at least CF_DIRECT_RUNS
// runs of 32) the shuffles cost more than they save and every lane adds its own
// values directly (same-address lanes are serialised by the atomic unit).
// Returns true on the lanes that must add.
#ifndef CF_DIRECT_RUNS
#define CF_DIRECT_RUNS 16
#endif
__device__ __forceinline__ bool seg_sum6(int key, float v[6], int lane) {
  const unsigned full = 0xffffffffu;
  const int prev = __shfl_up_sync(full, key, 1);
#if CF_NEG_HEADS
  // lanes without a body to add to (static / chain side, key < 0) are runs of
  // their own: a warp of floor contacts needs no sums at all
  const bool head = lane == 0 || prev != key || key < 0;
#else
  const bool head = lane == 0 || prev != key;
#endif
  const unsigned heads = __ballot_sync(full, head);
  if (__popc(heads) >= CF_DIRECT_RUNS) return true;  // warp-uniform: direct adds
  const int next = __shfl_down_sync(full, key, 1);
  const bool tail = lane == 31 || next != key;
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

// ---- S6 accumulation: 64-bit fixed point in shared memory ----------------
// sm_100a has no native shared-memory fp32 add (atomicAdd compiles to a CAS
// loop), but native 32-bit integer atomics.  Each value is added as the 64-bit
// integer x = round(v * 2^e); integer addition is associative, so the result
// does not depend on the order in which warps arrive: the step is bitwise
// deterministic.  The scale 2^e is per body and per component group:
// e = exponent(m^-1) + 33 for the linear part, exponent(max diag I_w^-1) + 33
// for the angular part, i.e. a velocity resolution of about 2^-33 (1.2e-10).
// Carry form (default, CF_FX_SPLIT=0): lo/hi words of one 64-bit integer, the
// hi add takes the carry out of the lo add.  Split form (CF_FX_SPLIT=1, a
// variant): the lo plane receives the low 16 bits of x (unsigned) and the hi
// plane x >> 16, so neither atomic needs the other's result (no carry, no
// returned value); the sum is hi * 2^16 + lo exactly while a world has at most
// 65536 contacts (lo < 2^32) and |x| < 2^47 per add.  Both forms check every
// add against fx_threshold (below), so a sum can never wrap.
#ifndef CF_FX_SPLIT
#define CF_FX_SPLIT 0  // split: -0.6 us on C4 but its range is 2^15 times smaller (variant only)
#endif
static constexpr int kMaxWorldContacts = CF_FX_SPLIT ? 65536 : 0x7fffffff;
__device__ __forceinline__ int fx_exp(float inv) {
  const int e = inv > 0.f ? ((__float_as_int(inv) >> 23) & 0xff) - 127 : 0;
  return max(-90, min(90, e + 33));
}
__device__ __forceinline__ float fx_pow2(int e) { return __int_as_float((e + 127) << 23); }
// Body scales: 2^(exponent(inv) + 33) straight from the bits of inv (0 <= inv <
// 2^94, enforced by comfree_load_scene; inv = 0 gives 2^-94) and the exact
// inverse of such a power of two.
__device__ __forceinline__ float fx_scale(float inv) {
  return __int_as_float((__float_as_int(inv) & 0x7f800000) + (33 << 23));
}
__device__ __forceinline__ float fx_inv(float scale) { return __int_as_float((254 << 23) - __float_as_int(scale)); }
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void fx_add(unsigned* lo, int* hi, float v, float scale) {
#if CF_XU_TEST  // timing probe only (wrong beyond 2^31): is the 64-bit conversion on the XU pipe the limiter?
  const long long x = (long long)__float2int_rn(v * scale);
#else
  const long long x = __float2ll_rn(v * scale);
#endif
#if CF_FX_SPLIT
  atomicAdd(lo, (unsigned)x & 0xffffu);
  atomicAdd(hi, (int)(x >> 16));
#else
  const unsigned xl = (unsigned)x;
  const unsigned old = atomicAdd(lo, xl);
  int h;  // hi word + carry out of (old + xl): two instructions with the carry flag
  asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.s32 %0, %3, 0;\n\t}"
      : "=r"(h) : "r"(old), "r"(xl), "r"((int)(x >> 32)));
  atomicAdd(hi, h);
#endif
}
// The six components of one body: every lo-word atomic first (their return
// latencies overlap), then the carries and the six hi-word atomics -- instead
// of lo, wait, carry, hi per component (atomics keep program order, so the
// order of the source is the order of issue).
#ifndef CF_FX_BATCH
#define CF_FX_BATCH 1
#endif
#ifndef CF_HI_SKIP
#define CF_HI_SKIP 0
#endif
template <class LoAddr, class HiAddr>
__device__ __forceinline__ void fx_add6(LoAddr lo_of, HiAddr hi_of, const float v[6], float sl, float sa) {
#if CF_FX_SPLIT || !CF_FX_BATCH
#pragma unroll
  for (int q = 0; q < 6; ++q) fx_add(lo_of(q), hi_of(q), v[q], q < 3 ? sl : sa);
#else
  long long x[6];
  unsigned old[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) x[q] = __float2ll_rn(v[q] * (q < 3 ? sl : sa));
#pragma unroll
  for (int q = 0; q < 6; ++q) old[q] = atomicAdd(lo_of(q), (unsigned)x[q]);
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    int h;
    asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.s32 %0, %3, 0;\n\t}"
        : "=r"(h) : "r"(old[q]), "r"((unsigned)x[q]), "r"((int)(x[q] >> 32)));
#if CF_HI_SKIP  // skip a zero hi add (most adds): measured 57.32 vs 56.77 us, so not the default
    if (h != 0) atomicAdd(hi_of(q), h);
#else
    atomicAdd(hi_of(q), h);
#endif
  }
#endif
}

// Per-add range.  Every add is |x| = |v| * scale < thr, thr = 2^62 / (2 n_c + 2)
// for a world of n_c contacts (a body receives at most 2 n_c adds per
// component), so no sum can wrap and the 64-bit total stays below 2^62; the
// split form also needs |x| < 2^47.  The lanes keep a NaN-propagating running
// maximum of |v| * scale (max.NaN: a NaN impulse, which the float-to-int
// conversion would turn into 0, poisons it) and compare it once after the loop.
__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fx_mag(const float v[6], float sl, float sa) {
  const float ml = max_nan(max_nan(fabsf(v[0]), fabsf(v[1])), fabsf(v[2]));
  const float ma = max_nan(max_nan(fabsf(v[3]), fabsf(v[4])), fabsf(v[5]));
  return max_nan(ml * sl, ma * sa);
}
__device__ __forceinline__ float fx_threshold(int64_t n_contacts) {
  // carry form: the 64-bit sum stays below 2^62; split form: the hi plane's sum
  // of x >> 16 stays below 2^31, i.e. sum |x| < 2^47
  return (CF_FX_SPLIT ? 1.40737488e14f : 4.61168602e18f) / (float)(2 * n_contacts + 2);
}
__device__ __forceinline__ float fx_get(unsigned lo, int hi, float inv_scale) {
#if CF_FX_SPLIT
  const long long x = ((long long)hi << 16) + (long long)lo;
#else
  const long long x = (long long)(((unsigned long long)(unsigned)hi << 32) | (unsigned long long)lo);
#endif
  return __ll2float_rn(x) * inv_scale;
}

// S0 fused into the step for sorted input: one warp finds the first index with
// world id >= key0 and >= key1 in the sorted id array by 32-way search (each
// round one coalesced probe per lane; both searches advance together).
__device__ __forceinline__ int ld_id(const int32_t* p) {
  int r;
  asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
// Exact-guess probe: 16 lanes per key read a[g - 8, g + 8) around the uniform
// guess g = key n / n_keys (a[-1] = -inf, a[n] = +inf); issued early, consumed
// by lower_bound2 (worlds of equal size resolve with this one access).
__device__ __forceinline__ int probe_issue(const int32_t* a, int64_t n, int64_t n_keys, int64_t key0, int64_t key1,
                                           int lane) {
  const int64_t key = (lane >> 4) ? key1 : key0;
  const int64_t pp = (n_keys > 0 ? key * n / n_keys : 0) - 8 + (lane & 15);
  return pp < 0 ? INT_MIN : (pp < n ? ld_id(a + pp) : INT_MAX);
}
__device__ __forceinline__ void lower_bound2(const int32_t* a, int64_t n, int64_t n_keys, int64_t key0, int64_t key1,
                                             int lane, int probe, int64_t& r0, int64_t& r1) {
  const unsigned full = 0xffffffffu;
  int64_t lo0 = 0, hi0 = n, lo1 = 0, hi1 = n;  // answers in [lo, hi]
  {  // exact-guess round (probe_issue)
    const int64_t key = (lane >> 4) ? key1 : key0;
    const bool q = (int64_t)probe < key;
    const unsigned b = __ballot_sync(full, q);
    const unsigned b0 = b & 0xffffu, b1 = b >> 16;
    const int64_t g0 = (n_keys > 0 ? key0 * n / n_keys : 0) - 8, g1 = (n_keys > 0 ? key1 * n / n_keys : 0) - 8;
    // resolved when the window holds both a "< key" and a ">= key" position, or
    // touches an end of the array on the matching side
    const bool ok0 = (b0 & 1u) && !(b0 >> 15);
    const bool ok1 = (b1 & 1u) && !(b1 >> 15);
    if (ok0) lo0 = hi0 = g0 + __popc(b0);  // a resolved key keeps this answer in every later
    if (ok1) lo1 = hi1 = g1 + __popc(b1);  // round (adjacent worlds agree even on unsorted ids)
    if (ok0 && ok1) {
      r0 = lo0;
      r1 = lo1;
      return;
    }
  }
  const bool done0 = lo0 == hi0, done1 = lo1 == hi1;
  {  // first round: 16 lanes per key probe a window around the uniform guess k n / n_keys
    const int64_t avg = n_keys > 0 ? n / n_keys : n;
    const int64_t hw = 2 * avg + 32;
    const int half = lane >> 4, l = lane & 15;
    const int64_t key = half ? key1 : key0;
    int64_t g = (n_keys > 0 ? key * n / n_keys : 0) - hw;
    g = g < 0 ? 0 : (g > n ? n : g);
    const int64_t width = (2 * hw < n - g) ? 2 * hw : n - g;
    const int64_t step = (width + 15) / 16 > 0 ? (width + 15) / 16 : 1;
    const int64_t pp = g + l * step;
    const bool q = pp < n && ld_id(a + pp) < key;
    const unsigned b = __ballot_sync(full, q);
    const int k0 = __popc(b & 0xffffu), k1 = __popc(b >> 16);
    const int64_t g0 = __shfl_sync(full, g, 0), s0 = __shfl_sync(full, step, 0);
    const int64_t g1 = __shfl_sync(full, g, 16), s1 = __shfl_sync(full, step, 16);
    if (!done0) {
      if (k0 == 0) { lo0 = 0; hi0 = g0; }
      else if (k0 < 16) { lo0 = g0 + (k0 - 1) * s0 + 1; hi0 = g0 + k0 * s0; }
      else { lo0 = g0 + 15 * s0 + 1; hi0 = n; }
      if (lo0 > n) lo0 = n;
      if (hi0 > n) hi0 = n;
    }
    if (!done1) {
      if (k1 == 0) { lo1 = 0; hi1 = g1; }
      else if (k1 < 16) { lo1 = g1 + (k1 - 1) * s1 + 1; hi1 = g1 + k1 * s1; }
      else { lo1 = g1 + 15 * s1 + 1; hi1 = n; }
      if (lo1 > n) lo1 = n;
      if (hi1 > n) hi1 = n;
    }
  }
  while (hi0 - lo0 > 32 || hi1 - lo1 > 32) {
    const int64_t st0 = hi0 - lo0 > 32 ? (hi0 - lo0 + 31) / 32 : 1;
    const int64_t st1 = hi1 - lo1 > 32 ? (hi1 - lo1 + 31) / 32 : 1;
    const int64_t p0 = lo0 + lane * st0, p1 = lo1 + lane * st1;
    const bool q0 = p0 < hi0 && ld_id(a + p0) < key0;
    const bool q1 = p1 < hi1 && ld_id(a + p1) < key1;
    const int k0 = __popc(__ballot_sync(full, q0)), k1 = __popc(__ballot_sync(full, q1));
    if (hi0 - lo0 > 32) {
      const int64_t nlo = k0 ? lo0 + (k0 - 1) * st0 + 1 : lo0;
      const int64_t pk = lo0 + k0 * st0;
      hi0 = k0 == 0 ? lo0 : (k0 < 32 && pk < hi0 ? pk : hi0);
      lo0 = nlo;
    }
    if (hi1 - lo1 > 32) {
      const int64_t nlo = k1 ? lo1 + (k1 - 1) * st1 + 1 : lo1;
      const int64_t pk = lo1 + k1 * st1;
      hi1 = k1 == 0 ? lo1 : (k1 < 32 && pk < hi1 ? pk : hi1);
      lo1 = nlo;
    }
  }
  const int64_t p0 = lo0 + lane, p1 = lo1 + lane;
  const bool q0 = p0 < hi0 && ld_id(a + p0) < key0;
  const bool q1 = p1 < hi1 && ld_id(a + p1) < key1;
  r0 = lo0 + __popc(__ballot_sync(full, q0));
  r1 = lo1 + __popc(__ballot_sync(full, q1));
}

// Exact-diagonal impedance (Eq. (11), reading R24): one side's share of the
// facet's diagonal entry J~_f M^-1 J~_f^T for a facet row g = (gl, ga) acting on
// the contact twist.  Free body (record ix; static sides read the all-zero
// record): J_x^T g = (gl, r x gl + ga), M_x^-1 = diag(m^-1 I, I_w^-1).
__device__ __forceinline__ float side_quad_free(const float4* rec, int Bp, int ix, float3 r, float3 gl, float3 ga) {
  const float4 r0 = rec[ix], r1 = rec[Bp + ix], r2 = rec[2 * Bp + ix], r3 = rec[3 * Bp + ix];
  const float3 c = cross3(r, gl);
  const float3 u = make_float3(c.x + ga.x, c.y + ga.y, c.z + ga.z);
  const float Ixx = r1.w, Iyy = r2.w, Izz = r3.x, Ixy = r3.y, Ixz = r3.z, Iyz = r3.w;
  const float3 Iu = make_float3(Ixx * u.x + Ixy * u.y + Ixz * u.z, Ixy * u.x + Iyy * u.y + Iyz * u.z,
                                Ixz * u.x + Iyz * u.y + Izz * u.z);
  return r0.w * dot3(gl, gl) + dot3(u, Iu);
}
// Chain side: y = J_lin^T gl + J_ang^T ga over the chain's DoFs, y^T (L L^T)^-1 y.
__device__ __forceinline__ float side_quad_tree(const float4* jr, int64_t stride, const float* Ls, int nd, float3 gl,
                                                float3 ga) {
  const float gv[3] = {gl.x, gl.y, gl.z}, av[3] = {ga.x, ga.y, ga.z};
  float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int kk = 0; kk < 3; ++kk) {
    const float4 jl = jr[(size_t)kk * stride], ja = jr[(size_t)(kk + 3) * stride];
    y.x += jl.x * gv[kk] + ja.x * av[kk];
    y.y += jl.y * gv[kk] + ja.y * av[kk];
    y.z += jl.z * gv[kk] + ja.z * av[kk];
    y.w += jl.w * gv[kk] + ja.w * av[kk];
  }
  return chol_quad(Ls, nd, y);
}

// S6 for one side: run aggregation inside the warp, then the run's last lane
// adds its total (6 values) to the body's fixed-point accumulators.
// Accumulator of component q of body k: (lo, hi) words adjacent, so one
// address serves both atomics (planes of Bp uint2 per component).
#ifndef CF_ACC_PLANES
#define CF_ACC_PLANES 0
#endif
#if CF_ACC_PLANES  // lo words in planes 0-5, hi words in planes 6-11 (all 32 banks per plane)
#define ACC_LO(q, k) (accl + (q) * Bp + (k))
#define ACC_HI(q, k) (reinterpret_cast<int*>(accl) + (6 + (q)) * Bp + (k))
#else
#define ACC_LO(q, k) (accl + 2 * ((q) * Bp + (k)))
#define ACC_HI(q, k) (reinterpret_cast<int*>(accl) + 2 * ((q) * Bp + (k)) + 1)
#endif

template <bool RUNS, bool OWN>
__device__ __forceinline__ void scatter_side(unsigned* accl, const float4* rec, int Bp, int key, float v[6], int lane,
                                             float im_own, float dm_own, float& mag) {
  const bool tail = (!RUNS || seg_sum6(key, v, lane)) && key >= 0;
  if (tail) {
    // scales: OWN = from the run's last lane's own side-a record (registers of
    // S2; that lane's body is the run's body), else reloaded from shared memory
    // (chain variants, where the extra live registers cost more)
    float im = im_own, dmax = dm_own;
    if (!OWN) {
      const float* r = reinterpret_cast<const float*>(rec);
      im = r[4 * key + 3];
      dmax = fmaxf(fmaxf(r[4 * (Bp + key) + 3], r[4 * (2 * Bp + key) + 3]), r[4 * (3 * Bp + key)]);
    }
    const float sl = fx_scale(im), sa = fx_scale(dmax);
    mag = max_nan(mag, fx_mag(v, sl, sa));
    fx_add6([&](int q) { return ACC_LO(q, key); }, [&](int q) { return ACC_HI(q, key); }, v, sl, sa);
  }
}

// S6 for a side whose body record is still in registers (direct adds, no runs):
// the scales come from the lane's own m^-1 and max diag I_w^-1.
__device__ __forceinline__ void scatter_own(unsigned* accl, int Bp, int key, const float v[6], float im,
                                            float dmax, float& mag) {
  if (key >= 0) {
    const float sl = fx_scale(im), sa = fx_scale(dmax);
    mag = max_nan(mag, fx_mag(v, sl, sa));
    fx_add6([&](int q) { return ACC_LO(q, key); }, [&](int q) { return ACC_HI(q, key); }, v, sl, sa);
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// L2 prefetch of a world the step will reach later (its slab planes 0-12 and
// its first contacts), issued by one thread through the bulk-copy engine.
#ifndef CF_PF_CONTACTS
#define CF_PF_CONTACTS 512
#endif
__device__ __forceinline__ void prefetch_world_l2(const StepParams& P, int64_t w) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.slab + (size_t)w * P.sc.slab),
               "r"((uint32_t)(N_BODY_PLANES * P.sc.Bp * sizeof(float))) : "memory");
  if (CF_PF_CONTACTS > 0 && P.off) {
    const int64_t c0 = P.off[w], c1 = P.off[w + 1];
    const int64_t n = c1 - c0 < CF_PF_CONTACTS ? c1 - c0 : CF_PF_CONTACTS;
    if (n > 0) {
      const uint32_t nb = (uint32_t)(n * 16);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.c0 + c0), "r"(nb) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.c1 + c0), "r"(nb) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.c2 + c0), "r"(nb) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.c3 + c0), "r"(nb) : "memory");
    }
  }
}

// One world's step (S0-S8) by the world group `group` (WPW warps) of the CTA.
// stg: the world's slab planes 0-12 already staged in shared memory (the
// persistent kernel's TMA bulk copy), else null (S1 and S7 read the slab in HBM).
// GMEM: the world's working set (body records, fixed-point accumulators, chain
// data) lives in a global scratch slab (P.gscratch, L2-resident) instead of
// shared memory, for worlds too large for a CTA's 227 KB (about 2070 bodies):
// the same code with global loads and global integer atomics.
// Contact of the collision front-end's staging area (STG, comfree_step_collided):
// the placed record (point, phi), (normal, pair key g1 << 16 | g2) expanded to
// the step's four streams: the tangent of the normal exactly as the
// front-end's emit pass computes it (IEEE operations in its order, no
// contraction, so the step sees bit-identical records), the geometry's
// friction coefficients and condim, the bodies of the pair's geoms.
__device__ __forceinline__ void stg_expand(const StepParams& P, const float4 b, float4& c1, float4& c2, int4& c3) {
  const float nx = b.x, ny = b.y, nz = b.z;
  const uint32_t key = __float_as_uint(b.w);
  const int g1 = (int)(key >> 16), g2 = (int)(key & 0xffffu);
  const float sg = copysignf(1.f, nz);
  const float a = __fdiv_rn(-1.f, __fadd_rn(sg, nz));
  const float bb = __fmul_rn(__fmul_rn(nx, ny), a);
  const float t1x = __fadd_rn(1.f, __fmul_rn(__fmul_rn(__fmul_rn(sg, nx), nx), a));
  const float t1y = __fmul_rn(sg, bb), t1z = __fmul_rn(-sg, nx);
  c1 = make_float4(nx, ny, nz, P.st_mu_t);
  c2 = make_float4(t1x, t1y, t1z, P.st_mu_tor);
  c3 = make_int4(__ldg(&P.st_geom[g1].y), __ldg(&P.st_geom[g2].y), __float_as_int(P.st_mu_rol), P.st_condim);
}

template <int CW, int WPW, bool FAST, bool TREES, bool IMP, bool GMEM = false, bool STG = false>
__device__ __forceinline__ void world_step(const StepParams& P, float* smem, const int64_t w, const int group,
                                           const float* stg) {
  const SceneDev& sc = P.sc;
  const GroupLayout GL = group_layout(sc);
  constexpr int kGT = WPW * 32;
  const int gt = threadIdx.x % kGT;
  const int lane = threadIdx.x & 31;

  TL_MARK(0);
  float* G = GMEM ? P.gscratch + (size_t)w * GL.total : smem + (size_t)group * GL.total;
  float4* rec = reinterpret_cast<float4*>(G + GL.rec);
  unsigned* accl = reinterpret_cast<unsigned*>(G + GL.accl);
  float4* tq = reinterpret_cast<float4*>(G + GL.tq);
  float4* tqp = reinterpret_cast<float4*>(G + GL.tqp);
  float* tL = G + GL.tL;
  unsigned* tacl = reinterpret_cast<unsigned*>(G + GL.tacl);
  int* tach = reinterpret_cast<int*>(G + GL.tach);
  float* red = G + GL.red;
  int64_t* rng = reinterpret_cast<int64_t*>(red + 12);
  const int B = sc.B, Bp = sc.Bp, T = sc.T, nd = sc.nd;
  float* slab = P.slab + (size_t)w * sc.slab;
  const float dt = P.dt;
  const bool stats = IMP && P.wstats != nullptr;  // IMP: per-facet impulses and/or statistics requested

  // S0 (sorted input, fused): the first warp of the group issues its range probe
  // now and resolves it after its share of S1 (the probe's latency overlaps S1).
  int probe = 0;
  // contacts in use: the device-side count when given (the streams' capacity is P.n_contacts)
  const int64_t ncon = P.n_dev ? min(*P.n_dev, P.n_contacts) : P.n_contacts;
  if (P.world_sorted && (CF_EARLY_RANGE || gt < 32)) probe = probe_issue(P.world_sorted, ncon, P.n_worlds, w, w + 1, lane);
#ifndef CF_SELF_PF
#define CF_SELF_PF 1  // C4: 56.3 -> 55.4 us (profiles/r02_ab_kernel.txt)
#endif
  // the world's own slab planes requested into L2 by one bulk prefetch at the
  // start, so S1's second round of body loads waits on L2 rather than HBM
  if (CF_SELF_PF && gt == 0 && !stg && !GMEM)
    bulk_prefetch_l2(slab, (uint32_t)(N_BODY_PLANES * Bp * sizeof(float)));
  const float k = P.k, kappa_g = P.kappa;
  int n_active = 0;
  float max_pen = 0.f;
  float4 C0 = make_float4(0.f, 0.f, 0.f, 0.f), C1 = C0, C2 = C0;
  int4 C3 = make_int4(-1, -1, 0, 0);
  int base = gt & ~31;
  // ---------------- S1: smooth prediction (Kernel I) ----------------
  // record B (Bp >= B + 1) stays all zero: static and chain sides read it in S2
  if (gt < 4) rec[gt * Bp + B] = make_float4(0.f, 0.f, 0.f, 0.f);
  // body i: x, q, v, omega from the slab planes (from `stg` instead of the slab
  // for planes 0-11 when given), omega_z and the scene parameters passed in.
  // (Staging planes 0-11 with cp.async into the accumulator region before S1
  // was measured neutral on C4 and slower on C3.)
  auto s1_body = [&](int i, const float* stg, float omz, float im, float3 ib, float3 ibi) {
    const float* sp = stg ? stg + i : slab + i;
    const size_t pb = (size_t)Bp;
    const float3 x = make_float3(sp[0 * pb], sp[1 * pb], sp[2 * pb]);
    const float4 q = make_float4(sp[3 * pb], sp[4 * pb], sp[5 * pb], sp[6 * pb]);
    const float3 v = make_float3(sp[7 * pb], sp[8 * pb], sp[9 * pb]);
    const float3 om = make_float3(sp[10 * pb], sp[11 * pb], omz);
    // rotation of the normalised quaternion (reading R15)
    const float qn = rsqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    const float qw = q.x * qn, qx = q.y * qn, qy = q.z * qn, qz = q.w * qn;
    const float R00 = 1.f - 2.f * (qy * qy + qz * qz), R01 = 2.f * (qx * qy - qw * qz), R02 = 2.f * (qx * qz + qw * qy);
    const float R10 = 2.f * (qx * qy + qw * qz), R11 = 1.f - 2.f * (qx * qx + qz * qz), R12 = 2.f * (qy * qz - qw * qx);
    const float R20 = 2.f * (qx * qz - qw * qy), R21 = 2.f * (qy * qz + qw * qx), R22 = 1.f - 2.f * (qx * qx + qy * qy);
    // Iw^-1 = R diag(ib) R^T
    const float Ixx = R00 * R00 * ib.x + R01 * R01 * ib.y + R02 * R02 * ib.z;
    const float Iyy = R10 * R10 * ib.x + R11 * R11 * ib.y + R12 * R12 * ib.z;
    const float Izz = R20 * R20 * ib.x + R21 * R21 * ib.y + R22 * R22 * ib.z;
    const float Ixy = R00 * R10 * ib.x + R01 * R11 * ib.y + R02 * R12 * ib.z;
    const float Ixz = R00 * R20 * ib.x + R01 * R21 * ib.y + R02 * R22 * ib.z;
    const float Iyz = R10 * R20 * ib.x + R11 * R21 * ib.y + R12 * R22 * ib.z;
    float3 fl = make_float3(0.f, 0.f, 0.f), ta = make_float3(0.f, 0.f, 0.f);
    if (P.f_ext) {
      const float* fe = P.f_ext + ((size_t)w * B + i) * 6;
      fl = make_float3(fe[0], fe[1], fe[2]);
      ta = make_float3(fe[3], fe[4], fe[5]);
    }
    float3 vs = v;
    if (im > 0.f) {  // gravity only on translating bodies (reading R14)
      vs.x += (im * fl.x + P.g[0]) * dt;
      vs.y += (im * fl.y + P.g[1]) * dt;
      vs.z += (im * fl.z + P.g[2]) * dt;
    }
    // bias c = omega x (Iw omega), Iw = R diag(1/ib) R^T on unlocked axes
    // (ibi = I_b = 1/I_b^-1, 0 on locked axes, precomputed per scene)
    float3 wl = make_float3(R00 * om.x + R10 * om.y + R20 * om.z, R01 * om.x + R11 * om.y + R21 * om.z,
                            R02 * om.x + R12 * om.y + R22 * om.z);
    wl.x *= ibi.x;
    wl.y *= ibi.y;
    wl.z *= ibi.z;
    const float3 Iwo = make_float3(R00 * wl.x + R01 * wl.y + R02 * wl.z, R10 * wl.x + R11 * wl.y + R12 * wl.z,
                                   R20 * wl.x + R21 * wl.y + R22 * wl.z);
    const float3 gy = cross3(om, Iwo);
    const float3 rh = make_float3(ta.x - gy.x, ta.y - gy.y, ta.z - gy.z);
    const float3 ws = make_float3(om.x + (Ixx * rh.x + Ixy * rh.y + Ixz * rh.z) * dt,
                                  om.y + (Ixy * rh.x + Iyy * rh.y + Iyz * rh.z) * dt,
                                  om.z + (Ixz * rh.x + Iyz * rh.y + Izz * rh.z) * dt);
    rec[i] = make_float4(vs.x, vs.y, vs.z, im);
    rec[Bp + i] = make_float4(ws.x, ws.y, ws.z, Ixx);
    rec[2 * Bp + i] = make_float4(x.x, x.y, x.z, Iyy);
    rec[3 * Bp + i] = make_float4(Izz, Ixy, Ixz, Iyz);
  };
  auto s1_params = [&](int i, float& omz, float& im, float3& ib, float3& ibi) {
    const size_t pb = (size_t)Bp;
    omz = (stg ? stg : slab)[12 * pb + i];
    im = sc.inv_mass[i];
    ib = make_float3(sc.inv_inertia[i], sc.inv_inertia[pb + i], sc.inv_inertia[2 * pb + i]);
    ibi = make_float3(sc.inertia[i], sc.inertia[pb + i], sc.inertia[2 * pb + i]);
  };
#pragma unroll kS1Unroll
  for (int i = gt; i < B; i += kGT) {
    float omz, im;
    float3 ib, ibi;
    s1_params(i, omz, im, ib, ibi);
    s1_body(i, stg, omz, im, ib, ibi);
  }
  TL_MARK(5);
  // S0: the contact range of this world (CF_EARLY_RANGE: every warp resolves it
  // itself and issues its first contact loads before the group barrier;
  // otherwise the first warp resolves it and shares it through shared memory)
  int64_t e_b0 = 0, e_b1 = 0;
  if (CF_EARLY_RANGE && P.world_sorted) {
    lower_bound2(P.world_sorted, ncon, P.n_worlds, w, w + 1, lane, probe, e_b0, e_b1);
    if (e_b1 < e_b0) e_b1 = e_b0;  // unsorted ids (reported below)
  }
  if (P.world_sorted && gt < 32) {
    int64_t b0, b1;
    if (CF_EARLY_RANGE) { b0 = e_b0; b1 = e_b1; }
    else lower_bound2(P.world_sorted, ncon, P.n_worlds, w, w + 1, lane, probe, b0, b1);
    TL_MARK(4);
    if (lane == 0) {
      rng[0] = b0;
      rng[1] = b1;
      P.off_out[w] = b0;
      if (w == P.n_worlds - 1) P.off_out[w + 1] = b1;
      // coverage: ids below 0 precede world 0, ids >= n_worlds follow the last world
      if ((w == 0 && b0 != 0) || (w == P.n_worlds - 1 && b1 != ncon)) atomicOr(P.err, ERR_WORLD_RANGE);
      if (b1 < b0) {  // only possible when the ids are not sorted
        atomicOr(P.err, ERR_UNSORTED);
        rng[1] = b0;
      }
    }
  }
  int64_t cbeg = 0;
  int nloc = 0;
  int WID = (int)w;  // world id of the prefetched contact (fused S0 check)
  if (CF_EARLY_RANGE) {  // first contact of this lane in flight across the barrier
    cbeg = P.world_sorted ? e_b0 : P.off[w];
    nloc = (int)((P.world_sorted ? e_b1 : P.off[w + 1]) - cbeg);
    if (base + lane < nloc) {
      const int64_t g = cbeg + base + lane;
      C0 = ld_stream(P.c0 + g); C1 = ld_stream(P.c1 + g); C2 = ld_stream(P.c2 + g); C3 = ld_stream(P.c3 + g);
      if (P.world_sorted) WID = ld_id(P.world_sorted + g);
    }
  }
  {  // zero the accumulators (12 Bp words = 3 Bp uint4)
    uint4* z = reinterpret_cast<uint4*>(accl);
    for (int q = gt; q < 3 * Bp; q += kGT) z[q] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (TREES) {
    for (int t = gt; t < T; t += kGT) {
      const float* Lg = P.tree_L + ((size_t)w * T + t) * 10;
      float* Ls = tL + 16 * t;
#pragma unroll
      for (int k = 0; k < 10; ++k) Ls[k] = Lg[k];
      float dmax = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        Ls[10 + k] = k < nd ? 1.0f / Lg[tri(k, k)] : 0.f;
        dmax = fmaxf(dmax, Ls[10 + k] * Ls[10 + k]);
      }
      Ls[14] = __int_as_float(fx_exp(dmax));  // fixed-point exponent of this chain's impulses
      float x[4] = {0.f, 0.f, 0.f, 0.f}, qd[4] = {0.f, 0.f, 0.f, 0.f};
      const float* qv = slab + N_BODY_PLANES * Bp + sc.Qp + t * nd;
      const float* tau = P.tree_tau + (size_t)w * sc.Q + t * nd;
      float qq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nd) { x[j] = tau[j]; qd[j] = qv[j]; qq[j] = qv[j - sc.Qp]; }
      tqp[t] = make_float4(qq[0], qq[1], qq[2], qq[3]);
      chol_solve(Ls, nd, x);
      tq[t] = make_float4(qd[0] + x[0] * dt, qd[1] + x[1] * dt, qd[2] + x[2] * dt, qd[3] + x[3] * dt);
#pragma unroll
      for (int k = 0; k < 4; ++k) { tacl[4 * t + k] = 0u; tach[4 * t + k] = 0; }
    }
  }
  if (gt < 8) red[gt] = 0.f;
  group_sync<WPW, CW>(group);
  TL_MARK(1);
  // The world the CTA slot that frees next will start (P.pf_ahead worlds on:
  // the resident world slots of the grid) into L2 while this world runs, so
  // that world's prologue does not wait on HBM.
  if (P.pf_ahead > 0 && gt == 0 && !stg && w + P.pf_ahead < P.n_worlds) prefetch_world_l2(P, w + P.pf_ahead);

  // Contact range of this world.
  // STG: from the front-end's status word: a world whose records stayed in
  // the staging area reads them there (placed order, local indices); a world
  // the front-end wrote in place (more records than the staging area) reads
  // the public streams from its base, up to the whole-pair cut of the capacity
  bool staged = false;
  const float4* S0p = nullptr;
  const float4* S1p = nullptr;
  if (STG) {
    const unsigned long long sw = P.st_status[w];
    const int64_t total = (int64_t)(sw & ST_VAL);
    staged = !(sw & ST_DONE);
    if (staged) {
      cbeg = 0;
      nloc = (int)total;
      S0p = P.st_base + ((size_t)w * 4 + 2) * P.st_cap;
      S1p = S0p + P.st_cap;
    } else {
      cbeg = P.st_fbase[w];
      const int64_t cut = *P.st_cut;
      nloc = (int)max((int64_t)0, min(total, cut - cbeg));
    }
  } else if (!CF_EARLY_RANGE) {
    cbeg = P.world_sorted ? rng[0] : P.off[w];
    nloc = (int)((P.world_sorted ? rng[1] : P.off[w + 1]) - cbeg);
  }
  if (!STG && !P.world_sorted) {  // caller's off[]: monotone, inside [0, n], off[0] = 0, off[W] = n
    const int64_t cend = cbeg + nloc;
    if (cbeg < 0 || nloc < 0 || cend > ncon || (w == 0 && cbeg != 0) || (w == P.n_worlds - 1 && cend != ncon)) {
      if (gt == 0) atomicOr(P.err, ERR_WORLD_RANGE);
      cbeg = 0;
      nloc = 0;
    }
  }
  const float4* C0p = P.c0 + cbeg;
  const float4* C1p = P.c1 + cbeg;
  const float4* C2p = P.c2 + cbeg;
  const int4* C3p = P.c3 + cbeg;
  if (nloc > kMaxWorldContacts && gt == 0) atomicOr(P.err, ERR_WORLD_CONTACTS);  // S6 lo-plane bound
  float fx_mag_max = 0.f;  // S6: running max of |value| * scale over this lane's adds (NaN-propagating)
  const int32_t* Wp = P.world_sorted ? P.world_sorted + cbeg : nullptr;

  // ---------------- S2-S6: contacts ----------------
  // Warp-uniform loop: lane l of warp j handles local contact base + l; base
  // advances by the group's thread count; the next contact is prefetched.
  if (STG && staged) {
    if (base + lane < nloc) { C0 = ld_stream(S0p + base + lane); C1 = ld_stream(S1p + base + lane); }
  } else if (!CF_EARLY_RANGE && base + lane < nloc) {
    const int j = base + lane;
    C0 = ld_stream(C0p + j); C1 = ld_stream(C1p + j); C2 = ld_stream(C2p + j); C3 = ld_stream(C3p + j);
    if (Wp) WID = ld_id(Wp + j);
  }
#ifndef CF_ROLL_PF
#define CF_ROLL_PF 0
#endif
  for (; base < nloc; base += kGT) {
    const int j = base + lane;
#if CF_ROLL_PF
    // rolling bulk L2 prefetch: the group's contact block CF_ROLL_PF iterations
    // ahead, one bulk request per stream from the group's first lane
    if (gt == 0) {
      const int64_t pb = (int64_t)base + (int64_t)CF_ROLL_PF * kGT;
      if (pb < nloc) {
        const int64_t cnt = (nloc - pb) < kGT ? (nloc - pb) : kGT;
        const uint32_t nb = (uint32_t)(cnt * 16);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.c0 + cbeg + pb), "r"(nb) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.c1 + cbeg + pb), "r"(nb) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.c2 + cbeg + pb), "r"(nb) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.c3 + cbeg + pb), "r"(nb) : "memory");
      }
    }
#endif
    // Next-contact prefetch: free-body variants load it once this contact's
    // fields are dead (after S5), so the loads reuse the same registers (no
    // copies); chain variants load it here, at the top of the iteration.
#ifndef CF_EARLY_PF
#define CF_EARLY_PF 0
#endif
    constexpr bool kLatePrefetch = !TREES && !CF_EARLY_PF;
    const float4 c0 = C0;
    float4 c1 = C1, c2 = C2;
    int4 c3 = C3;
    if (STG && staged) stg_expand(P, C1, c1, c2, c3);
    const int wid = WID;
    auto prefetch_next = [&]() {  // index clamped: no branch
      const int jn = min(j + kGT, nloc - 1);
      if (STG && staged) {
        C0 = ld_stream(S0p + jn);
        C1 = ld_stream(S1p + jn);
        return;
      }
      // global index made opaque so the stream addresses are formed from the
      // kernel parameters each time (no per-stream 64-bit pointers held live)
      int64_t g = cbeg + jn;
      asm volatile("" : "+l"(g));
      if (!(CF_EARLY_C0 && kLatePrefetch)) C0 = ld_stream(P.c0 + g);
      C1 = ld_stream(P.c1 + g); C2 = ld_stream(P.c2 + g);
      if (!(CF_EARLY_C3 && kLatePrefetch && FAST)) {
        C3 = ld_stream(P.c3 + g);
        if (P.world_sorted) WID = ld_id(P.world_sorted + g);
      }
#if CF_L2AHEAD
      // one iteration further: pull the contact after next into L2 (no registers), so
      // the register prefetch above waits on L2 rather than HBM latency
      {
        int64_t g2 = cbeg + min(j + 2 * kGT, nloc - 1);
        asm volatile("" : "+l"(g2));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.c0 + g2));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.c1 + g2));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.c2 + g2));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.c3 + g2));
      }
#endif
    };
    if (!kLatePrefetch) prefetch_next();

    int ida = c3.x, idb = c3.y;
    const int cd = c3.w;
    // ids: free body in [0, B), static -1, chain -(2+t) with J rows; condim in {1,3,4,6}
    const int lo = TREES ? -1 - T : -1;
    const bool cd_ok = (unsigned)cd < 8u && ((0x5Au >> (cd & 7)) & 1u);
    const bool ids_ok = ida >= lo && idb >= lo && ida < B && idb < B && (ida != -1 || idb != -1) &&
                        (!TREES || P.jrow != nullptr || (ida >= -1 && idb >= -1));
    const bool in_range = j < nloc;
    const bool valid = in_range && cd_ok && ids_ok;
    const bool unsorted = in_range && wid != (int)w;  // fused S0 check
    if (__any_sync(0xffffffffu, (in_range && !valid) || unsorted)) {  // rare: one uniform branch
      if (unsorted) atomicOr(P.err, ERR_UNSORTED);
      if (in_range && !valid) atomicOr(P.err, cd_ok ? ERR_BODY_RANGE : ERR_CONDIM);
    }
    if (!valid) { ida = -1; idb = -1; }
    const float3 p = make_float3(c0.x, c0.y, c0.z);
    // S2: relative twist of b w.r.t. a, and the traces of S3.  Each side's
    // point velocity, angular velocity and trace are formed on their own and
    // combined once (no accumulation into zero-initialised sums).
    float3 vs2[2], ws2[2], rs2[2];
    float trs2[2], ims2[2], dms2[2];
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int id = side ? idb : ida;
      // free body (branch-free: a static or chain side reads the all-zero record B,
      // whose velocity, inverse mass and inverse inertia contribute exactly 0)
      const int ix = id >= 0 ? id : B;
      const float4 r0 = rec[ix], r1 = rec[Bp + ix], r2 = rec[2 * Bp + ix], r3 = rec[3 * Bp + ix];
      const float3 r = make_float3(p.x - r2.x, p.y - r2.y, p.z - r2.z);
      const float3 wxr = cross3(make_float3(r1.x, r1.y, r1.z), r);
      vs2[side] = make_float3(r0.x + wxr.x, r0.y + wxr.y, r0.z + wxr.z);
      ws2[side] = make_float3(r1.x, r1.y, r1.z);
      // tr(J M^-1 J^T) of the linear point Jacobian: 3 im + tr(I)|r|^2 - r^T I r
      const float Ixx = r1.w, Iyy = r2.w, Izz = r3.x, Ixy = r3.y, Ixz = r3.z, Iyz = r3.w;
      const float3 Ir = make_float3(Ixx * r.x + Ixy * r.y + Ixz * r.z, Ixy * r.x + Iyy * r.y + Iyz * r.z,
                                    Ixz * r.x + Iyz * r.y + Izz * r.z);
      trs2[side] = fmaf(3.f, r0.w, fmaf(Ixx + Iyy + Izz, dot3(r, r), -dot3(r, Ir)));
      rs2[side] = r;
      ims2[side] = r0.w;
      dms2[side] = fmaxf(fmaxf(Ixx, Iyy), Izz);
      if (TREES && id < -1) {
        const int t = -2 - id;
        const float4 qd = tq[t];
        const float* Ls = tL + 16 * t;
        const float4* jr = P.jrow + (size_t)(side * 6) * P.n_contacts + cbeg + j;
        float vp[3], wp[3];
        float trc = 0.f;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const float4 jl = ld_stream(jr + (size_t)kk * P.n_contacts);
          const float4 ja = ld_stream(jr + (size_t)(kk + 3) * P.n_contacts);
          vp[kk] = dot4(jl, qd);
          wp[kk] = dot4(ja, qd);
          trc += chol_quad(Ls, nd, jl);
        }
        // the all-zero record contributed exactly 0 above
        vs2[side] = make_float3(vp[0], vp[1], vp[2]);
        ws2[side] = make_float3(wp[0], wp[1], wp[2]);
        trs2[side] = trc;
      }
    }
    const float3 vrel = make_float3(vs2[1].x - vs2[0].x, vs2[1].y - vs2[0].y, vs2[1].z - vs2[0].z);
    const float3 wrel = make_float3(ws2[1].x - ws2[0].x, ws2[1].y - ws2[0].y, ws2[1].z - ws2[0].z);
    const float tr = trs2[0] + trs2[1];
    const float3 ra = rs2[0], rb = rs2[1];
    const float ima = ims2[0], dma = dms2[0], imb = ims2[1], dmb = dms2[1];  // S6 scales
    if (CF_EARLY_C3 && kLatePrefetch && FAST && !(STG && staged)) {  // the next contact's ids first: the loop head waits on them
      int64_t g = cbeg + min(j + kGT, nloc - 1);
      asm volatile("" : "+l"(g));
      C3 = ld_stream(P.c3 + g);
      if (CF_EARLY_C0) C0 = ld_stream(P.c0 + g);
      if (P.world_sorted) WID = ld_id(P.world_sorted + g);
    }
    // S3-S5, computed for every lane (invalid lanes are masked by select at the end)
    float3 f, tau = make_float3(0.f, 0.f, 0.f);
    {
      const float phi = c0.w;
      const float3 n = make_float3(c1.x, c1.y, c1.z);
      const float3 t1 = make_float3(c2.x, c2.y, c2.z);
      const float mu_t = c1.w;
      const float3 t2 = cross3(n, t1);
      const float un = dot3(n, vrel);
      if (stats) max_pen = fmaxf(max_pen, valid ? -phi : 0.f);
      // S3: M(phi) (Eq. (12)-(13))
      const float r = impedance_r<FAST>(P, phi);
      const float Mc = r * rcp_approx((1.f - r) * tr);
      // S4: Lambda_f = Mc (A + kappa mu (d . w))_+,  A = -k phi - kappa u_n,
      // with the contact's own (k_user, d_user) when given
      float kc = k, kappa = kappa_g;
      if (P.kd) {  // warp-uniform
        const float2 kd = P.kd[cbeg + min(j, max(nloc - 1, 0))];
        kc = kd.x;
        kappa = kd.x * P.dt + kd.y;
        // Eq. (11)'s split k dt : d (exact_diag == 1) needs kappa > 0
        if (valid && !(kd.x >= 0.f && kd.y >= 0.f && kd.x < INFINITY && kd.y < INFINITY &&
                       (FAST || P.exact_diag != 1 || kappa > 0.f)))
          atomicOr(P.err, ERR_IMPEDANCE);
      }
      const float A = -kc * phi - kappa * un;
      float N = 0.f, F1 = 0.f, F2 = 0.f;
      float* out = nullptr;
      if (IMP && P.impulses && valid) {
        const int64_t c = cbeg + j;
        const int64_t orig = P.perm ? (int64_t)P.perm[c] : c;
        const int64_t fb = P.foff[orig];
        const int nf = cd == 1 ? 1 : P.n_t + (cd >= 4 ? 2 : 0) + (cd == 6 ? P.n_rol : 0);
        if (fb + nf <= P.impulses_cap) out = P.impulses + fb;
        else atomicOr(P.err, ERR_IMPULSE_CAP);
      }
      const float wt1 = dot3(t1, vrel), wt2 = dot3(t2, vrel);
      int act_t = 0;
      channel2<FAST ? 4 : 0, IMP>(A, kappa * mu_t, wt1, wt2, P.dir_t, P.n_t, N, F1, F2, act_t,
                                   cd == 1 ? nullptr : out, Mc);
      if (cd == 1) {  // normal facet only: one row J_n
        N = fmaxf(A, 0.f);
        F1 = 0.f;
        F2 = 0.f;
        act_t = N > 0.f;
        if (IMP && out) out[0] = Mc * N;
      }
      if (stats) n_active += valid ? act_t : 0;
      if (!FAST && P.exact_diag) {  // warp-uniform: a facet's own diagonal entry A_f per facet
        // every facet f: row g_f = (gl, ga), s_f = g_f . (v_rel, w_rel),
        // A_f = J~_f M^-1 J~_f^T and Lambda_f = M_f (-k phi - kappa s_f)_+ with
        //   exact_diag 1, Eq. (11) literally (K_f dt + D_f = 1/(dt A_f), split
        //                 k dt : d, reading R24): M_f = 1 / (kappa A_f);
        //   exact_diag 2, Eq. (12) with the facet diagonal (reading R28):
        //                 M_f = r/(1-r) / A_f;
        // the contact wrench is (sum Lambda_f gl, sum Lambda_f ga)
        const bool eq11 = P.exact_diag == 1;
        const float rho = r * rcp_approx(1.f - r);
        const float mu_tor = c2.w, mu_rol = __int_as_float(c3.z);
        const int nf = cd == 1 ? 1 : P.n_t + (cd >= 4 ? 2 : 0) + (cd == 6 ? P.n_rol : 0);
        const int ixa = ida >= 0 ? ida : B, ixb = idb >= 0 ? idb : B;
        float3 fs = make_float3(0.f, 0.f, 0.f), ts = make_float3(0.f, 0.f, 0.f);
        int act = 0;
        for (int fi = 0; fi < nf; ++fi) {
          float3 gl = n, ga = make_float3(0.f, 0.f, 0.f);
          if (cd != 1) {
            if (fi < P.n_t) {
              const float2 d = P.dir_t[fi];
              gl = make_float3(n.x - mu_t * (d.x * t1.x + d.y * t2.x), n.y - mu_t * (d.x * t1.y + d.y * t2.y),
                               n.z - mu_t * (d.x * t1.z + d.y * t2.z));
            } else if (fi < P.n_t + 2) {
              const float sg = fi == P.n_t ? -mu_tor : mu_tor;
              ga = make_float3(sg * n.x, sg * n.y, sg * n.z);
            } else {
              const float2 d = P.dir_r[fi - P.n_t - 2];
              ga = make_float3(-mu_rol * (d.x * t1.x + d.y * t2.x), -mu_rol * (d.x * t1.y + d.y * t2.y),
                               -mu_rol * (d.x * t1.z + d.y * t2.z));
            }
          }
          const float sf = dot3(gl, vrel) + dot3(ga, wrel);
          float Af = side_quad_free(rec, Bp, ixa, ra, gl, ga) + side_quad_free(rec, Bp, ixb, rb, gl, ga);
          if (TREES) {
#pragma unroll
            for (int side = 0; side < 2; ++side) {
              const int id = side ? idb : ida;
              if (id < -1) {
                const float4* jr = P.jrow + (size_t)(side * 6) * P.n_contacts + cbeg + j;
                Af += side_quad_tree(jr, P.n_contacts, tL + 16 * (-2 - id), nd, gl, ga);
              }
            }
          }
          const float Lf = (eq11 ? rcp_approx(kappa * Af) : rho * rcp_approx(Af)) * fmaxf(-kc * phi - kappa * sf, 0.f);
          fs = make_float3(fs.x + Lf * gl.x, fs.y + Lf * gl.y, fs.z + Lf * gl.z);
          ts = make_float3(ts.x + Lf * ga.x, ts.y + Lf * ga.y, ts.z + Lf * ga.z);
          act += Lf > 0.f;
          if (IMP && out) out[fi] = Lf;
        }
        if (stats) n_active += valid ? act - act_t : 0;
        f = valid ? fs : make_float3(0.f, 0.f, 0.f);
        tau = valid ? ts : make_float3(0.f, 0.f, 0.f);
      } else {
      if (__any_sync(0xffffffffu, valid && cd >= 4)) {
        float Mt = 0.f, R1 = 0.f, R2 = 0.f;
        const float mu_tor = c2.w, mu_rol = __int_as_float(c3.z);
        if (cd >= 4) {
          const float wtor = dot3(n, wrel);
          float Lp, Lm;
          facet_pair(A, kappa * mu_tor * wtor, Lp, Lm, Mt);
          N += Lp + Lm;
          int act = (Lp > 0.f) + (Lm > 0.f);
          if (IMP && out) { out[P.n_t] = Mc * Lp; out[P.n_t + 1] = Mc * Lm; }
          if (cd == 6) {
            const float wr1 = dot3(t1, wrel), wr2 = dot3(t2, wrel);
            channel2<0, IMP>(A, kappa * mu_rol, wr1, wr2, P.dir_r, P.n_rol, N, R1, R2, act,
                             out ? out + P.n_t + 2 : nullptr, Mc);
          }
          if (stats) n_active += valid ? act : 0;
        }
        // S5 (angular part): tau = -Mc (mu_tor Mt n + mu_rol R . (t1, t2))
        const float mt = -mu_tor * Mt * Mc, mr1 = -mu_rol * R1 * Mc, mr2 = -mu_rol * R2 * Mc;
        tau = make_float3(mt * n.x + mr1 * t1.x + mr2 * t2.x, mt * n.y + mr1 * t1.y + mr2 * t2.y,
                          mt * n.z + mr1 * t1.z + mr2 * t2.z);
        if (!valid) tau = make_float3(0.f, 0.f, 0.f);
      }
      // S5: f = Mc (N n - mu_t F . (t1, t2))
      const float fn = Mc * N, ft1 = -mu_t * F1 * Mc, ft2 = -mu_t * F2 * Mc;
      f = make_float3(fn * n.x + ft1 * t1.x + ft2 * t2.x, fn * n.y + ft1 * t1.y + ft2 * t2.y,
                      fn * n.z + ft1 * t1.z + ft2 * t2.z);
      if (!valid) f = make_float3(0.f, 0.f, 0.f);
      }
    }
    if (kLatePrefetch) prefetch_next();
    // S6: scatter J^T (f, tau).  Free bodies get (f, r x f + tau) per side:
    // the warp sums runs of equal body ids (contacts sorted by body pair make
    // them long), then each run's last lane adds the total in fixed point.
    {
      const float3 ma = cross3(ra, f), mb = cross3(rb, f);
      float va[6] = {-f.x, -f.y, -f.z, -(ma.x + tau.x), -(ma.y + tau.y), -(ma.z + tau.z)};
      scatter_side<true, !TREES>(accl, rec, Bp, ida >= 0 ? ida : -1, va, lane, ima, dma, fx_mag_max);
      float vb[6] = {f.x, f.y, f.z, mb.x + tau.x, mb.y + tau.y, mb.z + tau.z};
#if CF_PROBE_B  // timing probe only (wrong results): side b adds to 32 distinct, bank-disjoint bodies
      for (int q = 0; q < 6; ++q) vb[q] *= 0.f;
      scatter_own(accl, Bp, idb >= 0 ? lane % B : -1, vb, imb, dmb, fx_mag_max);
#else
      scatter_own(accl, Bp, idb >= 0 ? idb : -1, vb, imb, dmb, fx_mag_max);
#endif
    }
    if (TREES) {
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int id = side ? idb : ida;
        if (id < -1) {  // chain side: J_lin^T f + J_ang^T tau into its DoFs
          const float sg = side ? 1.f : -1.f;
          const int t = -2 - id;
          const float4* jr = P.jrow + (size_t)(side * 6) * P.n_contacts + cbeg + j;
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
          const float scl = fx_pow2(__float_as_int(tL[16 * t + 14]));
          fx_mag_max = max_nan(fx_mag_max, max_nan(max_nan(fabsf(s4.x), fabsf(s4.y)), max_nan(fabsf(s4.z), fabsf(s4.w))) * scl);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            if (jj < nd) fx_add(tacl + 4 * t + jj, tach + 4 * t + jj, sg * sv[jj], scl);
        }
      }
    }
  }
  group_sync<WPW, CW>(group);
  TL_MARK(2);

  // ---------------- S7: velocity correction + integration (Kernel IV) ----------------
  float ke = 0.f;
  // S6 range: every add of this lane below the world's per-add bound (NaN fails)
  bool nonfinite = P.check_finite && !(fx_mag_max < fx_threshold(nloc));
  for (int i = gt; i < B; i += kGT) {
    const float4 r0 = rec[i], r1 = rec[Bp + i], r2 = rec[2 * Bp + i], r3 = rec[3 * Bp + i];
    float* sp = slab + i;
    const size_t pb = (size_t)Bp;
    const float* sq = stg ? stg + i : sp;  // step-start orientation
    const float4 q = make_float4(sq[3 * pb], sq[4 * pb], sq[5 * pb], sq[6 * pb]);
    const float im = r0.w;
    const float Ixx = r1.w, Iyy = r2.w, Izz = r3.x, Ixy = r3.y, Ixz = r3.z, Iyz = r3.w;
    const float isl = fx_inv(fx_scale(im)), isa = fx_inv(fx_scale(fmaxf(fmaxf(Ixx, Iyy), Izz)));
    int hi[6];
    unsigned range = 0u;
#pragma unroll
    for (int q6 = 0; q6 < 6; ++q6) {
      hi[q6] = *ACC_HI(q6, i);
      range |= (unsigned)hi[q6] + (1u << 30);  // bit 31 set: |hi| >= 2^30, fixed-point range exceeded
    }
    if (P.check_finite) nonfinite |= (range >> 31) != 0u;
    const float4 a0 = make_float4(fx_get(*ACC_LO(0, i), hi[0], isl), fx_get(*ACC_LO(1, i), hi[1], isl),
                                  fx_get(*ACC_LO(2, i), hi[2], isl), fx_get(*ACC_LO(3, i), hi[3], isa));
    const float2 a1 = make_float2(fx_get(*ACC_LO(4, i), hi[4], isa), fx_get(*ACC_LO(5, i), hi[5], isa));
    const float3 v = make_float3(r0.x + im * a0.x, r0.y + im * a0.y, r0.z + im * a0.z);
    const float3 om = make_float3(r1.x + Ixx * a0.w + Ixy * a1.x + Ixz * a1.y,
                                  r1.y + Ixy * a0.w + Iyy * a1.x + Iyz * a1.y,
                                  r1.z + Ixz * a0.w + Iyz * a1.x + Izz * a1.y);
    const float3 x = make_float3(r2.x + v.x * dt, r2.y + v.y * dt, r2.z + v.z * dt);
    // q+ = normalize(exp(omega dt / 2) (x) q), world-frame omega
    const float3 th = make_float3(om.x * dt, om.y * dt, om.z * dt);
    const float a2 = dot3(th, th);
    float s, ch;
    if (a2 < 0.0625f) {  // |omega dt| < 1/4: sin(h)/(2h), cos(h) by series, h = |omega dt|/2 (error < 1e-10)
      const float h2 = 0.25f * a2;
      s = 0.5f * (1.f - h2 * (1.f / 6.f - h2 * (1.f / 120.f - h2 * (1.f / 5040.f))));
      ch = 1.f - h2 * (0.5f - h2 * (1.f / 24.f - h2 * (1.f / 720.f)));
    } else {
      const float ang = sqrtf(a2);
      float sh;
      sincosf(0.5f * ang, &sh, &ch);
      s = sh / ang;
    }
    const float ew = ch, ex = s * th.x, ey = s * th.y, ez = s * th.z;
    float nw = ew * q.x - ex * q.y - ey * q.z - ez * q.w;
    float nx = ew * q.y + ex * q.x + ey * q.w - ez * q.z;
    float ny = ew * q.z - ex * q.w + ey * q.x + ez * q.y;
    float nz = ew * q.w + ex * q.z - ey * q.y + ez * q.x;
    const float inv = rsqrtf(nw * nw + nx * nx + ny * ny + nz * nz);
    nw *= inv; nx *= inv; ny *= inv; nz *= inv;
    sp[0 * pb] = x.x; sp[1 * pb] = x.y; sp[2 * pb] = x.z;
    sp[3 * pb] = nw; sp[4 * pb] = nx; sp[5 * pb] = ny; sp[6 * pb] = nz;
    sp[7 * pb] = v.x; sp[8 * pb] = v.y; sp[9 * pb] = v.z;
    sp[10 * pb] = om.x; sp[11 * pb] = om.y; sp[12 * pb] = om.z;
    if (P.check_finite) {
      const float chk = x.x + x.y + x.z + v.x + v.y + v.z + om.x + om.y + om.z + nw + nx + ny + nz;
      nonfinite |= !isfinite(chk);
    }
    if (stats) {
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
  if (TREES) {
    for (int t = gt; t < T; t += kGT) {
      const float* Ls = tL + 16 * t;
      const float isc = fx_pow2(-__float_as_int(Ls[14]));
      float x[4];
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) x[k4] = fx_get(tacl[4 * t + k4], tach[4 * t + k4], isc);
      chol_solve(Ls, nd, x);
      const float4 qs = tq[t], q0 = tqp[t];
      const float qsv[4] = {qs.x, qs.y, qs.z, qs.w}, q0v[4] = {q0.x, q0.y, q0.z, q0.w};
      float* qp = slab + N_BODY_PLANES * Bp + t * nd;
      float* qv = slab + N_BODY_PLANES * Bp + sc.Qp + t * nd;
      float qdn[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < nd) {
          qdn[j] = qsv[j] + x[j];
          qv[j] = qdn[j];
          const float qn = q0v[j] + qdn[j] * dt;
          qp[j] = qn;
          if (P.check_finite) nonfinite |= !isfinite(qn + qdn[j]);
        }
      }
      if (stats) {  // 1/2 qd^T L L^T qd
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          float y = 0.f;
#pragma unroll
          for (int j = i2; j < 4; ++j) y += j < nd ? Ls[tri(j, i2)] * qdn[j] : 0.f;
          ke += i2 < nd ? 0.5f * y * y : 0.f;
        }
      }
    }
  }
  TL_MARK(3);
  if (nonfinite) {
    atomicOr(P.err, ERR_NONFINITE);
    atomicMin(P.first_bad, (unsigned long long)(P.world_base + w));
  }
  if (stats) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      n_active += __shfl_xor_sync(0xffffffffu, n_active, o);
      max_pen = fmaxf(max_pen, __shfl_xor_sync(0xffffffffu, max_pen, o));
      ke += __shfl_xor_sync(0xffffffffu, ke, o);
    }
    if (lane == 0) {  // integer counters are order-free; energy is summed in warp order below
      atomicAdd(reinterpret_cast<int*>(&red[0]), n_active);
      atomicMax(reinterpret_cast<int*>(&red[1]), __float_as_int(fmaxf(max_pen, 0.f)));
      red[16 + (gt >> 5)] = ke;
    }
    group_sync<WPW, CW>(group);
    if (gt == 0) {
      comfree_world_stats ws;
      ws.contacts = nloc;
      ws.active_facets = *reinterpret_cast<int*>(&red[0]);
      ws.max_penetration = __int_as_float(*reinterpret_cast<int*>(&red[1]));
      float kes = 0.f;
      for (int q8 = 0; q8 < WPW; ++q8) kes += red[16 + q8];
      ws.kinetic_energy = kes;
      P.wstats[w] = ws;
    }
  }
}

template <int CW, int WPW, bool FAST, bool TREES, bool IMP, bool GMEM = false, bool STG = false>
__global__ void __launch_bounds__(CW * 32, CW == kWarps ? CF_MINB : (CW == 16 ? 2 : (CW == 32 ? 1 : 16))) k_step(const __grid_constant__ StepParams P) {
  extern __shared__ float4 smem4[];
  constexpr int kGroups = CW / WPW;
  const int group = threadIdx.x / (WPW * 32);
  const int64_t w = (int64_t)blockIdx.x * kGroups + group;
  if (w >= P.n_worlds) return;  // whole group leaves together
  world_step<CW, WPW, FAST, TREES, IMP, GMEM, STG>(P, reinterpret_cast<float*>(smem4), w, group, nullptr);
}

// ---- persistent variant: CTAs that step their worlds in turn ----
// CTA b (one world group of WPW warps) steps worlds b, b + G, b + 2G, ... (G =
// the grid, sized to the CTAs the SMs hold at once).  While it runs world k,
// one elected thread prepares world k + G:
//   STAGE: the Tensor Memory Accelerator's bulk copy engine (cp.async.bulk,
//          completion counted on an mbarrier) brings the next world's slab
//          planes 0-12 (x, q, v, omega: 52 B per body, one contiguous range)
//          into the second of two shared-memory staging buffers, so S1 of the
//          next world starts from shared memory;
//   else:  the next world's slab is prefetched into L2
//          (cp.async.bulk.prefetch.L2);
// and in both cases the first contacts of the next world are prefetched into
// L2.  The next world's prologue then no longer waits on HBM latency, which in
// the one-world-per-CTA kernel stalls every SM at the start and again when the
// second wave of CTAs starts together.
#ifndef CF_PERSIST_PF_CONTACTS
#define CF_PERSIST_PF_CONTACTS 512  // contacts of the next world prefetched into L2 (per stream)
#endif
template <bool STAGE>
__device__ __forceinline__ void prepare_world(const StepParams& P, float* buf, uint64_t* bar, int64_t w) {
  const uint32_t bytes = (uint32_t)(N_BODY_PLANES * P.sc.Bp * sizeof(float));
  const float* src = P.slab + (size_t)w * P.sc.slab;
  if (STAGE) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of buf precede the async write
    mbar_expect_tx(bar, bytes);
    bulk_g2s(buf, src, bytes, bar);
  } else {
    bulk_prefetch_l2(src, bytes);
  }
  if (CF_PERSIST_PF_CONTACTS > 0 && P.off) {  // the first contacts of the next world into L2
    const int64_t c0 = P.off[w], c1 = P.off[w + 1];
    const int64_t n = c1 - c0 < CF_PERSIST_PF_CONTACTS ? c1 - c0 : CF_PERSIST_PF_CONTACTS;
    if (n > 0) {
      const uint32_t nb = (uint32_t)(n * 16);
      bulk_prefetch_l2(P.c0 + c0, nb);
      bulk_prefetch_l2(P.c1 + c0, nb);
      bulk_prefetch_l2(P.c2 + c0, nb);
      bulk_prefetch_l2(P.c3 + c0, nb);
    }
  }
}

// Worlds are handed out by a global ticket counter (P.queue[0]), one world
// ahead: a CTA that finishes early takes the next unclaimed world, so the SMs
// stay balanced whichever CTAs they hold.  The last CTA to finish resets the
// counters for the next launch (stream order makes the reset visible to it).
template <int WPW, bool STAGE, bool FAST, bool IMP>
__global__ void __launch_bounds__(WPW * 32, 32 / WPW) k_step_persist(const __grid_constant__ StepParams P) {
  extern __shared__ float4 smem4[];
  __shared__ int64_t s_next;
  float* smem = reinterpret_cast<float*>(smem4);
  const GroupLayout GL = group_layout(P.sc);
  const int stage_f = STAGE ? N_BODY_PLANES * P.sc.Bp : 0;
  float* buf0 = smem + GL.total;
  float* buf1 = buf0 + stage_f;
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf1 + stage_f);
  int64_t w = 0, nxt = 0;
  if (threadIdx.x == 0) {
    w = atomicAdd(&P.queue[0], 1);
    nxt = atomicAdd(&P.queue[0], 1);
    if (STAGE) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (w < P.n_worlds) prepare_world<true>(P, buf0, &bar[0], w);
    }
    s_next = w;
  }
  __syncthreads();
  w = s_next;
  for (int k = 0; w < P.n_worlds; ++k) {
    const int b = k & 1;
    // the next world: staged into the other buffer (free: its last reader, the
    // previous world's S7, finished before the barrier that ended that world)
    // or prefetched into L2
    if (threadIdx.x == 0 && nxt < P.n_worlds) prepare_world<STAGE>(P, b ? buf0 : buf1, &bar[b ^ 1], nxt);
    if (STAGE) mbar_wait(&bar[b], (uint32_t)((k >> 1) & 1));
    world_step<WPW, WPW, FAST, false, IMP>(P, smem, w, 0, STAGE ? (b ? buf1 : buf0) : nullptr);
    if (threadIdx.x == 0) {
      s_next = nxt;
      nxt = nxt < P.n_worlds ? atomicAdd(&P.queue[0], 1) : nxt;
    }
    __syncthreads();  // S7 done with rec / acc / the staging buffer before the next world
    w = s_next;
    __syncthreads();  // s_next read before it is rewritten
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&P.queue[1], 1) == (int)gridDim.x - 1) {  // last CTA: reset for the next launch
      P.queue[0] = 0;
      P.queue[1] = 0;
    }
  }
}

template <int WPW, bool STAGE, bool FAST, bool IMP>
cudaError_t launch_persist_variant(const StepParams& p, cudaStream_t s, int n_sm) {
  const size_t smem = persist_smem_bytes(p.sc, STAGE);
  cudaError_t e = cudaFuncSetAttribute(k_step_persist<WPW, STAGE, FAST, IMP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step_persist<WPW, STAGE, FAST, IMP>, WPW * 32, smem);
  if (e != cudaSuccess) return e;
  const int64_t slots = (int64_t)n_sm * (per_sm > 0 ? per_sm : 1);
  const unsigned grid = (unsigned)(p.n_worlds < slots ? p.n_worlds : slots);
  if (grid == 0) return cudaSuccess;
  k_step_persist<WPW, STAGE, FAST, IMP><<<grid, WPW * 32, smem, s>>>(p);
  return cudaGetLastError();
}

template <int CW, int WPW, bool FAST, bool TREES, bool IMP, bool GMEM = false, bool STG = false>
cudaError_t launch_variant(const StepParams& p, cudaStream_t s) {
  const int groups = CW / WPW;
  const size_t smem = GMEM ? 0 : (size_t)groups * group_layout(p.sc).total * sizeof(float);
  const unsigned grid = (unsigned)((p.n_worlds + groups - 1) / groups);
  if (grid == 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_step<CW, WPW, FAST, TREES, IMP, GMEM, STG>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  StepParams q = p;
  q.pf_ahead = 0;
  const char* pf = getenv("COMFREE_PF");  // opt-in (measured +1.6 us on C4): next-world L2 prefetch
  if (pf && atoi(pf) != 0) {
    int dev = 0, n_sm = 0, per_sm = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step<CW, WPW, FAST, TREES, IMP, GMEM, STG>, CW * 32, smem) == cudaSuccess &&
        (int64_t)grid > (int64_t)n_sm * per_sm)
      q.pf_ahead = (int64_t)n_sm * per_sm * groups;  // worlds resident at once
  }
  k_step<CW, WPW, FAST, TREES, IMP, GMEM, STG><<<grid, CW * 32, smem, s>>>(q);
  return cudaGetLastError();
}

// FAST = the 4-facet tangential cone with the default power p = 2 (dense piles);
// every other configuration takes the general facet loop and __powf.
template <int CW, int WPW>
cudaError_t launch_cfg(const StepParams& p, cudaStream_t s) {
    const bool trees = p.sc.T > 0, imp = p.impulses != nullptr || p.wstats != nullptr;
  if (WPW == kWarps && p.gscratch) {  // worlds beyond shared memory: the global-scratch variant (general facets)
    if (trees) return imp ? launch_variant<CW, WPW, false, true, true, true>(p, s) : launch_variant<CW, WPW, false, true, false, true>(p, s);
    return imp ? launch_variant<CW, WPW, false, false, true, true>(p, s) : launch_variant<CW, WPW, false, false, false, true>(p, s);
  }
  if (p.st_status) {  // contacts from the front-end's staging area (comfree_step_collided: FAST, no chains, no outputs)
    if (trees || imp || !(p.n_t == 4 && p.power_is_2 && !p.exact_diag) || p.gscratch) return cudaErrorInvalidValue;
    return launch_variant<CW, WPW, true, false, false, false, true>(p, s);
  }
  if (p.n_t == 4 && p.power_is_2 && !p.exact_diag) {
    if (trees) return imp ? launch_variant<CW, WPW, true, true, true>(p, s) : launch_variant<CW, WPW, true, true, false>(p, s);
    return imp ? launch_variant<CW, WPW, true, false, true>(p, s) : launch_variant<CW, WPW, true, false, false>(p, s);
  }
  if (trees) return imp ? launch_variant<CW, WPW, false, true, true>(p, s) : launch_variant<CW, WPW, false, true, false>(p, s);
  return imp ? launch_variant<CW, WPW, false, false, true>(p, s) : launch_variant<CW, WPW, false, false, false>(p, s);
}

template <int WPW>
cudaError_t launch_wpw(const StepParams& p, cudaStream_t s) {
  return launch_cfg<kWarps, WPW>(p, s);
}

}  // namespace cf
