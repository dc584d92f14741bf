// capi.cpp — host side of the C ABI (include/comfree.h): validation,
// library-owned device memory, stream-ordered dispatch of S0 and the fused
// step kernel, host-buffer staging and latched device errors.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "comfree.h"
#include "internal.h"

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

cudaError_t ensure(DevBuf& b, size_t bytes) {
  if (b.p && b.cap >= bytes) return cudaSuccess;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  size_t nb = std::max<size_t>(256, bytes + bytes / 4);
  cudaError_t e = cudaMalloc(&b.p, nb);
  if (e == cudaSuccess) b.cap = nb;
  return e;
}

void release(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
}

int64_t round4(int64_t x) { return (x + 3) & ~int64_t(3); }

}  // namespace

struct comfree_ctx {
  comfree_config cfg{};
  int device = 0;
  std::string err;
  bool loaded = false;
  cf::SceneDev sc{};
  int64_t W = 0;
  float* slab = nullptr;
  float* inv_mass = nullptr;
  float* inv_inertia = nullptr;
  comfree_world_stats* wstats = nullptr;
  int* d_err = nullptr;
  int* d_queue = nullptr;  // persistent step kernel's world queue: [ticket, CTAs done] (self-resetting)
  unsigned long long* d_first_bad = nullptr;
  // S0 scratch
  DevBuf off, keys, perm, iota, s0, s1, s2, s3, sj, skd, nf, foff, cub_tmp;
  // host-input staging
  DevBuf in_world, in_off, in_c0, in_c1, in_c2, in_c3, in_jrow, in_kd, in_fext, in_L, in_tau, imp;
  DevBuf st_tmp;
  DevBuf gscratch;  // step working sets of worlds beyond shared memory
  // COMFREE_MEM_HOST_ASYNC: two staging slots, a copy-in and a copy-out stream
  struct AsyncSlot {
    DevBuf world, off, c0, c1, c2, c3, jrow, kd, fext, L, tau, out;
  } aslot[2];
  int a_in = 0, a_out = 0;               // next slot of comfree_step / comfree_get_state
  cudaStream_t s_h2d = nullptr, s_h2d2 = nullptr, s_d2h = nullptr;  // two copy-in streams (two copy engines)
  cudaEvent_t ev_h2d2[2] = {nullptr, nullptr};
  cudaEvent_t ev_entry = nullptr, ev_h2d[2] = {nullptr, nullptr}, ev_conv[2] = {nullptr, nullptr},
              ev_d2h[2] = {nullptr, nullptr};
  // articulated upstream: device copy of the chain model (comfree_load_articulation)
  DevBuf art;
  bool art_loaded = false;
  // collision front-end: device geometry (comfree_load_geometry) and scan scratch
  DevBuf geo, col_counts, col_offs, col_tmp, col_frames;
  DevBuf bp_status, bp_queue, bp_count, bp_stage;   // broadphase mode scratch
  // comfree_step_collided: library-owned contact streams (records of worlds the
  // front-end writes in place), per-world in-place bases, and the staged-source
  // description the step picks up (active only inside that call)
  DevBuf fs_world, fs_c0, fs_c1, fs_c2, fs_c3, fs_link, bp_fbase;
  int64_t* bp_fbase_hook = nullptr;  // set by comfree_step_collided for its collide call
  struct {
    bool active = false;
    const unsigned long long* status = nullptr;
    const float4* stage = nullptr;
    int64_t cap = 0;
    const int64_t* fbase = nullptr;
    const int64_t* cut = nullptr;
  } stg;
  int32_t n_geoms = 0, n_pairs = 0;
  float col_margin = 0.f, col_mu[3] = {0.f, 0.f, 0.f};
  int32_t col_condim = 3;
  bool geo_loaded = false;
  int64_t launches = 0;
  int64_t last_first = 0, last_nw = 0, last_nc = 0;
  bool last_sorted_copy = false;
  bool stats_valid = false;
  float2 dir_t[32], dir_r[32];
  // instrumentation: event pairs recorded on the step's stream
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_step, ev_seg;  // indices into ev_pool
  size_t ev_used = 0;
};

namespace {

comfree_status fail(comfree_ctx* ctx, comfree_status s, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return s;
}

#define CUDA_TRY(ctx, expr)                                                                  \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(ctx, COMFREE_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),   \
                  __FILE__, __LINE__);                                                       \
  } while (0)

bool finite(float x) { return std::isfinite(x); }

// Eq. (7): symmetric unit directions d_j = (cos 2 pi j/n, sin 2 pi j/n); exact
// zeros / ones where the angle is a multiple of a quarter turn.
void directions(int n, float2* out) {
  for (int j = 0; j < 32; ++j) out[j] = make_float2(0.f, 0.f);
  for (int j = 0; j < n && j < 32; ++j) {
    double th = 2.0 * M_PI * j / n;
    double c = std::cos(th), s = std::sin(th);
    if (std::fabs(c) < 1e-12) c = 0.0;
    if (std::fabs(s) < 1e-12) s = 0.0;
    if (std::fabs(std::fabs(c) - 1.0) < 1e-12) c = c > 0 ? 1.0 : -1.0;
    if (std::fabs(std::fabs(s) - 1.0) < 1e-12) s = s > 0 ? 1.0 : -1.0;
    out[j] = make_float2((float)c, (float)s);
  }
}

// Lazily created streams / events of the asynchronous host path.
cudaError_t async_init(comfree_ctx* ctx) {
  if (ctx->s_h2d) return cudaSuccess;
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->s_h2d2, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_entry, cudaEventDisableTiming);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&ctx->ev_h2d[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_h2d2[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_conv[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_d2h[k], cudaEventDisableTiming);
  }
  return e;
}

comfree_status check_latched(comfree_ctx* ctx, cudaStream_t s) {
  CUDA_TRY(ctx, cudaStreamSynchronize(s));
  int e = 0;
  unsigned long long bad = ~0ull;
  CUDA_TRY(ctx, cudaMemcpy(&e, ctx->d_err, sizeof e, cudaMemcpyDeviceToHost));
  if (e == 0) return COMFREE_OK;
  CUDA_TRY(ctx, cudaMemcpy(&bad, ctx->d_first_bad, sizeof bad, cudaMemcpyDeviceToHost));
  const int zero = 0;
  const unsigned long long none = ~0ull;
  CUDA_TRY(ctx, cudaMemcpy(ctx->d_err, &zero, sizeof zero, cudaMemcpyHostToDevice));
  CUDA_TRY(ctx, cudaMemcpy(ctx->d_first_bad, &none, sizeof none, cudaMemcpyHostToDevice));
  if (e & cf::ERR_CONTACT_CAP)
    return fail(ctx, COMFREE_ERR_CAPACITY, "collide: more contacts than the output capacity (flags 0x%x)", e);
  if (e & cf::ERR_CANDIDATES)
    return fail(ctx, COMFREE_ERR_CAPACITY, "collide: more broadphase candidate pairs in a world than fit shared memory (flags 0x%x)", e);
  if (e & (cf::ERR_UNSORTED | cf::ERR_WORLD_RANGE | cf::ERR_BODY_RANGE | cf::ERR_CONDIM | cf::ERR_IMPULSE_CAP |
           cf::ERR_IMPEDANCE | cf::ERR_WORLD_CONTACTS | cf::ERR_ARTICULATION))
    return fail(ctx, COMFREE_ERR_VALIDATION, "device validation failed (flags 0x%x):%s%s%s%s%s%s%s%s", e,
                (e & cf::ERR_UNSORTED) ? " contacts not sorted by world;" : "",
                (e & cf::ERR_WORLD_RANGE) ? " world id out of range or off[] inconsistent;" : "",
                (e & cf::ERR_BODY_RANGE) ? " body id out of range or chain side without J rows;" : "",
                (e & cf::ERR_CONDIM) ? " condim not in {1,3,4,6};" : "",
                (e & cf::ERR_IMPULSE_CAP) ? " impulses buffer too small;" : "",
                (e & cf::ERR_IMPEDANCE) ? " per-contact impedance negative or non-finite;" : "",
                (e & cf::ERR_WORLD_CONTACTS) ? " more than 65536 contacts in one world;" : "",
                (e & cf::ERR_ARTICULATION) ? " articulation: M(q) not positive definite or bad chain/link id;" : "");
  return fail(ctx, COMFREE_ERR_NONFINITE, "non-finite state (or impulse beyond the fixed-point range) in world %lld",
              (long long)bad);
}

// Copy a caller buffer to device staging when it lives on the host.
template <typename T>
comfree_status stage(comfree_ctx* ctx, DevBuf& buf, const T* src, size_t count, int loc, cudaStream_t s,
                     const T** out) {
  if (!src || loc == COMFREE_MEM_DEVICE) {
    *out = src;
    return COMFREE_OK;
  }
  CUDA_TRY(ctx, ensure(buf, count * sizeof(T)));
  // HOST_ASYNC: s is the context's copy-in stream, buf the step's staging slot
  CUDA_TRY(ctx, cudaMemcpyAsync(buf.p, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
  *out = static_cast<const T*>(buf.p);
  return COMFREE_OK;
}

cudaEvent_t next_event(comfree_ctx* ctx, int* idx) {
  if (ctx->ev_used == ctx->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    ctx->ev_pool.push_back(e);
  }
  *idx = (int)ctx->ev_used;
  return ctx->ev_pool[ctx->ev_used++];
}

}  // namespace

#ifdef CF_BP_TIMELINE
extern "C" int comfree_debug_bp_timeline(comfree_ctx* ctx, unsigned long long* host, int64_t n_worlds) {
  return cudaMemcpy(host, ctx->col_frames.p, (size_t)n_worlds * 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}
#endif
#ifdef CF_TIMELINE
// Tuning builds only: per-CTA phase timestamps of the last step launch.
static unsigned* g_tl = nullptr;
static unsigned* cf_debug_timeline_buf() {
  if (!g_tl) cudaMalloc(&g_tl, sizeof(unsigned) * 8 * (1 << 20));
  return g_tl;
}
extern "C" int comfree_debug_timeline(unsigned* host, int64_t n_ctas) {
  if (!g_tl) return -1;
  return (int)cudaMemcpy(host, g_tl, sizeof(unsigned) * 8 * n_ctas, cudaMemcpyDeviceToHost);
}
#endif

extern "C" {

int comfree_abi_version(void) { return COMFREE_ABI_VERSION; }

const char* comfree_status_string(comfree_status s) {
  switch (s) {
    case COMFREE_OK: return "ok";
    case COMFREE_ERR_INVALID_ARGUMENT: return "invalid argument";
    case COMFREE_ERR_VALIDATION: return "validation error";
    case COMFREE_ERR_CAPACITY: return "capacity exceeded";
    case COMFREE_ERR_NONFINITE: return "non-finite state";
    case COMFREE_ERR_CUDA: return "CUDA error";
    case COMFREE_ERR_STATE: return "invalid call order";
  }
  return "unknown status";
}

comfree_status comfree_default_config(comfree_config* c) {
  if (!c) return COMFREE_ERR_INVALID_ARGUMENT;
  c->k_user = 0.1f;
  c->d_user = 0.001f;
  c->r_min = 0.9f;    // P:233 defaults
  c->r_max = 0.95f;
  c->width = 0.001f;
  c->midpoint = 0.5f;
  c->power = 2.0f;
  c->n_t = 4;
  c->n_rol = 4;
  c->gravity[0] = 0.f;
  c->gravity[1] = 0.f;
  c->gravity[2] = -9.81f;
  c->flags = 0;
  return COMFREE_OK;
}

comfree_status comfree_validate_config(const comfree_config* c) {
  if (!c) return COMFREE_ERR_INVALID_ARGUMENT;
  bool ok = finite(c->k_user) && c->k_user > 0 && finite(c->d_user) && c->d_user >= 0;
  ok = ok && c->r_min > 0 && c->r_min <= c->r_max && c->r_max < 1;
  ok = ok && finite(c->width) && c->width > 0 && c->midpoint > 0 && c->midpoint < 1;
  ok = ok && finite(c->power) && c->power >= 1;
  ok = ok && c->n_t >= 4 && c->n_t <= 32 && c->n_t % 2 == 0;
  ok = ok && c->n_rol >= 2 && c->n_rol <= 32 && c->n_rol % 2 == 0;
  ok = ok && finite(c->gravity[0]) && finite(c->gravity[1]) && finite(c->gravity[2]);
  // one impedance model at a time
  ok = ok && !((c->flags & COMFREE_FLAG_EXACT_DIAGONAL) && (c->flags & COMFREE_FLAG_FACET_DIAGONAL));
  return ok ? COMFREE_OK : COMFREE_ERR_VALIDATION;
}

static constexpr float kMaxInv = 1e27f;

comfree_status comfree_validate_scene(const comfree_scene* s) {
  if (!s) return COMFREE_ERR_INVALID_ARGUMENT;
  if (s->n_bodies < 0 || s->n_trees < 0) return COMFREE_ERR_VALIDATION;
  if (s->n_bodies > 0 && (!s->inv_mass || !s->inv_inertia)) return COMFREE_ERR_INVALID_ARGUMENT;
  if (s->n_trees > 0 && (s->tree_ndof < 1 || s->tree_ndof > 4)) return COMFREE_ERR_VALIDATION;
  for (int i = 0; i < s->n_bodies; ++i) {
    // finite, >= 0 and <= kMaxInv (the S6 fixed-point scale 2^(exponent + 33) stays a normal float)
    if (!(finite(s->inv_mass[i]) && s->inv_mass[i] >= 0 && s->inv_mass[i] <= kMaxInv)) return COMFREE_ERR_VALIDATION;
    for (int k = 0; k < 3; ++k)
      if (!(finite(s->inv_inertia[3 * i + k]) && s->inv_inertia[3 * i + k] >= 0 && s->inv_inertia[3 * i + k] <= kMaxInv))
        return COMFREE_ERR_VALIDATION;
  }
  return COMFREE_OK;
}

int32_t comfree_facets_per_contact(const comfree_config* c, int32_t condim) {
  if (!c) return -1;
  switch (condim) {
    case 1: return 1;
    case 3: return c->n_t;
    case 4: return c->n_t + 2;
    case 6: return c->n_t + 2 + c->n_rol;
  }
  return -1;
}

comfree_status comfree_create(const comfree_config* cfg, int device, comfree_ctx** out) {
  if (!cfg || !out) return COMFREE_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  comfree_status v = comfree_validate_config(cfg);
  if (v != COMFREE_OK) return v;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return COMFREE_ERR_CUDA;
  }
  comfree_ctx* ctx = new (std::nothrow) comfree_ctx();
  if (!ctx) return COMFREE_ERR_CAPACITY;
  ctx->cfg = *cfg;
  ctx->device = device;
  directions(cfg->n_t, ctx->dir_t);
  directions(cfg->n_rol, ctx->dir_r);
  if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(&ctx->d_err, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&ctx->d_first_bad, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&ctx->d_queue, 2 * sizeof(int)) != cudaSuccess) {
    delete ctx;
    return COMFREE_ERR_CUDA;
  }
  const unsigned long long none = ~0ull;
  cudaMemset(ctx->d_err, 0, sizeof(int));
  cudaMemset(ctx->d_queue, 0, 2 * sizeof(int));
  cudaMemcpy(ctx->d_first_bad, &none, sizeof none, cudaMemcpyHostToDevice);
  *out = ctx;
  return COMFREE_OK;
}

static comfree_status set_state_impl(comfree_ctx* ctx, int64_t first, int64_t nw, const comfree_state* in,
                                     cudaStream_t s) {
  const cf::SceneDev& sc = ctx->sc;
  const float *pos = in ? in->pos : nullptr, *quat = in ? in->quat : nullptr, *vel = in ? in->vel : nullptr,
              *om = in ? in->omega : nullptr, *qp = in ? in->qpos : nullptr, *qv = in ? in->qvel : nullptr;
  if (in && in->location == COMFREE_MEM_HOST) {
    const size_t nb = (size_t)nw * sc.B, nq = (size_t)nw * sc.Q;
    const size_t total = nb * 13 + nq * 2;
    CUDA_TRY(ctx, ensure(ctx->st_tmp, std::max<size_t>(1, total) * sizeof(float)));
    float* d = static_cast<float*>(ctx->st_tmp.p);
    float* dp[6] = {d, d + 3 * nb, d + 7 * nb, d + 10 * nb, d + 13 * nb, d + 13 * nb + nq};
    const float* hp[6] = {pos, quat, vel, om, qp, qv};
    const size_t cnt[6] = {3 * nb, 4 * nb, 3 * nb, 3 * nb, nq, nq};
    const float* res[6];
    for (int k = 0; k < 6; ++k) {
      res[k] = nullptr;
      if (hp[k] && cnt[k]) {
        CUDA_TRY(ctx, cudaMemcpyAsync(dp[k], hp[k], cnt[k] * sizeof(float), cudaMemcpyHostToDevice, s));
        res[k] = dp[k];
      }
    }
    pos = res[0]; quat = res[1]; vel = res[2]; om = res[3]; qp = res[4]; qv = res[5];
  }
  CUDA_TRY(ctx, cf::launch_public_to_slab(pos, quat, vel, om, qp, qv, nw, sc, ctx->slab + (size_t)first * sc.slab, s));
  ctx->launches += 1;
  if (in && in->location == COMFREE_MEM_HOST) CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return COMFREE_OK;
}

comfree_status comfree_load_scene(comfree_ctx* ctx, const comfree_scene* scene, int64_t n_worlds,
                                  const comfree_state* initial) {
  if (!ctx || !scene || n_worlds < 0) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "load_scene: bad argument");
  comfree_status v = comfree_validate_scene(scene);
  if (v != COMFREE_OK) return fail(ctx, v, "load_scene: scene violates an invariant (masses, inertias >= 0, 1 <= tree_ndof <= 4)");
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  if (ctx->slab) { cudaFree(ctx->slab); ctx->slab = nullptr; }
  if (ctx->inv_mass) { cudaFree(ctx->inv_mass); ctx->inv_mass = nullptr; }
  if (ctx->inv_inertia) { cudaFree(ctx->inv_inertia); ctx->inv_inertia = nullptr; }
  if (ctx->wstats) { cudaFree(ctx->wstats); ctx->wstats = nullptr; }
  ctx->loaded = false;
  cf::SceneDev& sc = ctx->sc;
  sc.B = scene->n_bodies;
  sc.Bp = (int)round4(scene->n_bodies + 1);  // + the all-zero body record the step reads for static sides
  sc.T = scene->n_trees;
  sc.nd = scene->n_trees ? scene->tree_ndof : 0;
  sc.Q = sc.T * sc.nd;
  sc.Qp = (int)round4(sc.Q);
  sc.slab = cf::N_BODY_PLANES * sc.Bp + 2 * sc.Qp;
  ctx->W = n_worlds;
  const size_t slab_bytes = std::max<size_t>(16, (size_t)n_worlds * sc.slab * sizeof(float));
  CUDA_TRY(ctx, cudaMalloc(&ctx->slab, slab_bytes));
  CUDA_TRY(ctx, cudaMalloc(&ctx->inv_mass, sc.Bp * sizeof(float)));
  CUDA_TRY(ctx, cudaMalloc(&ctx->inv_inertia, 6 * sc.Bp * sizeof(float)));
  CUDA_TRY(ctx, cudaMalloc(&ctx->wstats, std::max<int64_t>(1, n_worlds) * sizeof(comfree_world_stats)));
  std::string h(7 * sc.Bp * sizeof(float), '\0');
  float* hm = reinterpret_cast<float*>(&h[0]);
  for (int i = 0; i < sc.Bp; ++i) {
    hm[i] = i < sc.B ? scene->inv_mass[i] : 0.f;
    for (int k = 0; k < 3; ++k) {
      const float ib = i < sc.B ? scene->inv_inertia[3 * i + k] : 0.f;
      hm[sc.Bp + k * sc.Bp + i] = ib;
      hm[4 * sc.Bp + k * sc.Bp + i] = ib > 0.f ? 1.0f / ib : 0.f;
    }
  }
  CUDA_TRY(ctx, cudaMemcpy(ctx->inv_mass, hm, sc.Bp * sizeof(float), cudaMemcpyHostToDevice));
  CUDA_TRY(ctx, cudaMemcpy(ctx->inv_inertia, hm + sc.Bp, 6 * sc.Bp * sizeof(float), cudaMemcpyHostToDevice));
  sc.inv_mass = ctx->inv_mass;
  sc.inv_inertia = ctx->inv_inertia;
  sc.inertia = ctx->inv_inertia + 3 * sc.Bp;
  ctx->loaded = true;
  comfree_status st = set_state_impl(ctx, 0, n_worlds, initial, 0);
  if (st != COMFREE_OK) return st;
  CUDA_TRY(ctx, cudaDeviceSynchronize());
  ctx->stats_valid = false;
  return COMFREE_OK;
}

// Warps per world.  An SM holds 32 warps of the step kernel (64 registers) and
// as many worlds as fit its 228 KB of shared memory; the world group gets the
// warps the SM can spare per resident world (rounded up to a power of two),
// but no more than its work needs (about one lane per contact or body).
// Measured on B200 (profiles/r01_wpw_sweep.txt): B = 500 -> 8 at every contact
// count, pile-lite (B = 100, 400 contacts) -> 2, hand (20 contacts) -> 1.
static int pick_wpw(const cf::SceneDev& sc, int64_t n_contacts, int64_t n_worlds) {
  const int64_t avgc = n_worlds ? n_contacts / n_worlds : 0;
  const int64_t work = std::max<int64_t>(sc.B + sc.T, avgc);
  const int cap = work <= 32 ? 1 : work <= 64 ? 2 : work <= 128 ? 4 : 8;
  const size_t world_smem = cf::step_smem_bytes(sc, 8) + 256;   // one group per CTA at 8 warps
  const int64_t worlds_per_sm = std::max<int64_t>(1, (int64_t)(228 * 1024 / world_smem));
  int want = 1;
  while (want < 8 && want * worlds_per_sm < 32) want *= 2;
  int wpw = std::min(want, cap);
  while (wpw < 8 && cf::step_smem_bytes(sc, wpw) > 200 * 1024) wpw *= 2;
  return wpw;
}

comfree_status comfree_step(comfree_ctx* ctx, const comfree_worlds* wd, const comfree_contacts* c, float dt,
                            void* stream) {
  if (!ctx) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "step before load_scene");
  if (!wd || !c) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step: null descriptor");
  if (!(dt > 0) || !finite(dt)) return fail(ctx, COMFREE_ERR_VALIDATION, "step: dt must be finite and > 0");
  const int64_t first = wd->first_world, nw = wd->n_worlds, n = c->n_contacts;
  if (first < 0 || nw < 0 || first + nw > ctx->W) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step: world range outside the loaded batch");
  if (n < 0 || n > INT32_MAX) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step: n_contacts out of range");
  if (n > 0 && (!c->c0 || !c->c1 || !c->c2 || !c->c3)) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step: contact streams required");
  if (n > 0 && !c->off && !c->world) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step: world[] or off[] required");
  const cf::SceneDev& sc = ctx->sc;
  if (sc.T > 0 && nw > 0 && (!wd->tree_L || !wd->tree_tau)) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step: chains need tree_L and tree_tau");
  if (c->location != COMFREE_MEM_DEVICE && c->location != COMFREE_MEM_HOST && c->location != COMFREE_MEM_HOST_ASYNC)
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step: bad contacts location");
  if ((c->location == COMFREE_MEM_HOST_ASYNC) != (wd->location == COMFREE_MEM_HOST_ASYNC) &&
      !(c->location == COMFREE_MEM_HOST_ASYNC && !wd->f_ext && !wd->tree_L && !wd->tree_tau))
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step: HOST_ASYNC contacts and world inputs go together");
  if (c->location == COMFREE_MEM_HOST_ASYNC && (c->impulses || c->foff || c->n_device))
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step: HOST_ASYNC takes no impulses / foff / n_device");
  if (c->impulses && c->impulses_capacity < 0) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step: impulses_capacity");
  if (c->n_device && (!(c->flags & COMFREE_CONTACTS_SORTED) || !c->world || c->off || c->impulses || c->foff ||
                      c->location != COMFREE_MEM_DEVICE))
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT,
                "step: n_device needs sorted DEVICE contacts with world[] and no off[] / impulses / foff");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const bool async_io = c->location == COMFREE_MEM_HOST_ASYNC;
  const int loc = async_io ? COMFREE_MEM_HOST : c->location;
  const bool host_io = !async_io && ((loc == COMFREE_MEM_HOST) || (wd->location == COMFREE_MEM_HOST));
  // HOST_ASYNC: the inputs go to staging slot a_in over the copy-in stream,
  // which first waits for the caller's stream to reach this call (so slot
  // a_in's previous user, two steps back, has finished with it); the caller's
  // stream then waits for the copies, and the call returns without a sync.
  cudaStream_t s_stage = s;
  comfree_ctx::AsyncSlot* as = nullptr;
  int aslot = 0;
  if (async_io) {
    CUDA_TRY(ctx, async_init(ctx));
    aslot = ctx->a_in;
    ctx->a_in ^= 1;
    as = &ctx->aslot[aslot];
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_entry, s));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->s_h2d, ctx->ev_entry, 0));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->s_h2d2, ctx->ev_entry, 0));
    s_stage = ctx->s_h2d;
  }

  // ---- stage inputs ----
  const int32_t* world = nullptr;
  const int64_t* off_in = nullptr;
  const float *c0 = nullptr, *c1 = nullptr, *c2 = nullptr, *jrow = nullptr;
  const int32_t* c3 = nullptr;
  comfree_status st;
  DevBuf& b_world = as ? as->world : ctx->in_world;
  DevBuf& b_off = as ? as->off : ctx->in_off;
  DevBuf& b_c0 = as ? as->c0 : ctx->in_c0;
  DevBuf& b_c1 = as ? as->c1 : ctx->in_c1;
  DevBuf& b_c2 = as ? as->c2 : ctx->in_c2;
  DevBuf& b_c3 = as ? as->c3 : ctx->in_c3;
  DevBuf& b_jrow = as ? as->jrow : ctx->in_jrow;
  DevBuf& b_kd = as ? as->kd : ctx->in_kd;
  DevBuf& b_fext = as ? as->fext : ctx->in_fext;
  DevBuf& b_L = as ? as->L : ctx->in_L;
  DevBuf& b_tau = as ? as->tau : ctx->in_tau;
  if ((st = stage(ctx, b_world, c->off ? nullptr : c->world, (size_t)n, loc, s_stage, &world)) != COMFREE_OK) return st;
  if ((st = stage(ctx, b_off, c->off, (size_t)nw + 1, loc, s_stage, &off_in)) != COMFREE_OK) return st;
  if ((st = stage(ctx, b_c0, c->c0, (size_t)n * 4, loc, s_stage, &c0)) != COMFREE_OK) return st;
  if ((st = stage(ctx, b_c1, c->c1, (size_t)n * 4, loc, s_stage, &c1)) != COMFREE_OK) return st;
  // streams c2, c3 over the second copy-in stream (a second copy engine)
  cudaStream_t s_stage2 = async_io ? ctx->s_h2d2 : s;
  if ((st = stage(ctx, b_c2, c->c2, (size_t)n * 4, loc, s_stage2, &c2)) != COMFREE_OK) return st;
  if ((st = stage(ctx, b_c3, c->c3, (size_t)n * 4, loc, s_stage2, &c3)) != COMFREE_OK) return st;
  if ((st = stage(ctx, b_jrow, c->jrow, (size_t)n * 48, loc, s_stage, &jrow)) != COMFREE_OK) return st;
  const float* kdp = nullptr;
  if ((st = stage(ctx, b_kd, c->kd, (size_t)n * 2, loc, s_stage, &kdp)) != COMFREE_OK) return st;
  const float *fext = nullptr, *tL = nullptr, *ttau = nullptr;
  const int wloc = async_io ? COMFREE_MEM_HOST : wd->location;
  if ((st = stage(ctx, b_fext, wd->f_ext, (size_t)nw * sc.B * 6, wloc, s_stage, &fext)) != COMFREE_OK) return st;
  if ((st = stage(ctx, b_L, sc.T ? wd->tree_L : nullptr, (size_t)nw * sc.T * 10, wloc, s_stage, &tL)) != COMFREE_OK) return st;
  if ((st = stage(ctx, b_tau, sc.T ? wd->tree_tau : nullptr, (size_t)nw * sc.Q, wloc, s_stage, &ttau)) != COMFREE_OK) return st;
  if (async_io) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_h2d[aslot], ctx->s_h2d));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_h2d2[aslot], ctx->s_h2d2));
    CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_h2d[aslot], 0));
    CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_h2d2[aslot], 0));
  }

  // ---- S0: segmentation ----
  const int64_t* off = off_in;
  const int32_t* perm = nullptr;
  const float4 *k0 = (const float4*)c0, *k1 = (const float4*)c1, *k2 = (const float4*)c2, *kj = (const float4*)jrow;
  const float2* kk = (const float2*)kdp;
  const int4* k3 = (const int4*)c3;
  ctx->last_sorted_copy = false;
  const int32_t* fused_world = nullptr;
  int seg_e0 = -1, seg_e1 = -1;
  const bool stg_mode = ctx->stg.active;  // contacts from the front-end's staging area (comfree_step_collided)
  if (!off && ctx->timing && !(c->flags & COMFREE_CONTACTS_SORTED) && !stg_mode) {
    cudaEvent_t e = next_event(ctx, &seg_e0);
    if (e) cudaEventRecord(e, s);
  }
  if (!off && !stg_mode) {
    CUDA_TRY(ctx, ensure(ctx->off, (size_t)(nw + 1) * sizeof(int64_t)));
    int64_t* doff = static_cast<int64_t*>(ctx->off.p);
    if ((c->flags & COMFREE_CONTACTS_SORTED) && (n > 0 || c->n_device)) {
      // fused S0: the step kernel locates each world's range and verifies the ids
      fused_world = world;
    } else if (c->flags & COMFREE_CONTACTS_SORTED) {
      // no contacts (world[] may be null): every offset is 0
      CUDA_TRY(ctx, cf::launch_offsets_sorted(world, 0, nw, doff, ctx->d_err, s));
    } else {
      CUDA_TRY(ctx, ensure(ctx->keys, std::max<size_t>(1, n) * sizeof(int32_t)));
      CUDA_TRY(ctx, ensure(ctx->perm, std::max<size_t>(1, n) * sizeof(int32_t)));
      CUDA_TRY(ctx, ensure(ctx->iota, std::max<size_t>(1, n) * sizeof(int32_t)));
      size_t tb = 0;
      CUDA_TRY(ctx, cf::sort_by_world(world, n, nw, nullptr, nullptr, nullptr, nullptr, &tb, s));
      CUDA_TRY(ctx, ensure(ctx->cub_tmp, tb));
      tb = ctx->cub_tmp.cap;
      CUDA_TRY(ctx, cf::launch_check_world_range(world, n, nw, ctx->d_err, s));
      CUDA_TRY(ctx, cf::launch_iota(static_cast<int32_t*>(ctx->iota.p), n, s));
      if (n > 0)
        CUDA_TRY(ctx, cf::sort_by_world(world, n, nw, static_cast<int32_t*>(ctx->keys.p), static_cast<int32_t*>(ctx->perm.p),
                                        static_cast<int32_t*>(ctx->iota.p), ctx->cub_tmp.p, &tb, s));
      CUDA_TRY(ctx, cf::launch_offsets_sorted(static_cast<int32_t*>(ctx->keys.p), n, nw, doff, ctx->d_err, s));
      CUDA_TRY(ctx, ensure(ctx->s0, std::max<size_t>(1, n) * 16));
      CUDA_TRY(ctx, ensure(ctx->s1, std::max<size_t>(1, n) * 16));
      CUDA_TRY(ctx, ensure(ctx->s2, std::max<size_t>(1, n) * 16));
      CUDA_TRY(ctx, ensure(ctx->s3, std::max<size_t>(1, n) * 16));
      if (jrow) CUDA_TRY(ctx, ensure(ctx->sj, std::max<size_t>(1, n) * 16 * 12));
      if (kk) CUDA_TRY(ctx, ensure(ctx->skd, std::max<size_t>(1, n) * 8));
      CUDA_TRY(ctx, cf::launch_gather_contacts(static_cast<int32_t*>(ctx->perm.p), n, k0, k1, k2, k3, kj, kk,
                                               (float4*)ctx->s0.p, (float4*)ctx->s1.p, (float4*)ctx->s2.p,
                                               (int4*)ctx->s3.p, jrow ? (float4*)ctx->sj.p : nullptr,
                                               kk ? (float2*)ctx->skd.p : nullptr, s));
      ctx->launches += 5;
      k0 = (const float4*)ctx->s0.p; k1 = (const float4*)ctx->s1.p; k2 = (const float4*)ctx->s2.p;
      k3 = (const int4*)ctx->s3.p; kj = jrow ? (const float4*)ctx->sj.p : nullptr;
      kk = kk ? (const float2*)ctx->skd.p : nullptr;
      perm = static_cast<int32_t*>(ctx->perm.p);
      ctx->last_sorted_copy = true;
    }
    off = doff;
    if (seg_e0 >= 0) {
      cudaEvent_t e = next_event(ctx, &seg_e1);
      if (e) {
        cudaEventRecord(e, s);
        ctx->ev_seg.push_back({seg_e0, seg_e1});
      }
    }
  }

  // ---- facet offsets for impulse output ----
  const int64_t* foff = nullptr;
  float* imp = nullptr;
  int64_t imp_cap = 0;
  if (c->impulses || c->foff) {
    CUDA_TRY(ctx, ensure(ctx->foff, (size_t)(n + 1) * sizeof(int64_t)));
    CUDA_TRY(ctx, ensure(ctx->nf, (size_t)(n + 1) * sizeof(int32_t)));
    size_t tb = 0;
    CUDA_TRY(ctx, cf::facet_offsets(nullptr, n, ctx->cfg.n_t, ctx->cfg.n_rol, nullptr, nullptr, nullptr, &tb, nullptr, s));
    CUDA_TRY(ctx, ensure(ctx->cub_tmp, std::max(tb, ctx->cub_tmp.cap)));
    tb = ctx->cub_tmp.cap;
    CUDA_TRY(ctx, cf::facet_offsets((const int4*)c3, n, ctx->cfg.n_t, ctx->cfg.n_rol, static_cast<int32_t*>(ctx->nf.p),
                                    static_cast<int64_t*>(ctx->foff.p), ctx->cub_tmp.p, &tb, ctx->d_err, s));
    ctx->launches += 2;
    foff = static_cast<const int64_t*>(ctx->foff.p);
    if (c->impulses) {
      imp_cap = c->impulses_capacity;
      if (loc == COMFREE_MEM_HOST) {
        CUDA_TRY(ctx, ensure(ctx->imp, std::max<size_t>(1, imp_cap) * sizeof(float)));
        imp = static_cast<float*>(ctx->imp.p);
      } else {
        imp = c->impulses;
      }
    }
  }

  // ---- fused step ----
  cf::StepParams P{};
  const comfree_config& cf_ = ctx->cfg;
  P.k = cf_.k_user;
  P.d = cf_.d_user;
  P.kappa = cf_.k_user * dt + cf_.d_user;
  P.dt = dt;
  P.r_min = cf_.r_min;
  P.r_span = cf_.r_max - cf_.r_min;
  P.inv_width = 1.0f / cf_.width;
  P.mid = cf_.midpoint;
  P.inv_mid = 1.0f / cf_.midpoint;
  P.inv_1m_mid = 1.0f / (1.0f - cf_.midpoint);
  P.power = cf_.power;
  P.power_is_2 = cf_.power == 2.0f;
  for (int k = 0; k < 3; ++k) P.g[k] = cf_.gravity[k];
  P.n_t = cf_.n_t;
  P.n_rol = cf_.n_rol;
  std::memcpy(P.dir_t, ctx->dir_t, sizeof P.dir_t);
  std::memcpy(P.dir_r, ctx->dir_r, sizeof P.dir_r);
  P.sc = sc;
  P.slab = ctx->slab + (size_t)first * sc.slab;
  P.n_worlds = nw;
  P.f_ext = fext;
  P.tree_L = tL;
  P.tree_tau = ttau;
  P.off = off;
  P.world_sorted = fused_world;
  P.off_out = fused_world ? const_cast<int64_t*>(off) : nullptr;
  P.c0 = k0; P.c1 = k1; P.c2 = k2; P.c3 = k3; P.jrow = kj; P.kd = kk;
  P.n_contacts = n;
  P.n_dev = c->n_device;
  P.perm = perm;
  P.foff = foff;
  P.impulses = imp;
  P.impulses_cap = imp_cap;
  P.wstats = (cf_.flags & COMFREE_FLAG_STATS) ? ctx->wstats + first : nullptr;
  P.err = ctx->d_err;
  P.first_bad = ctx->d_first_bad;
  P.queue = ctx->d_queue;
  P.world_base = first;
  P.check_finite = !(cf_.flags & COMFREE_FLAG_NO_FINITE_CHECK);
  P.exact_diag = (cf_.flags & COMFREE_FLAG_EXACT_DIAGONAL) ? 1 : ((cf_.flags & COMFREE_FLAG_FACET_DIAGONAL) ? 2 : 0);
#ifdef CF_TIMELINE
  P.timeline = cf_debug_timeline_buf();
#endif
  if (stg_mode) {
    P.st_status = ctx->stg.status;
    P.st_base = ctx->stg.stage;
    P.st_cap = ctx->stg.cap;
    P.st_fbase = ctx->stg.fbase;
    P.st_cut = ctx->stg.cut;
    P.st_geom = static_cast<const int4*>(ctx->geo.p);
    P.st_mu_t = ctx->col_mu[0];
    P.st_mu_tor = ctx->col_mu[1];
    P.st_mu_rol = ctx->col_mu[2];
    P.st_condim = ctx->col_condim;
  }
  int wpw = pick_wpw(sc, n, nw);
  if (const char* e = getenv("COMFREE_WPW")) {  // tuning override (1, 2, 4, 8 or 16 warps per world)
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) wpw = v;
  }
  const size_t smem_need = cf::step_smem_bytes(sc, wpw);
  P.gscratch = nullptr;
  if (smem_need > 227 * 1024) {
    // the world's working set does not fit a CTA's shared memory: one CTA of 8
    // warps per world over a global (L2-resident) scratch slab
    wpw = 8;
    CUDA_TRY(ctx, ensure(ctx->gscratch, std::max<int64_t>(1, nw) * cf::step_world_floats(sc) * sizeof(float)));
    P.gscratch = static_cast<float*>(ctx->gscratch.p);
  }
  int st_e0 = -1, st_e1 = -1;
  if (ctx->timing) {
    cudaEvent_t e = next_event(ctx, &st_e0);
    if (e) cudaEventRecord(e, s);
  }
  // Opt-in (COMFREE_PERSIST=1, big free-body worlds): the persistent kernel
  // (CTAs stepping their worlds in turn, the next world TMA-staged or
  // L2-prefetched).  Measured slower than one CTA per world on C4 in every
  // mode (profiles/r02_ab_kernel.txt), so not the default.
  bool persist = false;
  if (const char* e = getenv("COMFREE_PERSIST"))
    persist = atoi(e) != 0 && sc.T == 0 && wpw == 8 && !stg_mode && cf::step_persist_smem_bytes(sc) <= 227 * 1024;
  if (persist) {
    CUDA_TRY(ctx, cf::launch_step_persist(P, s));
  } else {
    CUDA_TRY(ctx, cf::launch_step(P, wpw, s));
  }
  if (st_e0 >= 0) {
    cudaEvent_t e = next_event(ctx, &st_e1);
    if (e) {
      cudaEventRecord(e, s);
      ctx->ev_step.push_back({st_e0, st_e1});
    }
  }
  ctx->launches += nw > 0 ? 1 : 0;
  ctx->last_first = first;
  ctx->last_nw = nw;
  ctx->last_nc = n;
  ctx->stats_valid = (cf_.flags & COMFREE_FLAG_STATS) != 0;

  // ---- outputs to host ----
  if (c->foff && foff) {
    CUDA_TRY(ctx, cudaMemcpyAsync(c->foff, foff, (size_t)(n + 1) * sizeof(int64_t),
                                  loc == COMFREE_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
  }
  if (c->impulses && loc == COMFREE_MEM_HOST && imp_cap > 0) {
    CUDA_TRY(ctx, cudaMemcpyAsync(c->impulses, imp, (size_t)imp_cap * sizeof(float), cudaMemcpyDeviceToHost, s));
  }
  if (host_io) return check_latched(ctx, s);
  return COMFREE_OK;
}

static comfree_status get_state_impl(comfree_ctx* ctx, int64_t first, int64_t nw, comfree_state* out,
                                     cudaStream_t s) {
  const cf::SceneDev& sc = ctx->sc;
  const float* src = ctx->slab + (size_t)first * sc.slab;
  if (out->location == COMFREE_MEM_HOST_ASYNC) {
    // public layout into staging slot a_out on the caller's stream (after that
    // slot's previous copy-out), then copied out on the copy-out stream; the
    // caller's stream does not wait for the copy (comfree_wait_async)
    CUDA_TRY(ctx, async_init(ctx));
    const int k = ctx->a_out;
    ctx->a_out ^= 1;
    const size_t nb = (size_t)nw * sc.B, nq = (size_t)nw * sc.Q;
    CUDA_TRY(ctx, ensure(ctx->aslot[k].out, std::max<size_t>(1, nb * 13 + nq * 2) * sizeof(float)));
    float* d = static_cast<float*>(ctx->aslot[k].out.p);
    float* dp[6] = {d, d + 3 * nb, d + 7 * nb, d + 10 * nb, d + 13 * nb, d + 13 * nb + nq};
    float* hp[6] = {out->pos, out->quat, out->vel, out->omega, out->qpos, out->qvel};
    const size_t cnt[6] = {3 * nb, 4 * nb, 3 * nb, 3 * nb, nq, nq};
    CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_d2h[k], 0));
    CUDA_TRY(ctx, cf::launch_slab_to_public(src, nw, sc, hp[0] ? dp[0] : nullptr, hp[1] ? dp[1] : nullptr,
                                            hp[2] ? dp[2] : nullptr, hp[3] ? dp[3] : nullptr,
                                            hp[4] ? dp[4] : nullptr, hp[5] ? dp[5] : nullptr, s));
    ctx->launches += 1;
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_conv[k], s));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_conv[k], 0));
    for (int q = 0; q < 6; ++q)
      if (hp[q] && cnt[q])
        CUDA_TRY(ctx, cudaMemcpyAsync(hp[q], dp[q], cnt[q] * sizeof(float), cudaMemcpyDeviceToHost, ctx->s_d2h));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_d2h[k], ctx->s_d2h));
    return COMFREE_OK;
  }
  if (out->location == COMFREE_MEM_DEVICE) {
    CUDA_TRY(ctx, cf::launch_slab_to_public(src, nw, sc, out->pos, out->quat, out->vel, out->omega, out->qpos, out->qvel, s));
    ctx->launches += 1;
    return COMFREE_OK;
  }
  const size_t nb = (size_t)nw * sc.B, nq = (size_t)nw * sc.Q;
  CUDA_TRY(ctx, ensure(ctx->st_tmp, std::max<size_t>(1, nb * 13 + nq * 2) * sizeof(float)));
  float* d = static_cast<float*>(ctx->st_tmp.p);
  float* dp[6] = {d, d + 3 * nb, d + 7 * nb, d + 10 * nb, d + 13 * nb, d + 13 * nb + nq};
  float* hp[6] = {out->pos, out->quat, out->vel, out->omega, out->qpos, out->qvel};
  const size_t cnt[6] = {3 * nb, 4 * nb, 3 * nb, 3 * nb, nq, nq};
  CUDA_TRY(ctx, cf::launch_slab_to_public(src, nw, sc, hp[0] ? dp[0] : nullptr, hp[1] ? dp[1] : nullptr,
                                          hp[2] ? dp[2] : nullptr, hp[3] ? dp[3] : nullptr,
                                          hp[4] ? dp[4] : nullptr, hp[5] ? dp[5] : nullptr, s));
  ctx->launches += 1;
  for (int k = 0; k < 6; ++k)
    if (hp[k] && cnt[k])
      CUDA_TRY(ctx, cudaMemcpyAsync(hp[k], dp[k], cnt[k] * sizeof(float), cudaMemcpyDeviceToHost, s));
  return COMFREE_OK;
}

comfree_status comfree_get_state(comfree_ctx* ctx, int64_t first, int64_t nw, comfree_state* out, void* stream) {
  if (!ctx || !out) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "get_state before load_scene");
  if (first < 0 || nw < 0 || first + nw > ctx->W) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "get_state: range");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  comfree_status st = get_state_impl(ctx, first, nw, out, s);
  if (st != COMFREE_OK) return st;
  if (out->location == COMFREE_MEM_HOST_ASYNC) return COMFREE_OK;  // errors surface at comfree_check
  return check_latched(ctx, s);
}

comfree_status comfree_wait_async(comfree_ctx* ctx, void* stream) {
  if (!ctx) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->s_h2d) return COMFREE_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  for (int k = 0; k < 2; ++k) {
    CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_h2d[k], 0));
    CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_h2d2[k], 0));
    CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_d2h[k], 0));
  }
  return COMFREE_OK;
}

comfree_status comfree_load_articulation(comfree_ctx* ctx, const comfree_articulation* a) {
  if (!ctx || !a) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "load_articulation before load_scene");
  const cf::SceneDev& sc = ctx->sc;
  if (a->n_trees != sc.T || a->tree_ndof != sc.nd || sc.T == 0)
    return fail(ctx, COMFREE_ERR_VALIDATION, "load_articulation: %d chains x %d DoFs, the scene has %d x %d",
                a->n_trees, a->tree_ndof, sc.T, sc.nd);
  if (!a->base || !a->axis || !a->length || !a->mass || !a->inertia || !a->armature)
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "load_articulation: null array");
  const int T = sc.T, nd = sc.nd, per = 3 + 7 * nd;
  std::vector<float> h((size_t)T * per);
  for (int t = 0; t < T; ++t) {
    float* m = h.data() + (size_t)t * per;
    for (int k = 0; k < 3; ++k) m[k] = a->base[3 * t + k];
    for (int j = 0; j < nd; ++j) {
      const int tj = t * nd + j;
      float* mj = m + 3 + 7 * j;
      const float ax = a->axis[3 * tj], ay = a->axis[3 * tj + 1], az = a->axis[3 * tj + 2];
      const float nrm = std::sqrt(ax * ax + ay * ay + az * az);
      if (!(std::fabs(nrm - 1.f) < 1e-3f)) return fail(ctx, COMFREE_ERR_VALIDATION, "load_articulation: axis not unit");
      mj[0] = ax / nrm; mj[1] = ay / nrm; mj[2] = az / nrm;
      mj[3] = a->length[tj]; mj[4] = a->mass[tj]; mj[5] = a->inertia[tj]; mj[6] = a->armature[tj];
      for (int k = 3; k < 7; ++k)
        if (!(finite(mj[k]) && mj[k] >= 0.f)) return fail(ctx, COMFREE_ERR_VALIDATION, "load_articulation: negative or non-finite link parameter");
    }
  }
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  CUDA_TRY(ctx, ensure(ctx->art, h.size() * sizeof(float)));
  CUDA_TRY(ctx, cudaMemcpy(ctx->art.p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  ctx->art_loaded = true;
  return COMFREE_OK;
}

comfree_status comfree_articulation_update(comfree_ctx* ctx, int64_t first, int64_t nw, const float* tau_ext,
                                           float* tree_L, float* tree_tau, int64_t n, const int64_t* n_device,
                                           const int32_t* world, const float* c0, const int32_t* c3,
                                           const int32_t* link, float* jrow, void* stream) {
  if (!ctx) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->art_loaded) return fail(ctx, COMFREE_ERR_STATE, "articulation_update before load_articulation");
  if (first < 0 || nw < 0 || first + nw > ctx->W) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "articulation_update: world range");
  if (nw > 0 && (!tree_L || !tree_tau)) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "articulation_update: tree_L / tree_tau required");
  if (n < 0 || n > INT32_MAX) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "articulation_update: n_contacts");
  if (n > 0 && (!world || !c0 || !c3 || !link || !jrow))
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "articulation_update: contact arrays required");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const cf::SceneDev& sc = ctx->sc;
  const float* slab = ctx->slab + (size_t)first * sc.slab;
  const float* model = static_cast<const float*>(ctx->art.p);
  CUDA_TRY(ctx, cf::launch_upstream(model, sc, slab, nw, tau_ext, ctx->cfg.gravity, tree_L, tree_tau, n, n_device,
                                    world, reinterpret_cast<const float4*>(c0), reinterpret_cast<const int4*>(c3), link,
                                    reinterpret_cast<float4*>(jrow), ctx->d_err, s));
  ctx->launches += (nw > 0 || n > 0);
  return COMFREE_OK;
}

comfree_status comfree_load_geometry(comfree_ctx* ctx, const comfree_geometry* g) {
  if (!ctx || !g) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "load_geometry before load_scene");
  const int G = g->n_geoms, P = g->n_pairs;
  if (G < 0 || P < 0 || (G > 0 && (!g->kind || !g->body || !g->link || !g->size || !g->local)) || (P > 0 && !g->pairs))
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "load_geometry: arrays");
  if (!(g->margin >= 0.f && finite(g->margin)) || !(g->mu[0] >= 0.f && g->mu[1] >= 0.f && g->mu[2] >= 0.f) ||
      !(g->condim == 1 || g->condim == 3 || g->condim == 4 || g->condim == 6))
    return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: margin, friction or condim");
  const cf::SceneDev& sc = ctx->sc;
  std::vector<int4> gi(G > 0 ? G : 1);
  std::vector<float4> gs(G > 0 ? G : 1), gl(G > 0 ? G : 1);
  bool chains = false;
  for (int k = 0; k < G; ++k) {
    const int kind = g->kind[k], body = g->body[k], link = g->link[k];
    if (kind < 0 || kind > 3 || body >= sc.B || body < -1 - sc.T) return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: geom %d kind/body", k);
    if (body < -1 && (link < 0 || link >= sc.nd)) return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: geom %d link", k);
    if (kind == 2 && body != -1) return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: planes must be static");
    chains |= body < -1;
    const float* sz = g->size + 3 * k;
    const float* lc = g->local + 3 * k;
    if (kind == 2) {
      const float nrm = std::sqrt(sz[0] * sz[0] + sz[1] * sz[1] + sz[2] * sz[2]);
      if (!(std::fabs(nrm - 1.f) < 1e-3f)) return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: plane normal not unit");
    } else if (!(sz[0] > 0.f && (kind == 0 || (kind == 3 && sz[1] > 0.f) || (sz[1] > 0.f && sz[2] > 0.f)))) {
      return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: geom %d size", k);
    }
    gi[k] = make_int4(kind, body, link, 0);
    gs[k] = make_float4(sz[0], sz[1], sz[2], 0.f);
    gl[k] = make_float4(lc[0], lc[1], lc[2], 0.f);
  }
  std::vector<int2> pr(P > 0 ? P : 1);
  for (int k = 0; k < P; ++k) {
    const int a = g->pairs[2 * k], b = g->pairs[2 * k + 1];
    if (a < 0 || a >= G || b < 0 || b >= G) return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: pair %d index", k);
    const int ka = g->kind[a], kb = g->kind[b];
    // supported: plane-{sphere, box, capsule} and every pair of {sphere, box, capsule}
    const bool ok = kb != 2 && ka >= 0 && kb >= 0;
    if (!ok) return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: pair %d kinds %d-%d not supported", k, ka, kb);
    if (g->body[a] == g->body[b] && g->body[a] >= 0)
      return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: pair %d on one body", k);
    pr[k] = make_int2(a, b);
  }
  if (chains && !ctx->art_loaded) return fail(ctx, COMFREE_ERR_STATE, "load_geometry: chain geoms need load_articulation first");
  if (P == 0) {  // broadphase mode (reading R32): planes lead the geom list, geom ids fit 16 bits
    bool seen_other = false;
    for (int k = 0; k < G; ++k) {
      if (g->kind[k] != 2) seen_other = true;
      else if (seen_other) return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: without pairs, planes must come first");
    }
    if (G > 65535) return fail(ctx, COMFREE_ERR_VALIDATION, "load_geometry: at most 65535 geoms");
  }
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const size_t bytes = (size_t)gi.size() * (sizeof(int4) + 2 * sizeof(float4)) + pr.size() * sizeof(int2);
  CUDA_TRY(ctx, ensure(ctx->geo, bytes));
  char* base = static_cast<char*>(ctx->geo.p);
  CUDA_TRY(ctx, cudaMemcpy(base, gi.data(), gi.size() * sizeof(int4), cudaMemcpyHostToDevice));
  CUDA_TRY(ctx, cudaMemcpy(base + gi.size() * sizeof(int4), gs.data(), gs.size() * sizeof(float4), cudaMemcpyHostToDevice));
  CUDA_TRY(ctx, cudaMemcpy(base + gi.size() * (sizeof(int4) + sizeof(float4)), gl.data(), gl.size() * sizeof(float4),
                           cudaMemcpyHostToDevice));
  CUDA_TRY(ctx, cudaMemcpy(base + gi.size() * (sizeof(int4) + 2 * sizeof(float4)), pr.data(), pr.size() * sizeof(int2),
                           cudaMemcpyHostToDevice));
  ctx->n_geoms = G;
  ctx->n_pairs = P;
  ctx->col_margin = g->margin;
  for (int k = 0; k < 3; ++k) ctx->col_mu[k] = g->mu[k];
  ctx->col_condim = g->condim;
  ctx->geo_loaded = true;
  return COMFREE_OK;
}

comfree_status comfree_collide(comfree_ctx* ctx, int64_t first, int64_t nw, int64_t capacity, int32_t* world,
                               float* c0, float* c1, float* c2, int32_t* c3, int32_t* link, int64_t* n_out,
                               int64_t* n_device, void* stream) {
  if (!ctx || (!n_out && !n_device)) return COMFREE_ERR_INVALID_ARGUMENT;
  if (n_out) *n_out = 0;
  if (!ctx->geo_loaded) return fail(ctx, COMFREE_ERR_STATE, "collide before load_geometry");
  if (first < 0 || nw < 0 || first + nw > ctx->W) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "collide: world range");
  if (capacity < 0 || (capacity > 0 && (!world || !c0 || !c1 || !c2 || !c3 || !link)))
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "collide: output arrays");
  if (nw * (int64_t)ctx->n_pairs * 17 >= INT32_MAX) return fail(ctx, COMFREE_ERR_CAPACITY, "collide: too many candidate pairs");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  cf::CollideParams P{};
  P.sc = ctx->sc;
  P.slab = ctx->slab + (size_t)first * ctx->sc.slab;
  P.model = static_cast<const float*>(ctx->art.p);
  const size_t G = ctx->n_geoms > 0 ? ctx->n_geoms : 1;
  char* base = static_cast<char*>(ctx->geo.p);
  P.geom = reinterpret_cast<const int4*>(base);
  P.size = reinterpret_cast<const float4*>(base + G * sizeof(int4));
  P.local = reinterpret_cast<const float4*>(base + G * (sizeof(int4) + sizeof(float4)));
  P.pairs = reinterpret_cast<const int2*>(base + G * (sizeof(int4) + 2 * sizeof(float4)));
  P.n_pairs = ctx->n_pairs;
  P.n_worlds = nw;
  P.first_world = first;
  P.margin = ctx->col_margin;
  P.mu_t = ctx->col_mu[0];
  P.mu_tor = ctx->col_mu[1];
  P.mu_rol = ctx->col_mu[2];
  P.condim = ctx->col_condim;
  P.c0 = reinterpret_cast<float4*>(c0);
  P.c1 = reinterpret_cast<float4*>(c1);
  P.c2 = reinterpret_cast<float4*>(c2);
  P.c3 = reinterpret_cast<int4*>(c3);
  P.world = world;
  P.link = reinterpret_cast<int2*>(link);
  P.n_geoms = ctx->n_geoms;
  if (ctx->n_pairs == 0) {
    // broadphase mode (reading R32): one kernel, candidates found per world
    int np2 = 1;
    while (np2 < ctx->n_geoms + 1) np2 <<= 1;  // as collide_broadphase
    const size_t fixed = cf::collide_bp_smem(ctx->n_geoms, 0, np2);
    // candidate capacity: two CTAs per SM when that leaves room for 8
    // candidates per geom (a dense pile has ~7), else one CTA per SM (the
    // kernel's static shared memory, ~5 KB, comes on top of each)
    int64_t room = (int64_t)(108 * 1024) - (int64_t)fixed;
    if (room / 10 < 8 * (int64_t)ctx->n_geoms) room = (int64_t)(220 * 1024) - (int64_t)fixed;
    // (at least collide_bp_min_cap: the candidate list's storage holds the
    // sort's and the sweep's scratch before the candidates)
    const int min_cap = (cf::collide_bp_min_cap(ctx->n_geoms, np2) + 7) & ~7;
    const int cap_c = (int)std::max<int64_t>(std::max(1024, min_cap), std::min<int64_t>(room / 10 & ~7, 65535));
    if (cf::collide_bp_smem(ctx->n_geoms, cap_c, np2) > 227 * 1024)
      return fail(ctx, COMFREE_ERR_CAPACITY, "collide: %d geoms per world exceed the broadphase's shared memory", ctx->n_geoms);
    CUDA_TRY(ctx, ensure(ctx->bp_status, (std::max<int64_t>(1, nw) + (std::max<int64_t>(1, nw) + 255) / 256) * sizeof(unsigned long long)));  // + group sums
    CUDA_TRY(ctx, ensure(ctx->bp_queue, 8 * sizeof(int)));
    CUDA_TRY(ctx, ensure(ctx->bp_count, 2 * sizeof(int64_t)));
    int64_t* cnt = static_cast<int64_t*>(ctx->bp_count.p);
#ifdef CF_BP_TIMELINE
    CUDA_TRY(ctx, ensure(ctx->col_frames, std::max<size_t>(1, (size_t)nw) * 16 * sizeof(unsigned long long)));
    P.frames = static_cast<float4*>(ctx->col_frames.p);
#endif
    // staged records per world: 16 per geom (the settled pile: ~10 per geom),
    // found order and placed (two areas of 2 x stage_cap float4)
    static const int stage_env = [] {  // test override of the staging size (exercises the second pass)
      const char* e = getenv("COMFREE_BP_STAGE_CAP");
      return e ? atoi(e) : 0;
    }();
    const int stage_cap = stage_env > 0 ? stage_env : (int)std::min<int64_t>(16 * (int64_t)ctx->n_geoms + 256, 1 << 20);
    CUDA_TRY(ctx, ensure(ctx->bp_stage, std::max<int64_t>(1, nw) * 4 * (size_t)stage_cap * sizeof(float4)));
    CUDA_TRY(ctx, cf::collide_broadphase(P, cap_c, capacity, static_cast<unsigned long long*>(ctx->bp_status.p),
                                         static_cast<int*>(ctx->bp_queue.p), n_device ? n_device : cnt, cnt + 1,
                                         ctx->d_err, static_cast<float4*>(ctx->bp_stage.p), stage_cap, s,
                                         ctx->bp_fbase_hook));
    if (ctx->bp_fbase_hook) {  // comfree_step_collided: the step reads the staged records
      ctx->stg.status = static_cast<const unsigned long long*>(ctx->bp_status.p);
      ctx->stg.stage = static_cast<const float4*>(ctx->bp_stage.p);
      ctx->stg.cap = stage_cap;
      ctx->stg.fbase = ctx->bp_fbase_hook;
      ctx->stg.cut = reinterpret_cast<const int64_t*>(static_cast<int*>(ctx->bp_queue.p) + 2);
      ctx->launches += 1;
      return COMFREE_OK;
    }
    ctx->launches += 2;
    if (n_device) return COMFREE_OK;
    int64_t h[2] = {0, 0};
    CUDA_TRY(ctx, cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(ctx, cudaStreamSynchronize(s));
    *n_out = h[1];
    if (h[1] > capacity) {
      int zero = 0;
      CUDA_TRY(ctx, cudaMemcpy(ctx->d_err, &zero, sizeof zero, cudaMemcpyHostToDevice));  // reported here instead
      return fail(ctx, COMFREE_ERR_CAPACITY, "collide: %lld contacts, capacity %lld", (long long)h[1], (long long)capacity);
    }
    return check_latched(ctx, s);
  }
  const size_t m = (size_t)nw * ctx->n_pairs + 1;
  CUDA_TRY(ctx, ensure(ctx->col_frames, std::max<size_t>(1, (size_t)nw * ctx->n_geoms) * 3 * sizeof(float4)));
  P.frames = static_cast<float4*>(ctx->col_frames.p);
  CUDA_TRY(ctx, cf::collide_frames(P, s));
  ctx->launches += 1;
  CUDA_TRY(ctx, ensure(ctx->col_counts, m * sizeof(int32_t)));
  CUDA_TRY(ctx, ensure(ctx->col_offs, m * sizeof(int32_t)));
  size_t tb = 0;
  CUDA_TRY(ctx, cf::collide_count_scan(P, nullptr, nullptr, nullptr, &tb, s));
  CUDA_TRY(ctx, ensure(ctx->col_tmp, tb > 0 ? tb : 1));
  tb = ctx->col_tmp.cap;
  int32_t* offs = static_cast<int32_t*>(ctx->col_offs.p);
  CUDA_TRY(ctx, cf::collide_count_scan(P, static_cast<int32_t*>(ctx->col_counts.p), offs, ctx->col_tmp.p, &tb, s));
  ctx->launches += 2;
  if (n_device) {  // asynchronous: count on the device, overflow latched as COMFREE_ERR_CAPACITY
    CUDA_TRY(ctx, cf::collide_emit(P, offs, capacity, n_device, ctx->d_err, s));
    ctx->launches += 1;
    return COMFREE_OK;
  }
  int32_t total = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&total, offs + (m - 1), sizeof total, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(ctx, cudaStreamSynchronize(s));
  *n_out = total;
  if (total > capacity) return fail(ctx, COMFREE_ERR_CAPACITY, "collide: %d contacts, capacity %lld", total, (long long)capacity);
  CUDA_TRY(ctx, cf::collide_emit(P, offs, capacity, nullptr, nullptr, s));
  ctx->launches += 1;
  return COMFREE_OK;
}

// One full step from the geometry (comfree.h): the broadphase without its emit
// pass, then the step reading each world's staged records (the STG kernel), or
// collide + step on library-owned streams when the staged kernel does not
// cover the configuration.
comfree_status comfree_step_collided(comfree_ctx* ctx, const comfree_worlds* wd, int64_t capacity, float dt,
                                     void* stream) {
  if (!ctx) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "step_collided before load_scene");
  if (!ctx->geo_loaded) return fail(ctx, COMFREE_ERR_STATE, "step_collided before load_geometry");
  if (!wd) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step_collided: null worlds");
  if (ctx->n_pairs != 0) return fail(ctx, COMFREE_ERR_STATE, "step_collided: the geometry has a candidate list (broadphase mode only)");
  if (ctx->sc.T != 0) return fail(ctx, COMFREE_ERR_STATE, "step_collided: scenes with chains take collide + articulation_update + step");
  if (wd->location != COMFREE_MEM_DEVICE) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step_collided: DEVICE world inputs");
  if (capacity <= 0 || capacity > INT32_MAX) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step_collided: capacity");
  const int64_t first = wd->first_world, nw = wd->n_worlds;
  if (first < 0 || nw < 0 || first + nw > ctx->W) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "step_collided: world range");
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const size_t cap = (size_t)capacity;
  CUDA_TRY(ctx, ensure(ctx->fs_world, cap * sizeof(int32_t)));
  CUDA_TRY(ctx, ensure(ctx->fs_c0, cap * 16));
  CUDA_TRY(ctx, ensure(ctx->fs_c1, cap * 16));
  CUDA_TRY(ctx, ensure(ctx->fs_c2, cap * 16));
  CUDA_TRY(ctx, ensure(ctx->fs_c3, cap * 16));
  CUDA_TRY(ctx, ensure(ctx->fs_link, cap * 8));
  CUDA_TRY(ctx, ensure(ctx->bp_count, 2 * sizeof(int64_t)));
  int64_t* ndev = static_cast<int64_t*>(ctx->bp_count.p);
  const comfree_config& c = ctx->cfg;
  const bool staged_ok = c.n_t == 4 && c.power == 2.0f &&
                         !(c.flags & (COMFREE_FLAG_EXACT_DIAGONAL | COMFREE_FLAG_FACET_DIAGONAL | COMFREE_FLAG_STATS)) &&
                         cf::step_smem_bytes(ctx->sc, 8) <= 227 * 1024;
  if (staged_ok) {
    CUDA_TRY(ctx, ensure(ctx->bp_fbase, std::max<int64_t>(1, nw) * sizeof(int64_t)));
    ctx->bp_fbase_hook = static_cast<int64_t*>(ctx->bp_fbase.p);
  }
  comfree_status st = comfree_collide(ctx, first, nw, capacity, static_cast<int32_t*>(ctx->fs_world.p),
                                      static_cast<float*>(ctx->fs_c0.p), static_cast<float*>(ctx->fs_c1.p),
                                      static_cast<float*>(ctx->fs_c2.p), static_cast<int32_t*>(ctx->fs_c3.p),
                                      static_cast<int32_t*>(ctx->fs_link.p), nullptr, ndev, stream);
  ctx->bp_fbase_hook = nullptr;
  if (st != COMFREE_OK) return st;
  comfree_contacts cd{};
  cd.world = static_cast<const int32_t*>(ctx->fs_world.p);
  cd.c0 = static_cast<const float*>(ctx->fs_c0.p);
  cd.c1 = static_cast<const float*>(ctx->fs_c1.p);
  cd.c2 = static_cast<const float*>(ctx->fs_c2.p);
  cd.c3 = static_cast<const int32_t*>(ctx->fs_c3.p);
  cd.flags = COMFREE_CONTACTS_SORTED;
  cd.location = COMFREE_MEM_DEVICE;
  cd.n_contacts = capacity;
  if (!staged_ok) {
    cd.n_device = ndev;
    return comfree_step(ctx, wd, &cd, dt, stream);
  }
  ctx->stg.active = true;
  st = comfree_step(ctx, wd, &cd, dt, stream);
  ctx->stg.active = false;
  return st;
}

comfree_status comfree_mppi_sample(comfree_ctx* ctx, int32_t P, int32_t N, int32_t H, const float* plan, float sigma,
                                   float lo, float hi, uint64_t seed, uint64_t iteration, float* U, void* stream) {
  if (!ctx) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "mppi_sample before load_scene");
  if (P < 0 || N < 1 || H < 1 || (P > 0 && (!plan || !U))) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "mppi_sample: sizes / arrays");
  if (!(sigma > 0.f) || !(lo <= hi)) return fail(ctx, COMFREE_ERR_VALIDATION, "mppi_sample: sigma > 0 and lo <= hi");
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  CUDA_TRY(ctx, cf::mppi_sample(plan, P, N, H, ctx->sc.Q, sigma, lo, hi, seed, iteration, U, static_cast<cudaStream_t>(stream)));
  ctx->launches += P > 0;
  return COMFREE_OK;
}

comfree_status comfree_mppi_control(comfree_ctx* ctx, int64_t first, int64_t nw, const float* U, int32_t t, int32_t H,
                                    float kp, float kd, float* command, float* tau, void* stream) {
  if (!ctx) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "mppi_control before load_scene");
  if (first < 0 || nw < 0 || first + nw > ctx->W || t < 0 || t >= H || (nw > 0 && (!U || !command || !tau)))
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "mppi_control: range / arrays");
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  CUDA_TRY(ctx, cf::mppi_control(ctx->sc, ctx->slab + (size_t)first * ctx->sc.slab, nw, U, t, H, kp, kd, command, tau,
                                 static_cast<cudaStream_t>(stream)));
  ctx->launches += nw > 0;
  return COMFREE_OK;
}

static comfree_status mppi_cost_params(comfree_ctx* ctx, int64_t first, int64_t nw, int32_t n_samples,
                                       const comfree_mppi_task* task, int32_t terminal, const float* J,
                                       cf::MppiCostParams& C);

comfree_status comfree_mppi_cost_control(comfree_ctx* ctx, int64_t first, int64_t nw, int32_t n_samples,
                                         const comfree_mppi_task* task, float* J, const float* U, int32_t t,
                                         int32_t H, float kp, float kd, float* command, float* tau, void* stream) {
  if (!ctx || !task) return COMFREE_ERR_INVALID_ARGUMENT;
  if (t < 0 || t >= H || (nw > 0 && (!U || !command || !tau)))
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "mppi_cost_control: step / arrays");
  cf::MppiCostParams C{};
  comfree_status st = mppi_cost_params(ctx, first, nw, n_samples, task, 0, J, C);
  if (st != COMFREE_OK) return st;
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  CUDA_TRY(ctx, cf::mppi_cost_control(C, J, U, t, H, kp, kd, command, tau, static_cast<cudaStream_t>(stream)));
  ctx->launches += nw > 0;
  return COMFREE_OK;
}

static comfree_status mppi_cost_params(comfree_ctx* ctx, int64_t first, int64_t nw, int32_t n_samples,
                                       const comfree_mppi_task* task, int32_t terminal, const float* J,
                                       cf::MppiCostParams& C) {
  if (!ctx->art_loaded) return fail(ctx, COMFREE_ERR_STATE, "mppi_cost before load_articulation");
  if (first < 0 || nw < 0 || first + nw > ctx->W || n_samples < 1 || (nw > 0 && !J))
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "mppi_cost: range / arrays");
  if (task->object_body < 0 || task->object_body >= ctx->sc.B || !task->target_pos || !task->target_quat || !task->q_ref)
    return fail(ctx, COMFREE_ERR_VALIDATION, "mppi_cost: object body / targets");
  C.sc = ctx->sc;
  C.slab = ctx->slab + (size_t)first * ctx->sc.slab;
  C.model = static_cast<const float*>(ctx->art.p);
  C.n_worlds = nw;
  C.n_samples = n_samples;
  C.obj = task->object_body;
  C.target_pos = task->target_pos;
  C.target_quat = task->target_quat;
  C.q_ref = task->q_ref;
  for (int k = 0; k < 6; ++k) C.w[k] = task->w[k];
  C.omega_fallen = task->omega_fallen;
  C.z_fallen = task->z_fallen;
  C.phi1 = task->phi1;
  C.phi2 = task->phi2;
  C.terminal = terminal != 0;
  return COMFREE_OK;
}

comfree_status comfree_mppi_cost(comfree_ctx* ctx, int64_t first, int64_t nw, int32_t n_samples,
                                 const comfree_mppi_task* task, int32_t terminal, float* J, void* stream) {
  if (!ctx || !task) return COMFREE_ERR_INVALID_ARGUMENT;
  cf::MppiCostParams C{};
  comfree_status st = mppi_cost_params(ctx, first, nw, n_samples, task, terminal, J, C);
  if (st != COMFREE_OK) return st;
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  CUDA_TRY(ctx, cf::mppi_cost(C, J, static_cast<cudaStream_t>(stream)));
  ctx->launches += nw > 0;
  return COMFREE_OK;
}

comfree_status comfree_mppi_update(comfree_ctx* ctx, int32_t P, int32_t N, int32_t H, const float* J, const float* U,
                                   float lambda, float lo, float hi, float* plan, float* weights, void* stream) {
  if (!ctx) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "mppi_update before load_scene");
  if (P < 0 || N < 1 || H < 1 || (P > 0 && (!J || !U || !plan))) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "mppi_update: sizes / arrays");
  if (!(lambda > 0.f) || !(lo <= hi)) return fail(ctx, COMFREE_ERR_VALIDATION, "mppi_update: lambda > 0 and lo <= hi");
  if ((size_t)N * sizeof(float) > 48 * 1024) return fail(ctx, COMFREE_ERR_CAPACITY, "mppi_update: more than 12288 samples per problem");
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  CUDA_TRY(ctx, cf::mppi_update(J, U, P, N, H, ctx->sc.Q, lambda, lo, hi, plan, weights, static_cast<cudaStream_t>(stream)));
  ctx->launches += P > 0;
  return COMFREE_OK;
}

comfree_status comfree_mppi_update_shift(comfree_ctx* ctx, int32_t P, int32_t N, int32_t H, const float* J,
                                         const float* U, float lambda, float lo, float hi, float* plan, float* weights,
                                         float* u0, void* stream) {
  if (!ctx) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "mppi_update_shift before load_scene");
  if (P < 0 || N < 1 || H < 1 || (P > 0 && (!J || !U || !plan || !u0)))
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "mppi_update_shift: sizes / arrays");
  if (!(lambda > 0.f) || !(lo <= hi)) return fail(ctx, COMFREE_ERR_VALIDATION, "mppi_update_shift: lambda > 0 and lo <= hi");
  if ((size_t)N * sizeof(float) > 48 * 1024) return fail(ctx, COMFREE_ERR_CAPACITY, "mppi_update_shift: more than 12288 samples per problem");
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  CUDA_TRY(ctx, cf::mppi_update(J, U, P, N, H, ctx->sc.Q, lambda, lo, hi, plan, weights, static_cast<cudaStream_t>(stream), u0));
  ctx->launches += P > 0;
  return COMFREE_OK;
}

comfree_status comfree_set_state_broadcast(comfree_ctx* ctx, int64_t first, int64_t n_src, int64_t repeat,
                                           const comfree_state* in, void* stream) {
  if (!ctx || !in) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "set_state_broadcast before load_scene");
  if (first < 0 || n_src < 0 || repeat < 1 || first + n_src * repeat > ctx->W)
    return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "set_state_broadcast: range");
  const cf::SceneDev& sc = ctx->sc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const float *pos = in->pos, *quat = in->quat, *vel = in->vel, *om = in->omega, *qp = in->qpos, *qv = in->qvel;
  if (in->location == COMFREE_MEM_HOST) {  // the n_src source states only go over PCIe
    const size_t nb = (size_t)n_src * sc.B, nq = (size_t)n_src * sc.Q;
    CUDA_TRY(ctx, ensure(ctx->st_tmp, std::max<size_t>(1, nb * 13 + nq * 2) * sizeof(float)));
    float* d = static_cast<float*>(ctx->st_tmp.p);
    float* dp[6] = {d, d + 3 * nb, d + 7 * nb, d + 10 * nb, d + 13 * nb, d + 13 * nb + nq};
    const float* hp[6] = {pos, quat, vel, om, qp, qv};
    const size_t cnt[6] = {3 * nb, 4 * nb, 3 * nb, 3 * nb, nq, nq};
    const float* res[6];
    for (int k = 0; k < 6; ++k) {
      res[k] = nullptr;
      if (hp[k] && cnt[k]) {
        CUDA_TRY(ctx, cudaMemcpyAsync(dp[k], hp[k], cnt[k] * sizeof(float), cudaMemcpyHostToDevice, s));
        res[k] = dp[k];
      }
    }
    pos = res[0]; quat = res[1]; vel = res[2]; om = res[3]; qp = res[4]; qv = res[5];
  }
  CUDA_TRY(ctx, cf::launch_public_to_slab(pos, quat, vel, om, qp, qv, n_src * repeat, sc,
                                          ctx->slab + (size_t)first * sc.slab, s, repeat));
  ctx->launches += 1;
  if (in->location == COMFREE_MEM_HOST) CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return COMFREE_OK;
}

comfree_status comfree_set_state(comfree_ctx* ctx, int64_t first, int64_t nw, const comfree_state* in, void* stream) {
  if (!ctx || !in) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "set_state before load_scene");
  if (first < 0 || nw < 0 || first + nw > ctx->W) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "set_state: range");
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  return set_state_impl(ctx, first, nw, in, static_cast<cudaStream_t>(stream));
}

comfree_status comfree_get_world_stats(comfree_ctx* ctx, int64_t first, int64_t nw, comfree_world_stats* out,
                                       int32_t location, void* stream) {
  if (!ctx || !out) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "get_world_stats before load_scene");
  if (!ctx->stats_valid) return fail(ctx, COMFREE_ERR_STATE, "no statistics: set COMFREE_FLAG_STATS and step");
  if (first < 0 || nw < 0 || first + nw > ctx->W) return fail(ctx, COMFREE_ERR_INVALID_ARGUMENT, "get_world_stats: range");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(ctx, cudaMemcpyAsync(out, ctx->wstats + first, (size_t)nw * sizeof(comfree_world_stats),
                                location == COMFREE_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
  return check_latched(ctx, s);
}

comfree_status comfree_get_stats(comfree_ctx* ctx, comfree_stats* out, void* stream) {
  if (!ctx || !out) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "get_stats before load_scene");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::memset(out, 0, sizeof *out);
  out->n_worlds = ctx->last_nw;
  out->first_nonfinite_world = -1;
  CUDA_TRY(ctx, cudaStreamSynchronize(s));
  int e = 0;
  unsigned long long bad = ~0ull;
  CUDA_TRY(ctx, cudaMemcpy(&e, ctx->d_err, sizeof e, cudaMemcpyDeviceToHost));
  CUDA_TRY(ctx, cudaMemcpy(&bad, ctx->d_first_bad, sizeof bad, cudaMemcpyDeviceToHost));
  if (e & cf::ERR_NONFINITE) out->first_nonfinite_world = (int64_t)bad;
  if (ctx->stats_valid && ctx->last_nw > 0) {
    std::string h((size_t)ctx->last_nw * sizeof(comfree_world_stats), '\0');
    comfree_world_stats* ws = reinterpret_cast<comfree_world_stats*>(&h[0]);
    CUDA_TRY(ctx, cudaMemcpy(ws, ctx->wstats + ctx->last_first, h.size(), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < ctx->last_nw; ++i) {
      out->contacts += ws[i].contacts;
      out->active_facets += ws[i].active_facets;
      out->max_penetration = std::max(out->max_penetration, ws[i].max_penetration);
      out->kinetic_energy += ws[i].kinetic_energy;
    }
  }
  return check_latched(ctx, s);
}

comfree_status comfree_segment_info(comfree_ctx* ctx, int64_t* off, int32_t* perm, void* stream) {
  if (!ctx || !off) return COMFREE_ERR_INVALID_ARGUMENT;
  if (!ctx->loaded) return fail(ctx, COMFREE_ERR_STATE, "segment_info before load_scene");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CUDA_TRY(ctx, cudaStreamSynchronize(s));
  if (!ctx->off.p) return fail(ctx, COMFREE_ERR_STATE, "segment_info: last step had caller-supplied off[]");
  CUDA_TRY(ctx, cudaMemcpy(off, ctx->off.p, (size_t)(ctx->last_nw + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (perm) {
    if (ctx->last_sorted_copy) {
      CUDA_TRY(ctx, cudaMemcpy(perm, ctx->perm.p, (size_t)ctx->last_nc * sizeof(int32_t), cudaMemcpyDeviceToHost));
    } else {
      for (int64_t i = 0; i < ctx->last_nc; ++i) perm[i] = (int32_t)i;
    }
  }
  return check_latched(ctx, s);
}

comfree_status comfree_set_timing(comfree_ctx* ctx, int enable) {
  if (!ctx) return COMFREE_ERR_INVALID_ARGUMENT;
  ctx->timing = enable != 0;
  return COMFREE_OK;
}

comfree_status comfree_check(comfree_ctx* ctx, void* stream) {
  if (!ctx) return COMFREE_ERR_INVALID_ARGUMENT;
  return check_latched(ctx, static_cast<cudaStream_t>(stream));
}

comfree_status comfree_get_timing(comfree_ctx* ctx, double out[3]) {
  if (!ctx || !out) return COMFREE_ERR_INVALID_ARGUMENT;
  out[0] = out[1] = out[2] = 0.0;
  for (auto& pr : ctx->ev_step) {
    float ms = 0.f;
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev_pool[pr.second]));
    CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->ev_pool[pr.first], ctx->ev_pool[pr.second]));
    out[0] += ms;
    out[2] += 1.0;
  }
  for (auto& pr : ctx->ev_seg) {
    float ms = 0.f;
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev_pool[pr.second]));
    CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->ev_pool[pr.first], ctx->ev_pool[pr.second]));
    out[1] += ms;
  }
  ctx->ev_step.clear();
  ctx->ev_seg.clear();
  ctx->ev_used = 0;
  return COMFREE_OK;
}

int64_t comfree_kernel_launches(const comfree_ctx* ctx) { return ctx ? ctx->launches : -1; }

void comfree_destroy(comfree_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  DevBuf* bufs[] = {&ctx->off, &ctx->keys, &ctx->perm, &ctx->iota, &ctx->s0, &ctx->s1, &ctx->s2, &ctx->s3,
                    &ctx->sj, &ctx->skd, &ctx->nf, &ctx->foff, &ctx->cub_tmp, &ctx->in_world, &ctx->in_off, &ctx->in_c0,
                    &ctx->in_c1, &ctx->in_c2, &ctx->in_c3, &ctx->in_jrow, &ctx->in_kd, &ctx->in_fext, &ctx->in_L,
                    &ctx->in_tau, &ctx->imp, &ctx->st_tmp, &ctx->art, &ctx->geo, &ctx->col_counts,
                    &ctx->col_offs, &ctx->col_tmp, &ctx->col_frames, &ctx->bp_status, &ctx->bp_queue, &ctx->bp_count, &ctx->bp_stage, &ctx->gscratch};
  for (DevBuf* b : bufs) release(*b);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->slab) cudaFree(ctx->slab);
  if (ctx->inv_mass) cudaFree(ctx->inv_mass);
  if (ctx->inv_inertia) cudaFree(ctx->inv_inertia);
  if (ctx->wstats) cudaFree(ctx->wstats);
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->d_first_bad) cudaFree(ctx->d_first_bad);
  if (ctx->d_queue) cudaFree(ctx->d_queue);
  for (auto& sl : ctx->aslot)
    for (DevBuf* b : {&sl.world, &sl.off, &sl.c0, &sl.c1, &sl.c2, &sl.c3, &sl.jrow, &sl.kd, &sl.fext, &sl.L, &sl.tau, &sl.out})
      if (b->p) cudaFree(b->p);
  if (ctx->s_h2d) cudaStreamDestroy(ctx->s_h2d);
  if (ctx->s_d2h) cudaStreamDestroy(ctx->s_d2h);
  if (ctx->s_h2d2) cudaStreamDestroy(ctx->s_h2d2);
  for (cudaEvent_t e : {ctx->ev_entry, ctx->ev_h2d[0], ctx->ev_h2d[1], ctx->ev_h2d2[0], ctx->ev_h2d2[1],
                        ctx->ev_conv[0], ctx->ev_conv[1],
                        ctx->ev_d2h[0], ctx->ev_d2h[1]})
    if (e) cudaEventDestroy(e);
  delete ctx;
}

const char* comfree_last_error(const comfree_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

}  // extern "C"
