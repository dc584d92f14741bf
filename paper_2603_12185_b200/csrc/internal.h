// internal.h — device-side parameter blocks and kernel launchers of the
// ComFree-Sim step (not part of the ABI; see include/comfree.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "comfree.h"

namespace cf {

// Device error word bits (latched, surfaced by the next synchronising call).
enum : int {
  ERR_NONFINITE = 1,
  ERR_UNSORTED = 2,     // COMFREE_CONTACTS_SORTED promised but world[] decreases
  ERR_WORLD_RANGE = 4,  // world id outside [0, n_worlds)
  ERR_BODY_RANGE = 8,   // body id out of range / tree side without J rows
  ERR_CONDIM = 16,      // condim not in {1,3,4,6}
  ERR_IMPULSE_CAP = 32, // impulses buffer too small
  ERR_IMPEDANCE = 64,   // per-contact (k_user, d_user) negative or non-finite
  ERR_WORLD_CONTACTS = 128, // more contacts in one world than the S6 fixed-point bound (65536)
  ERR_ARTICULATION = 256,   // articulated upstream: M(q) not positive definite, or a bad chain/link id
  ERR_CONTACT_CAP = 512,    // collision front-end (device count): more contacts than the capacity
  ERR_CANDIDATES = 1024     // broadphase: more candidate pairs in one world than the shared-memory list holds
};

// State slab: per world, 13 planes of Bp floats (px py pz qw qx qy qz vx vy vz
// wx wy wz) followed by 2 planes of Qp floats (qpos, qvel).  Bp, Qp are
// multiples of 4 so each plane is 16-byte aligned; Bp >= B + 1 (body record B
// of the step's shared memory is the all-zero record of static sides).
enum { PL_PX = 0, PL_QW = 3, PL_VX = 7, PL_WX = 10, N_BODY_PLANES = 13 };

struct SceneDev {
  int B, Bp, T, nd, Q, Qp;
  int slab;                     // floats per world
  const float* inv_mass;        // [Bp]
  const float* inv_inertia;     // [3][Bp]
  const float* inertia;         // [3][Bp] principal I_b (1 / inv_inertia, 0 where locked)
};

struct StepParams {
  // Eq. (12)-(13) parameters
  float k, d, kappa, dt;
  float r_min, r_span, inv_width, mid, inv_mid, inv_1m_mid, power;
  int power_is_2;
  float g[3];
  int n_t, n_rol;
  float2 dir_t[32];             // (cos, sin)(2 pi j / n_t), Eq. (7)
  float2 dir_r[32];
  SceneDev sc;
  float* slab;                  // world 0 of the step range
  int64_t n_worlds;
  const float* f_ext;           // [n_worlds][B][6] or null
  const float* tree_L;          // [n_worlds][T][10]
  const float* tree_tau;        // [n_worlds][Q]
  // contacts, grouped by world (possibly a permuted copy)
  const int64_t* off;           // [n_worlds + 1]
  const int32_t* world_sorted;  // fused S0: sorted world ids (then off is computed in-kernel), or null
  int64_t* off_out;             // fused S0: receives off[n_worlds + 1]
  const float4* c0;
  const float4* c1;
  const float4* c2;
  const int4* c3;
  const float4* jrow;           // [12][n_contacts] or null
  const float2* kd;             // [n_contacts] per-contact (k_user, d_user) or null
  int64_t n_contacts;           // stream length (capacity when n_dev is given)
  const int64_t* n_dev;         // device-side count of contacts in use, or null
  const int32_t* perm;          // sorted position -> input index, or null (identity)
  const int64_t* foff;          // [n_contacts + 1] facet offsets (input order) or null
  float* impulses;              // or null
  int64_t impulses_cap;
  comfree_world_stats* wstats;  // [n_worlds] or null
  int* err;                     // device error word
  unsigned long long* first_bad;// min world id with a non-finite state
  int* queue;                   // persistent kernel: [next world ticket, CTAs done], 0 between launches
  int64_t pf_ahead;             // > 0: prefetch world w + pf_ahead into L2 during world w (resident world slots)
  float* gscratch;              // non-null: per-world working set in global memory (worlds beyond shared memory)
  int64_t world_base;           // absolute id of world 0 of the range (error reporting)
  int check_finite;
  int exact_diag;               // per-facet impedance, general variants only: 1 Eq. (11) (COMFREE_FLAG_EXACT_DIAGONAL),
                                // 2 Eq. (12) with the facet diagonal (COMFREE_FLAG_FACET_DIAGONAL)
  unsigned* timeline;           // CF_TIMELINE builds only: per CTA (smid, t0, t1, t2, t3) globaltimer ns
  // contacts from the collision front-end's staging area (comfree_step_collided), else st_status null
  const unsigned long long* st_status;  // [n_worlds] broadphase status words: ST_VAL total, ST_DONE written in place
  const float4* st_base;        // world w's placed records: st_base + (4 w + 2) st_cap (point, phi), + st_cap (normal, key)
  int64_t st_cap;
  const int64_t* st_fbase;      // [n_worlds] base offset in c0..c3 of a world written in place
  const int64_t* st_cut;        // whole-pair cut of the in-place records (the capacity)
  const int4* st_geom;          // geom table (kind, body, link, -)
  float st_mu_t, st_mu_tor, st_mu_rol;
  int st_condim;
};
// broadphase status word fields (collide.cu's chained-scan words)
constexpr unsigned long long ST_DONE = 1ull << 61, ST_VAL = (1ull << 61) - 1;

// Launchers (return cudaError_t of the launch).
cudaError_t launch_step(const StepParams& p, int warps_per_world, cudaStream_t s);
size_t step_world_floats(const SceneDev& sc);  // floats of one world's working set (shared or global)
// persistent variant (free bodies only): one 32-warp CTA per SM, worlds staged by TMA
cudaError_t launch_step_persist(const StepParams& p, cudaStream_t s);
size_t step_persist_smem_bytes(const SceneDev& sc);
size_t step_smem_bytes(const SceneDev& sc, int warps_per_world);

// S0
cudaError_t launch_offsets_sorted(const int32_t* world, int64_t n, int64_t n_worlds, int64_t* off,
                                  int* err, cudaStream_t s);
cudaError_t launch_check_world_range(const int32_t* world, int64_t n, int64_t n_worlds, int* err,
                                     cudaStream_t s);
cudaError_t sort_by_world(const int32_t* world, int64_t n, int64_t n_worlds, int32_t* keys_out,
                          int32_t* perm_out, int32_t* iota_tmp, void* temp, size_t* temp_bytes,
                          cudaStream_t s);
cudaError_t launch_gather_contacts(const int32_t* perm, int64_t n, const float4* c0, const float4* c1,
                                   const float4* c2, const int4* c3, const float4* jrow, const float2* kd,
                                   float4* o0, float4* o1, float4* o2, int4* o3, float4* ojrow, float2* okd,
                                   cudaStream_t s);
cudaError_t facet_offsets(const int4* c3, int64_t n, int n_t, int n_rol, int32_t* nf_tmp,
                          int64_t* foff, void* temp, size_t* temp_bytes, int* err, cudaStream_t s);
cudaError_t launch_iota(int32_t* out, int64_t n, cudaStream_t s);

// articulated upstream (articulation.cu); model: per chain base[3] + per joint
// (axis[3], length, mass, inertia, armature), slab: world 0 of the range
cudaError_t launch_upstream(const float* model, const SceneDev& sc, const float* slab, int64_t n_worlds,
                            const float* tau_ext, const float g[3], float* L_out, float* tau_out, int64_t n,
                            const int64_t* n_dev, const int32_t* world, const float4* c0, const int4* c3,
                            const int32_t* link, float4* jrow, int* err, cudaStream_t s);

// collision front-end (collide.cu)
struct CollideParams {
  SceneDev sc;
  const float* slab;          // world 0 of the range
  const float* model;         // articulation model (chain-link geoms) or null
  const int4* geom;           // [G] (kind, body, link, 0)
  const float4* size;         // [G]
  const float4* local;        // [G]
  const int2* pairs;          // [P]
  int n_pairs;
  int64_t n_worlds, first_world;
  float margin, mu_t, mu_tor, mu_rol;
  int condim;
  float4* c0;
  float4* c1;
  float4* c2;
  int4* c3;
  int32_t* world;
  int2* link;
  float4* frames;             // [n_worlds][n_geoms][3] geom world frames (rows of R | x), filled by the frame pass
  int n_geoms;
};
cudaError_t collide_frames(const CollideParams& P, cudaStream_t s);
// Broadphase mode (no candidate list): one CTA per world finds the candidates
// (sort-and-sweep on grown AABBs) and emits their contacts with a chained scan
// over worlds.  status [n_worlds] and queue [4 ints] are scratch; n_dev gets
// the count of whole pairs within `capacity`, total (optional) every contact.
size_t collide_bp_smem(int n_geoms, int cap_c, int np2);
int collide_bp_min_cap(int n_geoms, int np2);
// stage: [n_worlds][2][stage_cap] float4 scratch for the records of the single
// narrowphase pass (a world with more records evaluates the narrowphase again).
// fbase non-null (comfree_step_collided): no emit pass; the staged records stay
// in `stage` for the step and a world written in place stores its base in fbase.
cudaError_t collide_broadphase(const CollideParams& P, int cap_c, int64_t capacity, unsigned long long* status,
                               int* queue, int64_t* n_dev, int64_t* total, int* err, float4* stage, int stage_cap,
                               cudaStream_t s, int64_t* fbase = nullptr);
cudaError_t collide_count_scan(const CollideParams& P, int32_t* counts, int32_t* offs, void* temp,
                               size_t* temp_bytes, cudaStream_t s);
// n_dev != null: also stores the (clamped) total for the asynchronous mode
cudaError_t collide_emit(const CollideParams& P, const int32_t* offs, int64_t capacity, int64_t* n_dev, int* err,
                         cudaStream_t s);

// MPPI (mppi.cu)
struct MppiCostParams {
  SceneDev sc;
  const float* slab;          // world 0 of the range
  const float* model;         // articulation model (fingertips)
  int64_t n_worlds;
  int n_samples;              // world w belongs to problem w / n_samples
  int obj;                    // object body index
  const float* target_pos;    // [P][3]
  const float* target_quat;   // [P][4]
  const float* q_ref;         // [Q]
  float w[6];
  float omega_fallen, z_fallen, phi1, phi2;
  int terminal;
};
cudaError_t mppi_sample(const float* plan, int P, int N, int H, int Q, float sigma, float lo, float hi, uint64_t seed,
                        uint64_t iteration, float* U, cudaStream_t s);
cudaError_t mppi_control(const SceneDev& sc, const float* slab, int64_t W, const float* U, int t, int H, float kp,
                         float kd, float* command, float* tau, cudaStream_t s);
cudaError_t mppi_cost(const MppiCostParams& C, float* J, cudaStream_t s);
cudaError_t mppi_cost_control(const MppiCostParams& C, float* J, const float* U, int t, int H, float kp, float kd,
                              float* command, float* tau, cudaStream_t s);
// u0 != null: also the receding-horizon shift -- u0[P][Q] = the new plan's first
// action, plan stores the new plan advanced by one step (last step 0)
cudaError_t mppi_update(const float* J, const float* U, int P, int N, int H, int Q, float lambda, float lo, float hi,
                        float* plan, float* weights, cudaStream_t s, float* u0 = nullptr);

// state layout conversion
cudaError_t launch_public_to_slab(const float* pos, const float* quat, const float* vel,
                                  const float* omega, const float* qpos, const float* qvel,
                                  int64_t n_worlds, const SceneDev& sc, float* slab, cudaStream_t s, int64_t repeat = 1);
cudaError_t launch_slab_to_public(const float* slab, int64_t n_worlds, const SceneDev& sc,
                                  float* pos, float* quat, float* vel, float* omega, float* qpos,
                                  float* qvel, cudaStream_t s);

}  // namespace cf
