/*
 * comfree.h — C ABI of the B200-native ComFree-Sim contact-resolution step.
 *
 * One call of comfree_step() runs, for every world and every contact, the
 * complementarity-free contact-resolution step of arXiv 2603.12185 (PAPER.md
 * §III, Algorithm 1):
 *   S0  world segmentation of the contact set C               ("the detected contact set C")
 *   S1  smooth prediction  v_s = v + M^-1 (tau - c) dt          Eq. (2)
 *   S2  contact kinematics (v_c, omega_c) = J v_s               Eq. (4)-(5) P:109-123
 *   S3  dual-cone impedance K = k M(phi)/dt, D = d M(phi)/dt    Eq. (12)-(13) P:209-233
 *   S4  per-facet closed-form impulse                           Eq. (7)-(9) P:142-180
 *         lambda = ( -K (J~ v_s dt + phi) - D J~ v_s )_+   (sign of Eq. (9); Alg. 1 P:260 is garbled)
 *   S5  facet impulses -> contact wrench (sum_f J~_f^T Lambda_f regrouped)
 *   S6  per-world scatter of J^T Lambda (Kernel III)
 *   S7  v+ = v_s + M^-1 p (Eq. (10)) and semi-implicit integration
 *   S8  articulated chains: M^-1 through per-chain Cholesky factors
 * with lambda a step-averaged wrench and Lambda = lambda dt the impulse.
 *
 * Conventions (see DESIGN.md for every reading of the paper):
 *  - fp32 everywhere on the device; quaternions (w,x,y,z) scalar first;
 *    angular velocities in the world frame.
 *  - Body ids inside a contact: >= 0 free 6-DoF body of the world,
 *    -1 static (world-fixed), -(2+t) articulated chain t (J rows supplied).
 *  - The normal n points from side a to side b; J v = motion of b relative
 *    to a, so n . v_c > 0 separates.  phi > 0 separated, < 0 penetrating.
 *  - condim (MuJoCo style): 1 normal only, 3 + tangential (n_t facets),
 *    4 + torsional (2 facets), 6 + rolling (n_rol facets).  Facet order per
 *    contact: tangential j = 0..n_t-1 with d_j = (cos 2 pi j/n_t, sin 2 pi j/n_t)
 *    in the (t1, t2 = n x t1) basis, then torsional (+1, -1), then rolling.
 *
 * Ownership: the library owns world state and scratch (allocated in
 * comfree_load_scene).  Every other buffer belongs to the caller and is only
 * borrowed for the stream-ordered duration of the call.  Device pointers
 * must be 16-byte aligned where a float4 stream is named.
 *
 * Streams: all work is enqueued on the caller's stream (a cudaStream_t passed
 * as void*, NULL = legacy default stream).  No call synchronises except
 * comfree_get_state / comfree_get_stats / comfree_get_world_stats /
 * comfree_segment_info and calls given HOST buffers.
 *
 * Errors: no C++ exception crosses the ABI.  Argument and validation errors
 * are returned synchronously.  Errors detected on the device (non-finite
 * state, unsorted contacts under COMFREE_CONTACTS_SORTED, out-of-range ids)
 * are latched and returned by the next synchronising call; the message is in
 * comfree_last_error().  A context is not thread-safe: single owner.
 */
#ifndef COMFREE_H
#define COMFREE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COMFREE_ABI_VERSION 2  /* 2: comfree_contacts.kd */

typedef enum {
  COMFREE_OK = 0,
  COMFREE_ERR_INVALID_ARGUMENT = 1, /* NULL / out-of-range argument */
  COMFREE_ERR_VALIDATION = 2,       /* config or scene violates a documented invariant */
  COMFREE_ERR_CAPACITY = 3,         /* allocation failed or size limit exceeded */
  COMFREE_ERR_NONFINITE = 4,        /* a world produced a non-finite state (or overflowed S6) */
  COMFREE_ERR_CUDA = 5,             /* CUDA runtime error */
  COMFREE_ERR_STATE = 6             /* call out of order (e.g. step before load_scene) */
} comfree_status;

/* memory location of caller buffers */
/* COMFREE_MEM_HOST_ASYNC: page-locked (pinned) HOST buffers, copied without
 * synchronising.  comfree_step stages contacts and world inputs into one of
 * two device slots over the context's copy-in stream (which first waits for
 * the caller's stream to reach the call) and makes the caller's stream wait
 * for the copies; comfree_get_state converts the state on the caller's stream
 * and copies it out over the context's copy-out stream, without making the
 * caller's stream wait.  So step k + 1's upload overlaps step k's kernel and
 * download.  The caller keeps a step's input buffers unchanged, and reads the
 * output buffers only after comfree_wait_async(ctx, stream) plus a
 * synchronisation of `stream` (or comfree_check).  Errors surface at the next
 * comfree_check / synchronising call.  Not with impulses, foff or n_device. */
enum { COMFREE_MEM_DEVICE = 0, COMFREE_MEM_HOST = 1, COMFREE_MEM_HOST_ASYNC = 2 };

/* comfree_config.flags */
enum {
  COMFREE_FLAG_STATS = 1u << 0,         /* per-world statistics every step */
  COMFREE_FLAG_DETERMINISTIC = 1u << 1, /* accepted, no effect: every step is bitwise deterministic
                                           (fixed-point accumulation, see comfree_step) */
  COMFREE_FLAG_NO_FINITE_CHECK = 1u << 2,
  /* Eq. (11) instead of the heuristic of Eq. (12): every facet f
   * takes K_f dt + D_f = 1 / (dt A_f) with its own diagonal entry
   * A_f = J~_f M^-1 J~_f^T, split K_f dt : D_f = k dt : d (DESIGN.md reading
   * R24), i.e. Lambda_f = (-k phi - kappa s_f)_+ / (kappa A_f), kappa = k dt + d
   * (per-contact (k, d) pairs must then have kappa > 0, else
   * COMFREE_ERR_VALIDATION).  Costs one quadratic form per facet and side
   * (general kernel variant). */
  COMFREE_FLAG_EXACT_DIAGONAL = 1u << 3,
  /* Eq. (12) with the facet's own diagonal entry in place of the trace
   * heuristic (reading R28, not Eq. (11)): M_f = r/(1-r) / A_f,
   * K_f = k M_f/dt, D_f = d M_f/dt.  Exclusive with EXACT_DIAGONAL. */
  COMFREE_FLAG_FACET_DIAGONAL = 1u << 4
};

/* comfree_contacts.flags */
enum {
  COMFREE_CONTACTS_SORTED = 1u << 0     /* world[] is non-decreasing (verified on device) */
};

typedef struct comfree_ctx comfree_ctx;   /* opaque, single owner */

/* Global parameters.  Eq. (12) k_user, d_user; Eq. (13) r_min,
 * r_max, width w, midpoint m, power p (MuJoCo solimp defaults
 * 0.9, 0.95, 0.001, 0.5, 2); Eq. (7) facet counts n_t, n_rol (even, n_t >= 4,
 * n_rol >= 2; the torsional channel always has 2 facets); gravity acts on
 * every free body with inv_mass > 0 (part of tau - c in Eq. (2)).
 * Validation: k_user > 0, d_user >= 0, 0 < r_min <= r_max < 1, width > 0,
 * 0 < midpoint < 1, power >= 1, n_t, n_rol even, 4 <= n_t <= 32,
 * 2 <= n_rol <= 32, finite gravity. */
typedef struct {
  float k_user, d_user;
  float r_min, r_max, width, midpoint, power;
  int32_t n_t, n_rol;
  float gravity[3];
  uint32_t flags;
} comfree_config;

/* Per-scene body parameters shared by every world (HOST pointers, copied).
 * 0 <= inv_mass[i] <= 1e27 and 0 <= inv_inertia[i][0..2] <= 1e27 (principal
 * body-frame inverse inertia; 0 locks that DoF; the upper bound keeps the S6
 * fixed-point scales normal floats).  Articulated chains: n_trees chains of
 * tree_ndof in 1..4 DoFs each; their inertia comes per step as Cholesky
 * factors in comfree_worlds (the upstream CRBA is not part of this step). */
typedef struct {
  int32_t n_bodies;
  const float* inv_mass;     /* [n_bodies] */
  const float* inv_inertia;  /* [n_bodies][3] */
  int32_t n_trees;
  int32_t tree_ndof;
} comfree_scene;

/* World state in the public layout (row-major, world-major):
 *   pos [W][n_bodies][3], quat [W][n_bodies][4], vel [W][n_bodies][3],
 *   omega [W][n_bodies][3], qpos [W][Q], qvel [W][Q] with Q = n_trees*tree_ndof
 * (qpos/qvel may be NULL when Q == 0).  location: COMFREE_MEM_*. */
typedef struct {
  float* pos;
  float* quat;
  float* vel;
  float* omega;
  float* qpos;
  float* qvel;
  int32_t location;
} comfree_state;

/* Which worlds one step advances, and their per-step non-contact inputs. */
typedef struct {
  int64_t first_world;       /* step worlds [first_world, first_world + n_worlds) */
  int64_t n_worlds;
  const float* f_ext;        /* [n_worlds][n_bodies][6] world-frame force | torque, or NULL */
  const float* tree_L;       /* [n_worlds][n_trees][10] packed lower-triangular Cholesky
                                factor of each chain's M, L[i(i+1)/2 + j]; required if n_trees */
  const float* tree_tau;     /* [n_worlds][Q] tau - c of the chains; required if n_trees */
  int32_t location;
} comfree_worlds;

/* The detected contact set C, contact-major SoA float4 streams:
 *   c0[n] = (p.x, p.y, p.z, phi)      contact point (world), signed gap
 *   c1[n] = (n.x, n.y, n.z, mu_t)     unit normal a->b, tangential friction
 *   c2[n] = (t1.x, t1.y, t1.z, mu_tor) unit first tangent (orthogonal to n),
 *                                      torsional friction (a length)
 *   c3[n] = (body_a, body_b, bits(mu_rol), condim)  int32 x 4
 *   jrow [12][n][4]: stream s = side*6 + row (side 0 = a, 1 = b): rows 0-2
 *       linear velocity of the contact point, rows 3-5 angular velocity, of
 *       an articulated side, one column per chain DoF; NULL if no chains.
 *   kd [n][2] (optional, NULL = use the config's pair): per-contact
 *       (k_user, d_user) replacing the global pair of Eq. (12), for
 *       user-set or learned impedance; finite and >= 0
 *       (checked on the device, reported as COMFREE_ERR_VALIDATION).
 * Segmentation (S0): if off != NULL contacts are grouped by world and
 * off[n_worlds + 1] is their CSR (no S0 work).  Otherwise world[n] (relative
 * to first_world) is used; with COMFREE_CONTACTS_SORTED it must be
 * non-decreasing (checked) and only offsets are built; without it contacts
 * are stably sorted by world on the device.
 * Outputs (optional): impulses[F] = Lambda_f (N s) of every facet, at
 * foff[c] + facet for contact c in input order; foff[n + 1] its exclusive
 * prefix (int64).  Output pointers follow `location`. */
typedef struct {
  int64_t n_contacts;
  const int32_t* world;
  const int64_t* off;
  const float* c0;
  const float* c1;
  const float* c2;
  const int32_t* c3;
  const float* jrow;
  const float* kd;
  float* impulses;
  int64_t* foff;
  int64_t impulses_capacity; /* elements available at impulses (checked) */
  uint32_t flags;
  int32_t location;
  /* optional DEVICE count of the contacts in use (<= n_contacts, which is then
   * the length / stride of every stream), e.g. from comfree_collide in its
   * asynchronous mode: no host round trip, graph-capturable.  Needs sorted
   * DEVICE contacts with world[], no off[], impulses or foff. */
  const int64_t* n_device;
} comfree_contacts;

/* Aggregate statistics of the last step. */
typedef struct {
  int64_t n_worlds;
  int64_t contacts;
  int64_t active_facets;          /* facets with Lambda > 0 */
  float max_penetration;          /* max(0, -phi) over contacts */
  double kinetic_energy;          /* sum over worlds, after the step */
  int64_t first_nonfinite_world;  /* -1 if none */
} comfree_stats;

/* Per-world statistics record (COMFREE_FLAG_STATS). */
typedef struct {
  int32_t contacts;
  int32_t active_facets;
  float max_penetration;
  float kinetic_energy;
} comfree_world_stats;

/* ---- API ---------------------------------------------------------------- */

int comfree_abi_version(void);
const char* comfree_status_string(comfree_status s);

/* Fill *cfg with the paper's defaults (k=0.1, d=0.001 as in P:390; solimp
 * defaults; n_t = n_rol = 4; gravity (0,0,-9.81); flags 0).  CPU only. */
comfree_status comfree_default_config(comfree_config* cfg);

/* Check a config against the invariants above without touching the GPU. */
comfree_status comfree_validate_config(const comfree_config* cfg);

/* Check scene parameters (HOST) without touching the GPU. */
comfree_status comfree_validate_scene(const comfree_scene* scene);

/* Facets per contact for a condim under cfg (Eq. (7)-(8) facet sets); -1 if
 * condim is not one of 1, 3, 4, 6. */
int32_t comfree_facets_per_contact(const comfree_config* cfg, int32_t condim);

/* Create a context on CUDA device `cuda_device`.  *out owned by the caller,
 * release with comfree_destroy. */
comfree_status comfree_create(const comfree_config* cfg, int cuda_device, comfree_ctx** out);

/* Allocate state for n_worlds copies of the scene and set the initial state
 * (any location; NULL -> zero velocities, identity orientations, zero
 * positions).  Synchronous. */
comfree_status comfree_load_scene(comfree_ctx* ctx, const comfree_scene* scene, int64_t n_worlds,
                                  const comfree_state* initial);

/* One step of duration dt > 0 for the worlds in *worlds with contacts *c.
 * Asynchronous on `stream` when every buffer is on the device.
 * Deterministic: the J^T lambda scatter (S6) accumulates each body's
 * generalized impulse in 64-bit fixed point (scale 2^(exponent(m^-1)+33)
 * linear, 2^(exponent(max diag I_w^-1)+33) angular, i.e. a velocity
 * resolution near 1e-10) with integer atomics, so the result is bitwise
 * identical run to run for the same input (contact order included).  Every
 * add is bounded by 2^62 / (2 n_c + 2) for a world of n_c contacts (about
 * 2^17 m/s of velocity change per contact at 2000 contacts), so no sum can
 * wrap; an add beyond the bound, or a non-finite impulse (from a non-finite
 * contact record), is reported as COMFREE_ERR_NONFINITE for its world. */
comfree_status comfree_step(comfree_ctx* ctx, const comfree_worlds* worlds,
                            const comfree_contacts* c, float dt, void* stream);

/* Copy the state of worlds [first_world, first_world + n_worlds) out to *out
 * (public layout, arrays sized for n_worlds).  Synchronises `stream`,
 * surfaces latched device errors. */
comfree_status comfree_get_state(comfree_ctx* ctx, int64_t first_world, int64_t n_worlds,
                                  comfree_state* out, void* stream);

/* Overwrite the state of worlds [first_world, first_world + n_worlds)
 * (snapshots, MPPI resets). */
comfree_status comfree_set_state(comfree_ctx* ctx, int64_t first_world, int64_t n_worlds,
                                  const comfree_state* in, void* stream);

/* World first_world + i (0 <= i < n_src * repeat) takes source state i / repeat
 * of *in (n_src worlds in the public layout, HOST or DEVICE): e.g. MPPI's
 * live states broadcast to every rollout world of their problem, with only
 * the n_src source states crossing PCIe (the replication runs on the device). */
comfree_status comfree_set_state_broadcast(comfree_ctx* ctx, int64_t first_world, int64_t n_src, int64_t repeat,
                                           const comfree_state* in, void* stream);

/* ---- Articulated upstream ----------------------------
 * The step takes each chain's Cholesky factor of M(q), tau - c(q, v) and the
 * J rows of chain-side contacts as inputs (Eq. (1)-(2), P:80-97;
 * Eq. (4)-(5)).  For serial hinge chains these can be computed on
 * the device from the state with the two calls below.
 *
 * Chain t starts at base[t] with the world frame's orientation; joint j
 * rotates about axis[t][j] (unit, in the frame of the link before it; the
 * base frame for j = 0); link j extends length[t][j] along its local +z,
 * has mass[t][j] at mid-length and isotropic rotational inertia inertia[t][j]
 * about its centre of mass; armature[t][j] adds to M's diagonal:
 *   M(q) = diag(armature) + sum_l m_l Jv_l^T Jv_l + I_l Jw_l^T Jw_l,
 *   c(q, v) = the Coriolis/centrifugal/gravity bias (gravity from the config).
 * HOST arrays, copied; n_trees / tree_ndof must equal the loaded scene's. */
typedef struct {
  int32_t n_trees, tree_ndof;
  const float* base;      /* [T][3] */
  const float* axis;      /* [T][nd][3] */
  const float* length;    /* [T][nd] */
  const float* mass;      /* [T][nd] */
  const float* inertia;   /* [T][nd] */
  const float* armature;  /* [T][nd] */
} comfree_articulation;

/* Validate and copy the chain model to the device (after load_scene).
 * COMFREE_ERR_VALIDATION on a size mismatch, a non-unit axis or a negative
 * link parameter. */
comfree_status comfree_load_articulation(comfree_ctx* ctx, const comfree_articulation* art);

/* For worlds [first_world, first_world + n_worlds), from the current state's
 * chain q, v (the step-start pose, reading R17): tree_L[n_worlds][T][10]
 * (packed Cholesky factor of M(q)) and tree_tau[n_worlds][Q] = tau_ext - c
 * (tau_ext [n_worlds][Q] or NULL).  For the n contacts (world ids world[n],
 * absolute; c0[n][4] points; c3[n][4] body ids as in comfree_contacts; link
 * [n][2] link index of each side, read for chain sides only): the chain-side
 * J rows at the contact point into jrow[12][n][4] (the comfree_contacts.jrow
 * layout; rows of other sides are not written).  All pointers DEVICE,
 * asynchronous on `stream`; errors (M not positive definite, bad chain or
 * link id) are reported by the next synchronising call as
 * COMFREE_ERR_VALIDATION. */
comfree_status comfree_articulation_update(comfree_ctx* ctx, int64_t first_world, int64_t n_worlds,
                                           const float* tau_ext, float* tree_L, float* tree_tau,
                                           int64_t n_contacts, const int64_t* n_device, const int32_t* world,
                                           const float* c0, const int32_t* c3, const int32_t* link, float* jrow,
                                           void* stream);

/* ---- Collision front-end -------------------------------
 * Primitive narrowphase over a candidate pair list shared by every world,
 * emitting the step's contact records (the paper takes them from MJWarp's
 * collision; records as PAPER.md P:244-246).  Geom k: kind[k] 0 sphere
 * (size[k][0] = radius), 1 box (size = half extents along the frame's axes),
 * 2 plane (static; size = unit normal, local[k][0] = offset, n . x = offset),
 * 3 capsule (size = (radius, half length), segment along the frame's z);
 * attached to body[k] (>= 0 free body, -1 world, -(2+t) chain t at link[k],
 * which needs comfree_load_articulation) at local[k] in that frame.  Pair p =
 * (pairs[2p], pairs[2p+1]) = (g1, g2): plane first with a sphere, box or
 * capsule, or any two of sphere / box / capsule (box-box by vertex-face,
 * capsule-box by the capsule's end spheres: DESIGN.md R25; at most 16
 * contacts per pair); the contact normal points from g1 to g2
 * (body_a = body of g1), phi is the signed surface distance, the point the
 * midpoint of the two surface points, t1 the branch-free basis of Duff et al.
 * (2017); a pair emits when phi < margin (plane-box: every corner below).
 * Every contact carries mu[0..2] = (mu_t, mu_tor, mu_rol) and condim.
 * HOST arrays, copied. */
typedef struct {
  int32_t n_geoms, n_pairs;
  const int32_t* kind;    /* [G] */
  const int32_t* body;    /* [G] */
  const int32_t* link;    /* [G] (chain geoms) */
  const float* size;      /* [G][3] */
  const float* local;     /* [G][3] */
  const int32_t* pairs;   /* [P][2] */
  float margin;
  float mu[3];
  int32_t condim;
} comfree_geometry;

/* Validate and copy the geometry (after load_scene, and load_articulation
 * when chain geoms are present).  COMFREE_ERR_VALIDATION on bad kinds, bodies,
 * links, sizes, unsupported pair kinds, margin / friction / condim. */
comfree_status comfree_load_geometry(comfree_ctx* ctx, const comfree_geometry* geo);

/* Contacts of worlds [first_world, first_world + n_worlds) at the current
 * state into DEVICE arrays of `capacity` records: world[n] (ids relative to
 * first_world, as comfree_step takes them; sorted), c0/c1/c2 [n][4], c3 [n][4] (the comfree_contacts streams) and
 * link [n][2] (link index of chain sides, for comfree_articulation_update);
 * world-major, candidate-pair order within a world (deterministic).
 * With n_device == NULL: synchronises `stream` once to read the count into
 * *n_contacts (HOST); COMFREE_ERR_CAPACITY (with *n_contacts set) when it
 * exceeds capacity.  With n_device (DEVICE int64): asynchronous, the count
 * (clamped to capacity) goes to *n_device for comfree_contacts.n_device and
 * comfree_articulation_update; an overflow is reported as
 * COMFREE_ERR_CAPACITY by the next synchronising call. */
comfree_status comfree_collide(comfree_ctx* ctx, int64_t first_world, int64_t n_worlds, int64_t capacity,
                               int32_t* world, float* c0, float* c1, float* c2, int32_t* c3, int32_t* link,
                               int64_t* n_contacts, int64_t* n_device, void* stream);

/* One full step from the geometry: comfree_collide (the broadphase mode of
 * reading R32 and the narrowphase, §II, §IV) followed by
 * comfree_step (Alg. 1) on worlds [first_world, first_world +
 * n_worlds), with the contact records kept where the front-end leaves them:
 * the step reads each world's placed records (point, phi, normal, geom pair:
 * 32 B) from the front-end's staging area and expands them (tangent,
 * friction, condim, bodies) as the emit pass would, so no public contact
 * streams are written or read.  The state is bit-identical to comfree_collide
 * + comfree_step (the step's result does not depend on the contacts' memory
 * layout).  A world with more records than the staging area is written in
 * place into library-owned streams of `capacity` records (whole pairs; an
 * overflow sets COMFREE_ERR_CAPACITY, reported by the next synchronising
 * call).  Requires a geometry without a candidate list (broadphase mode) and
 * a scene without chains; `worlds` as comfree_step takes it (DEVICE inputs).
 * Configurations the staged kernel does not cover (general facet sets,
 * per-facet impedance, statistics) run comfree_collide + comfree_step on the
 * library-owned streams instead.  Asynchronous, graph-capturable. */
comfree_status comfree_step_collided(comfree_ctx* ctx, const comfree_worlds* worlds, int64_t capacity, float dt,
                                     void* stream);

/* ---- MPPI on the batched step -------------------------
 * PAPER.md §V, Eq. (14)-(15), P:490-512 (reading R27).  The rollout
 * worlds of a context are P problems x N samples, world w belonging to problem
 * w / N; plans and samples are DEVICE arrays in DoF-minor layout: plan
 * [P][H][Q], U [P][N][H][Q] (Q = the scene's chain DoFs).  A control step is
 * mppi_sample, then for t = 0..H-1 {mppi_cost (running), mppi_control,
 * collide / articulation_update / step}, mppi_cost (terminal), mppi_update. */
typedef struct {
  int32_t object_body;       /* the manipulated free body */
  const float* target_pos;   /* [P][3] DEVICE */
  const float* target_quat;  /* [P][4] DEVICE (w, x, y, z) */
  const float* q_ref;        /* [Q] DEVICE home pose */
  float w[6];                /* Eq. (15): quat, |dx|, |dy|, |dz|, fingertip-object, joint */
  float omega_fallen, z_fallen;  /* Omega, fallen when p_z < z_fallen */
  float phi1, phi2;          /* terminal V */
} comfree_mppi_task;

/* U = clip(plan + eps, lo, hi), eps_k = sigma sqrt(-2 ln(1 - u1)) cos(2 pi u2)
 * with u1, u2 the top 24 bits of SplitMix64(seed + 2k), SplitMix64(seed + 2k + 1)
 * over 2^24 and k = iteration * (P N H Q) + the element index (counter-based:
 * reproducible, independent of launch shape).  sigma > 0, lo <= hi. */
comfree_status comfree_mppi_sample(comfree_ctx* ctx, int32_t n_problems, int32_t n_samples, int32_t horizon,
                                   const float* plan, float sigma, float lo, float hi, uint64_t seed,
                                   uint64_t iteration, float* U, void* stream);

/* Incremental position control for worlds [first_world, +n_worlds): command
 * [n_worlds][Q] += U[w][t], then tau[n_worlds][Q] = kp (command - q) - kd qdot
 * from the current state (pass tau as tau_ext to comfree_articulation_update). */
comfree_status comfree_mppi_control(comfree_ctx* ctx, int64_t first_world, int64_t n_worlds, const float* U,
                                    int32_t t, int32_t horizon, float kp, float kd, float* command, float* tau,
                                    void* stream);

/* J[n_worlds] += Eq. (15)'s running cost c(x) (terminal = 0) or terminal V(x)
 * (terminal = 1) of the current state of each world (fingertips = chain tips
 * from the loaded articulation; needs comfree_load_articulation). */
comfree_status comfree_mppi_cost(comfree_ctx* ctx, int64_t first_world, int64_t n_worlds, int32_t n_samples,
                                 const comfree_mppi_task* task, int32_t terminal, float* J, void* stream);

/* comfree_mppi_cost (running, terminal = 0) and comfree_mppi_control of the
 * same rollout step t in one launch (both read the current state only). */
comfree_status comfree_mppi_cost_control(comfree_ctx* ctx, int64_t first_world, int64_t n_worlds,
                                         int32_t n_samples, const comfree_mppi_task* task, float* J,
                                         const float* U, int32_t t, int32_t horizon, float kp, float kd,
                                         float* command, float* tau, void* stream);

/* Per problem: w_i = exp(-(J_i - min J)/lambda) / sum (weights [P][N] or
 * NULL), plan[P][H][Q] = clip(sum_i w_i U_i, lo, hi).  lambda > 0; N <= 12288. */
comfree_status comfree_mppi_update(comfree_ctx* ctx, int32_t n_problems, int32_t n_samples, int32_t horizon,
                                   const float* J, const float* U, float lambda, float lo, float hi, float* plan,
                                   float* weights, void* stream);

/* comfree_mppi_update plus the receding-horizon shift, in the same launch:
 * u0[P][Q] (DEVICE) receives the new plan's first action and plan[P][H][Q]
 * the new plan advanced by one step (its last step 0).  A problem whose costs
 * are all non-finite keeps its plan (shifted the same way). */
comfree_status comfree_mppi_update_shift(comfree_ctx* ctx, int32_t n_problems, int32_t n_samples, int32_t horizon,
                                         const float* J, const float* U, float lambda, float lo, float hi, float* plan,
                                         float* weights, float* u0, void* stream);

/* Aggregate statistics of the last step (requires COMFREE_FLAG_STATS for
 * contacts / facets / penetration / energy; the non-finite check is always
 * on unless COMFREE_FLAG_NO_FINITE_CHECK).  Synchronises. */
comfree_status comfree_get_stats(comfree_ctx* ctx, comfree_stats* out, void* stream);

/* Per-world statistics of the last step into out[n_worlds] (location).  */
comfree_status comfree_get_world_stats(comfree_ctx* ctx, int64_t first_world, int64_t n_worlds,
                                       comfree_world_stats* out, int32_t location, void* stream);

/* S0 results of the last step (device scratch copied to HOST arrays):
 * off[n_worlds + 1] int64, perm[n_contacts] int32 (stable world order; the
 * identity when the input was already grouped).  Synchronises. */
comfree_status comfree_segment_info(comfree_ctx* ctx, int64_t* off, int32_t* perm, void* stream);

/* Synchronise `stream` and surface the device errors latched by earlier
 * asynchronous calls (collision overflow, device validation, non-finite
 * state), then clear them: COMFREE_OK when none.  A cheap check (one 4-byte
 * read) for loops that never call comfree_get_* (e.g. MPPI control steps). */
comfree_status comfree_check(comfree_ctx* ctx, void* stream);

/* Make `stream` wait (on the device, no host sync) for every copy the
 * COMFREE_MEM_HOST_ASYNC path has enqueued so far, so that an event recorded
 * on `stream` afterwards, or a synchronisation of `stream`, covers them. */
comfree_status comfree_wait_async(comfree_ctx* ctx, void* stream);

/* Instrumentation: while enabled, every comfree_step records CUDA events on
 * its own stream around the S0 kernels and around the fused step kernel. */
comfree_status comfree_set_timing(comfree_ctx* ctx, int enable);

/* Sums of the recorded device durations since the previous call, in ms:
 * out[0] fused step kernel, out[1] S0 kernels, out[2] number of fused-step
 * launches timed.  Synchronises the recorded events; clears the record. */
comfree_status comfree_get_timing(comfree_ctx* ctx, double out[3]);

/* Number of kernels this context has launched so far (instrumentation). */
int64_t comfree_kernel_launches(const comfree_ctx* ctx);

void comfree_destroy(comfree_ctx* ctx);
const char* comfree_last_error(const comfree_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* COMFREE_H */
