/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.  Plain fp64 CPU oracle of the
 * ComFree-Sim contact-resolution step (arXiv 2603.12185, §III).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this.  It shares no code, header, table or
 * helper with the CUDA path (paper_2603_12185_b200/csrc, include/comfree.h).
 *
 * Data layout (public exchange format, also produced by harness/scenes.py):
 *   per world w, body i:  pos[w][i][3], quat[w][i][4] (w,x,y,z), vel[w][i][3],
 *                         omega[w][i][3]  (world-frame angular velocity)
 *   per world w, tree DoF: qpos[w][Q], qvel[w][Q]   (Q = n_trees * tree_ndof)
 *   per contact c:  c0[c] = (p.x, p.y, p.z, phi)      contact point, signed gap
 *                   c1[c] = (n.x, n.y, n.z, mu_t)     normal a->b, tangential mu
 *                   c2[c] = (t1.x, t1.y, t1.z, mu_tor) first tangent, torsional mu
 *                   body_a[c], body_b[c]: >=0 free body, -1 static, -(2+t) tree t
 *                   mu_rol[c], condim[c] in {1,3,4,6}
 *                   jrow[c][side][6][4]: rows 0-2 linear point-velocity Jacobian,
 *                   rows 3-5 angular-velocity Jacobian of an articulated side,
 *                   columns = the tree's DoFs (only read for tree sides).
 */
#ifndef COMFREE_ORACLE_H
#define COMFREE_ORACLE_H
#include <stdint.h>

typedef struct {
  double k_user, d_user;                         /* Eq. (12) */
  double r_min, r_max, width, midpoint, power;   /* Eq. (13) */
  int32_t n_t, n_rol;                            /* Eq. (7) facet counts */
  double gravity[3];
  double dt;
  int32_t exact_diagonal;   /* 0: M(phi) of Eq. (12) (trace heuristic);
                               1: Eq. (11) literally (reading R24): per facet
                               K_f dt + D_f = 1/(dt A_f), A_f = J~_f M^-1 J~_f^T,
                               split K_f dt : D_f = k dt : d;
                               2: Eq. (12) with the facet diagonal (reading R28):
                               M_f = r/(1-r) / A_f, K_f = k M_f/dt, D_f = d M_f/dt */
} orc_config;

typedef struct {
  int32_t n_bodies;            /* free 6-DoF bodies per world */
  const double* inv_mass;      /* [n_bodies] */
  const double* inv_inertia;   /* [n_bodies][3] principal body-frame I^-1 */
  int32_t n_trees;             /* articulated chains per world */
  int32_t tree_ndof;           /* DoFs per chain, 1..4 */
} orc_scene;

/* Status codes. */
enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ENONFINITE = 2 };

/* S0: world segmentation with plain loops.  off[n_worlds+1], perm[n] (stable
 * by world id), foff[n+1] (exclusive prefix of facets per contact, in input
 * order). */
int orc_segment(int64_t n_contacts, const int32_t* world, int64_t n_worlds,
                const int32_t* condim, int32_t n_t, int32_t n_rol,
                int64_t* off, int32_t* perm, int64_t* foff);

/* Facets per contact for a condim (Eq. (7)-(8) facet sets, reading A11). */
int orc_facets_per_contact(int32_t condim, int32_t n_t, int32_t n_rol);

/* One step of Algorithm 1 (Kernels I-IV; sign per Eq. (9)) plus
 * the semi-implicit integrator, in place on the state arrays.
 * impulses: [F] Lambda_f = lambda_f * dt in foff order, or NULL.
 * wrench:   [n][6] per-contact (f_c, tau_c) on body b, or NULL.
 * stats:    [n_worlds][5] (contacts, active facets, max penetration, KE,
 *           non-finite flag), or NULL.
 * kd:       [n][2] per-contact (k_user, d_user) replacing the global pair in
 *           Eq. (12) (user-set or learned impedance), or NULL.
 * n_threads > 1 parallelises across worlds only (timing driver).       */
int orc_step(const orc_config* cfg, const orc_scene* scene, int64_t n_worlds,
             double* pos, double* quat, double* vel, double* omega,
             double* qpos, double* qvel,
             const double* f_ext, const double* tree_L, const double* tree_tau,
             int64_t n_contacts, const int32_t* world,
             const double* c0, const double* c1, const double* c2,
             const int32_t* body_a, const int32_t* body_b,
             const double* mu_rol, const int32_t* condim, const double* jrow,
             const double* kd,
             double* impulses, double* wrench, double* stats, int n_threads);

/* Pieces exposed for the pins (same code the step uses). */
double orc_gamma(double x, double m, double p);                 /* Eq. (13b) */
double orc_r(double phi, const orc_config* cfg);                /* Eq. (13a) */
double orc_facet_lambda(double K, double D, double s, double phi, double dt); /* Eq. (9) */

#endif
