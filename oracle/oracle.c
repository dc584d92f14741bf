/*
 * oracle.c — TEST INFRASTRUCTURE ONLY: the plain, slow, fp64 CPU oracle of
 * the ComFree-Sim contact-resolution step (arXiv 2603.12185).
 *
 * Written from PAPER.md, step by step in the paper's order and notation:
 *   Kernel I   smooth prediction          Eq. (2)  P:91-97,  Alg.1
 *   Kernel II  per-contact, per-facet     Eq. (4)-(9), (12)-(13)
 *              closed-form impulse        P:109-180, Alg.1
 *              (sign of Eq. (9), not the garbled Alg.1 line P:260; R1)
 *   Kernel III p += J~^T lambda dt        Alg.1, Eq. (10)
 *   Kernel IV  v+ = v_s + M^-1 p          Eq. (10), Alg.1
 *   integration (semi-implicit Euler, exp-map quaternion; "same time
 *              integration" as MJWarp; reading R15 in DESIGN.md)
 *
 * No blocking, fusion or regrouping: each facet's row J~_f is formed as a
 * contact-space covector g_f, J~_f v = g_f . (J_b v - J_a v), and its
 * transpose is applied literally per facet.  The trace in M(phi) is formed as
 * the trace of the 3x3 matrix J_i M^-1 J_i^T (reading R6), not a closed form.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
 * --impl reference) may load this library.  It shares nothing with the CUDA
 * path.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* small linear algebra, written out                                  */
/* ------------------------------------------------------------------ */
static double dot3(const double* a, const double* b) { return a[0]*b[0] + a[1]*b[1] + a[2]*b[2]; }
static void cross3(const double* a, const double* b, double* o) {
  double x = a[1]*b[2] - a[2]*b[1];
  double y = a[2]*b[0] - a[0]*b[2];
  double z = a[0]*b[1] - a[1]*b[0];
  o[0] = x; o[1] = y; o[2] = z;
}
/* 3x3 row-major */
static void matvec3(const double* M, const double* x, double* o) {
  for (int i = 0; i < 3; ++i) o[i] = M[3*i]*x[0] + M[3*i+1]*x[1] + M[3*i+2]*x[2];
}
static void matmul3(const double* A, const double* B, double* C) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += A[3*i+k] * B[3*k+j];
      C[3*i+j] = s;
    }
}
static void transpose3(const double* A, double* T) {
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) T[3*j+i] = A[3*i+j];
}
/* rotation matrix of the quaternion (w,x,y,z), scalar first,
 * normalised first: stored fp32 quaternions are unit only to ~1e-7, and a
 * non-orthogonal R would make R diag(I^-1) R^T differ from (R diag(I) R^T)^-1
 * (reading R15 in DESIGN.md). */
static void quat_to_R(const double* q0, double* R) {
  double nq = sqrt(q0[0]*q0[0] + q0[1]*q0[1] + q0[2]*q0[2] + q0[3]*q0[3]);
  double w = q0[0] / nq, x = q0[1] / nq, y = q0[2] / nq, z = q0[3] / nq;
  R[0] = 1 - 2*(y*y + z*z); R[1] = 2*(x*y - w*z);     R[2] = 2*(x*z + w*y);
  R[3] = 2*(x*y + w*z);     R[4] = 1 - 2*(x*x + z*z); R[5] = 2*(y*z - w*x);
  R[6] = 2*(x*z - w*y);     R[7] = 2*(y*z + w*x);     R[8] = 1 - 2*(x*x + y*y);
}
/* R diag(d) R^T */
static void rot_diag(const double* R, const double* d, double* out) {
  double D[9] = {d[0],0,0, 0,d[1],0, 0,0,d[2]}, RD[9], RT[9];
  matmul3(R, D, RD);
  transpose3(R, RT);
  matmul3(RD, RT, out);
}
/* skew matrix [r]x such that [r]x y = r x y */
static void skew3(const double* r, double* S) {
  S[0] = 0;     S[1] = -r[2]; S[2] = r[1];
  S[3] = r[2];  S[4] = 0;     S[5] = -r[0];
  S[6] = -r[1]; S[7] = r[0];  S[8] = 0;
}
/* Hamilton product a (x) b, scalar first */
static void quat_mul(const double* a, const double* b, double* o) {
  double w = a[0]*b[0] - a[1]*b[1] - a[2]*b[2] - a[3]*b[3];
  double x = a[0]*b[1] + a[1]*b[0] + a[2]*b[3] - a[3]*b[2];
  double y = a[0]*b[2] - a[1]*b[3] + a[2]*b[0] + a[3]*b[1];
  double z = a[0]*b[3] + a[1]*b[2] - a[2]*b[1] + a[3]*b[0];
  o[0] = w; o[1] = x; o[2] = y; o[3] = z;
}

/* packed lower-triangular 4x4 Cholesky factor, row-major: L(i,j) = L[i(i+1)/2 + j] */
static double Lget(const double* L, int i, int j) { return L[i*(i+1)/2 + j]; }
/* x <- M^-1 x with M = L L^T (forward then backward substitution) */
static void tree_minv(const double* L, int nd, double* x) {
  double y[4];
  for (int i = 0; i < nd; ++i) {
    double s = x[i];
    for (int j = 0; j < i; ++j) s -= Lget(L, i, j) * y[j];
    y[i] = s / Lget(L, i, i);
  }
  for (int i = nd - 1; i >= 0; --i) {
    double s = y[i];
    for (int j = i + 1; j < nd; ++j) s -= Lget(L, j, i) * x[j];
    x[i] = s / Lget(L, i, i);
  }
}

/* ------------------------------------------------------------------ */
/* Eq. (13): gap-dependent scaling r(|phi|), MuJoCo impedance curve    */
/* ------------------------------------------------------------------ */
double orc_gamma(double x, double m, double p) {
  /* Eq. (13b); x clamped to [0,1] by the caller (reading R7) */
  if (x < m) return m * pow(x / m, p);
  return 1.0 - (1.0 - m) * pow((1.0 - x) / (1.0 - m), p);
}
double orc_r(double phi, const orc_config* cfg) {
  /* Eq. (13a): r = r_min + (r_max - r_min) gamma(x), x = |phi| / w */
  double x = fabs(phi) / cfg->width;
  if (x > 1.0) x = 1.0;
  return cfg->r_min + (cfg->r_max - cfg->r_min) * orc_gamma(x, cfg->midpoint, cfg->power);
}
/* Eq. (9): lambda = ( -K (s dt + phi) - D s )_+ */
double orc_facet_lambda(double K, double D, double s, double phi, double dt) {
  double v = -K * (s * dt + phi) - D * s;
  return v > 0.0 ? v : 0.0;
}

int orc_facets_per_contact(int32_t condim, int32_t n_t, int32_t n_rol) {
  switch (condim) {
    case 1: return 1;                 /* normal only */
    case 3: return n_t;               /* tangential channel */
    case 4: return n_t + 2;           /* + torsional {+1,-1} */
    case 6: return n_t + 2 + n_rol;   /* + rolling */
    default: return -1;
  }
}

int orc_segment(int64_t n, const int32_t* world, int64_t n_worlds,
                const int32_t* condim, int32_t n_t, int32_t n_rol,
                int64_t* off, int32_t* perm, int64_t* foff) {
  for (int64_t w = 0; w <= n_worlds; ++w) off[w] = 0;
  for (int64_t c = 0; c < n; ++c) {
    if (world[c] < 0 || world[c] >= n_worlds) return ORC_EINVAL;
    off[world[c] + 1] += 1;
  }
  for (int64_t w = 0; w < n_worlds; ++w) off[w + 1] += off[w];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_worlds + 1));
  for (int64_t w = 0; w <= n_worlds; ++w) fill[w] = off[w];
  for (int64_t c = 0; c < n; ++c) perm[fill[world[c]]++] = (int32_t)c;  /* stable */
  free(fill);
  foff[0] = 0;
  for (int64_t c = 0; c < n; ++c) {
    int nf = orc_facets_per_contact(condim[c], n_t, n_rol);
    if (nf < 0) return ORC_EINVAL;
    foff[c + 1] = foff[c] + nf;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* per-world step                                                      */
/* ------------------------------------------------------------------ */
typedef struct {
  /* per-body, step-start pose quantities */
  double Iw_inv[9];   /* R diag(I_b^-1) R^T */
  double vs[3], ws[3];/* smooth-predicted velocities, Eq. (2) */
  double p_lin[3], p_ang[3]; /* accumulated generalized impulse, Kernel III */
} body_work;

/* side kinematics: point velocity and angular velocity of the contact point
 * on side x (J_x v_s), and the trace tr(J_x M^-1 J_x^T) of its 3-row linear
 * point Jacobian (reading R6: static -> 0). */
static void side_velocity(int32_t id, const double* p, const double* pos_w, const body_work* bw,
                          const double* qd_s, int nd, const double* J, double* vpt, double* wang) {
  if (id == -1) { vpt[0] = vpt[1] = vpt[2] = 0; wang[0] = wang[1] = wang[2] = 0; return; }
  if (id >= 0) {
    const double* x = pos_w + 3 * id;
    double r[3] = {p[0] - x[0], p[1] - x[1], p[2] - x[2]}, wxr[3];
    cross3(bw[id].ws, r, wxr);
    for (int k = 0; k < 3; ++k) { vpt[k] = bw[id].vs[k] + wxr[k]; wang[k] = bw[id].ws[k]; }
    return;
  }
  int t = -2 - id;
  const double* qd = qd_s + t * nd;
  for (int k = 0; k < 3; ++k) {
    double sl = 0, sa = 0;
    for (int j = 0; j < nd; ++j) { sl += J[k*4 + j] * qd[j]; sa += J[(3+k)*4 + j] * qd[j]; }
    vpt[k] = sl; wang[k] = sa;
  }
}

static double side_trace(int32_t id, const double* p, const double* pos_w, const double* inv_mass,
                         const body_work* bw, const double* Lw, int nd, const double* J) {
  if (id == -1) return 0.0;
  if (id >= 0) {
    /* J_lin = [ I_3 , -[r]x ] over (v, omega);  M^-1 = diag(inv_m I_3, Iw^-1).
     * J M^-1 J^T = inv_m I_3 + [r]x Iw^-1 [r]x^T ; take its trace. */
    const double* x = pos_w + 3 * id;
    double r[3] = {p[0] - x[0], p[1] - x[1], p[2] - x[2]};
    double S[9], ST[9], SI[9], SIS[9];
    skew3(r, S);
    transpose3(S, ST);
    matmul3(S, bw[id].Iw_inv, SI);
    matmul3(SI, ST, SIS);
    double im = inv_mass[id];
    return (im + SIS[0]) + (im + SIS[4]) + (im + SIS[8]);
  }
  int t = -2 - id;
  const double* L = Lw + 10 * t;
  double tr = 0.0;
  for (int k = 0; k < 3; ++k) {      /* tr = sum_k J_k M^-1 J_k^T */
    double y[4] = {0, 0, 0, 0};
    for (int j = 0; j < nd; ++j) y[j] = J[k*4 + j];
    tree_minv(L, nd, y);
    for (int j = 0; j < nd; ++j) tr += J[k*4 + j] * y[j];
  }
  return tr;
}

/* g J_x M_x^-1 J_x^T g^T for a facet row g = (gl, ga) acting on the contact
 * twist, restricted to side x (its contribution to the diagonal entry
 * J~_f M^-1 J~_f^T of Eq. (11); a side's sign drops out). */
static double side_quad(int32_t id, const double* p, const double* pos_w, const double* inv_mass,
                        const body_work* bw, const double* Lw, int nd, const double* J,
                        const double gl[3], const double ga[3]) {
  if (id == -1) return 0.0;
  if (id >= 0) {
    /* J_x^T g = (gl, r x gl + ga) for a free body; M_x^-1 = diag(inv_m I_3, Iw^-1) */
    const double* x = pos_w + 3 * id;
    double r[3] = {p[0] - x[0], p[1] - x[1], p[2] - x[2]}, u[3], Iu[3];
    cross3(r, gl, u);
    for (int k = 0; k < 3; ++k) u[k] += ga[k];
    matvec3(bw[id].Iw_inv, u, Iu);
    return inv_mass[id] * dot3(gl, gl) + dot3(u, Iu);
  }
  /* tree: y = J_lin^T gl + J_ang^T ga over the chain's DoFs; y^T (L L^T)^-1 y */
  int t = -2 - id;
  double y[4] = {0, 0, 0, 0}, z[4] = {0, 0, 0, 0};
  for (int j = 0; j < nd; ++j) {
    for (int k = 0; k < 3; ++k) y[j] += J[k*4 + j] * gl[k] + J[(3+k)*4 + j] * ga[k];
    z[j] = y[j];
  }
  tree_minv(Lw + 10 * t, nd, z);
  double q = 0.0;
  for (int j = 0; j < nd; ++j) q += y[j] * z[j];
  return q;
}

/* apply J_x^T (f, tau) * sign to side x's generalized impulse */
static void side_scatter(int32_t id, double sign, const double* p, const double* pos_w,
                         body_work* bw, double* p_tree, int nd, const double* J,
                         const double* f, const double* tau) {
  if (id == -1) return;
  if (id >= 0) {
    /* J_x^T (f, tau) = (f, r x f + tau) for a free body */
    const double* x = pos_w + 3 * id;
    double r[3] = {p[0] - x[0], p[1] - x[1], p[2] - x[2]}, rxf[3];
    cross3(r, f, rxf);
    for (int k = 0; k < 3; ++k) {
      bw[id].p_lin[k] += sign * f[k];
      bw[id].p_ang[k] += sign * (rxf[k] + tau[k]);
    }
    return;
  }
  int t = -2 - id;
  double* pt = p_tree + t * nd;
  for (int j = 0; j < nd; ++j) {
    double s = 0;
    for (int k = 0; k < 3; ++k) s += J[k*4 + j] * f[k] + J[(3+k)*4 + j] * tau[k];
    pt[j] += sign * s;
  }
}

static int step_world(const orc_config* cfg, const orc_scene* sc, int64_t w,
                      double* pos, double* quat, double* vel, double* omega,
                      double* qpos, double* qvel,
                      const double* f_ext, const double* tree_L, const double* tree_tau,
                      int64_t c_begin, int64_t c_end, const int32_t* perm,
                      const double* c0, const double* c1, const double* c2,
                      const int32_t* body_a, const int32_t* body_b,
                      const double* mu_rol, const int32_t* condim, const double* jrow,
                      const double* kd,
                      const int64_t* foff, double* impulses, double* wrench, double* stats) {
  const int B = sc->n_bodies, T = sc->n_trees, nd = sc->tree_ndof, Q = T * nd;
  const double dt = cfg->dt;
  double* pos_w = pos + (size_t)w * B * 3;
  double* quat_w = quat + (size_t)w * B * 4;
  double* vel_w = vel + (size_t)w * B * 3;
  double* om_w = omega + (size_t)w * B * 3;
  double* qp_w = Q ? qpos + (size_t)w * Q : NULL;
  double* qv_w = Q ? qvel + (size_t)w * Q : NULL;
  const double* L_w = T ? tree_L + (size_t)w * T * 10 : NULL;
  const double* tau_w = Q ? tree_tau + (size_t)w * Q : NULL;

  body_work* bw = (body_work*)calloc((size_t)(B > 0 ? B : 1), sizeof(body_work));
  double qd_s[64], p_tree[64];
  if (Q > 64) { free(bw); return ORC_EINVAL; }

  /* ---- Kernel I: smooth prediction, Eq. (2) v_s = v + M^-1 (tau - c) dt ---- */
  for (int i = 0; i < B; ++i) {
    const double im = sc->inv_mass[i];
    const double* Ibi = sc->inv_inertia + 3 * i;
    double R[9];
    quat_to_R(quat_w + 4 * i, R);
    rot_diag(R, Ibi, bw[i].Iw_inv);
    const double* fe = f_ext ? f_ext + ((size_t)w * B + i) * 6 : NULL;
    /* linear: M^-1 (f + m g) = inv_m f + g (gravity only on translating bodies, reading R14) */
    for (int k = 0; k < 3; ++k) {
      double a = (im > 0.0) ? (im * (fe ? fe[k] : 0.0) + cfg->gravity[k]) : 0.0;
      bw[i].vs[k] = vel_w[3*i + k] + a * dt;
    }
    /* angular: omega_s = omega + Iw^-1 (tau - omega x (Iw omega)) dt; c = gyroscopic term.
     * Iw = R diag(I_b) R^T with I_b = 1/I_b^-1 on unlocked axes, 0 on locked ones. */
    double Ib[3];
    for (int k = 0; k < 3; ++k) Ib[k] = Ibi[k] > 0.0 ? 1.0 / Ibi[k] : 0.0;
    double Iw[9], Iwo[3], gyro[3], rhs[3], dw[3];
    rot_diag(R, Ib, Iw);
    matvec3(Iw, om_w + 3 * i, Iwo);
    cross3(om_w + 3 * i, Iwo, gyro);
    for (int k = 0; k < 3; ++k) rhs[k] = (fe ? fe[3 + k] : 0.0) - gyro[k];
    matvec3(bw[i].Iw_inv, rhs, dw);
    for (int k = 0; k < 3; ++k) bw[i].ws[k] = om_w[3*i + k] + dw[k] * dt;
  }
  for (int t = 0; t < T; ++t) {
    double x[4] = {0, 0, 0, 0};
    for (int j = 0; j < nd; ++j) x[j] = tau_w[t*nd + j];
    tree_minv(L_w + 10 * t, nd, x);                       /* M^-1 (tau - c) */
    for (int j = 0; j < nd; ++j) qd_s[t*nd + j] = qv_w[t*nd + j] + x[j] * dt;
  }
  for (int j = 0; j < Q; ++j) p_tree[j] = 0.0;

  /* ---- Kernel II + III, per contact in input order ---- */
  int64_t n_active = 0;
  double max_pen = 0.0;
  const double k = cfg->k_user, d = cfg->d_user;
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t q = c_begin; q < c_end; ++q) {
    const int64_t c = perm[q];
    const double* P = c0 + 4 * c;
    const double p[3] = {P[0], P[1], P[2]}, phi = P[3];
    const double n[3] = {c1[4*c], c1[4*c+1], c1[4*c+2]}, mu_t = c1[4*c+3];
    const double t1[3] = {c2[4*c], c2[4*c+1], c2[4*c+2]}, mu_tor = c2[4*c+3];
    double t2[3];
    cross3(n, t1, t2);                                    /* t2 = n x t1 */
    const int32_t a = body_a[c], b = body_b[c];
    const double* Ja = jrow ? jrow + (size_t)c * 48 : NULL;
    const double* Jb = jrow ? jrow + (size_t)c * 48 + 24 : NULL;
    if (-phi > max_pen) max_pen = -phi;

    /* Eq. (4)-(5): relative contact twist (v_c, omega_c) = J v_s, b relative to a */
    double va[3], wa[3], vb[3], wb[3], vc[3], wc[3];
    side_velocity(a, p, pos_w, bw, qd_s, nd, Ja, va, wa);
    side_velocity(b, p, pos_w, bw, qd_s, nd, Jb, vb, wb);
    for (int i = 0; i < 3; ++i) { vc[i] = vb[i] - va[i]; wc[i] = wb[i] - wa[i]; }

    /* Eq. (12)-(13): M(phi) = r/(1-r) / (tr_a + tr_b); K = k M/dt, D = d M/dt */
    double tr = side_trace(a, p, pos_w, sc->inv_mass, bw, L_w, nd, Ja)
              + side_trace(b, p, pos_w, sc->inv_mass, bw, L_w, nd, Jb);
    double r = orc_r(phi, cfg);
    double Mphi = r / (1.0 - r) / tr;
    /* per-contact (k_user, d_user) when given, else the global pair */
    const double kc = kd ? kd[2 * c] : k, dc = kd ? kd[2 * c + 1] : d;
    double K = kc * Mphi / dt, D = dc * Mphi / dt;

    /* Eq. (7)-(8): facets. Each facet row J~_f acts on the contact twist through
     * g_f = (g_lin, g_ang):  J~_f v = g_lin . v_c + g_ang . omega_c           */
    double f_c[3] = {0, 0, 0}, tau_c[3] = {0, 0, 0};
    int nf = orc_facets_per_contact(condim[c], cfg->n_t, cfg->n_rol);
    if (nf < 0) { free(bw); return ORC_EINVAL; }
    for (int f = 0; f < nf; ++f) {
      double gl[3] = {n[0], n[1], n[2]}, ga[3] = {0, 0, 0};   /* J_n */
      if (condim[c] != 1) {
        if (f < cfg->n_t) {                 /* tangential: J_n - mu_t d_j^T J_t */
          double th = two_pi * f / cfg->n_t, dj[2] = {cos(th), sin(th)};
          for (int i = 0; i < 3; ++i) gl[i] -= mu_t * (dj[0] * t1[i] + dj[1] * t2[i]);
        } else if (f < cfg->n_t + 2) {      /* torsional: J_n - mu_tor (+-1) J_tor */
          double dj = (f == cfg->n_t) ? 1.0 : -1.0;
          for (int i = 0; i < 3; ++i) ga[i] -= mu_tor * dj * n[i];
        } else {                            /* rolling: J_n - mu_rol d_j^T J_rol */
          int j = f - cfg->n_t - 2;
          double th = two_pi * j / cfg->n_rol, dj[2] = {cos(th), sin(th)};
          for (int i = 0; i < 3; ++i) ga[i] -= mu_rol[c] * (dj[0] * t1[i] + dj[1] * t2[i]);
        }
      }
      double s = dot3(gl, vc) + dot3(ga, wc);                 /* s = J~ v_s */
      double Kf = K, Df = D;
      if (cfg->exact_diagonal) {  /* this facet's own diagonal entry A_f = J~_f M^-1 J~_f^T */
        double A = side_quad(a, p, pos_w, sc->inv_mass, bw, L_w, nd, Ja, gl, ga)
                 + side_quad(b, p, pos_w, sc->inv_mass, bw, L_w, nd, Jb, gl, ga);
        if (cfg->exact_diagonal == 1) {
          /* Eq. (11), literally: K_f dt + D_f = 1 / (dt A_f), split in
           * the user's ratio K_f dt : D_f = k dt : d (reading R24)            */
          double kap = kc * dt + dc;
          Kf = (kc / kap) / (dt * A);
          Df = (dc / kap) / (dt * A);
        } else {
          /* Eq. (12) with the facet diagonal in place of the trace (reading R28) */
          double Mf = r / (1.0 - r) / A;
          Kf = kc * Mf / dt;
          Df = dc * Mf / dt;
        }
      }
      double lam = orc_facet_lambda(Kf, Df, s, phi, dt);      /* Eq. (9) */
      double Lam = lam * dt;                                  /* impulse, Eq. (10) */
      if (Lam > 0.0) n_active++;
      if (impulses) impulses[foff[c] + f] = Lam;
      /* Kernel III: p += J~_f^T Lam = J_b^T (g Lam) - J_a^T (g Lam) */
      double fl[3], fa[3];
      for (int i = 0; i < 3; ++i) { fl[i] = gl[i] * Lam; fa[i] = ga[i] * Lam; }
      side_scatter(b, +1.0, p, pos_w, bw, p_tree, nd, Jb, fl, fa);
      side_scatter(a, -1.0, p, pos_w, bw, p_tree, nd, Ja, fl, fa);
      for (int i = 0; i < 3; ++i) { f_c[i] += fl[i]; tau_c[i] += fa[i]; }
    }
    if (wrench) for (int i = 0; i < 3; ++i) { wrench[6*c + i] = f_c[i]; wrench[6*c + 3 + i] = tau_c[i]; }
  }

  /* ---- Kernel IV: v+ = v_s + M^-1 p ; then integrate ---- */
  int bad = 0;
  double ke = 0.0;
  for (int i = 0; i < B; ++i) {
    const double im = sc->inv_mass[i];
    double dw[3];
    matvec3(bw[i].Iw_inv, bw[i].p_ang, dw);
    double* v = vel_w + 3 * i;
    double* om = om_w + 3 * i;
    double* x = pos_w + 3 * i;
    double* qq = quat_w + 4 * i;
    for (int k2 = 0; k2 < 3; ++k2) {
      v[k2] = bw[i].vs[k2] + im * bw[i].p_lin[k2];
      om[k2] = bw[i].ws[k2] + dw[k2];
      x[k2] = x[k2] + v[k2] * dt;
    }
    /* q+ = normalize(q_exp(omega+ dt) (x) q), world-frame omega */
    double th[3] = {om[0] * dt, om[1] * dt, om[2] * dt};
    double ang = sqrt(dot3(th, th));
    double e[4] = {1, 0, 0, 0};
    if (ang > 0.0) {
      double s = sin(0.5 * ang) / ang;
      e[0] = cos(0.5 * ang); e[1] = s * th[0]; e[2] = s * th[1]; e[3] = s * th[2];
    }
    double qn[4];
    quat_mul(e, qq, qn);
    double nrm = sqrt(qn[0]*qn[0] + qn[1]*qn[1] + qn[2]*qn[2] + qn[3]*qn[3]);
    for (int k2 = 0; k2 < 4; ++k2) qq[k2] = qn[k2] / nrm;
    /* kinetic energy with step-end velocities, step-start inertia */
    const double* Ibi = sc->inv_inertia + 3 * i;
    if (im > 0.0) ke += 0.5 * dot3(v, v) / im;
    double R[9], Ib[3], Iw[9], Iwo[3];
    quat_to_R(qq, R);
    for (int k2 = 0; k2 < 3; ++k2) Ib[k2] = Ibi[k2] > 0.0 ? 1.0 / Ibi[k2] : 0.0;
    rot_diag(R, Ib, Iw);
    matvec3(Iw, om, Iwo);
    ke += 0.5 * dot3(om, Iwo);
    for (int k2 = 0; k2 < 3; ++k2) if (!isfinite(v[k2]) || !isfinite(om[k2]) || !isfinite(x[k2])) bad = 1;
    for (int k2 = 0; k2 < 4; ++k2) if (!isfinite(qq[k2])) bad = 1;
  }
  for (int t = 0; t < T; ++t) {
    double x[4] = {0, 0, 0, 0};
    for (int j = 0; j < nd; ++j) x[j] = p_tree[t*nd + j];
    tree_minv(L_w + 10 * t, nd, x);
    for (int j = 0; j < nd; ++j) {
      double* qd = qv_w + t*nd + j;
      *qd = qd_s[t*nd + j] + x[j];
      qp_w[t*nd + j] += *qd * dt;
      if (!isfinite(*qd) || !isfinite(qp_w[t*nd + j])) bad = 1;
    }
    /* KE = 1/2 qd^T L L^T qd */
    const double* L = L_w + 10 * t;
    for (int i = 0; i < nd; ++i) {
      double y = 0;
      for (int j = i; j < nd; ++j) y += Lget(L, j, i) * qv_w[t*nd + j];
      ke += 0.5 * y * y;
    }
  }
  if (stats) {
    double* st = stats + 5 * w;
    st[0] = (double)(c_end - c_begin);
    st[1] = (double)n_active;
    st[2] = max_pen;
    st[3] = ke;
    st[4] = bad ? 1.0 : 0.0;
  }
  free(bw);
  return bad ? ORC_ENONFINITE : ORC_OK;
}

int orc_step(const orc_config* cfg, const orc_scene* sc, int64_t n_worlds,
             double* pos, double* quat, double* vel, double* omega,
             double* qpos, double* qvel,
             const double* f_ext, const double* tree_L, const double* tree_tau,
             int64_t n, const int32_t* world,
             const double* c0, const double* c1, const double* c2,
             const int32_t* body_a, const int32_t* body_b,
             const double* mu_rol, const int32_t* condim, const double* jrow,
             const double* kd,
             double* impulses, double* wrench, double* stats, int n_threads) {
  if (!cfg || !sc || n_worlds < 0 || n < 0 || !(cfg->dt > 0)) return ORC_EINVAL;
  if (sc->n_trees > 0 && (sc->tree_ndof < 1 || sc->tree_ndof > 4 || !tree_L || !tree_tau)) return ORC_EINVAL;
  for (int64_t c = 0; c < n; ++c) {
    /* per-contact impedance: finite and non-negative, like the global pair */
    if (kd && !(kd[2 * c] >= 0.0 && kd[2 * c + 1] >= 0.0 && kd[2 * c] < HUGE_VAL && kd[2 * c + 1] < HUGE_VAL))
      return ORC_EINVAL;
    /* Eq. (11)'s split k dt : d needs k dt + d > 0 */
    if (cfg->exact_diagonal == 1 && !((kd ? kd[2 * c] : cfg->k_user) * cfg->dt + (kd ? kd[2 * c + 1] : cfg->d_user) > 0.0))
      return ORC_EINVAL;
    int32_t ids[2] = {body_a[c], body_b[c]};
    for (int s = 0; s < 2; ++s) {
      int32_t id = ids[s];
      if (id >= sc->n_bodies) return ORC_EINVAL;
      if (id <= -2 && (-2 - id >= sc->n_trees || !jrow)) return ORC_EINVAL;
    }
    if (ids[0] == -1 && ids[1] == -1) return ORC_EINVAL;
  }
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_worlds + 1));
  int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int64_t* foff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int rc = orc_segment(n, world, n_worlds, condim, cfg->n_t, cfg->n_rol, off, perm, foff);
  if (rc != ORC_OK) { free(off); free(perm); free(foff); return rc; }
  int status = ORC_OK;
#ifdef _OPENMP
  if (n_threads < 1) n_threads = 1;
  #pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads)
#endif
  for (int64_t w = 0; w < n_worlds; ++w) {
    int s = step_world(cfg, sc, w, pos, quat, vel, omega, qpos, qvel, f_ext, tree_L, tree_tau,
                       off[w], off[w + 1], perm, c0, c1, c2, body_a, body_b, mu_rol, condim, jrow, kd,
                       foff, impulses, wrench, stats);
    if (s != ORC_OK) {
#ifdef _OPENMP
      #pragma omp critical
#endif
      { if (status == ORC_OK || s == ORC_EINVAL) status = s; }
    }
  }
  (void)n_threads;
  free(off); free(perm); free(foff);
  return status;
}
