"""TEST INFRASTRUCTURE ONLY — oracle of the articulated upstream of the step
(SURVEY §8(f) rank 2): for the serial hinge chains of a harness.types.
Articulation, the quantities Eq. (1)-(2) of PAPER.md takes as given
per step -- the joint-space inertia M(q), the bias c(q, v) ("Coriolis/
centrifugal/gravity"), the Cholesky factor of M the step consumes, and
the contact Jacobian rows J(q) of a point on a link (Eq. (4)-(5)).

Plain fp64 numpy, the definitions written out; no blocking, no fusion.  Shares
no code with the CUDA path.  Only tests/ (and bench.py's reference leg) use it.

  forward kinematics  R_{-1} = I, o_{-1} = base;  for joint j:
                      a_j = R_{j-1} axis_j (world axis), R_j = Rot(a_j, q_j) R_{j-1},
                      origin_j = o_{j-1}, d_j = R_j e_z, com_j = origin_j + l_j d_j / 2,
                      o_j = origin_j + l_j d_j  (o_{nd-1} is the fingertip)
  link Jacobians      Jv_l[:, i] = a_i x (com_l - origin_i), Jw_l[:, i] = a_i   (i <= l)
  inertia             M = diag(armature) + sum_l m_l Jv_l^T Jv_l + I_l Jw_l^T Jw_l
                      (so 1/2 v^T M v is the chain's kinetic energy)
  bias                c = sum_l Jv_l^T m_l (a_l - g) + Jw_l^T I_l alpha_l, where
                      (a_l, alpha_l) are the COM / angular accelerations of link l
                      at acceleration 0 (velocity-product terms), from the
                      Newton-Euler forward recursion; isotropic link inertia has
                      no gyroscopic term
  contact rows        point p on link l: J_lin[:, i] = a_i x (p - origin_i),
                      J_ang[:, i] = a_i (i <= l), 0 beyond l
Pinned in tests/test_oracle_articulation.py against finite differences of the
kinematics, the kinetic energy and the Euler-Lagrange equations.
"""
from __future__ import annotations

import numpy as np


def rot(axis, theta):
    """Rodrigues rotation about a unit axis."""
    k = np.asarray(axis, float)
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + np.sin(theta) * K + (1 - np.cos(theta)) * K @ K


def fk_frames(art, t, q):
    """World joint axes a (nd,3), joint origins (nd,3), link COMs (nd,3), tip (3,)
    and link rotations R (nd,3,3)."""
    nd = art.tree_ndof
    R = np.eye(3)
    o = np.asarray(art.base[t], float).copy()
    axes, origins, coms, Rs = np.zeros((nd, 3)), np.zeros((nd, 3)), np.zeros((nd, 3)), np.zeros((nd, 3, 3))
    for j in range(nd):
        a = R @ np.asarray(art.axis[t, j], float)
        R = rot(a, q[j]) @ R
        axes[j], origins[j], Rs[j] = a, o, R
        d = R @ np.array([0.0, 0.0, 1.0])
        coms[j] = o + 0.5 * float(art.length[t, j]) * d
        o = o + float(art.length[t, j]) * d
    return axes, origins, coms, o, Rs


def fk(art, t, q):
    axes, origins, coms, tip, _ = fk_frames(art, t, q)
    return axes, origins, coms, tip


def link_jacobians(axes, origins, coms):
    nd = axes.shape[0]
    Jv, Jw = np.zeros((nd, 3, nd)), np.zeros((nd, 3, nd))
    for l in range(nd):
        for i in range(l + 1):
            Jv[l, :, i] = np.cross(axes[i], coms[l] - origins[i])
            Jw[l, :, i] = axes[i]
    return Jv, Jw


def mass_matrix(art, t, q):
    axes, origins, coms, _ = fk(art, t, q)
    Jv, Jw = link_jacobians(axes, origins, coms)
    M = np.diag(np.asarray(art.armature[t], float))
    for l in range(art.tree_ndof):
        M = M + float(art.mass[t, l]) * Jv[l].T @ Jv[l] + float(art.inertia[t, l]) * Jw[l].T @ Jw[l]
    return M


def bias(art, t, q, v, gravity):
    """c(q, v): Newton-Euler forward pass at zero joint acceleration, then the
    link forces projected on the joints through the link Jacobians."""
    nd = art.tree_ndof
    axes, origins, coms, _ = fk(art, t, q)
    Jv, Jw = link_jacobians(axes, origins, coms)
    g = np.asarray(gravity, float)
    w = np.zeros(3)          # angular velocity of the link before joint j
    al = np.zeros(3)         # its angular acceleration
    acc_o = np.zeros(3)      # acceleration of joint j's origin
    c = np.zeros(nd)
    for j in range(nd):
        a = axes[j]
        wj = w + a * v[j]
        alj = al + np.cross(w, a * v[j])                      # d/dt (a_j v_j) with v-dot = 0
        # COM acceleration of link j: origin acceleration + alpha x r + w x (w x r)
        r = coms[j] - origins[j]
        acc_com = acc_o + np.cross(alj, r) + np.cross(wj, np.cross(wj, r))
        F = float(art.mass[t, j]) * (acc_com - g)
        N = float(art.inertia[t, j]) * alj
        c += Jv[j].T @ F + Jw[j].T @ N
        # next joint origin = this link's far end (twice the COM offset)
        r_end = 2.0 * r
        acc_o = acc_o + np.cross(alj, r_end) + np.cross(wj, np.cross(wj, r_end))
        w, al = wj, alj
    return c


def point_rows(art, t, q, link, p):
    """6 x nd rows: point velocity (rows 0-2) and angular velocity (rows 3-5) of
    link `link` at world point p, per joint velocity."""
    axes, origins, _, _ = fk(art, t, q)
    J = np.zeros((6, art.tree_ndof))
    for i in range(link + 1):
        J[0:3, i] = np.cross(axes[i], np.asarray(p, float) - origins[i])
        J[3:6, i] = axes[i]
    return J


def upstream(art, qpos, qvel, gravity, tau_ext=None):
    """Per world and chain: packed Cholesky factors (W,T,10) and tau - c (W,Q)."""
    W = qpos.shape[0]
    T, nd = art.n_trees, art.tree_ndof
    L = np.zeros((W, T, 10))
    tau = np.zeros((W, T * nd))
    for w in range(W):
        for t in range(T):
            q = np.asarray(qpos[w, t * nd:(t + 1) * nd], float)
            v = np.asarray(qvel[w, t * nd:(t + 1) * nd], float)
            Lt = np.linalg.cholesky(mass_matrix(art, t, q))
            for i in range(nd):
                for j in range(i + 1):
                    L[w, t, i * (i + 1) // 2 + j] = Lt[i, j]
            te = np.zeros(nd) if tau_ext is None else np.asarray(tau_ext[w, t * nd:(t + 1) * nd], float)
            tau[w, t * nd:(t + 1) * nd] = te - bias(art, t, q, v, gravity)
    return L, tau
