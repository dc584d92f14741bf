"""TEST INFRASTRUCTURE ONLY — oracle B: the step in dense generalized
coordinates, for small instances (a handful of bodies / contacts).

Independent of oracle A (oracle.c): it assembles the joint-space inertia M,
the contact Jacobian J and the facet rows J~ (Eq. (8))
as dense matrices over the generalized velocity of the whole world, evaluates
the trace in M(phi) as trace(J_i M^-1 J_i^T) with numpy.linalg.solve
(reading R6), and applies Eq. (10) as v+ = v_s + solve(M, J~^T Lambda).
No closed forms, no per-body regrouping.

Also holds ``enumerate_activation``: brute force over all 2^F activation
patterns of the clamp (.)_+ in Eq. (9), written as the complementarity problem
Lambda >= 0, Lambda - a >= 0, Lambda (Lambda - a) = 0, which must have exactly
one solution because the update decouples across facets.
"""
from __future__ import annotations

import itertools

import numpy as np

from harness.types import Config, Contacts, Inputs, Scene, State


def _quat_R(q):
    w, x, y, z = np.asarray(q, float) / np.linalg.norm(np.asarray(q, float))
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def _skew(r):
    return np.array([[0, -r[2], r[1]], [r[2], 0, -r[0]], [-r[1], r[0], 0]])


def _unpack_L(Lp, nd):
    L = np.zeros((nd, nd))
    for i in range(nd):
        for j in range(i + 1):
            L[i, j] = Lp[i * (i + 1) // 2 + j]
    return L


def _gamma(x, m, p):
    # Eq. (13b)
    return m * (x / m) ** p if x < m else 1 - (1 - m) * ((1 - x) / (1 - m)) ** p


def world_system(cfg: Config, scene: Scene, state: State, w: int, inputs: Inputs | None):
    """Dense M (nv x nv), generalized force tau - c (nv), velocity v (nv)."""
    inputs = inputs or Inputs()
    B, T, nd = scene.n_bodies, scene.n_trees, scene.tree_ndof
    nv = 6 * B + T * nd
    M = np.zeros((nv, nv))
    h = np.zeros(nv)
    v = np.zeros(nv)
    g = np.asarray(cfg.gravity, float)
    for i in range(B):
        im = float(scene.inv_mass[i])
        Ib = 1.0 / np.asarray(scene.inv_inertia[i], float)
        R = _quat_R(np.asarray(state.quat[w, i], float))
        Iw = R @ np.diag(Ib) @ R.T
        m = 1.0 / im
        M[6 * i:6 * i + 3, 6 * i:6 * i + 3] = m * np.eye(3)
        M[6 * i + 3:6 * i + 6, 6 * i + 3:6 * i + 6] = Iw
        om = np.asarray(state.omega[w, i], float)
        fe = np.zeros(6) if inputs.f_ext is None else np.asarray(inputs.f_ext[w, i], float)
        h[6 * i:6 * i + 3] = fe[:3] + m * g                      # tau: applied + gravity
        h[6 * i + 3:6 * i + 6] = fe[3:] - np.cross(om, Iw @ om)  # minus bias c (gyroscopic)
        v[6 * i:6 * i + 3] = state.vel[w, i]
        v[6 * i + 3:6 * i + 6] = om
    for t in range(T):
        L = _unpack_L(np.asarray(inputs.tree_L[w, t], float), nd)
        sl = slice(6 * B + t * nd, 6 * B + (t + 1) * nd)
        M[sl, sl] = L @ L.T
        h[sl] = inputs.tree_tau[w, t * nd:(t + 1) * nd]
        v[sl] = state.qvel[w, t * nd:(t + 1) * nd]
    return M, h, v


def side_jacobian(scene: Scene, state: State, w: int, side: int, p, jrow_side):
    """6 x nv Jacobian mapping generalized velocity to (point velocity, angular
    velocity) of the contact point on one side (Eq. (4)-(5))."""
    B, T, nd = scene.n_bodies, scene.n_trees, scene.tree_ndof
    nv = 6 * B + T * nd
    J = np.zeros((6, nv))
    if side == -1:
        return J
    if side >= 0:
        r = np.asarray(p, float) - np.asarray(state.pos[w, side], float)
        J[0:3, 6 * side:6 * side + 3] = np.eye(3)
        J[0:3, 6 * side + 3:6 * side + 6] = -_skew(r)     # omega x r = -[r]x omega
        J[3:6, 6 * side + 3:6 * side + 6] = np.eye(3)
        return J
    t = -2 - side
    J[:, 6 * B + t * nd:6 * B + (t + 1) * nd] = np.asarray(jrow_side, float)[:, :nd]
    return J


def facet_rows(cfg: Config, n, t1, mu_t, mu_tor, mu_rol, condim, Jc):
    """Rows J~_f (Eq. (7)-(8)) in channel order t, tor, rol."""
    t2 = np.cross(n, t1)
    Jn = n @ Jc[0:3]
    if condim == 1:
        return [Jn]
    Jt = np.stack([t1 @ Jc[0:3], t2 @ Jc[0:3]])
    rows = []
    for j in range(cfg.n_t):
        d = np.array([np.cos(2 * np.pi * j / cfg.n_t), np.sin(2 * np.pi * j / cfg.n_t)])
        rows.append(Jn - mu_t * (d @ Jt))
    if condim >= 4:
        Jtor = n @ Jc[3:6]
        rows.append(Jn - mu_tor * Jtor)
        rows.append(Jn + mu_tor * Jtor)
    if condim == 6:
        Jr = np.stack([t1 @ Jc[3:6], t2 @ Jc[3:6]])
        for j in range(cfg.n_rol):
            d = np.array([np.cos(2 * np.pi * j / cfg.n_rol), np.sin(2 * np.pi * j / cfg.n_rol)])
            rows.append(Jn - mu_rol * (d @ Jr))
    return rows


def dense_world_step(cfg: Config, scene: Scene, state: State, contacts: Contacts,
                     w: int, inputs: Inputs | None = None):
    """Velocities after the step for world w, plus per-facet impulses in
    contact input order.  Returns (v_plus (nv,), Lambda list, aux dict)."""
    M, h, v = world_system(cfg, scene, state, w, inputs)
    dt = cfg.dt
    v_s = v + np.linalg.solve(M, h) * dt                        # Eq. (2)
    rows, phis, Ks, Ds, a_list = [], [], [], [], []
    for c in np.nonzero(np.asarray(contacts.world) == w)[0]:
        p = np.asarray(contacts.c0[c, :3], float)
        phi = float(contacts.c0[c, 3])
        n = np.asarray(contacts.c1[c, :3], float)
        t1 = np.asarray(contacts.c2[c, :3], float)
        jr = None if contacts.jrow is None else contacts.jrow[c]
        Ja = side_jacobian(scene, state, w, int(contacts.body_a[c]), p, None if jr is None else jr[0])
        Jb = side_jacobian(scene, state, w, int(contacts.body_b[c]), p, None if jr is None else jr[1])
        Jc = Jb - Ja                                             # b relative to a
        # M(phi): traces of the 3-row linear point Jacobians
        tr = 0.0
        for Jx in (Ja, Jb):
            Jl = Jx[0:3]
            if np.any(Jl):
                tr += float(np.trace(Jl @ np.linalg.solve(M, Jl.T)))
        x = min(abs(phi) / cfg.width, 1.0)
        r = cfg.r_min + (cfg.r_max - cfg.r_min) * _gamma(x, cfg.midpoint, cfg.power)
        Mphi = r / (1 - r) / tr
        ku, du = (cfg.k_user, cfg.d_user) if getattr(contacts, "kd", None) is None else \
            (float(contacts.kd[c, 0]), float(contacts.kd[c, 1]))   # per-contact pair
        K, D = ku * Mphi / dt, du * Mphi / dt                       # Eq. (12)
        for row in facet_rows(cfg, n, t1, float(contacts.c1[c, 3]), float(contacts.c2[c, 3]),
                              float(contacts.mu_rol[c]), int(contacts.condim[c]), Jc):
            s = row @ v_s
            Kf, Df = K, D
            imp = getattr(cfg, "impedance", "heuristic")
            if imp == "exact_diagonal":
                # Eq. (11): K_f dt + D_f = (1/dt) (J~_f M^-1 J~_f^T)^-1 in
                # diagonal form, split K_f dt : D_f = k dt : d (reading R24)
                A = float(row @ np.linalg.solve(M, row))
                total = 1.0 / (dt * A)
                Kf = total * (ku * dt / (ku * dt + du)) / dt
                Df = total * (du / (ku * dt + du))
            elif imp == "facet_diagonal":
                # Eq. (12) with this facet's diagonal entry in place of the trace (reading R28)
                A = float(row @ np.linalg.solve(M, row))
                Mf = r / (1 - r) / A
                Kf, Df = ku * Mf / dt, du * Mf / dt
            rows.append(row)
            phis.append(phi)
            Ks.append(Kf)
            Ds.append(Df)
            a_list.append(-Kf * (s * dt + phi) - Df * s)         # Eq. (9) before the clamp
    if rows:
        Jt = np.stack(rows)
        lam = np.maximum(np.asarray(a_list), 0.0)
        Lam = lam * dt
        v_plus = v_s + np.linalg.solve(M, Jt.T @ Lam)            # Eq. (10)
    else:
        Lam = np.zeros(0)
        v_plus = v_s
    return v_plus, Lam, dict(a=np.asarray(a_list), v_s=v_s, M=M,
                             rows=np.stack(rows) if rows else np.zeros((0, len(v))))


def enumerate_activation(a: np.ndarray):
    """All activation patterns sigma in {0,1}^F of the clamp in Eq. (9):
    Lambda_f = a_f on active facets, 0 otherwise; keep the ones with
    Lambda >= 0, Lambda - a >= 0 (complementarity form of (x)_+).
    Returns the list of consistent Lambda vectors."""
    F = len(a)
    sols = []
    for sigma in itertools.product((0, 1), repeat=F):
        sg = np.asarray(sigma, bool)
        lam = np.where(sg, a, 0.0)
        if np.all(lam >= 0) and np.all(lam - a >= 0):
            sols.append(lam)
    return sols
