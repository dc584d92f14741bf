"""Pins for the articulated-upstream oracle (oracle/articulation.py, SURVEY
§8(f) rank 2): M(q), c(q, v), the Cholesky factor and the contact rows J(q)
of Eq. (1)-(5) for serial hinge chains, each checked against
something other than its own formula.  CPU only.

- forward kinematics: straight and single-bend chains have closed-form tips;
- link and contact Jacobians equal central finite differences of the
  forward kinematics (points carried rigidly by their link);
- 1/2 v^T M v equals the kinetic energy summed from finite-difference COM
  velocities and link angular velocities (from rotation-matrix differences);
- c(q, v) equals the Euler-Lagrange bias d/dt(dL/dv) - dL/dq at zero
  acceleration, assembled from finite differences of M(q) and of the
  potential energy (independent of the Newton-Euler recursion);
- the config-3 generator's Cholesky factors are this model's.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import articulation as ar
from harness import scenes

ART = scenes.hand_articulation()
G = np.array([0.0, 0.0, -9.81])
EPS = 1e-6


def _rand_q(rng):
    return rng.uniform([-0.3, 0.0, 0.0, 0.0], [0.3, 1.2, 1.2, 1.2])


def test_fk_closed_forms():
    L = ART.length[1]
    base = ART.base[1]
    tip = ar.fk(ART, 1, np.zeros(4))[3]
    np.testing.assert_allclose(tip, base + np.array([0, 0, L.sum()]), atol=1e-15)
    tip = ar.fk(ART, 1, np.array([0.7, 0.0, 0.0, 0.0]))[3]          # spin about the chain's own axis
    np.testing.assert_allclose(tip, base + np.array([0, 0, L.sum()]), atol=1e-15)
    phi = 0.4
    tip = ar.fk(ART, 1, np.array([0.0, phi, 0.0, 0.0]))[3]          # bend at joint 1 about y
    exp = base + np.array([0, 0, L[0]]) + L[1:].sum() * np.array([np.sin(phi), 0, np.cos(phi)])
    np.testing.assert_allclose(tip, exp, atol=1e-15)


@pytest.mark.parametrize("seed", range(5))
def test_jacobians_are_fk_derivatives(seed):
    rng = np.random.default_rng(seed)
    t = seed % 4
    q = _rand_q(rng)
    axes, origins, coms, tip, Rs = ar.fk_frames(ART, t, q)
    Jv, Jw = ar.link_jacobians(axes, origins, coms)
    link = seed % 4
    p0 = origins[link] + Rs[link] @ rng.normal(0, 0.01, 3)           # a point on that link
    local = Rs[link].T @ (p0 - origins[link])
    J = ar.point_rows(ART, t, q, link, p0)
    for i in range(4):
        dq = np.zeros(4)
        dq[i] = EPS
        fp, fm = ar.fk_frames(ART, t, q + dq), ar.fk_frames(ART, t, q - dq)
        for l in range(4):
            np.testing.assert_allclose((fp[2][l] - fm[2][l]) / (2 * EPS), Jv[l, :, i], atol=1e-8)
        pp = fp[1][link] + fp[4][link] @ local
        pm = fm[1][link] + fm[4][link] @ local
        np.testing.assert_allclose((pp - pm) / (2 * EPS), J[0:3, i], atol=1e-8)
        dR = (fp[4][link] - fm[4][link]) / (2 * EPS) @ Rs[link].T     # [w]x for a unit joint rate
        np.testing.assert_allclose([dR[2, 1], dR[0, 2], dR[1, 0]], J[3:6, i], atol=1e-8)


@pytest.mark.parametrize("seed", range(5))
def test_mass_matrix_is_kinetic_energy(seed):
    rng = np.random.default_rng(10 + seed)
    t = seed % 4
    q, v = _rand_q(rng), rng.normal(0, 1.0, 4)
    M = ar.mass_matrix(ART, t, q)
    fp, fm = ar.fk_frames(ART, t, q + EPS * v), ar.fk_frames(ART, t, q - EPS * v)
    Rs = ar.fk_frames(ART, t, q)[4]
    ke = 0.5 * float(np.sum(ART.armature[t] * v * v))
    for l in range(4):
        vc = (fp[2][l] - fm[2][l]) / (2 * EPS)
        W = (fp[4][l] - fm[4][l]) / (2 * EPS) @ Rs[l].T
        w = np.array([W[2, 1], W[0, 2], W[1, 0]])
        ke += 0.5 * ART.mass[t, l] * vc @ vc + 0.5 * ART.inertia[t, l] * w @ w
    assert 0.5 * v @ M @ v == pytest.approx(ke, rel=1e-8)
    np.testing.assert_allclose(M, M.T, atol=1e-18)
    assert np.all(np.linalg.eigvalsh(M) > 0)


@pytest.mark.parametrize("seed", range(6))
def test_bias_is_euler_lagrange(seed):
    rng = np.random.default_rng(20 + seed)
    t = seed % 4
    q, v = _rand_q(rng), rng.normal(0, 2.0, 4)
    c = ar.bias(ART, t, q, v, G)
    h = 1e-5

    def V(qq):  # potential energy -sum m g . com
        return -sum(ART.mass[t, l] * G @ ar.fk(ART, t, qq)[2][l] for l in range(4))

    Mdot = (ar.mass_matrix(ART, t, q + h * v) - ar.mass_matrix(ART, t, q - h * v)) / (2 * h)
    el = Mdot @ v
    for i in range(4):
        dq = np.zeros(4)
        dq[i] = h
        dM = (ar.mass_matrix(ART, t, q + dq) - ar.mass_matrix(ART, t, q - dq)) / (2 * h)
        el[i] += -0.5 * v @ dM @ v + (V(q + dq) - V(q - dq)) / (2 * h)
    np.testing.assert_allclose(c, el, rtol=1e-6, atol=1e-9)


def test_gravity_only_bias_and_cholesky():
    q = np.array([0.1, 0.5, 0.3, 0.2])
    c = ar.bias(ART, 2, q, np.zeros(4), G)
    axes, origins, coms, _ = ar.fk(ART, 2, q)
    Jv, _ = ar.link_jacobians(axes, origins, coms)
    np.testing.assert_allclose(c, -sum(ART.mass[2, l] * Jv[l].T @ G for l in range(4)), atol=1e-15)
    L, tau = ar.upstream(ART, np.tile(q, 4)[None], np.zeros((1, 16)), G)
    for t in range(4):
        Lt = np.zeros((4, 4))
        for i in range(4):
            for j in range(i + 1):
                Lt[i, j] = L[0, t, i * (i + 1) // 2 + j]
        np.testing.assert_allclose(Lt @ Lt.T, ar.mass_matrix(ART, t, q), rtol=1e-12, atol=1e-18)


def test_c3_generator_uses_this_model():
    scene, st, c, inp = scenes.c3_hand(n_worlds=3)
    L, _ = ar.upstream(ART, st.qpos.astype(np.float64), st.qvel.astype(np.float64), G)
    np.testing.assert_allclose(inp.tree_L, L, rtol=2e-6, atol=1e-7)
