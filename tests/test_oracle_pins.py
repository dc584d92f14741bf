"""Pins of the fp64 oracle against what the paper and the mathematics fix
(SURVEY §8(c) P1-P14).  CPU only.

Every test here checks oracle.c (through its ctypes wrapper) against a value
that does not come from oracle.c: a printed/hand-derived example
(tests/golden/spec_examples.json, each with its citation), a closed form
derived from Eq. (9)-(13) evaluated independently in tests/_helpers.py, an
invariant, or the dense generalized-coordinate oracle B (oracle/dense.py).
"""
from __future__ import annotations

import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import dense
from harness import scenes
from harness.collide import Friction, Geom, Plane, WorldGeometry, collide_batch
from harness.types import Config, Contacts, Inputs, Scene, State
from _helpers import (Mc_of, kappa, r_curve, rest_equilibrium, run_trajectory, sphere_tr)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
CFG = Config()
G = 9.81


def ostep(cfg, scene, st, c, inputs=None):
    out = oracle.step(cfg, scene, st, c, inputs)
    return out["state"], out


def single_contact(p, phi, n, t1, a, b, mu=(0.0, 0.0, 0.0), condim=1, world=0, jrow=None):
    return Contacts(np.array([world], np.int32), np.array([[*p, phi]], np.float32),
                    np.array([[*n, mu[0]]], np.float32), np.array([[*t1, mu[1]]], np.float32),
                    np.array([a], np.int32), np.array([b], np.int32),
                    np.array([mu[2]], np.float32), np.array([condim], np.int32), jrow)


# ------------------------------------------------------------------ P1
def test_p1_gamma_golden():
    g = GOLD["gamma"]
    for x, want in g["cases"]:
        assert oracle.gamma(x, g["m"], g["p"]) == pytest.approx(want, abs=1e-15)


def test_p1_r_golden_and_scaling_equivariance():
    for phi, want in GOLD["r"]["cases"]:
        assert oracle.r_of_phi(phi, CFG) == pytest.approx(want, abs=1e-15)
    rng = np.random.default_rng(1)
    for phi in rng.uniform(-2e-3, 2e-3, 200):
        # r depends on |phi|/w only: r(phi; w) = r(2 phi; 2 w)
        assert oracle.r_of_phi(phi, CFG) == oracle.r_of_phi(2 * phi, CFG.with_(width=2 * CFG.width))


def test_p1_gamma_exact_rational():
    """For p = 2 Eq. (13b) is a rational polynomial: compare to exact Fractions."""
    rng = np.random.default_rng(2)
    m = Fraction(1, 2)
    for _ in range(1000):
        x = Fraction(int(rng.integers(0, 2 ** 20)), 2 ** 20)
        want = m * (x / m) ** 2 if x < m else 1 - (1 - m) * ((1 - x) / (1 - m)) ** 2
        assert abs(oracle.gamma(float(x), 0.5, 2.0) - float(want)) <= 1e-15


def test_p1_gamma_continuity_monotone():
    xs = np.linspace(0, 1, 2001)
    for p in (1.0, 2.0, 3.5):
        for m in (0.2, 0.5, 0.8):
            v = np.array([oracle.gamma(x, m, p) for x in xs])
            assert np.all(np.diff(v) >= -1e-15)
            assert oracle.gamma(m - 1e-12, m, p) == pytest.approx(oracle.gamma(m, m, p), abs=1e-9)
    assert oracle.gamma(0.3, 0.5, 1.0) == pytest.approx(0.3, abs=1e-15)   # p = 1 is the identity


# ------------------------------------------------------------------ P4
def test_p4_facet_lambda_golden():
    for K, D, s, phi, dt, want in GOLD["facet_lambda"]["cases"]:
        assert oracle.facet_lambda(K, D, s, phi, dt) == pytest.approx(want, abs=1e-14)


# ------------------------------------------------------------------ P2
def _point_mass_world(n_bodies=1):
    scene = Scene(np.ones(n_bodies, np.float32), np.zeros((n_bodies, 3), np.float32))
    st = scenes.empty_state(1, n_bodies)
    return scene, st


@pytest.mark.parametrize("phi,rfac", [(0.0, 1.0), (-0.001, 19.0 / 9.0 / 1.0)])
def test_p2_mphi_point_mass(phi, rfac):
    """Unit point mass (rotation locked) on a static plane, contact at the COM:
    tr = 3, M(phi) = 9/3 = 3 at r = 0.9; at r = 0.95 the r/(1-r)
    factor is 19 instead of 9.  Read M through one normal facet:
    Lambda = M (-k phi - kappa s) with s = u_n."""
    cfg = CFG.with_(gravity=(0.0, 0.0, 0.0))
    scene, st = _point_mass_world()
    st.vel[0, 0] = (0, 0, -1.0)
    c = single_contact((0, 0, 0), phi, (0, 0, 1), (1, 0, 0), -1, 0)
    _, out = ostep(cfg, scene, st, c)
    M = GOLD["m_phi"]["point_mass_on_plane_r09"] * (GOLD["m_phi"]["ratio_r095_over_r09"] if phi else 1.0)
    phi32 = float(np.float32(phi))                       # the contact record is fp32
    want = M * (-cfg.k_user * phi32 - kappa(cfg) * (-1.0))
    assert out["impulses"][0] == pytest.approx(want, rel=1e-14)


def test_p2_mphi_two_point_masses():
    cfg = CFG.with_(gravity=(0.0, 0.0, 0.0))
    scene, st = _point_mass_world(2)
    st.vel[0, 0] = (0, 0, 0.5)
    st.vel[0, 1] = (0, 0, -0.5)
    c = single_contact((0, 0, 0), 0.0, (0, 0, 1), (1, 0, 0), 0, 1)
    _, out = ostep(cfg, scene, st, c)
    want = GOLD["m_phi"]["two_point_masses_r09"] * (-kappa(cfg) * (-1.0))
    assert out["impulses"][0] == pytest.approx(want, rel=1e-14)


# ------------------------------------------------------------------ P3 + integrator
def test_p3_smooth_prediction_gravity():
    scene, st = _point_mass_world()
    out, _ = ostep(CFG, scene, st, Contacts.empty())
    assert out.vel[0, 0, 2] == pytest.approx(GOLD["smooth_prediction"]["dvz"], abs=1e-15)
    assert out.pos[0, 0, 2] == pytest.approx(GOLD["smooth_prediction"]["dvz"] * CFG.dt, abs=1e-15)


def test_p3_principal_axis_spin_unchanged():
    cfg = CFG.with_(gravity=(0.0, 0.0, 0.0))
    scene = Scene(np.ones(1, np.float32), np.array([[1.0, 0.5, 1 / 3]], np.float32))
    for axis in range(3):
        st = scenes.empty_state(1, 1)
        st.omega[0, 0, axis] = 3.0
        out, _ = ostep(cfg, scene, st, Contacts.empty())
        np.testing.assert_allclose(out.omega[0, 0], st.omega[0, 0], atol=1e-15)


def test_p3_rest_unchanged():
    cfg = CFG.with_(gravity=(0.0, 0.0, 0.0))
    scene = Scene(np.ones(1, np.float32), np.array([[1.0, 0.5, 1 / 3]], np.float32))
    st = scenes.empty_state(1, 1)
    st.pos[0, 0] = (0.1, 0.2, 0.3)
    st.quat[0, 0] = np.array([0.5, 0.5, 0.5, 0.5], np.float32)
    out, _ = ostep(cfg, scene, st, Contacts.empty())
    np.testing.assert_allclose(out.pos[0, 0], st.pos[0, 0], atol=0)
    np.testing.assert_allclose(out.quat[0, 0], st.quat[0, 0], atol=1e-16)


def test_exp_map_golden():
    g = GOLD["exp_map"]
    scene = Scene(np.ones(1, np.float32), np.full((1, 3), 2.0, np.float32))
    st = scenes.empty_state(1, 1)
    st.vel[0, 0] = g["translate"]["v"]
    out, _ = ostep(CFG.with_(gravity=(0, 0, 0), dt=g["translate"]["dt"]), scene, st, Contacts.empty())
    np.testing.assert_allclose(out.pos[0, 0], g["translate"]["pos"], atol=1e-15)
    np.testing.assert_allclose(out.quat[0, 0], [1, 0, 0, 0], atol=1e-15)
    st = scenes.empty_state(1, 1)
    st.omega[0, 0] = np.array(g["half_turn"]["omega"], np.float32)
    out, _ = ostep(CFG.with_(gravity=(0, 0, 0), dt=g["half_turn"]["dt"]), scene, st, Contacts.empty())
    np.testing.assert_allclose(np.abs(out.quat[0, 0]), g["half_turn"]["quat_abs"], atol=1e-7)


def test_quaternion_norm_and_inertia_eigen():
    """|q| stays 1 to 1e-9 under random steps; the world inverse
    inertia keeps the body eigenvalues — observed through the velocity
    change from a known torque impulse."""
    rng = np.random.default_rng(5)
    cfg = CFG.with_(gravity=(0, 0, 0))
    Ib = np.array([[1.0, 2.0, 3.0]], np.float32)
    scene = Scene(np.ones(1, np.float32), Ib)
    st = scenes.empty_state(1, 1)
    st.omega[0, 0] = rng.normal(size=3)
    s = st
    for _ in range(2000):
        s, _ = ostep(cfg, scene, s, Contacts.empty())
        assert abs(np.linalg.norm(s.quat[0, 0]) - 1) < 1e-9
    # R diag(Ib^-1) R^T has eigenvalues Ib^-1: apply unit torque about each world axis
    st = scenes.empty_state(1, 1)
    q = rng.normal(size=4)
    st.quat[0, 0] = q / np.linalg.norm(q)
    cols = []
    for ax in range(3):
        f = np.zeros((1, 1, 6), np.float32)
        f[0, 0, 3 + ax] = 1.0
        o, _ = ostep(cfg.with_(dt=1.0), scene, st, Contacts.empty(), Inputs(f_ext=f))
        cols.append(o.omega[0, 0])
    Iinv = np.array(cols).T
    np.testing.assert_allclose(np.sort(np.linalg.eigvalsh(0.5 * (Iinv + Iinv.T))), [1, 2, 3], rtol=1e-6)
    np.testing.assert_allclose(Iinv, Iinv.T, atol=1e-7)


# ------------------------------------------------------------------ P5
def _sphere_setup(condim, cfg, mu=(0.0, 0.0, 0.0)):
    R, rho = 0.05, 1000.0
    geoms = [Geom("sphere", (R,))]
    scene = scenes.scene_from_geoms(geoms, rho)
    m = 1.0 / float(scene.inv_mass[0])
    I = 1.0 / float(scene.inv_inertia[0, 0])
    nF = oracle.facets_per_contact(condim, cfg.n_t, cfg.n_rol)
    phi, Mc = rest_equilibrium(m, 1, nF, sphere_tr(m, R, I), cfg)
    st = scenes.empty_state(1, 1)
    st.pos[0, 0] = (0, 0, R + phi)
    geo = WorldGeometry(geoms, [Plane()], Friction(*mu), condim=condim, margin=0.001)
    return scene, st, geo, m, I, phi, Mc, R


@pytest.mark.parametrize("condim,key", [(3, "sphere_condim3"), (6, "sphere_condim6_4_2_4")])
def test_p5_rest_equilibrium_sphere(condim, key):
    cfg = CFG
    scene, st, geo, m, I, phi, Mc, R = _sphere_setup(condim, cfg, (0.5, 0.01, 0.01))
    gold = GOLD["rest_equilibrium"][key]
    assert phi * 1e3 == pytest.approx(gold["phi_mm"], abs=5e-4)      # closed form vs survey print
    assert Mc == pytest.approx(gold["Mc"], rel=2e-5)
    st64 = st.astype(np.float64)
    st64.pos[0, 0, 2] = R + phi                                     # exact fp64 height
    c = collide_batch(geo, st64.pos, st64.quat)
    c.c0 = c.c0.astype(np.float64)
    c.c0[0, :3] = (0, 0, 0.5 * phi)
    c.c0[0, 3] = phi
    out = oracle.step(cfg, scene, st64, c)
    assert out["impulses"].sum() == pytest.approx(m * G * cfg.dt, rel=1e-12)
    assert np.max(np.abs(out["state"].vel)) < 1e-14
    assert np.max(np.abs(out["state"].omega)) < 1e-12


def test_p5_rest_equilibrium_box_4_corners():
    cfg = CFG
    h, m = 0.05, 1.0
    geoms = [Geom("box", (h, h, h))]
    scene = scenes.scene_from_geoms(geoms, masses=[m])
    I = 1.0 / float(scene.inv_inertia[0, 0])
    # corner contact point: r = (+-h, +-h, -(h + phi/2)) -> tr = 3/m + (|r|^2 * 3 - |r|^2)/I
    tr = lambda phi: 3 / m + 2 * (2 * h * h + (h + 0.5 * phi) ** 2) / I
    phi, Mc = rest_equilibrium(m, 4, cfg.n_t, tr, cfg)
    gold = GOLD["rest_equilibrium"]["box_4corners"]
    assert phi * 1e3 == pytest.approx(gold["phi_mm"], abs=5e-4)
    assert Mc == pytest.approx(gold["Mc"], rel=2e-5)
    st = scenes.empty_state(1, 1).astype(np.float64)
    st.pos[0, 0] = (0, 0, h + phi)
    geo = WorldGeometry(geoms, [Plane()], Friction(0.5, 0, 0), condim=3, margin=0.001)
    c = collide_batch(geo, st.pos, st.quat)
    c.c0 = c.c0.astype(np.float64)
    for i in range(c.n):
        c.c0[i, 2] = 0.5 * phi
        c.c0[i, 3] = phi
        c.c0[i, :2] = np.sign(c.c0[i, :2]) * h
    out = oracle.step(cfg, scene, st, c)
    assert c.n == 4
    assert out["impulses"].sum() == pytest.approx(m * G * cfg.dt, rel=1e-12)
    assert np.max(np.abs(out["state"].vel)) < 1e-14
    assert np.max(np.abs(out["state"].omega)) < 1e-12


# ------------------------------------------------------------------ P6
def _spin_run(condim, mu, w0, axis, steps):
    cfg = CFG
    scene, st, geo, m, I, phi, Mc, R = _sphere_setup(condim, cfg, mu)
    st = st.astype(np.float64)
    st.pos[0, 0, 2] = R + phi
    st.omega[0, 0, axis] = w0
    hist = []

    def stepfn(s, c):
        o = oracle.step(cfg, scene, s, c)
        return o["state"], o
    s, rec = run_trajectory(stepfn, geo, st, steps, record=lambda s, c, o: s.omega[0, 0, axis])
    return np.asarray(rec), Mc, I, phi


def test_p6_torsion_decay_closed_form():
    gold = GOLD["decay"]["torsion"]
    mu_tor = gold["mu_tor"]
    w, Mc, I, phi = _spin_run(6, (0.5, mu_tor, 0.01), gold["w0"], 2, 1000)
    fac = 1 - 2 * mu_tor ** 2 * Mc * kappa(CFG) / I          # both torsional facets active
    assert fac == pytest.approx(gold["factor"], abs=1e-8)
    want = gold["w0"] * fac ** np.arange(1, 1001)
    np.testing.assert_allclose(w, want, rtol=1e-10)
    assert w[-1] == pytest.approx(gold["w1000"], abs=2e-6)


def test_p6_rolling_decay_closed_form():
    gold = GOLD["decay"]["rolling"]
    mu_rol = gold["mu_rol"]
    w, Mc, I, phi = _spin_run(6, (0.0, 0.0, mu_rol), gold["w0"], 0, 1000)
    fac = 1 - 2 * mu_rol ** 2 * Mc * kappa(CFG) / I
    want = gold["w0"] * fac ** np.arange(1, 1001)
    np.testing.assert_allclose(w, want, rtol=1e-10)
    assert w[-1] == pytest.approx(gold["w1000"], abs=2e-6)


def test_p6_decay_monotone_in_mu():
    """decay responds monotonically to the coefficient."""
    ends = [_spin_run(6, (0.5, mu, 0.01), 20.0, 2, 200)[0][-1] for mu in (0.001, 0.005, 0.01)]
    assert ends[0] > ends[1] > ends[2]
    still = _spin_run(6, (0.5, 0.0, 0.01), 20.0, 2, 200)[0]
    np.testing.assert_allclose(still, 20.0, rtol=1e-12)                # mu_tor = 0 conserves spin


# ------------------------------------------------------------------ P7
def _block(mu=0.5, m=1.0, h=0.05, margin=0.001, n_t=4):
    geoms = [Geom("box", (h, h, h))]
    scene = scenes.scene_from_geoms(geoms, masses=[m], lock_rotation=True)
    geo = WorldGeometry(geoms, [Plane()], Friction(mu, 0, 0), condim=3, margin=margin)
    return scene, geo


def test_p7_single_active_facet_is_coulomb():
    """(i) when each contact's only active t-facet opposes slip, |F_t| = mu N exactly."""
    cfg = CFG
    scene, geo = _block(margin=0.01)
    st = scenes.empty_state(1, 1).astype(np.float64)
    st.pos[0, 0, 2] = 0.05 + 0.001                 # hovering: phi > kappa g dt / k
    st.vel[0, 0, 0] = 3.0
    c = collide_batch(geo, st.pos, st.quat, np.float64)
    out = oracle.step(cfg, scene, st, c)
    lam = out["impulses"].reshape(c.n, 4)
    # facet j=0 (d = +t1) is the one whose friction opposes +x slip
    assert np.all(lam[:, 1:] == 0) and np.all(lam[:, 0] > 0)
    wr = out["wrench"]
    N = wr[:, 2].sum()
    Ft = np.hypot(wr[:, 0].sum(), wr[:, 1].sum())
    assert Ft == pytest.approx(0.5 * N, rel=1e-12)


def test_p7_viscous_regime_closed_form():
    """(iii) at the rest equilibrium, with all four facets active, one step
    gives v+ = v (1 - 2 n_c mu^2 M_c kappa / m) and no vertical motion."""
    cfg = CFG
    mu, m, h = 0.5, 1.0, 0.05
    scene, geo = _block(mu, m, h)
    phi, Mc = rest_equilibrium(m, 4, 4, lambda p: 3.0 / m, cfg)
    st = scenes.empty_state(1, 1).astype(np.float64)
    st.pos[0, 0, 2] = h + phi
    v = 0.05
    st.vel[0, 0, 0] = v
    c = collide_batch(geo, st.pos, st.quat, np.float64)
    c.c0[:, 3] = phi
    out = oracle.step(cfg, scene, st, c)
    assert np.all(out["impulses"] > 0)
    want = v * (1 - 2 * 4 * mu ** 2 * Mc * kappa(cfg) / m)
    assert out["state"].vel[0, 0, 0] == pytest.approx(want, rel=1e-12)
    assert abs(out["state"].vel[0, 0, 2]) < 1e-14


def test_p7_coulomb_regime_deceleration():
    """(ii) above v_c the block hovers with one active facet per contact and
    decelerates at mu g (margin covers the hover gap)."""
    cfg = CFG
    gold = GOLD["sliding"]
    phi_b = kappa(cfg) * G * cfg.dt / cfg.k_user
    assert phi_b * 1e3 == pytest.approx(gold["phi_b_mm"], abs=1e-4)
    mu, m = 0.5, 1.0
    Mcb = Mc_of(phi_b, 3.0 / m, cfg)
    v_c = m * G * cfg.dt / (4 * Mcb * mu * kappa(cfg))
    assert v_c == pytest.approx(gold["v_c"], abs=2e-3)
    scene, geo = _block(mu, m, 0.05, margin=0.05)
    st = scenes.empty_state(1, 1).astype(np.float64)
    st.pos[0, 0, 2] = 0.05 + 0.0165
    st.vel[0, 0, 0] = 4.0

    def stepfn(s, c):
        o = oracle.step(cfg, scene, s, c)
        return o["state"], o
    v_prev = [st.vel[0, 0, 0]]

    def rec(s, c, o):
        r = (v_prev[0], s.vel[0, 0, 0], np.count_nonzero(o["impulses"] > 0), c.n, o["impulses"].sum())
        v_prev[0] = s.vel[0, 0, 0]
        return r
    s, recs = run_trajectory(stepfn, geo, st, 300, record=rec)
    r = np.array(recs)
    one = (r[:, 2] == r[:, 3]) & (r[:, 3] == 4)
    assert one.sum() > 100
    # every step with exactly one active facet per contact is Coulomb: dv = mu N / m
    np.testing.assert_allclose((r[one, 0] - r[one, 1]), mu * r[one, 4] / m, rtol=1e-9)
    # and the hover settles so that the windowed deceleration is mu g within 2 %
    v = r[:, 1]
    assert (v[99] - v[-1]) / (cfg.dt * (len(v) - 100)) == pytest.approx(mu * G, rel=0.02)


# ------------------------------------------------------------------ P8
def _incline_run(ratio, steps, margin=0.001):
    cfg = CFG
    mu, m, h = 0.5, 1.0, 0.05
    scene, st, geos, thetas = scenes.c2a_incline([ratio], mu=mu)
    for g in geos:
        g.margin = margin
    st = st.astype(np.float64)

    def stepfn(s, c):
        o = oracle.step(cfg, scene, s, c)
        return o["state"], o
    th = thetas[0]
    t1 = np.array([math.cos(th), 0, math.sin(th)])
    s, rec = run_trajectory(stepfn, geos, st, steps, record=lambda s, c, o: float(s.vel[0, 0] @ t1))
    return np.asarray(rec), th


def _creep_closed_form(th, cfg, mu=0.5, m=1.0, n_c=4):
    c, s = math.cos(th), math.sin(th)
    if math.tan(th) <= mu / 2:
        phi, Mc = rest_equilibrium(m, n_c, 4, lambda p: 3.0 / m, cfg, cos_t=c)
        return m * G * s * cfg.dt / (2 * n_c * mu ** 2 * Mc * kappa(cfg)) - G * s * cfg.dt
    lam_p = m * G * s * cfg.dt / (n_c * mu)
    lam_0 = m * G * cfg.dt / (2 * n_c) * (c - s / mu)
    # normal balance of the two side facets fixes phi: lam_0 = M_c(phi)(-k phi + kappa g c dt)
    from scipy.optimize import brentq
    f = lambda p: Mc_of(p, 3.0 / m, cfg) * (-cfg.k_user * p + kappa(cfg) * G * c * cfg.dt) - lam_0
    phi = brentq(f, -0.2, 0.05, xtol=1e-16)
    Mc = Mc_of(phi, 3.0 / m, cfg)
    return (lam_p - lam_0) / (mu * Mc * kappa(cfg)) - G * s * cfg.dt


@pytest.mark.parametrize("ratio,key,steps", [(0.25, "creep_tan_mu_over_4", 4000),
                                             (0.5, "creep_tan_mu_over_2", 4000), (0.75, None, 9000)])
def test_p8_incline_creep(ratio, key, steps):
    """Zero steady acceleration with a closed-form creep speed for
    tan(theta) <= mu (regime A: all facets active, tan <= mu/2; regime B:
    up-slope facet off); convergence is slow near tan -> mu."""
    u, th = _incline_run(ratio, steps)
    want = _creep_closed_form(th, CFG)
    if key:
        assert want == pytest.approx(GOLD["incline"][key], abs=2e-5)
    # down-slope creep is -t1; steady speed after convergence
    assert -u[-1] == pytest.approx(want, abs=1e-6)
    assert abs(u[-1] - u[-2]) < 1e-9                                 # zero steady acceleration


@pytest.mark.parametrize("ratio,key", [(1.1, "accel_tan_1.1mu"), (1.5, "accel_tan_1.5mu")])
def test_p8_incline_slip_acceleration(ratio, key):
    u, th = _incline_run(ratio, 3000, margin=1.0)
    want = G * (math.sin(th) - 0.5 * math.cos(th))
    assert want == pytest.approx(GOLD["incline"][key], abs=1e-4)
    acc = -(u[-1] - u[-501]) / (500 * CFG.dt)
    assert acc == pytest.approx(want, abs=1e-4)


# ------------------------------------------------------------------ P9
def test_p9_momentum_two_spheres():
    cfg = CFG.with_(gravity=(0, 0, 0))
    geoms = [Geom("sphere", (0.05,)), Geom("sphere", (0.05,))]
    scene = scenes.scene_from_geoms(geoms)
    st = scenes.empty_state(1, 2).astype(np.float64)
    st.pos[0, 0] = (0, 0, 0)
    st.pos[0, 1] = (0.0995, 0.01, 0)
    st.vel[0, 0] = (0.5, 0.0, 0.0)
    st.vel[0, 1] = (-0.3, 0.05, 0.0)
    geo = WorldGeometry(geoms, [], Friction(0.0, 0, 0), condim=1, margin=0.001, pairs=[(0, 1)])
    m = 1.0 / scene.inv_mass.astype(np.float64)
    p0 = (m[:, None] * st.vel[0]).sum(0)

    def stepfn(s, c):
        o = oracle.step(cfg, scene, s, c)
        return o["state"], o
    s, rec = run_trajectory(stepfn, geo, st, 1000, record=lambda s, c, o: (m[:, None] * s.vel[0]).sum(0))
    drift = np.max(np.abs(np.array(rec) - p0)) / np.linalg.norm(p0)
    assert drift < 1e-8
    assert s.vel[0, 0, 0] < 0.5                                      # they did collide


def test_p9_third_law_random():
    cfg = CFG.with_(gravity=(0, 0, 0))
    scene, st, c, inp = scenes.random_instance(11, n_worlds=4, n_bodies=4, contacts_per_world=10,
                                               static_frac=0.0, with_fext=False)
    out = oracle.step(cfg, scene, st, c)
    m = 1.0 / scene.inv_mass.astype(np.float64)
    dP = (m[None, :, None] * (out["state"].vel - st.vel.astype(np.float64))).sum(1)
    np.testing.assert_allclose(dP, 0.0, atol=1e-12 * np.abs(out["wrench"]).sum())


# ------------------------------------------------------------------ P10, P11, P12
def _channel_sums(Lam, c, cfg, k):
    """Per-channel normal part and friction vector from facet impulses
    (primal wrench), independent of oracle.c's regrouping."""
    cd = int(c.condim[k])
    out = {}
    if cd == 1:
        return {"n": (Lam.sum(), 0.0)}
    th = 2 * np.pi * np.arange(cfg.n_t) / cfg.n_t
    lt = Lam[:cfg.n_t]
    out["t"] = (lt.sum(), c.c1[k, 3] * np.hypot((lt * np.cos(th)).sum(), (lt * np.sin(th)).sum()))
    if cd >= 4:
        out["tor"] = (Lam[cfg.n_t:cfg.n_t + 2].sum(), c.c2[k, 3] * abs(Lam[cfg.n_t] - Lam[cfg.n_t + 1]))
    if cd == 6:
        th = 2 * np.pi * np.arange(cfg.n_rol) / cfg.n_rol
        lr = Lam[cfg.n_t + 2:]
        out["rol"] = (lr.sum(), c.mu_rol[k] * np.hypot((lr * np.cos(th)).sum(), (lr * np.sin(th)).sum()))
    return out


def test_p10_cone_membership_random():
    worst = 0.0
    count = 0
    for seed in range(40):
        for cfg in (CFG, CFG.with_(n_t=8, n_rol=8)):
            scene, st, c, inp = scenes.random_instance(100 + seed, n_worlds=5, n_bodies=6,
                                                       contacts_per_world=50)
            out = oracle.step(cfg, scene, st, c, inp)
            Lam, foff, wr = out["impulses"], out["foff"], out["wrench"]
            assert np.all(Lam >= 0)
            for k in range(c.n):
                L = Lam[foff[k]:foff[k + 1]]
                count += 1
                for ch, (Nch, Fch) in _channel_sums(L, c, cfg, k).items():
                    mu = {"t": c.c1[k, 3], "tor": c.c2[k, 3], "rol": c.mu_rol[k], "n": 0}[ch]
                    worst = min(worst, mu * Nch - Fch)
                # aggregate wrench from oracle.c against Eq. (3)
                n, t1 = c.c1[k, :3].astype(float), c.c2[k, :3].astype(float)
                t2 = np.cross(n, t1)
                N = wr[k, :3] @ n
                assert N == pytest.approx(L.sum(), rel=1e-6, abs=1e-14)
                if c.condim[k] >= 3:
                    assert np.hypot(wr[k, :3] @ t1, wr[k, :3] @ t2) <= c.c1[k, 3] * N * (1 + 1e-6) + 1e-15
                if c.condim[k] >= 4:
                    assert abs(wr[k, 3:] @ n) <= c.c2[k, 3] * N * (1 + 1e-6) + 1e-15
                if c.condim[k] == 6:
                    assert np.hypot(wr[k, 3:] @ t1, wr[k, 3:] @ t2) <= c.mu_rol[k] * N * (1 + 1e-6) + 1e-15
    assert count > 10000
    assert worst >= -1e-12


def test_p11_dual_cone_consistency():
    """Separated (phi > 0) and separating faster than any friction term on
    every facet -> all impulses zero (Eq. (6)-(9))."""
    cfg = CFG.with_(gravity=(0, 0, 0))
    scene, st = _point_mass_world(1)
    st.vel[0, 0] = (0.1, 0.05, 2.0)
    c = single_contact((0, 0, 0), 1e-4, (0, 0, 1), (1, 0, 0), -1, 0, mu=(0.5, 0.01, 0.01), condim=6)
    out = oracle.step(cfg, scene, st, c)
    assert np.all(out["impulses"] == 0)
    np.testing.assert_array_equal(out["state"].vel[0, 0], st.vel[0, 0].astype(np.float64))


def test_p12_decoupling_permutation_bitwise():
    scene, st, c, inp = scenes.random_instance(21, n_worlds=4, n_bodies=6, contacts_per_world=[9, 0, 17, 5])
    out = oracle.step(CFG, scene, st, c, inp)
    perm = np.random.default_rng(3).permutation(c.n)
    c2 = c.take(perm)
    out2 = oracle.step(CFG, scene, st, c2, inp)
    for new, old in enumerate(perm):
        a = out["impulses"][out["foff"][old]:out["foff"][old + 1]]
        b = out2["impulses"][out2["foff"][new]:out2["foff"][new + 1]]
        np.testing.assert_array_equal(a, b)


# ------------------------------------------------------------------ P13
@pytest.mark.parametrize("seed", range(12))
def test_p13_dense_oracle_agrees(seed):
    """oracle.c == dense generalized-coordinate oracle B on random 1-4 contact
    instances with free, static and articulated sides and every condim."""
    T = 2 if seed % 2 else 0
    n_con = 1 + seed % 4
    cfg = CFG if seed % 3 else CFG.with_(n_t=8, n_rol=6)
    scene, st, c, inp = scenes.random_instance(300 + seed, n_worlds=1, n_bodies=3,
                                               contacts_per_world=n_con, n_trees=T,
                                               tree_ndof=[4, 3][seed % 2])
    out = oracle.step(cfg, scene, st, c, inp)
    vB, LamB, aux = dense.dense_world_step(cfg, scene, st, c, 0, inp)
    # dense solves with M spanning 1e-5..1e1 (condition ~1e6) lose ~6 digits;
    # tolerances are relative to the size of the terms that cancel in Eq. (9)
    scale = np.max(np.abs(aux["a"])) * cfg.dt if len(aux["a"]) else 1.0
    np.testing.assert_allclose(out["impulses"], LamB, rtol=1e-9, atol=1e-10 * scale)
    B = scene.n_bodies
    vA = np.concatenate([np.concatenate([out["state"].vel[0, i], out["state"].omega[0, i]]) for i in range(B)]
                        + [out["state"].qvel[0]])
    np.testing.assert_allclose(vA, vB, rtol=1e-9, atol=1e-9 * np.max(np.abs(vB)))


@pytest.mark.parametrize("seed", range(6))
def test_p13_brute_force_enumeration_unique(seed):
    cfg = CFG
    scene, st, c, inp = scenes.random_instance(400 + seed, n_worlds=1, n_bodies=3,
                                               contacts_per_world=1 + seed % 4, condims=(1, 3, 4))
    out = oracle.step(cfg, scene, st, c, inp)
    _, LamB, aux = dense.dense_world_step(cfg, scene, st, c, 0, inp)
    if len(aux["a"]) > 16:
        pytest.skip("too many facets for 2^F enumeration")
    sols = dense.enumerate_activation(aux["a"])
    assert len(sols) >= 1
    scale = np.max(np.abs(aux["a"])) * cfg.dt
    for s in sols:                                   # all consistent patterns give one Lambda
        np.testing.assert_allclose(s * cfg.dt, out["impulses"], rtol=1e-9, atol=1e-10 * scale)
    if np.all(np.abs(aux["a"]) > 0):
        assert len(sols) == 1


# ------------------------------------------------------------------ P14
def test_p14_friction_dissipates_kinetic_energy():
    cfg = CFG
    scene, st, geo, m, I, phi, Mc, R = _sphere_setup(6, cfg, (0.5, 0.01, 0.01))
    st = st.astype(np.float64)
    st.omega[0, 0] = (0.0, 0.0, 15.0)

    def stepfn(s, c):
        o = oracle.step(cfg, scene, s, c)
        return o["state"], o
    s, rec = run_trajectory(stepfn, geo, st, 300, record=lambda s, c, o: o["stats"][0, 3])
    ke = np.asarray(rec)
    assert np.all(np.diff(ke) <= 1e-12)
    assert ke[-1] < ke[0]


# ------------------------------------------------------------------ S0 integers
def test_segment_plain_loops_vs_library():
    rng = np.random.default_rng(9)
    for W, n in ((1, 0), (5, 100), (64, 3000), (7, 1)):
        w = rng.integers(0, W, n).astype(np.int32)
        cd = rng.choice(np.array([1, 3, 4, 6], np.int32), n)
        c = Contacts(w, np.zeros((n, 4), np.float32), np.zeros((n, 4), np.float32),
                     np.zeros((n, 4), np.float32), np.zeros(n, np.int32), np.zeros(n, np.int32),
                     np.zeros(n, np.float32), cd)
        for cfg in (CFG, CFG.with_(n_t=8, n_rol=8)):
            off, perm, foff = oracle.segment(c, W, cfg)
            np.testing.assert_array_equal(perm, np.argsort(w, kind="stable"))
            np.testing.assert_array_equal(off, np.concatenate([[0], np.cumsum(np.bincount(w, minlength=W))]))
            nf = np.select([cd == 1, cd == 3, cd == 4, cd == 6], [1, cfg.n_t, cfg.n_t + 2, cfg.n_t + 2 + cfg.n_rol])
            np.testing.assert_array_equal(foff, np.concatenate([[0], np.cumsum(nf)]))
