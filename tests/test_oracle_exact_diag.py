"""Pins for the exact-diagonal impedance variant.

Eq. (11) fixes only the sum K dt + D = (1/dt)(J~ M^-1 J~^T)^-1 in
diagonal form; reading R24 splits it in the user's ratio
K_f dt : D_f = k dt : d, so with A_f = J~_f M^-1 J~_f^T and kappa = k dt + d
Eq. (9) gives Lambda_f = (-k phi - kappa s_f)_+ / (kappa A_f).  The facet
diagonal variant (reading R28: Eq. (12) with A_f in place of the trace,
M_f = r/(1-r) / A_f) is pinned as well.  CPU only.

- a single facet between two point masses: one step of Eq. (9)-(11) leaves
  the facet velocity at exactly J~ v+ = -(k dt / kappa) phi / dt (the facet is
  driven to the prediction-correction target, whatever its approach speed);
- a sphere on a plane: A_f = m^-1 (1 + mu^2 (1 + m R^2 / I)) for a tangential
  facet (the solid sphere makes it m^-1 (1 + 3.5 mu^2)) and m^-1 for the
  normal-only facet; the oracle's impulses equal (-k phi - kappa s)_+/(kappa A_f);
- two point masses under the facet-diagonal variant: exactly three times the
  heuristic (trace over 3 rows);
- the C oracle agrees with the dense oracle B (which forms the diagonal of
  J~ M^-1 J~^T with numpy.linalg.solve over whole-world matrices) on random
  worlds with free bodies, static sides and articulated chains, all condims;
- the variants change the result (neither is the heuristic in disguise).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import dense
from harness import scenes
from harness.collide import Friction, Geom, Plane, WorldGeometry, collide_batch
from harness.types import Config, Contacts, Scene

EX = Config(impedance="exact_diagonal")
FD = Config(impedance="facet_diagonal")
G = 9.81


def _r(phi, cfg):
    x = min(abs(phi) / cfg.width, 1.0)
    m, p = cfg.midpoint, cfg.power
    gam = m * (x / m) ** p if x < m else 1 - (1 - m) * ((1 - x) / (1 - m)) ** p
    return cfg.r_min + (cfg.r_max - cfg.r_min) * gam


@pytest.mark.parametrize("mu,condim,phi", [(0.5, 3, -0.0004), (1.0, 3, -0.0011), (0.7, 1, -0.0002)])
def test_sphere_on_plane_closed_form(mu, condim, phi):
    R, rho = 0.05, 1000.0
    geoms = [Geom("sphere", (R,))]
    scene = scenes.scene_from_geoms(geoms, rho)
    im = float(scene.inv_mass[0])
    i_inv = float(scene.inv_inertia[0, 0])            # isotropic: 1 / (2/5 m R^2)
    geo = WorldGeometry(geoms, [Plane()], Friction(mu, 0.0, 0.0), condim=condim, margin=0.001)
    st = scenes.empty_state(1, 1).astype(np.float64)
    st.pos[0, 0] = (0, 0, R + phi)
    c = collide_batch(geo, st.pos, st.quat)
    c.c0 = c.c0.astype(np.float64)
    c.c0[0, :3] = (0, 0, phi)                          # contact point on the sphere's axis
    c.c0[0, 3] = phi
    out = oracle.step(EX, scene, st, c)
    # closed form: r = p - x = (0, 0, -R); tangential row g = n - mu d, d in the
    # tangent plane, r x g = -mu r x d with |r x d| = R
    A = im * (1.0 + mu * mu) + i_inv * (mu * R) ** 2 if condim == 3 else im
    if condim == 3:
        assert A == pytest.approx(im * (1 + 3.5 * mu * mu), rel=1e-6)   # solid sphere (fp32 scene arrays)
    un = -G * EX.dt                                    # predicted normal velocity (b = sphere above)
    kappa = EX.k_user * EX.dt + EX.d_user
    lam = max(0.0, -EX.k_user * phi - kappa * un) / (kappa * A)
    nF = oracle.facets_per_contact(condim, EX.n_t, EX.n_rol)
    np.testing.assert_allclose(out["impulses"], np.full(nF, lam), rtol=1e-12)


def _two_point_masses(vz, phi):
    scene = Scene(inv_mass=np.array([2.0, 0.5]), inv_inertia=np.zeros((2, 3)))
    st = scenes.empty_state(1, 2).astype(np.float64)
    st.pos[0, 0] = (0, 0, 0)
    st.pos[0, 1] = (0, 0, 0.1)
    st.vel[0, 1] = (0, 0, vz)
    c = Contacts(world=np.array([0], np.int32), c0=np.array([[0, 0, 0.05, phi]]),
                 c1=np.array([[0, 0, 1, 0.0]]), c2=np.array([[1, 0, 0, 0.0]]),
                 body_a=np.array([0], np.int32), body_b=np.array([1], np.int32),
                 mu_rol=np.zeros(1), condim=np.array([1], np.int32))
    return scene, st, c


@pytest.mark.parametrize("vz,phi,k,d", [(-0.3, -0.0003, 0.1, 0.001), (0.01, -0.002, 0.5, 0.0),
                                        (-1.0, 0.0004, 0.2, 0.01), (-0.05, -0.001, 0.0, 0.003)])
def test_single_facet_reaches_the_eq11_target(vz, phi, k, d):
    """Two free point masses (I^-1 = 0), one normal facet, no gravity: A = 1/m_a
    + 1/m_b and the step ends with u_n+ = -(k dt/kappa) phi/dt exactly while
    the facet is active, i.e. Lambda = (-(k/kappa) phi - u_n)/A."""
    scene, st, c = _two_point_masses(vz, phi)
    cfg = EX.with_(gravity=(0.0, 0.0, 0.0), k_user=k, d_user=d)
    out = oracle.step(cfg, scene, st, c)
    kappa = k * cfg.dt + d
    target = -(k * cfg.dt / kappa) * phi / cfg.dt
    un_plus = out["state"].vel[0, 1, 2] - out["state"].vel[0, 0, 2]
    if target > vz:                                    # active: the clamp does not bind
        assert un_plus == pytest.approx(target, rel=1e-12, abs=1e-15)
        assert out["impulses"][0] == pytest.approx((target - vz) / 2.5, rel=1e-12)
    else:
        assert out["impulses"][0] == 0.0 and un_plus == pytest.approx(vz, rel=1e-15)


def test_eq11_needs_positive_kappa():
    scene, st, c = _two_point_masses(-0.1, -0.001)
    with pytest.raises(Exception):
        oracle.step(EX.with_(k_user=0.0, d_user=0.0), scene, st, c)


def test_point_masses_facet_diagonal_is_three_times_heuristic():
    """Facet-diagonal variant (R28), two free bodies with locked rotation,
    normal-only contact: J~ M^-1 J~^T = 1/m_a + 1/m_b, the heuristic trace is
    3 (1/m_a + 1/m_b)."""
    scene, st, c = _two_point_masses(-0.3, -0.0003)
    cfg = FD.with_(gravity=(0.0, 0.0, 0.0))
    ex = oracle.step(cfg, scene, st, c)["impulses"]
    he = oracle.step(cfg.with_(impedance="heuristic"), scene, st, c)["impulses"]
    r = _r(-0.0003, cfg)
    Mf = r / (1 - r) / (2.0 + 0.5)
    kappa = cfg.k_user * cfg.dt + cfg.d_user
    assert ex[0] == pytest.approx(Mf * (-cfg.k_user * -0.0003 - kappa * -0.3), rel=1e-12)
    assert ex[0] == pytest.approx(3.0 * he[0], rel=1e-12)


@pytest.mark.parametrize("cfg", [EX, FD], ids=["eq11", "facet_diag"])
@pytest.mark.parametrize("seed", range(10))
def test_exact_diagonal_dense_oracle_agrees(seed, cfg):
    T = 2 if seed % 2 else 0
    scene, st, c, inp = scenes.random_instance(1200 + seed, n_worlds=1, n_bodies=3,
                                               contacts_per_world=1 + seed % 4, n_trees=T,
                                               tree_ndof=[4, 3][seed % 2])
    out = oracle.step(cfg, scene, st, c, inp)
    vB, LamB, aux = dense.dense_world_step(cfg, scene, st, c, 0, inp)
    scale = np.max(np.abs(aux["a"])) * cfg.dt if len(aux["a"]) else 1.0
    np.testing.assert_allclose(out["impulses"], LamB, rtol=1e-9, atol=1e-10 * scale)
    B = scene.n_bodies
    vA = np.concatenate([np.concatenate([out["state"].vel[0, i], out["state"].omega[0, i]]) for i in range(B)]
                        + [out["state"].qvel[0]])
    np.testing.assert_allclose(vA, vB, rtol=1e-9, atol=1e-9 * np.max(np.abs(vB)))


@pytest.mark.parametrize("cfg", [EX, FD], ids=["eq11", "facet_diag"])
def test_exact_diagonal_differs_from_heuristic(cfg):
    scene, st, c, inp = scenes.random_instance(1300, n_worlds=2, n_bodies=4, contacts_per_world=[6, 9])
    a = oracle.step(cfg, scene, st, c, inp)["impulses"]
    b = oracle.step(cfg.with_(impedance="heuristic"), scene, st, c, inp)["impulses"]
    assert np.max(np.abs(a - b)) > 1e-3 * np.max(np.abs(b))
