"""Pins for the per-contact impedance variant: the
global (k_user, d_user) of Eq. (12) replaced by a per-contact pair, as the
paper's learned impedance does.  CPU only.

- a per-contact pair equal to the globals changes nothing, bit for bit;
- a resting sphere whose contact carries (k2, d2) settles at the P5 closed
  form evaluated with (k2, d2), not with the globals;
- the C oracle agrees with the dense oracle B given the same per-contact pairs;
- negative or non-finite pairs are rejected like invalid globals.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import dense
from harness import scenes
from harness.collide import Friction, Geom, Plane, WorldGeometry, collide_batch
from harness.types import Config
from _helpers import rest_equilibrium, sphere_tr

CFG = Config()
G = 9.81


def _with_kd(c, kd):
    c2 = c.take(np.arange(c.n))
    c2.kd = np.asarray(kd, np.float64).reshape(c.n, 2)
    return c2


@pytest.mark.parametrize("seed", range(4))
def test_kd_equal_to_globals_is_identity(seed):
    scene, st, c, inp = scenes.random_instance(900 + seed, n_worlds=4, n_bodies=5, contacts_per_world=[7, 0, 30, 12],
                                               n_trees=2 if seed % 2 else 0)
    a = oracle.step(CFG, scene, st, c, inp)
    b = oracle.step(CFG, scene, st, _with_kd(c, np.tile([CFG.k_user, CFG.d_user], (c.n, 1))), inp)
    for k in ("pos", "quat", "vel", "omega", "qpos", "qvel"):
        np.testing.assert_array_equal(getattr(a["state"], k), getattr(b["state"], k))
    np.testing.assert_array_equal(a["impulses"], b["impulses"])


@pytest.mark.parametrize("k2,d2", [(0.3, 0.004), (0.05, 0.0)])
def test_kd_rest_equilibrium_uses_the_contact_pair(k2, d2):
    """P5 with the contact's own pair: sum Lambda = m g dt and v+ = 0 at
    phi*(k2, d2); at phi*(globals) the same contact does not balance."""
    R, rho = 0.05, 1000.0
    geoms = [Geom("sphere", (R,))]
    scene = scenes.scene_from_geoms(geoms, rho)
    m = 1.0 / float(scene.inv_mass[0])
    I = 1.0 / float(scene.inv_inertia[0, 0])
    nF = oracle.facets_per_contact(3, CFG.n_t, CFG.n_rol)
    phi2, _ = rest_equilibrium(m, 1, nF, sphere_tr(m, R, I), CFG.with_(k_user=k2, d_user=d2))
    phi1, _ = rest_equilibrium(m, 1, nF, sphere_tr(m, R, I), CFG)
    geo = WorldGeometry(geoms, [Plane()], Friction(0.5, 0.0, 0.0), condim=3, margin=0.001)
    for phi, balanced in ((phi2, True), (phi1, False)):
        st = scenes.empty_state(1, 1).astype(np.float64)
        st.pos[0, 0] = (0, 0, R + phi)
        c = collide_batch(geo, st.pos, st.quat)
        c.c0 = c.c0.astype(np.float64)
        c.c0[0, :3] = (0, 0, 0.5 * phi)
        c.c0[0, 3] = phi
        out = oracle.step(CFG, scene, st, _with_kd(c, [[k2, d2]]))
        total = out["impulses"].sum()
        if balanced:
            assert total == pytest.approx(m * G * CFG.dt, rel=1e-12)
            assert np.max(np.abs(out["state"].vel)) < 1e-14
        else:
            assert abs(total / (m * G * CFG.dt) - 1.0) > 1e-3


@pytest.mark.parametrize("seed", range(8))
def test_kd_dense_oracle_agrees(seed):
    T = 2 if seed % 2 else 0
    scene, st, c, inp = scenes.random_instance(950 + seed, n_worlds=1, n_bodies=3,
                                               contacts_per_world=1 + seed % 4, n_trees=T,
                                               tree_ndof=[4, 3][seed % 2])
    rng = np.random.default_rng(seed)
    c = _with_kd(c, np.stack([rng.uniform(0.02, 0.6, c.n), rng.uniform(0.0, 0.01, c.n)], 1))
    out = oracle.step(CFG, scene, st, c, inp)
    vB, LamB, aux = dense.dense_world_step(CFG, scene, st, c, 0, inp)
    scale = np.max(np.abs(aux["a"])) * CFG.dt if len(aux["a"]) else 1.0
    np.testing.assert_allclose(out["impulses"], LamB, rtol=1e-9, atol=1e-10 * scale)
    B = scene.n_bodies
    vA = np.concatenate([np.concatenate([out["state"].vel[0, i], out["state"].omega[0, i]]) for i in range(B)]
                        + [out["state"].qvel[0]])
    np.testing.assert_allclose(vA, vB, rtol=1e-9, atol=1e-9 * np.max(np.abs(vB)))


@pytest.mark.parametrize("bad", [(-0.1, 0.0), (0.1, -1e-3), (np.nan, 0.0), (np.inf, 0.0)])
def test_kd_invalid_pair_rejected(bad):
    scene, st, c, inp = scenes.random_instance(990, n_worlds=1, n_bodies=2, contacts_per_world=3)
    kd = np.tile([CFG.k_user, CFG.d_user], (c.n, 1))
    kd[1] = bad
    with pytest.raises(oracle.OracleError):
        oracle.step(CFG, scene, st, _with_kd(c, kd), inp)
