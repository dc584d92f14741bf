"""Pins for the MPPI oracle (oracle/mppi.py; SPEC
S:421-446).  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import mppi


def test_splitmix64_reference_values():
    # SplitMix64 from state 0: the first outputs of the reference generator
    # (Vigna's splitmix64.c: x += 0x9e37..., then the two xor-multiply rounds)
    x, outs = 0, []
    for _ in range(3):
        outs.append(mppi.splitmix64(x))
        x = (x + 0x9E3779B97F4A7C15) & mppi.M64
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_noise_moments():
    eps = mppi.noise(7, 0, 2, 64, 4, 16, 0.02)
    assert abs(eps.mean()) < 4 * 0.02 / np.sqrt(eps.size)
    assert eps.std() == pytest.approx(0.02, rel=0.05)
    assert np.all(mppi.noise(7, 0, 2, 64, 4, 16, 0.02) == eps)          # deterministic
    assert not np.all(mppi.noise(7, 1, 2, 64, 4, 16, 0.02) == eps)      # iteration changes the draw


def test_update_limits_and_shift_invariance():
    rng = np.random.default_rng(0)
    U = rng.uniform(-0.1, 0.1, (2, 8, 3, 4))
    J = rng.integers(0, 1024, (2, 8)) / 1024.0                          # dyadic: J + 123 is exact
    plan, w = mppi.update(J, U, 2e-3, -0.1, 0.1)
    np.testing.assert_allclose(w.sum(axis=1), 1.0)
    _, w2 = mppi.update(J + 123.0, U, 2e-3, -0.1, 0.1)
    np.testing.assert_array_equal(w, w2)                                 # bitwise under a constant shift
    J1 = J.copy()
    J1[:, 3] = -10.0                                                     # one cost far below the others
    plan1, w1 = mppi.update(J1, U, 2e-3, -0.1, 0.1)
    np.testing.assert_allclose(w1[:, 3], 1.0)
    np.testing.assert_allclose(plan1, U[:, 3], atol=1e-15)
    _, wu = mppi.update(J, U, 1e12, -0.1, 0.1)                          # lambda -> inf: uniform
    np.testing.assert_allclose(wu, 1.0 / 8, rtol=1e-9)


def test_cost_terms():
    task = dict(target_pos=[[0.0, 0.0, 0.05]], target_quat=[[1.0, 0, 0, 0]], q_ref=np.zeros(16),
                w=[1.0, 2.0, 3.0, 4.0, 5.0, 6.0], omega_fallen=100.0, z_fallen=0.03, phi1=7.0, phi2=8.0)
    half = np.sqrt(0.5)
    c = mppi.cost(task, np.array([0.01, -0.02, 0.04]), np.array([half, half, 0, 0]),
                  [np.array([0.01, -0.02, 0.05])] * 4, np.full(16, 0.1), 0, False)
    exp = 1.0 * 0.5 + 2 * 0.01 + 3 * 0.02 + 4 * 0.01 + 5 * 4 * 0.01 ** 2 + 6 * 16 * 0.01
    assert c == pytest.approx(exp, rel=1e-12)
    c = mppi.cost(task, np.array([0.0, 0.0, 0.02]), np.array([1.0, 0, 0, 0]), [np.zeros(3)] * 4, np.zeros(16), 0, False)
    assert c == pytest.approx(4 * 0.03 + 5 * 4 * 0.02 ** 2 + 100.0, rel=1e-12)
    v = mppi.cost(task, np.array([0.0, 0.03, 0.05]), np.array([half, 0, half, 0]), None, None, 0, True)
    assert v == pytest.approx(7.0 * 0.03 ** 2 + 8.0 * 0.5, rel=1e-12)


def test_update_non_finite_costs_reading_r29():
    """A diverged rollout (J = NaN or inf) gets weight 0 and the others are the
    update without it; a problem with no finite cost keeps its plan (R29)."""
    rng = np.random.default_rng(3)
    U = rng.uniform(-0.1, 0.1, (3, 6, 2, 4))
    J = rng.uniform(0.0, 0.01, (3, 6))
    prev = rng.uniform(-0.05, 0.05, (3, 2, 4))
    Jb = J.copy()
    Jb[0, 2] = np.nan
    Jb[1, 4] = np.inf
    Jb[2, :] = np.nan
    plan, w = mppi.update(Jb, U, 2e-3, -0.1, 0.1, plan_prev=prev)
    assert w[0, 2] == 0.0 and w[1, 4] == 0.0 and np.all(w[2] == 0.0)
    keep0 = [0, 1, 3, 4, 5]
    p0, w0 = mppi.update(J[:1, keep0], U[:1, keep0], 2e-3, -0.1, 0.1)
    np.testing.assert_allclose(w[0, keep0], w0[0], rtol=1e-15)
    np.testing.assert_allclose(plan[0], p0[0], rtol=1e-15)
    np.testing.assert_array_equal(plan[2], prev[2])
