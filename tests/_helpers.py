"""Test helpers: trajectory driver and closed forms used as oracle pins.

The closed forms below are derived from Eq. (9)-(13) of PAPER.md
for symmetric configurations; they are written in terms
of M_c and kappa = k dt + d and evaluated here with scalar root finding —
independently of oracle.c, which simulates the step.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.optimize import brentq

from harness.collide import collide_batch
from harness.types import Config, State


def run_trajectory(step_fn, geo, state: State, n_steps: int, record=None, dtype=None):
    """state_{k+1} = step_fn(state_k, contacts(state_k)); contacts from the
    shared CPU collision helper.  geo may be one WorldGeometry or a list (one
    per world)."""
    out = []
    s = state
    if dtype is None:
        dtype = np.float64 if state.pos.dtype == np.float64 else np.float32
    for _ in range(n_steps):
        if isinstance(geo, list):
            from harness.types import Contacts
            from harness.collide import collide
            parts = [collide(geo[w], s.pos[w], s.quat[w], w, dtype) for w in range(s.n_worlds)]
            c = Contacts.concat(parts)
        else:
            c = collide_batch(geo, s.pos, s.quat, dtype)
        s, aux = step_fn(s, c)
        if record is not None:
            out.append(record(s, c, aux))
    return s, out


# ---- impedance curve (Eq. (13)), evaluated exactly with rationals for p = 2
def r_curve(phi, cfg: Config):
    x = min(abs(phi) / cfg.width, 1.0)
    m, p = cfg.midpoint, cfg.power
    g = m * (x / m) ** p if x < m else 1 - (1 - m) * ((1 - x) / (1 - m)) ** p
    return cfg.r_min + (cfg.r_max - cfg.r_min) * g


def Mc_of(phi, tr, cfg):
    r = r_curve(phi, cfg)
    return r / (1 - r) / tr


def kappa(cfg):
    return cfg.k_user * cfg.dt + cfg.d_user


def rest_equilibrium(m, n_c, n_F, tr_fn, cfg, g=9.81, cos_t=1.0, lo=-0.2, hi=-1e-9):
    """phi* solving n_c n_F M_c(phi) (-k phi + kappa g cos dt) = m g cos dt
    (normal balance at rest): every facet carries
    Lambda = M_c(-k phi - kappa u_n) with u_n = -g cos(theta) dt."""
    dt = cfg.dt

    def f(phi):
        return n_c * n_F * Mc_of(phi, tr_fn(phi), cfg) * (-cfg.k_user * phi + kappa(cfg) * g * cos_t * dt) \
            - m * g * cos_t * dt
    phi = brentq(f, lo, hi, xtol=1e-16, rtol=1e-15, maxiter=500)
    return phi, Mc_of(phi, tr_fn(phi), cfg)


def sphere_tr(m, R, I):
    """tr of the 3-row linear point Jacobian for a contact point at depth
    R + phi/2 below the centre of an isotropic body: 3/m + 2|r|^2 / I."""
    return lambda phi: 3.0 / m + 2.0 * (R + 0.5 * phi) ** 2 / I
