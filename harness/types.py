"""Plain data containers shared by the input generators, the oracle wrapper and
the product binding.  They hold arrays only; none of the method's arithmetic
lives here ("Inputs").

Layouts (the public exchange format; PAPER.md P:244-246 lists what a contact
carries: gap phi_k, Jacobian rows, friction coefficients mu_k^s):

  State   pos (W,B,3)  quat (W,B,4) scalar-first  vel (W,B,3)  omega (W,B,3)
          qpos (W,Q)  qvel (W,Q)          Q = n_trees * tree_ndof
  Inputs  f_ext (W,B,6) world-frame force|torque or None
          tree_L (W,T,10) packed lower-triangular Cholesky factor of each
          chain's joint-space inertia (row-major, L[i(i+1)/2 + j])
          tree_tau (W,Q) applied minus bias generalized force (tau - c)
  Contacts (C,) world id; c0 (C,4) = (p, phi); c1 (C,4) = (n, mu_t);
          c2 (C,4) = (t1, mu_tor); body_a/body_b (C,) int32 with
          >=0 free body, -1 static, -(2+t) articulated chain t;
          mu_rol (C,); condim (C,) in {1,3,4,6};
          jrow (C,2,6,4) articulated-side Jacobian rows or None.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np


@dataclass
class Config:
    k_user: float = 0.1          # Eq. (12); value of P:390
    d_user: float = 0.001
    r_min: float = 0.9           # Eq. (13) defaults
    r_max: float = 0.95
    width: float = 0.001
    midpoint: float = 0.5
    power: float = 2.0
    n_t: int = 4                 # Eq. (7) symmetric direction counts
    n_rol: int = 4
    gravity: tuple = (0.0, 0.0, -9.81)
    dt: float = 0.002            # P:376 "we use dt=0.002s in all benchmarks"
    impedance: str = "heuristic" # "heuristic": M(phi) of Eq. (12); "exact_diagonal": Eq. (11) literally
                                 # (reading R24); "facet_diagonal": Eq. (12) with the facet diagonal (R28)

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


@dataclass
class Scene:
    inv_mass: np.ndarray                     # (B,)
    inv_inertia: np.ndarray                  # (B,3) principal body-frame I^-1
    n_trees: int = 0
    tree_ndof: int = 4

    @property
    def n_bodies(self) -> int:
        return int(self.inv_mass.shape[0])

    @property
    def n_tree_dofs(self) -> int:
        return int(self.n_trees * self.tree_ndof)


@dataclass
class Articulation:
    """Serial hinge chains shared by every world.  Chain t
    starts at base[t] with the world frame's orientation; joint j rotates about
    axis[t, j] given in the frame of the link before it (the base frame for
    j = 0); link j extends length[t, j] along its local +z, carries mass[t, j]
    with its centre of mass at mid-length and isotropic rotational inertia
    inertia[t, j] about it; armature[t, j] adds to the joint-space inertia's
    diagonal.  Data only (see oracle/articulation.py and include/comfree.h)."""
    base: np.ndarray                         # (T,3)
    axis: np.ndarray                         # (T,nd,3) unit, parent-link frame
    length: np.ndarray                       # (T,nd)
    mass: np.ndarray                         # (T,nd)
    inertia: np.ndarray                      # (T,nd) isotropic, about the link COM
    armature: np.ndarray                     # (T,nd)

    @property
    def n_trees(self) -> int:
        return int(self.base.shape[0])

    @property
    def tree_ndof(self) -> int:
        return int(self.length.shape[1])


@dataclass
class Geometry:
    """Collision geometry shared by every world (the front-end of SURVEY §8(f)
    rank 1).  Geom g is attached to body[g] (>= 0 free body, -1 static/world,
    -(2+t) chain t, link link[g]) at position local[g] in that frame; kind 0
    sphere (size[g, 0] = radius), 1 box (size = half extents, axes = the frame's),
    2 plane (static; size = unit normal, local[g, 0] = offset: n . x = offset).
    pairs (P,2) lists candidate geom pairs (g1, g2) tested in every world; the
    contact normal points from g1 to g2 (body_a = body of g1).  Data only."""
    kind: np.ndarray                         # (G,) int32
    body: np.ndarray                         # (G,) int32
    link: np.ndarray                         # (G,) int32
    size: np.ndarray                         # (G,3)
    local: np.ndarray                        # (G,3)
    pairs: np.ndarray                        # (P,2) int32, or None: broadphase mode (reading R32)
    margin: float = 0.001
    mu: tuple = (1.0, 0.005, 0.0001)         # (mu_t, mu_tor, mu_rol) of every contact
    condim: int = 3


@dataclass
class State:
    pos: np.ndarray
    quat: np.ndarray
    vel: np.ndarray
    omega: np.ndarray
    qpos: np.ndarray
    qvel: np.ndarray

    @property
    def n_worlds(self) -> int:
        return int(self.pos.shape[0])

    def copy(self) -> "State":
        return State(*(np.array(a, copy=True) for a in
                       (self.pos, self.quat, self.vel, self.omega, self.qpos, self.qvel)))

    def astype(self, dtype) -> "State":
        return State(*(np.ascontiguousarray(a, dtype=dtype) for a in
                       (self.pos, self.quat, self.vel, self.omega, self.qpos, self.qvel)))

    def world_slice(self, lo: int, hi: int) -> "State":
        return State(*(np.ascontiguousarray(a[lo:hi]) for a in
                       (self.pos, self.quat, self.vel, self.omega, self.qpos, self.qvel)))


@dataclass
class Inputs:
    f_ext: Optional[np.ndarray] = None       # (W,B,6)
    tree_L: Optional[np.ndarray] = None      # (W,T,10)
    tree_tau: Optional[np.ndarray] = None    # (W,Q)


@dataclass
class Contacts:
    world: np.ndarray                        # (C,) int32
    c0: np.ndarray                           # (C,4) f32: p.xyz, phi
    c1: np.ndarray                           # (C,4) f32: n.xyz, mu_t
    c2: np.ndarray                           # (C,4) f32: t1.xyz, mu_tor
    body_a: np.ndarray                       # (C,) int32
    body_b: np.ndarray                       # (C,) int32
    mu_rol: np.ndarray                       # (C,) f32
    condim: np.ndarray                       # (C,) int32
    jrow: Optional[np.ndarray] = None        # (C,2,6,4) f32
    meta: dict = field(default_factory=dict)
    kd: Optional[np.ndarray] = None          # (C,2) f32 per-contact (k_user, d_user), or None

    @property
    def n(self) -> int:
        return int(self.world.shape[0])

    def take(self, idx: np.ndarray) -> "Contacts":
        return Contacts(self.world[idx], self.c0[idx], self.c1[idx], self.c2[idx],
                        self.body_a[idx], self.body_b[idx], self.mu_rol[idx],
                        self.condim[idx], None if self.jrow is None else self.jrow[idx],
                        dict(self.meta), None if self.kd is None else self.kd[idx])

    @staticmethod
    def empty(with_jrow: bool = False) -> "Contacts":
        z4 = np.zeros((0, 4), np.float32)
        zi = np.zeros((0,), np.int32)
        return Contacts(zi.copy(), z4.copy(), z4.copy(), z4.copy(), zi.copy(), zi.copy(),
                        np.zeros((0,), np.float32), zi.copy(),
                        np.zeros((0, 2, 6, 4), np.float32) if with_jrow else None)

    @staticmethod
    def concat(parts: list) -> "Contacts":
        parts = [p for p in parts if p.n > 0] or parts[:1]
        jr = None
        if any(p.jrow is not None for p in parts):
            jr = np.concatenate([p.jrow if p.jrow is not None else
                                 np.zeros((p.n, 2, 6, 4), np.float32) for p in parts])
        kd = None
        if any(p.kd is not None for p in parts):
            raise ValueError("concat of contacts with per-contact impedance is not supported")
        return Contacts(*(np.concatenate([getattr(p, k) for p in parts]) for k in
                          ("world", "c0", "c1", "c2", "body_a", "body_b", "mu_rol", "condim")),
                        jr, {}, kd)
