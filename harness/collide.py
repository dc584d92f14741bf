"""Test-harness collision helper (NOT on the hot path).

Collision detection is upstream of the contact-resolution step (PAPER.md P:37,
P:274: ComFree-Sim reuses MJWarp's).  For trajectory tests both the oracle and
the CUDA path are fed contacts from this one CPU helper, recomputed from each
side's own state every step.  It is geometry only: it emits the contact
record (point, normal a->b, first tangent, signed gap phi, friction) and holds
none of the method's arithmetic.

Conventions (readings R16, R9):
  * normal points from body a to body b; phi > 0 separated, < 0 penetrating;
  * contact point = midpoint between the two surfaces (MuJoCo style);
  * t1 pivots on the smallest-magnitude normal component, so
    n = +z gives t1 = +x; callers may override t1 (incline tests align the
    facets with the slope).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .types import Contacts


def quat_R(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def tangent_frame(n):
    n = np.asarray(n, float)
    k = int(np.argmin(np.abs(n)))
    e = np.zeros(3)
    e[k] = 1.0
    t1 = e - np.dot(e, n) * n
    return t1 / np.linalg.norm(t1)


@dataclass
class Plane:
    normal: tuple = (0.0, 0.0, 1.0)
    offset: float = 0.0
    t1: Optional[tuple] = None       # facet alignment override


@dataclass
class Geom:
    kind: str                        # "sphere" | "box" | "capsule"
    size: tuple                      # sphere (R,), box (hx,hy,hz), capsule (R, half_len) along local z


@dataclass
class Friction:
    mu_t: float = 1.0
    mu_tor: float = 0.005
    mu_rol: float = 0.0001


@dataclass
class WorldGeometry:
    geoms: List[Geom]
    planes: List[Plane] = field(default_factory=lambda: [Plane()])
    friction: Friction = field(default_factory=Friction)
    condim: int = 3
    margin: float = 0.001
    pairs: Optional[list] = None     # explicit dynamic body pairs (a, b) to test
    box_pairs_aligned: bool = True   # box-box as face-on stacks


def _rec(out, p, phi, n, t1, a, b, fr: Friction, condim):
    out.append((p, phi, n, t1, a, b, fr, condim))


def _plane_contacts(pl: Plane, gi: int, g: Geom, x, q, fr, condim, margin, out):
    n = np.asarray(pl.normal, float)
    n = n / np.linalg.norm(n)
    t1 = np.asarray(pl.t1, float) if pl.t1 is not None else tangent_frame(n)
    if g.kind == "sphere":
        R = g.size[0]
        phi = float(np.dot(x, n) - pl.offset - R)
        if phi < margin:
            p = x - (R + 0.5 * phi) * n
            _rec(out, p, phi, n, t1, -1, gi, fr, condim)
    elif g.kind == "box":
        Rm = quat_R(q)
        h = np.asarray(g.size, float)
        corners = []
        for idx in range(8):
            s = np.array([1 if idx & 1 else -1, 1 if idx & 2 else -1, 1 if idx & 4 else -1], float)
            c = x + Rm @ (s * h)
            corners.append((float(np.dot(c, n) - pl.offset), idx, c))
        corners.sort(key=lambda t: (t[0], t[1]))
        for phi, _, c in corners[:4]:              # up to 4 deepest corners
            if phi < margin:
                _rec(out, c - 0.5 * phi * n, phi, n, t1, -1, gi, fr, condim)
    elif g.kind == "capsule":
        Rm = quat_R(q)
        R, hl = g.size
        axis = Rm @ np.array([0.0, 0.0, 1.0])
        for sgn in (-1.0, 1.0):                    # one contact per hemisphere
            cc = x + sgn * hl * axis
            phi = float(np.dot(cc, n) - pl.offset - R)
            if phi < margin:
                _rec(out, cc - (R + 0.5 * phi) * n, phi, n, t1, -1, gi, fr, condim)


def _pair_contacts(ga: Geom, xa, qa, gb: Geom, xb, qb, a, b, fr, condim, margin, out):
    if ga.kind == "sphere" and gb.kind == "sphere":
        d = xb - xa
        dist = float(np.linalg.norm(d))
        n = d / dist
        phi = dist - ga.size[0] - gb.size[0]
        if phi < margin:
            p = xa + (ga.size[0] + 0.5 * phi) * n
            _rec(out, p, phi, n, tangent_frame(n), a, b, fr, condim)
    elif ga.kind == "box" and gb.kind == "box":
        # stacked boxes: b rests on the top face of a (face normal = a's local +z)
        Ra, Rb = quat_R(qa), quat_R(qb)
        n = Ra @ np.array([0.0, 0.0, 1.0])
        top = float(np.dot(xa, n) + ga.size[2])
        hb = np.asarray(gb.size, float)
        corners = []
        for idx in range(8):
            s = np.array([1 if idx & 1 else -1, 1 if idx & 2 else -1, 1 if idx & 4 else -1], float)
            c = xb + Rb @ (s * hb)
            corners.append((float(np.dot(c, n) - top), idx, c))
        corners.sort(key=lambda t: (t[0], t[1]))
        t1 = Ra @ np.array([1.0, 0.0, 0.0])
        for phi, _, c in corners[:4]:
            if phi < margin:
                _rec(out, c - 0.5 * phi * n, phi, n, t1, a, b, fr, condim)
    else:
        raise NotImplementedError(f"pair {ga.kind}-{gb.kind}")


def collide(geo: WorldGeometry, pos, quat, world_id: int = 0, dtype=np.float32) -> Contacts:
    """Contacts of one world from body poses pos (B,3), quat (B,4)."""
    out = []
    B = len(geo.geoms)
    for i in range(B):
        for pl in geo.planes:
            _plane_contacts(pl, i, geo.geoms[i], np.asarray(pos[i], float),
                            np.asarray(quat[i], float), geo.friction, geo.condim, geo.margin, out)
    pairs = geo.pairs if geo.pairs is not None else []
    for a, b in pairs:
        _pair_contacts(geo.geoms[a], np.asarray(pos[a], float), np.asarray(quat[a], float),
                       geo.geoms[b], np.asarray(pos[b], float), np.asarray(quat[b], float),
                       a, b, geo.friction, geo.condim, geo.margin, out)
    n = len(out)
    if n == 0:
        return Contacts.empty()
    c0 = np.zeros((n, 4), dtype)
    c1 = np.zeros((n, 4), dtype)
    c2 = np.zeros((n, 4), dtype)
    ba = np.zeros(n, np.int32)
    bb = np.zeros(n, np.int32)
    mr = np.zeros(n, dtype)
    cd = np.zeros(n, np.int32)
    for k, (p, phi, nn, t1, a, b, fr, condim) in enumerate(out):
        c0[k] = (*p, phi)
        c1[k] = (*nn, fr.mu_t)
        c2[k] = (*t1, fr.mu_tor)
        ba[k], bb[k], mr[k], cd[k] = a, b, fr.mu_rol, condim
    return Contacts(np.full(n, world_id, np.int32), c0, c1, c2, ba, bb, mr, cd)


def collide_batch(geo: WorldGeometry, pos, quat, dtype=np.float32) -> Contacts:
    """Contacts of every world (same geometry, per-world poses); fp64 records
    for oracle-only trajectories, fp32 (the product's format) otherwise."""
    parts = [collide(geo, pos[w], quat[w], w, dtype) for w in range(pos.shape[0])]
    return Contacts.concat(parts)
