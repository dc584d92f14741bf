"""TEST INFRASTRUCTURE ONLY — oracle of the collision front-end (SURVEY §8(f)
rank 1): primitive narrowphase over a candidate pair list, emitting the
step's contact records (gap, frame, friction; the paper
takes them from MJWarp's collision).  Plain fp64 numpy, each pair
type written from its geometric definition; shares no code with the CUDA
path.

Conventions (R16, R25): the normal n points from geom g1 to geom g2
of a pair, body_a / body_b are their bodies; phi is the signed distance
between the surfaces (< 0 penetrating); the contact point is the midpoint
between the two surface points; a pair emits a contact when phi < margin.
The first tangent is the branch-free orthonormal basis of Duff et al. (2017):
s = sign(n_z) (+1 for n_z = +0), a = -1 / (s + n_z), b = n_x n_y a,
t1 = (1 + s n_x^2 a, s b, -s n_x).
  sphere-sphere  phi = |c2 - c1| - R1 - R2, n = (c2 - c1)/|c2 - c1|, p = c1 + (R1 + phi/2) n
  plane-sphere   phi = n . c - offset - R, p = c - (R + phi/2) n
  plane-box      every corner k with phi_k = n . corner_k - offset < margin,
                 p = corner_k - phi_k n / 2 (corner order: bit i of k picks the
                 sign of half extent i)
  sphere-box     (and box-sphere) c in the box frame; outside: closest point
                 q = clamp(c, -h, h), distance |c - q|, box normal (c - q)/|c - q|;
                 inside: the nearest face (smallest h_i - |c_i|, first on ties),
                 distance -(h_i - |c_i|), box normal sign(c_i) e_i;
                 phi = distance - R, p = midpoint of q_surface and c - R n_box
  capsules       (radius R, segment +-half_len along the frame's z, end -1 first)
                 plane-capsule: each end as a sphere; sphere-capsule: the closest
                 segment point as a sphere; capsule-capsule: the closest points of
                 the two segments (Ericson, Real-Time Collision Detection 5.1.9,
                 parallel when a e - b^2 <= 1e-12 a e: s = 0) as spheres;
                 capsule-box / box-capsule: each end as a sphere against the box
                 (reading R25: the capsule's side is not tested against the box)
  box-box        vertex-face (reading R25): every corner of g2 whose largest
                 signed face distance s = max_i (|c_i| - h_i) in g1's frame is below
                 the margin and lies within the other two face extents emits on
                 that face of g1 (n = sign(c_i) e_i, phi = s, p = corner - phi n/2),
                 then the corners of g1 against g2 (normal negated); edge-edge
                 contacts are not generated
"""
from __future__ import annotations

import numpy as np

from . import articulation as ar

SPHERE, BOX, PLANE, CAPSULE = 0, 1, 2, 3


def quat_R(q):
    w, x, y, z = np.asarray(q, float) / np.linalg.norm(np.asarray(q, float))
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def tangent(n):
    s = 1.0 if np.copysign(1.0, n[2]) > 0 else -1.0
    a = -1.0 / (s + n[2])
    b = n[0] * n[1] * a
    return np.array([1.0 + s * n[0] * n[0] * a, s * b, -s * n[0]])


def geom_frame(geo, g, state, w, art):
    """World rotation and position of geom g's frame origin + local offset."""
    body = int(geo.body[g])
    loc = np.asarray(geo.local[g], float)
    if body >= 0:
        R = quat_R(state.quat[w, body])
        return R, np.asarray(state.pos[w, body], float) + R @ loc
    if body == -1:
        return np.eye(3), loc
    t = -2 - body
    nd = art.tree_ndof
    q = np.asarray(state.qpos[w, t * nd:(t + 1) * nd], float)
    _, origins, _, _, Rs = ar.fk_frames(art, t, q)
    l = int(geo.link[g])
    return Rs[l], origins[l] + Rs[l] @ loc


def _sphere_box(c, Rs, Rb, xb, h):
    """phi, box-outward normal (world), box surface point (world) for sphere c, Rs."""
    cl = Rb.T @ (c - xb)
    if np.all(np.abs(cl) <= h):
        depth = h - np.abs(cl)
        i = int(np.argmin(depth))
        nl = np.zeros(3)
        nl[i] = 1.0 if cl[i] >= 0 else -1.0
        ql = cl.copy()
        ql[i] = nl[i] * h[i]
        dist = -float(depth[i])
    else:
        ql = np.clip(cl, -h, h)
        d = cl - ql
        dist = float(np.linalg.norm(d))
        nl = d / dist
    return dist - Rs, Rb @ nl, xb + Rb @ ql


def _segment(geo, g, state, w, art):
    R, c = geom_frame(geo, g, state, w, art)
    hl = float(geo.size[g, 1])
    ax = R @ np.array([0.0, 0.0, 1.0])
    return c - hl * ax, c + hl * ax


def _closest_on_segment(a, b, c):
    d = b - a
    t = float(np.clip((c - a) @ d / (d @ d), 0.0, 1.0))
    return a + t * d


def _closest_segments(p1, q1, p2, q2):
    d1, d2, r = q1 - p1, q2 - p2, p1 - p2
    a, e, f = d1 @ d1, d2 @ d2, d2 @ r
    c = d1 @ r
    b = d1 @ d2
    denom = a * e - b * b
    s = float(np.clip((b * f - c * e) / denom, 0.0, 1.0)) if denom > 1e-12 * a * e else 0.0
    t = (b * s + f) / e
    if t < 0.0:
        t, s = 0.0, float(np.clip(-c / a, 0.0, 1.0))
    elif t > 1.0:
        t, s = 1.0, float(np.clip((b - c) / a, 0.0, 1.0))
    return p1 + s * d1, p2 + t * d2


def _spheres(c1, R1, c2, R2, margin):
    d = c2 - c1
    dist = float(np.linalg.norm(d))
    n = d / dist
    phi = dist - R1 - R2
    return [(c1 + (R1 + 0.5 * phi) * n, phi, n)] if phi < margin else []


def _box_corners_on(RA, xA, hA, RB, xB, hB, margin, flip):
    """Corners of box B against the faces of box A (vertex-face)."""
    out = []
    for k in range(8):
        sgn = np.array([1.0 if k & 1 else -1.0, 1.0 if k & 2 else -1.0, 1.0 if k & 4 else -1.0])
        corner = xB + RB @ (sgn * hB)
        cl = RA.T @ (corner - xA)
        ex = np.abs(cl) - hA
        i = int(np.argmax(ex))
        s = float(ex[i])
        if s < margin and all(ex[j] <= 0.0 for j in range(3) if j != i):
            nl = np.zeros(3)
            nl[i] = 1.0 if cl[i] >= 0 else -1.0
            n = RA @ nl
            out.append((corner - 0.5 * s * n, s, -n if flip else n))
    return out


def pair_contacts(geo, pi, state, w, art):
    """Contacts of candidate pair pi in world w: list of (p, phi, n, body_a, body_b, link_a, link_b)."""
    g1, g2 = int(geo.pairs[pi, 0]), int(geo.pairs[pi, 1])
    k1, k2 = int(geo.kind[g1]), int(geo.kind[g2])
    ba, bb = int(geo.body[g1]), int(geo.body[g2])
    la = int(geo.link[g1]) if ba < -1 else 0
    lb = int(geo.link[g2]) if bb < -1 else 0
    out = []
    m = geo.margin
    if k1 == PLANE and k2 == CAPSULE:
        n = np.asarray(geo.size[g1], float)
        off = float(geo.local[g1, 0])
        Rr = float(geo.size[g2, 0])
        for e in _segment(geo, g2, state, w, art):
            phi = float(n @ e) - off - Rr
            if phi < m:
                out.append((e - (Rr + 0.5 * phi) * n, phi, n))
    elif CAPSULE in (k1, k2) and {k1, k2} <= {SPHERE, CAPSULE}:
        def pts(g, k, other):
            if k == SPHERE:
                return geom_frame(geo, g, state, w, art)[1]
            a, b = _segment(geo, g, state, w, art)
            return a, b
        R1, R2 = float(geo.size[g1, 0]), float(geo.size[g2, 0])
        if k1 == CAPSULE and k2 == CAPSULE:
            a1, b1 = _segment(geo, g1, state, w, art)
            a2, b2 = _segment(geo, g2, state, w, art)
            c1, c2 = _closest_segments(a1, b1, a2, b2)
        elif k1 == CAPSULE:
            a1, b1 = _segment(geo, g1, state, w, art)
            c2 = geom_frame(geo, g2, state, w, art)[1]
            c1 = _closest_on_segment(a1, b1, c2)
        else:
            c1 = geom_frame(geo, g1, state, w, art)[1]
            a2, b2 = _segment(geo, g2, state, w, art)
            c2 = _closest_on_segment(a2, b2, c1)
        out += _spheres(c1, R1, c2, R2, m)
    elif CAPSULE in (k1, k2) and BOX in (k1, k2):
        gc, gbx = (g1, g2) if k1 == CAPSULE else (g2, g1)
        Rb, xb = geom_frame(geo, gbx, state, w, art)
        Rr = float(geo.size[gc, 0])
        for e in _segment(geo, gc, state, w, art):
            phi, nbox, qs = _sphere_box(e, Rr, Rb, xb, np.asarray(geo.size[gbx], float))
            if phi < m:
                out.append((0.5 * (qs + (e - Rr * nbox)), phi, -nbox if k1 == CAPSULE else nbox))
    elif k1 == BOX and k2 == BOX:
        RA, xA = geom_frame(geo, g1, state, w, art)
        RB, xB = geom_frame(geo, g2, state, w, art)
        hA, hB = np.asarray(geo.size[g1], float), np.asarray(geo.size[g2], float)
        out += _box_corners_on(RA, xA, hA, RB, xB, hB, m, False)
        out += _box_corners_on(RB, xB, hB, RA, xA, hA, m, True)
    elif k1 == PLANE:
        n = np.asarray(geo.size[g1], float)
        off = float(geo.local[g1, 0])
        R2, x2 = geom_frame(geo, g2, state, w, art)
        if k2 == SPHERE:
            Rr = float(geo.size[g2, 0])
            phi = float(n @ x2) - off - Rr
            if phi < geo.margin:
                out.append((x2 - (Rr + 0.5 * phi) * n, phi, n))
        elif k2 == BOX:
            h = np.asarray(geo.size[g2], float)
            for k in range(8):
                s = np.array([1.0 if k & 1 else -1.0, 1.0 if k & 2 else -1.0, 1.0 if k & 4 else -1.0])
                corner = x2 + R2 @ (s * h)
                phi = float(n @ corner) - off
                if phi < geo.margin:
                    out.append((corner - 0.5 * phi * n, phi, n))
    elif k1 == SPHERE and k2 == SPHERE:
        _, c1 = geom_frame(geo, g1, state, w, art)
        _, c2 = geom_frame(geo, g2, state, w, art)
        R1, R2 = float(geo.size[g1, 0]), float(geo.size[g2, 0])
        d = c2 - c1
        dist = float(np.linalg.norm(d))
        n = d / dist
        phi = dist - R1 - R2
        if phi < geo.margin:
            out.append((c1 + (R1 + 0.5 * phi) * n, phi, n))
    elif {k1, k2} == {SPHERE, BOX}:
        gs, gbx = (g1, g2) if k1 == SPHERE else (g2, g1)
        _, c = geom_frame(geo, gs, state, w, art)
        Rb, xb = geom_frame(geo, gbx, state, w, art)
        Rr = float(geo.size[gs, 0])
        phi, nbox, qs = _sphere_box(c, Rr, Rb, xb, np.asarray(geo.size[gbx], float))
        if phi < geo.margin:
            p = 0.5 * (qs + (c - Rr * nbox))
            n = -nbox if k1 == SPHERE else nbox        # from g1 to g2
            out.append((p, phi, n))
    else:
        raise ValueError(f"unsupported pair kinds {k1}-{k2}")
    return [(p, phi, n, ba, bb, la, lb) for (p, phi, n) in out]


def collide(geo, state, art=None):
    """Contacts of every world, world-major, pair order within a world: a
    harness.types.Contacts (fp64 records) with meta['link'] (C,2)."""
    from harness.types import Contacts
    rows = []
    for w in range(state.n_worlds):
        for pi in range(geo.pairs.shape[0]):
            for rec in pair_contacts(geo, pi, state, w, art):
                rows.append((w,) + rec)
    n = len(rows)
    c0, c1, c2 = np.zeros((n, 4)), np.zeros((n, 4)), np.zeros((n, 4))
    world, ba, bb = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int32)
    link = np.zeros((n, 2), np.int32)
    for k, (w, p, phi, nn, a, b, la, lb) in enumerate(rows):
        c0[k] = (*p, phi)
        c1[k] = (*nn, geo.mu[0])
        c2[k] = (*tangent(nn), geo.mu[1])
        world[k], ba[k], bb[k] = w, a, b
        link[k] = (la, lb)
    c = Contacts(world, c0, c1, c2, ba, bb, np.full(n, geo.mu[2]), np.full(n, geo.condim, np.int32))
    c.meta["link"] = link
    return c
