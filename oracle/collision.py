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
                 capsule-box / box-capsule: each end as a sphere against the box,
                 then (reading R34) the segment point nearest the box centre,
                 a + t d with t = (x_box - a) . d / |d|^2, as a third sphere when
                 0 < t < 1 (a capsule lying across a box touches it there)
  box-box        vertex-face (reading R25): every corner of g2 whose largest
                 signed face distance s = max_i (|c_i| - h_i) in g1's frame is below
                 the margin and lies within the other two face extents emits on
                 that face of g1 (n = sign(c_i) e_i, phi = s, p = corner - phi n/2),
                 then the corners of g1 against g2 (normal negated); then edge-edge
                 (reading R33): the separating-axis test over the 15 axes (face
                 normals of g1, of g2, then the 9 edge cross products e1_i x e2_j,
                 i-major, skipped when |e1_i x e2_j| <= 1e-6) gives the overlap
                 o(L) = r1(L) + r2(L) - |L . (x2 - x1)|, r_b(L) = sum_k h_bk |L . R_b e_k|;
                 when the first axis of minimum overlap is an edge axis and
                 -o < margin, one contact: n = L oriented from g1 to g2, phi = -o,
                 p = the midpoint of the closest points (Ericson 5.1.9) of g1's edge
                 along e1_i through its support point in direction n and g2's edge
                 along e2_j through its support point in direction -n

Broadphase (reading R32, geometry without a candidate list): the candidates of
a world are every geom pair (g1 < g2, planes first in the geom list) whose geoms
are not on the same body / chain and not both static, and whose world AABBs,
grown by margin/2 on every side, overlap on all three axes (closed intervals);
a plane g1 is a candidate with g2 when g2's grown AABB reaches below
offset + margin/2 along the plane normal.  AABBs: sphere c +- R; box
x +- |R| h (element-wise |R|); capsule: the two end points +- R.  Candidate
order: (g1, g2) lexicographic.  Any pair with a contact (phi < margin) is a
candidate (the grown AABBs of two geoms within the margin overlap).
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


def _box_edge_edge(RA, xA, hA, RB, xB, hB, margin):
    """Reading R33: one edge-edge contact of boxes A (g1) and B (g2) when the
    separating-axis test's first minimum-overlap axis is an edge cross product."""
    d = xB - xA
    axes = [RA[:, i] for i in range(3)] + [RB[:, j] for j in range(3)]
    kinds = [None] * 6
    for i in range(3):
        for j in range(3):
            L = np.cross(RA[:, i], RB[:, j])
            nl = float(np.linalg.norm(L))
            if nl <= 1e-6:
                continue
            axes.append(L / nl)
            kinds.append((i, j))
    best, bo = None, None
    for k, L in enumerate(axes):
        rA = sum(hA[m] * abs(float(L @ RA[:, m])) for m in range(3))
        rB = sum(hB[m] * abs(float(L @ RB[:, m])) for m in range(3))
        o = rA + rB - abs(float(L @ d))
        if bo is None or o < bo:
            best, bo = k, o
    if kinds[best] is None or not (-bo < margin):
        return []
    i, j = kinds[best]
    n = axes[best] if float(axes[best] @ d) >= 0.0 else -axes[best]
    # support points: A towards +n, B towards -n; the edges through them
    pa = xA + sum((1.0 if float(n @ RA[:, m]) >= 0.0 else -1.0) * hA[m] * RA[:, m] for m in range(3) if m != i)
    pb = xB - sum((1.0 if float(n @ RB[:, m]) >= 0.0 else -1.0) * hB[m] * RB[:, m] for m in range(3) if m != j)
    c1, c2 = _closest_segments(pa - hA[i] * RA[:, i], pa + hA[i] * RA[:, i], pb - hB[j] * RB[:, j],
                               pb + hB[j] * RB[:, j])
    return [(0.5 * (c1 + c2), -bo, n)]


def aabb(geo, g, state, w, art):
    """World AABB (lo, hi) of geom g, grown by margin/2 (reading R32); planes: None."""
    k = int(geo.kind[g])
    if k == PLANE:
        return None
    R, x = geom_frame(geo, g, state, w, art)
    if k == SPHERE:
        e = np.full(3, float(geo.size[g, 0]))
        lo, hi = x - e, x + e
    elif k == BOX:
        e = np.abs(R) @ np.asarray(geo.size[g], float)
        lo, hi = x - e, x + e
    else:
        a, b = _segment(geo, g, state, w, art)
        r = float(geo.size[g, 0])
        lo, hi = np.minimum(a, b) - r, np.maximum(a, b) + r
    m = 0.5 * geo.margin
    return lo - m, hi + m


def _same_owner(geo, g1, g2):
    b1, b2 = int(geo.body[g1]), int(geo.body[g2])
    return b1 == b2                    # same free body, both static (-1), or the same chain


def broadphase(geo, state, w, art=None):
    """Candidate pairs of world w by the definition of reading R32 (every pair
    tested, no acceleration structure): list of (g1, g2), lexicographic."""
    G = len(geo.kind)
    kind = np.asarray(geo.kind)
    boxes = [aabb(geo, g, state, w, art) for g in range(G)]
    lo = np.array([b[0] if b is not None else np.zeros(3) for b in boxes])
    hi = np.array([b[1] if b is not None else np.zeros(3) for b in boxes])
    plane = kind == PLANE
    body = np.asarray(geo.body)
    # every pair (g1 < g2): grown AABBs overlap on all three axes
    ov = np.all((lo[:, None, :] <= hi[None, :, :]) & (lo[None, :, :] <= hi[:, None, :]), axis=2)
    # plane g1: g2's grown AABB reaches below offset + margin/2 along the normal
    for g1 in np.nonzero(plane)[0]:
        n = np.asarray(geo.size[g1], float)
        c, e = 0.5 * (lo + hi), 0.5 * (hi - lo)
        ov[g1] = (c @ n - e @ np.abs(n) - float(geo.local[g1, 0])) < 0.5 * geo.margin
    ok = ov & (body[:, None] != body[None, :]) & ~plane[None, :]
    ok &= np.triu(np.ones((G, G), bool), 1)
    ok[~plane[:, None] & plane[None, :]] = False
    return [(int(a), int(b)) for a, b in zip(*np.nonzero(ok))]


def pair_contacts(geo, pi, state, w, art, g12=None):
    """Contacts of candidate pair pi (or the geom pair g12) in world w: list of
    (p, phi, n, body_a, body_b, link_a, link_b)."""
    g1, g2 = g12 if g12 is not None else (int(geo.pairs[pi, 0]), int(geo.pairs[pi, 1]))
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
        a, b = _segment(geo, gc, state, w, art)
        pts = [a, b]
        d = b - a
        t = float((xb - a) @ d / (d @ d))              # the box centre projected onto the segment (R34)
        if 0.0 < t < 1.0:
            pts.append(a + t * d)
        for e in pts:
            phi, nbox, qs = _sphere_box(e, Rr, Rb, xb, np.asarray(geo.size[gbx], float))
            if phi < m:
                out.append((0.5 * (qs + (e - Rr * nbox)), phi, -nbox if k1 == CAPSULE else nbox))
    elif k1 == BOX and k2 == BOX:
        RA, xA = geom_frame(geo, g1, state, w, art)
        RB, xB = geom_frame(geo, g2, state, w, art)
        hA, hB = np.asarray(geo.size[g1], float), np.asarray(geo.size[g2], float)
        out += _box_corners_on(RA, xA, hA, RB, xB, hB, m, False)
        out += _box_corners_on(RB, xB, hB, RA, xA, hA, m, True)
        out += _box_edge_edge(RA, xA, hA, RB, xB, hB, m)
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
    bp = geo.pairs is None or len(geo.pairs) == 0       # broadphase mode (reading R32)
    for w in range(state.n_worlds):
        cands = broadphase(geo, state, w, art) if bp else [(int(a), int(b)) for a, b in geo.pairs]
        for g12 in cands:
            for rec in pair_contacts(geo, None, state, w, art, g12=g12):
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
