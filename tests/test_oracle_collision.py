"""Pins for the collision front-end oracle (oracle/collision.py, SURVEY §8(f)
rank 1): each primitive pair against closed-form distances, the contact
count of a resting box, frame orthonormality, rotation invariance, and
chain-attached geoms against the (pinned) forward kinematics.  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import collision as co
from oracle import articulation as ar
from harness import scenes
from harness.types import Geometry, State


def _state(pos, quat, qpos=None):
    pos = np.asarray(pos, float)[None]
    quat = np.asarray(quat, float)[None]
    B = pos.shape[1]
    q = np.zeros((1, 0)) if qpos is None else np.asarray(qpos, float)[None]
    return State(pos, quat, np.zeros((1, B, 3)), np.zeros((1, B, 3)), q, np.zeros_like(q))


def _geo(kind, body, size, local, pairs, margin=0.01):
    G = len(kind)
    return Geometry(np.array(kind, np.int32), np.array(body, np.int32), np.zeros(G, np.int32),
                    np.array(size, float), np.array(local, float), np.array(pairs, np.int32), margin=margin)


def test_plane_sphere_and_sphere_sphere():
    R = 0.05
    geo = _geo([2, 0, 0], [-1, 0, 1], [(0, 0, 1), (R, 0, 0), (0.02, 0, 0)], [(0, 0, 0)] * 3, [(0, 1), (1, 2)])
    st = _state([(0.1, 0.2, 0.049), (0.1, 0.2 + 0.069, 0.049)], [(1, 0, 0, 0)] * 2)
    c = co.collide(geo, st)
    assert c.n == 2
    np.testing.assert_allclose(c.c0[0], (0.1, 0.2, 0.5 * (0.049 - R), 0.049 - R), atol=1e-15)
    np.testing.assert_allclose(c.c1[0, :3], (0, 0, 1))
    np.testing.assert_allclose(c.c0[1, 3], 0.069 - R - 0.02, atol=1e-15)
    np.testing.assert_allclose(c.c1[1, :3], (0, 1, 0), atol=1e-15)
    np.testing.assert_allclose(c.c0[1, :3], (0.1, 0.2 + R + 0.5 * (0.069 - R - 0.02), 0.049), atol=1e-15)
    assert (c.body_a.tolist(), c.body_b.tolist()) == ([-1, 0], [0, 1])


def test_resting_box_on_plane_has_four_contacts():
    h = (0.05, 0.03, 0.02)
    geo = _geo([2, 1], [-1, 0], [(0, 0, 1), h], [(0, 0, 0)] * 2, [(0, 1)], margin=0.001)
    c = co.collide(geo, _state([(0.3, -0.1, 0.0195)], [(1, 0, 0, 0)]))
    assert c.n == 4
    np.testing.assert_allclose(c.c0[:, 3], -0.0005, atol=1e-15)
    np.testing.assert_allclose(sorted(map(tuple, np.round(c.c0[:, :2], 12))),
                               sorted([(0.3 + sx * 0.05, -0.1 + sy * 0.03) for sx in (-1, 1) for sy in (-1, 1)]))
    # tilted about x by 30 degrees and lifted: only the lowest edge's 2 corners are near the plane
    th = np.radians(30)
    q = (np.cos(th / 2), np.sin(th / 2), 0, 0)
    z = h[1] * np.sin(th) + h[2] * np.cos(th) - 0.0002
    c = co.collide(geo, _state([(0, 0, z)], [q]))
    assert c.n == 2
    np.testing.assert_allclose(c.c0[:, 3], -0.0002, atol=1e-12)


@pytest.mark.parametrize("c_local,expect", [
    ((0.0, 0.0, 0.08), 0.08 - 0.03 - 0.01),                    # face region
    ((0.05, 0.0, 0.06), np.hypot(0.02, 0.03) - 0.01),           # edge region
    ((0.05, 0.04, 0.07), np.sqrt(0.02**2 + 0.01**2 + 0.04**2) - 0.01),   # corner region
    ((0.0, 0.025, 0.01), -(0.03 - 0.025) - 0.01),               # inside, nearest face y
])
def test_sphere_box_distances(c_local, expect):
    h = (0.03, 0.03, 0.03)
    geo = _geo([0, 1], [1, 0], [(0.01, 0, 0), h], [(0, 0, 0)] * 2, [(0, 1)], margin=1.0)
    xb = np.array([0.2, -0.1, 0.3])
    for quat in ((1, 0, 0, 0), (np.cos(0.35), 0.3 * np.sin(0.35), -0.5 * np.sin(0.35), np.sqrt(0.66) * np.sin(0.35))):
        R = co.quat_R(quat)
        st = _state([xb, xb + R @ np.array(c_local)], [quat, (1, 0, 0, 0)])     # body 0 box, body 1 sphere
        c = co.collide(geo, st)
        assert c.n == 1
        assert c.c0[0, 3] == pytest.approx(expect, abs=1e-12)
        n = c.c1[0, :3]
        assert np.linalg.norm(n) == pytest.approx(1.0, abs=1e-12)
        # normal from the sphere (g1) to the box (g2): moving the sphere along -n
        # by delta increases phi by delta when outside
        if expect > 0:
            st2 = _state([xb, xb + R @ np.array(c_local) - 1e-6 * n], [quat, (1, 0, 0, 0)])
            assert co.collide(geo, st2).c0[0, 3] == pytest.approx(expect + 1e-6, abs=1e-11)


def test_tangent_frame_orthonormal():
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        t = co.tangent(n)
        assert abs(t @ n) < 1e-14 and abs(np.linalg.norm(t) - 1) < 1e-14
    np.testing.assert_allclose(co.tangent(np.array([0, 0, 1.0])), (1, 0, 0))


def test_chain_spheres_follow_forward_kinematics():
    art = scenes.hand_articulation()
    geo = scenes.hand_geometry(margin=10.0)              # every candidate pair emits
    rng = np.random.default_rng(3)
    q = rng.uniform([-0.3, 0, 0, 0] * 4, [0.3, 1.2, 1.2, 1.2] * 4)
    st = _state([(0.02, 0.0, 0.05)], [(1, 0, 0, 0)], q)
    c = co.collide(geo, st, art)
    assert c.n == 16 + 12 + 8
    for t in range(4):
        tip = ar.fk(art, t, q[4 * t:4 * t + 4])[3]
        k = 4 * t + 3                                     # pair (tip sphere of chain t, cube)
        assert c.body_a[k] == -2 - t and c.meta["link"][k, 0] == 3
        kp = 16 + 3 * t + 2                               # pair (palm, tip sphere of chain t)
        assert c.c0[kp, 3] == pytest.approx(tip[2] - 0.008, abs=1e-14)


def _q_axis_angle(axis, ang):
    axis = np.asarray(axis, float) / np.linalg.norm(axis)
    return (np.cos(ang / 2), *(np.sin(ang / 2) * axis))


def test_capsule_pairs_closed_forms():
    R, hl = 0.015, 0.02
    # tilted capsule above the plane: ends at z0 -+ hl cos(th)
    th = 0.6
    geo = _geo([2, 3], [-1, 0], [(0, 0, 1), (R, hl, 0)], [(0, 0, 0)] * 2, [(0, 1)], margin=0.05)
    c = co.collide(geo, _state([(0.1, 0.0, 0.03)], [_q_axis_angle((1, 0, 0), th)]))
    assert c.n == 2
    np.testing.assert_allclose(c.c0[:, 3], [0.03 - hl * np.cos(th) - R, 0.03 + hl * np.cos(th) - R], atol=1e-15)
    # sphere beside the capsule's side: distance = lateral offset - R - Rs
    geo = _geo([0, 3], [0, 1], [(0.01, 0, 0), (R, hl, 0)], [(0, 0, 0)] * 2, [(0, 1)], margin=0.05)
    c = co.collide(geo, _state([(0.03, 0.0, 0.005), (0, 0, 0)], [(1, 0, 0, 0)] * 2))
    assert c.n == 1 and c.c0[0, 3] == pytest.approx(0.03 - 0.01 - R, abs=1e-15)
    np.testing.assert_allclose(c.c1[0, :3], (-1, 0, 0), atol=1e-15)      # from the sphere to the capsule
    # perpendicular crossing capsules: distance between the axes minus the radii
    geo = _geo([3, 3], [0, 1], [(R, hl, 0), (R, hl, 0)], [(0, 0, 0)] * 2, [(0, 1)], margin=0.05)
    c = co.collide(geo, _state([(0, 0, 0), (0.004, 0.0, 0.027)], [(1, 0, 0, 0), _q_axis_angle((1, 0, 0), np.pi / 2)]))
    assert c.n == 1 and c.c0[0, 3] == pytest.approx(np.hypot(0.004, 0.027 - hl) - 2 * R, abs=1e-14)
    # parallel side by side: the s = 0 end of the first segment, distance = offset - 2R
    c = co.collide(geo, _state([(0, 0, 0), (0.028, 0.0, 0.005)], [(1, 0, 0, 0)] * 2))
    assert c.n == 1 and c.c0[0, 3] == pytest.approx(0.028 - 2 * R, abs=1e-15)
    # capsule standing on a box: both end spheres tested against the box
    geo = _geo([3, 1], [0, 1], [(R, hl, 0), (0.05, 0.05, 0.01)], [(0, 0, 0)] * 2, [(0, 1)], margin=0.005)
    c = co.collide(geo, _state([(0.0, 0.0, 0.01 + hl + R - 0.0007), (0, 0, 0)], [(1, 0, 0, 0)] * 2))
    assert c.n == 1 and c.c0[0, 3] == pytest.approx(-0.0007, abs=1e-14)
    np.testing.assert_allclose(c.c1[0, :3], (0, 0, -1), atol=1e-15)      # from the capsule (g1) to the box


def test_box_on_box_vertex_face():
    """A small box resting on a big one: its 4 bottom corners on the big box's
    top face, none of the big box's corners within the small box's faces."""
    hb, hs = (0.1, 0.1, 0.02), (0.02, 0.03, 0.01)
    geo = _geo([1, 1], [0, 1], [hb, hs], [(0, 0, 0)] * 2, [(0, 1)], margin=0.002)
    yaw = _q_axis_angle((0, 0, 1), 0.3)
    z = 0.02 + 0.01 - 0.0004
    c = co.collide(geo, _state([(0, 0, 0), (0.01, -0.02, z)], [(1, 0, 0, 0), yaw]))
    assert c.n == 4
    np.testing.assert_allclose(c.c0[:, 3], -0.0004, atol=1e-15)
    np.testing.assert_allclose(c.c1[:, :3], np.tile((0, 0, 1.0), (4, 1)), atol=1e-15)   # from g1 (big) to g2
    # the same pair listed the other way round: normals flip, points and gaps stay
    geo2 = _geo([1, 1], [1, 0], [hs, hb], [(0, 0, 0)] * 2, [(0, 1)], margin=0.002)
    c2 = co.collide(geo2, _state([(0, 0, 0), (0.01, -0.02, z)], [(1, 0, 0, 0), yaw]))
    assert c2.n == 4
    np.testing.assert_allclose(c2.c1[:, :3], np.tile((0, 0, -1.0), (4, 1)), atol=1e-15)
    np.testing.assert_allclose(sorted(c2.c0[:, 3]), sorted(c.c0[:, 3]), atol=1e-15)


# ---------------------------------------------------------------- broadphase (reading R32)
def _random_geometry(seed, n=12, with_plane=True, margin=0.01):
    from harness.types import Geometry
    rng = np.random.default_rng(seed)
    kind, body, size, local = [], [], [], []
    if with_plane:
        kind.append(co.PLANE); body.append(-1); size.append((0.0, 0.0, 1.0)); local.append((0.0, 0, 0))
    for i in range(n):
        k = int(rng.integers(0, 3))
        kk = [co.SPHERE, co.BOX, co.CAPSULE][k]
        kind.append(kk)
        body.append(i)
        size.append((rng.uniform(0.01, 0.03), 0, 0) if kk == co.SPHERE else
                    tuple(rng.uniform(0.008, 0.03, 3)) if kk == co.BOX else (rng.uniform(0.008, 0.02), rng.uniform(0.005, 0.03), 0))
        local.append((0.0, 0.0, 0.0))
    G = len(kind)
    return Geometry(np.array(kind, np.int32), np.array(body, np.int32), np.zeros(G, np.int32), np.array(size, float),
                    np.array(local, float), None, margin=margin, mu=(0.7, 0.01, 0.001), condim=3)


def _random_poses(seed, W, B, spread=0.08):
    from harness.types import State
    rng = np.random.default_rng(seed + 100)
    pos = rng.uniform([-spread, -spread, 0.0], [spread, spread, spread], (W, B, 3))
    quat = rng.normal(size=(W, B, 4))
    quat /= np.linalg.norm(quat, axis=2, keepdims=True)
    z = np.zeros((W, B, 3))
    return State(pos, quat, z, z.copy(), np.zeros((W, 0)), np.zeros((W, 0)))


@pytest.mark.parametrize("seed", range(4))
def test_broadphase_loses_no_contact(seed):
    """Conservativeness (R32): the contacts of the broadphase candidates equal
    those of every valid pair tested explicitly (same records, same order)."""
    from harness.types import Geometry
    geo = _random_geometry(seed)
    st = _random_poses(seed, 3, 12)
    G = len(geo.kind)
    allp = [(a, b) for a in range(G) for b in range(a + 1, G)
            if geo.body[a] != geo.body[b] and geo.kind[b] != co.PLANE]
    full = Geometry(geo.kind, geo.body, geo.link, geo.size, geo.local, np.array(allp, np.int32),
                    margin=geo.margin, mu=geo.mu, condim=geo.condim)
    a, b = co.collide(geo, st, None), co.collide(full, st, None)
    assert b.n > 10                                   # the scenes have contacts of several kinds
    np.testing.assert_array_equal(a.world, b.world)
    np.testing.assert_array_equal(a.body_a, b.body_a)
    np.testing.assert_array_equal(a.body_b, b.body_b)
    np.testing.assert_array_equal(a.c0, b.c0)
    np.testing.assert_array_equal(a.c1, b.c1)
    # and the broadphase prunes: fewer candidates than pairs
    assert all(len(co.broadphase(geo, st, w)) < len(allp) for w in range(3))


def _bounding_radius(geo, g):
    """Reading R32's bounding-sphere filter: sphere R, box |h|, capsule R +
    half length, about the geom's frame origin (R32)."""
    k, sz = int(geo.kind[g]), np.asarray(geo.size[g], float)
    return {co.SPHERE: sz[0], co.BOX: float(np.linalg.norm(sz)), co.CAPSULE: sz[0] + sz[1]}[k]


@pytest.mark.parametrize("seed", range(4))
def test_bounding_sphere_filter_keeps_every_contact_pair(seed):
    """The GPU broadphase drops a candidate whose grown bounding spheres do
    not overlap (|c1 - c2| > rho1 + rho2 + margin, R32).  Conservative: every
    non-plane pair the oracle finds a contact for (phi < margin) passes the
    test with room to spare; on the pile it still prunes AABB candidates."""
    from harness import scenes
    cases = [(_random_geometry(seed), _random_poses(seed, 3, 12), False)]
    if seed == 0:
        scene, st, _ = scenes.c4_pile(n_worlds=1, contacts_per_world=2000)
        cases.append((scenes.pile_geometry((10, 10, 5), broadphase=True), st.astype(np.float64), True))
    for geo, st, pile in cases:
        n_cand = n_pass = 0
        for w in range(st.n_worlds):
            for (g1, g2) in co.broadphase(geo, st, w):
                if geo.kind[g1] == co.PLANE:
                    continue
                c1 = co.geom_frame(geo, g1, st, w, None)[1]
                c2 = co.geom_frame(geo, g2, st, w, None)[1]
                slack = _bounding_radius(geo, g1) + _bounding_radius(geo, g2) + geo.margin - np.linalg.norm(c1 - c2)
                n_cand += 1
                n_pass += slack >= 0
                if co.pair_contacts(geo, None, st, w, None, g12=(g1, g2)):
                    assert slack > 0, (w, g1, g2, slack)
        if pile:
            assert n_pass < 0.7 * n_cand              # 3431 AABB candidates -> ~2100


def test_aabb_matches_brute_force_extremes():
    """Box AABB = min / max over its 8 corners; capsule AABB = ends +- R
    (checked against points sampled on the capsule surface); both grown by
    margin / 2."""
    geo = _random_geometry(5, n=20, with_plane=False, margin=0.004)
    st = _random_poses(5, 1, 20)
    rng = np.random.default_rng(9)
    for g in range(20):
        lo, hi = co.aabb(geo, g, st, 0, None)
        R, x = co.geom_frame(geo, g, st, 0, None)
        k = int(geo.kind[g])
        if k == co.BOX:
            h = geo.size[g]
            pts = np.array([x + R @ (np.array([sx, sy, sz]) * h) for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)])
            np.testing.assert_allclose(lo + 0.002, pts.min(0), atol=1e-15)
            np.testing.assert_allclose(hi - 0.002, pts.max(0), atol=1e-15)
        elif k == co.CAPSULE:
            r, hl = geo.size[g, 0], geo.size[g, 1]
            u = rng.normal(size=(20000, 3))
            u /= np.linalg.norm(u, axis=1, keepdims=True)
            ax = R[:, 2]
            ends = np.concatenate([x + hl * ax + r * u, x - hl * ax + r * u])
            assert np.all(ends >= lo + 0.002 - 1e-12) and np.all(ends <= hi - 0.002 + 1e-12)
            np.testing.assert_allclose(ends.min(0), lo + 0.002, atol=2e-4 * r / 0.01)
            np.testing.assert_allclose(ends.max(0), hi - 0.002, atol=2e-4 * r / 0.01)


def test_pile_broadphase_covers_the_lattice_neighbours():
    """Config-4 pile: every lattice-neighbour pair with a contact (the round-1
    fixed candidate list) is a broadphase candidate."""
    scene, st, _ = scenes.c4_pile(n_worlds=1, contacts_per_world=2000)
    geo = scenes.pile_geometry((10, 10, 5))
    so = st.astype(np.float64)
    with_contacts = {(int(a), int(b)) for a, b in geo.pairs
                     if co.pair_contacts(geo, None, so, 0, None, g12=(int(a), int(b)))}
    geo.pairs = None
    cand = set(co.broadphase(geo, so, 0))
    assert with_contacts and with_contacts <= cand


# ---------------------------------------------------------------- box-box edge-edge (reading R33)
def _box_overlap(RA, xA, hA, RB, xB, hB, L):
    rA = np.sum(hA * np.abs(L @ RA))
    rB = np.sum(hB * np.abs(L @ RB))
    return rA + rB - abs(L @ (xB - xA))


def _rand_R(rng):
    q = rng.normal(size=4)
    return co.quat_R(q / np.linalg.norm(q))


def test_box_edge_edge_depth_is_the_minimum_over_all_directions():
    """For interpenetrating boxes the penetration depth is the minimum overlap
    of the projections over ALL directions and the SAT's 15 axes attain it:
    densely sampled directions never go below R33's overlap, which is attained
    along the contact normal, itself perpendicular to an edge of each box."""
    rng = np.random.default_rng(11)
    u = rng.normal(size=(40000, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    found = 0
    for trial in range(200):
        RA, RB = _rand_R(rng), _rand_R(rng)
        hA, hB = rng.uniform(0.5, 1.5, 3), rng.uniform(0.5, 1.5, 3)
        xA = np.zeros(3)
        xB = rng.normal(size=3)
        xB *= (np.sum(hA) + np.sum(hB)) * 0.45 / np.linalg.norm(xB)
        out = co._box_edge_edge(RA, xA, hA, RB, xB, hB, 1e9)
        if not out:
            continue
        p, phi, n = out[0]
        ov = np.array([_box_overlap(RA, xA, hA, RB, xB, hB, L) for L in u])
        if phi > 0:                                   # separated along n: not a depth pin
            continue
        found += 1
        assert ov.min() >= -phi - 1e-9                # no direction overlaps less (minimality)
        assert abs(_box_overlap(RA, xA, hA, RB, xB, hB, n) + phi) < 1e-12   # attained along n
        assert abs(np.linalg.norm(n) - 1) < 1e-12 and n @ (xB - xA) >= 0
        # n is the cross product of one edge of each box
        assert min(abs(n @ RA[:, i]) for i in range(3)) < 1e-9
        assert min(abs(n @ RB[:, j]) for j in range(3)) < 1e-9
        if found >= 12:
            break
    assert found >= 12


def test_box_edge_edge_emitted_only_on_edge_axes_within_margin():
    """Face-on stacked boxes: the minimum-overlap axis is a face normal, so no
    edge-edge contact; boxes far apart along an edge axis: none either."""
    I = np.eye(3)
    h = np.ones(3)
    assert co._box_edge_edge(I, np.zeros(3), h, I, np.array([0.1, 0.2, 1.99]), h, 0.01) == []
    Rz = co.quat_R(np.array([np.cos(np.pi / 8), 0, 0, np.sin(np.pi / 8)]))
    Rx = co.quat_R(np.array([np.cos(np.pi / 8), np.sin(np.pi / 8), 0, 0]))
    assert co._box_edge_edge(Rz, np.zeros(3), h, Rx, np.array([0.0, 0.0, 10.0]), h, 0.01) == []


# ---------------------------------------------------------------- capsule side against a box (reading R34)
def test_capsule_lying_across_a_box_touches_in_the_middle():
    """A horizontal capsule (R 1 cm, half-length 5 cm) lying across a 2 cm box
    with both ends overhanging: the end spheres are far from the box, the
    segment point above the box centre gives the one contact, with the closed
    form phi = z_c - R - h_z and the normal +z (box -> capsule when the capsule
    is g2, so from g1 = box to g2 = capsule)."""
    from harness.types import Geometry, State
    geo = Geometry(np.array([co.BOX, co.CAPSULE], np.int32), np.array([0, 1], np.int32), np.zeros(2, np.int32),
                   np.array([(0.01, 0.01, 0.01), (0.01, 0.05, 0.0)]), np.zeros((2, 3)),
                   np.array([(0, 1)], np.int32), margin=0.001)
    z = 0.01 + 0.01 - 0.0004                         # 0.4 mm penetration
    q_cap = np.array([np.cos(np.pi / 4), 0.0, np.sin(np.pi / 4), 0.0])   # capsule axis z -> x
    st = State(np.array([[[0, 0, 0], [0.003, 0.0, z]]], float), np.array([[[1.0, 0, 0, 0], q_cap]]),
               np.zeros((1, 2, 3)), np.zeros((1, 2, 3)), np.zeros((1, 0)), np.zeros((1, 0)))
    c = co.collide(geo, st, None)
    assert c.n == 1
    np.testing.assert_allclose(c.c0[0, 3], z - 0.01 - 0.01, atol=1e-12)
    np.testing.assert_allclose(c.c1[0, :3], [0, 0, 1], atol=1e-12)
    np.testing.assert_allclose(c.c0[0, :2], [0.0, 0.0], atol=1e-12)   # above the box centre (t at x = 0)
    # the ends alone (round-1 reading) would have found nothing
    assert all(co._sphere_box(e, 0.01, np.eye(3), np.zeros(3), np.full(3, 0.01))[0] > 0.001
               for e in co._segment(geo, 1, st, 0, None))
