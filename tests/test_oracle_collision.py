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
