"""Pin for reading R3 (literal Eq. (12): K = k M(phi)/dt, D = d M(phi)/dt) from
the paper's drop test (Fig. "Penetration depths"): the table shows
the mean penetration depth falling as k_user rises (3.9 / 1.6 / 1.0 mm at
k = 0.1 / 0.3 / 0.5) and falling slightly as d_user rises from 0.001 to 0.005
(3-12 %).  (The text at P:280 says depth *increases* with k; the table says the
opposite -- reading R20 takes the table.)  The paper's scene (five 5x5 arrays
of mixed primitives on a box) and its MJWarp collision are out of scope; this
is the same experiment on a small scene the oracle runs in seconds: 3x3
columns of two stacked 5 cm cubes dropped from 1 cm onto the floor, 600 steps
at dt = 0.002, the depth of every penetrating contact recorded over the last
200 steps (after the drop has settled).  All six (k, d) settings of the table run as six worlds of one
oracle call through per-contact (k, d) pairs.  Under the dimensionally
consistent alternative K = k M/dt^2 the bodies float (depth ~ 0), so the trend
distinguishes the readings.  CPU only."""
from __future__ import annotations

import numpy as np

import oracle
from harness import scenes
from harness.collide import Friction, Geom, Plane, WorldGeometry, collide
from harness.types import Config, Contacts, State

SETTINGS = [(0.1, 0.001), (0.1, 0.005), (0.3, 0.001), (0.3, 0.005), (0.5, 0.001), (0.5, 0.005)]


def _drop_depths(steps=600, record_from=400):
    h = 0.025
    nx = 3
    geoms = [Geom("box", (h, h, h)) for _ in range(2 * nx * nx)]
    pairs = [(2 * i, 2 * i + 1) for i in range(nx * nx)]          # column i: box 2i below 2i+1
    geo = WorldGeometry(geoms, [Plane()], Friction(0.8, 0.005, 0.0001), condim=3, margin=0.002, pairs=pairs)
    scene = scenes.scene_from_geoms(geoms)
    W, B = len(SETTINGS), len(geoms)
    st = scenes.empty_state(W, B).astype(np.float64)
    for i in range(nx * nx):
        x, y = 0.08 * (i % nx), 0.08 * (i // nx)
        st.pos[:, 2 * i] = (x, y, h + 0.01)
        st.pos[:, 2 * i + 1] = (x, y, 3 * h + 0.012)
    cfg = Config()
    depths = [[] for _ in range(W)]
    for k in range(steps):
        parts = [collide(geo, st.pos[w], st.quat[w], w, np.float64) for w in range(W)]
        c = Contacts.concat(parts)
        c.kd = np.array([SETTINGS[w] for w in c.world], np.float64)
        if k >= record_from:
            for w in range(W):
                phi = c.c0[c.world == w, 3]
                depths[w].extend((-phi[phi < 0]).tolist())
        st = oracle.step(cfg, scene, st, c, None)["state"]
    return np.array([np.mean(d) for d in depths])


def test_drop_test_depth_trend_matches_table():
    d = _drop_depths() * 1e3                                       # mm
    by = {s: v for s, v in zip(SETTINGS, d)}
    # depth falls as k rises, for either damping (table rows 0.1 > 0.3 > 0.5)
    for dd in (0.001, 0.005):
        assert by[(0.1, dd)] > by[(0.3, dd)] > by[(0.5, dd)] > 0.0, d
    # more damping, less depth (table: 3.9 vs 3.8, 1.6 vs 1.4, 1.0 vs 0.9)
    for kk in (0.1, 0.3, 0.5):
        assert by[(kk, 0.005)] < by[(kk, 0.001)], d
    # the same millimetre scale as the table (3.9 / 1.6 / 1.0 mm at d = 0.001)
    assert 1.0 < by[(0.1, 0.001)] < 15.0 and 0.2 < by[(0.5, 0.001)] < 5.0, d
