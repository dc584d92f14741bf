"""GPU parity of the collision front-end (comfree_load_geometry /
comfree_collide) with the fp64 oracle
(oracle/collision.py): contact sets bit-exact (counts, world ids, body and
link ids, order), records within fp32 tolerance; then the closed-loop hand
(collide -> articulated upstream -> step on the GPU, every step) against the
same loop in the oracle."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import articulation as ar
from oracle import collision as co
from harness import scenes
from harness.types import Config, Geometry, Inputs, State
from _gpu import assert_close, compare_step, traj_assert

pytestmark = pytest.mark.gpu

CFG = Config()
ART = scenes.hand_articulation()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_12185_b200 as cf
    cf._lib.load()


def _tie_worlds(geo, st, art):
    """Worlds with a candidate within 2e-5 of the emission threshold (the fp32
    and fp64 decisions may differ there): excluded from the set comparison."""
    loose = Geometry(geo.kind, geo.body, geo.link, geo.size, geo.local, geo.pairs, margin=1e9, mu=geo.mu,
                     condim=geo.condim)
    allc = co.collide(loose, st, art)
    return set(allc.world[np.abs(allc.c0[:, 3] - geo.margin) < 2e-5].tolist())


def _compare(dc, link, ref, skip=()):
    """Contact sets equal (ids exact, same order), records within fp32 tolerance,
    on every world not in `skip`."""
    w = dc.world.cpu().numpy()
    gm = ~np.isin(w, list(skip))
    rm = ~np.isin(ref.world, list(skip))
    assert gm.sum() == rm.sum()
    c3 = dc.c3.cpu().numpy()[gm]
    np.testing.assert_array_equal(w[gm], ref.world[rm])
    np.testing.assert_array_equal(c3[:, 0], ref.body_a[rm])
    np.testing.assert_array_equal(c3[:, 1], ref.body_b[rm])
    np.testing.assert_array_equal(c3[:, 3], ref.condim[rm])
    np.testing.assert_array_equal(link.cpu().numpy()[gm], ref.meta["link"][rm])
    assert_close(dc.c0.cpu().numpy()[gm, :3], ref.c0[rm, :3], rtol=0, atol=2e-6, what="contact point")
    assert_close(dc.c0.cpu().numpy()[gm, 3], ref.c0[rm, 3], rtol=0, atol=1e-6, what="phi")
    assert_close(dc.c1.cpu().numpy()[gm], ref.c1[rm], rtol=0, atol=2e-5, what="normal, mu_t")
    assert_close(dc.c2.cpu().numpy()[gm], ref.c2[rm], rtol=0, atol=2e-5, what="t1, mu_tor")


def test_hand_contacts_match_oracle():
    import paper_2603_12185_b200 as cf
    scene, st, _, _ = scenes.c3_hand(n_worlds=128)
    geo = scenes.hand_geometry(margin=0.01)
    st64 = st.astype(np.float64)
    skip = _tie_worlds(geo, st64, ART)
    assert len(skip) < 8
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_articulation(ART)
    ctx.load_geometry(geo)
    dc, link = ctx.collide(capacity=128 * 40)
    ref = co.collide(geo, st64, ART)
    assert ref.n > 128                     # the test sees contacts of every kind
    _compare(dc, link, ref, skip)


@pytest.mark.parametrize("seed", range(3))
def test_random_spheres_boxes_plane(seed):
    """Free spheres and boxes above a plane, random poses; all supported pair kinds."""
    import paper_2603_12185_b200 as cf
    rng = np.random.default_rng(seed)
    W, B = 16, 6
    kind = [2] + [0, 1, 0, 1, 0, 1]
    body = [-1] + list(range(B))
    size = [(0, 0, 1.0)] + [(0.03, 0, 0), (0.04, 0.03, 0.02)] * 3
    geo = Geometry(np.array(kind, np.int32), np.array(body, np.int32), np.zeros(B + 1, np.int32),
                   np.array(size), np.zeros((B + 1, 3)),
                   np.array([(0, g) for g in range(1, B + 1)] + [(1, 3), (1, 2), (4, 5), (2, 3), (5, 6)], np.int32),
                   margin=0.02, mu=(0.7, 0.01, 0.001), condim=4)
    pos = rng.uniform([-0.04, -0.04, 0.0], [0.04, 0.04, 0.06], (W, B, 3))
    quat = rng.normal(size=(W, B, 4))
    quat /= np.linalg.norm(quat, axis=2, keepdims=True)
    st = State(pos, quat, np.zeros((W, B, 3)), np.zeros((W, B, 3)), np.zeros((W, 0)), np.zeros((W, 0)))
    st32 = st.astype(np.float32)
    st64 = st32.astype(np.float64)
    skip = _tie_worlds(geo, st64, None)
    from harness.types import Scene
    scene = Scene(np.full(B, 2.0, np.float32), np.full((B, 3), 500.0, np.float32))
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, W, st32)
    ctx.load_geometry(geo)
    dc, link = ctx.collide(capacity=W * 60)
    _compare(dc, link, co.collide(geo, st64, None), skip)


def test_capacity_and_validation():
    import paper_2603_12185_b200 as cf
    scene, st, _, _ = scenes.c3_hand(n_worlds=8)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 8, st)
    with pytest.raises(cf.ComfreeError) as ei:            # chain geoms before the articulation
        ctx.load_geometry(scenes.hand_geometry())
    assert ei.value.status == 6
    ctx.load_articulation(ART)
    bad = scenes.hand_geometry()
    bad.pairs = np.array([(1, 0)], np.int32)              # box-plane with the plane second: not supported
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.load_geometry(bad)
    assert ei.value.status == 2
    ctx.load_geometry(scenes.hand_geometry(margin=10.0))  # every candidate emits: 36 per world
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.collide(capacity=10)
    assert ei.value.status == 3


def test_closed_loop_hand():
    """collide -> articulated upstream -> step, every step, 25 steps, on the GPU
    and in the oracle; contact counts equal each step, every state element
    (pos, quat, vel, omega, chain q and qd) within the trajectory tolerance."""
    import paper_2603_12185_b200 as cf
    import torch
    scene, st, _, inp = scenes.c3_hand(n_worlds=16)
    geo = scenes.hand_geometry(margin=0.002)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_articulation(ART)
    ctx.load_geometry(geo)
    W, T, Q = st.n_worlds, 4, 16
    tL = torch.zeros((W, T, 10), device="cuda")
    tt = torch.zeros((W, Q), device="cuda")
    te = torch.from_numpy(np.ascontiguousarray(inp.tree_tau, np.float32)).cuda()
    so = st.astype(np.float64)
    for k in range(25):
        dc, link = ctx.collide(capacity=W * 40)
        ctx.articulation_update(tL, tt, dc, link, tau_ext=te)
        ctx.step(dc, Inputs(None, tL, tt), dt=CFG.dt)
        # oracle: same loop from its own state (fp32 records, like the product's)
        cref = co.collide(geo, so, ART)
        assert dc.n == cref.n, f"step {k}: {dc.n} vs {cref.n} contacts"
        L, tau = ar.upstream(ART, so.qpos, so.qvel, CFG.gravity, inp.tree_tau.astype(np.float64))
        J = np.zeros((cref.n, 2, 6, 4))
        for i in range(cref.n):
            for side, bid in enumerate((int(cref.body_a[i]), int(cref.body_b[i]))):
                if bid < -1:
                    t = -2 - bid
                    J[i, side] = ar.point_rows(ART, t, so.qpos[int(cref.world[i]), 4 * t:4 * t + 4],
                                               int(cref.meta["link"][i, side]), cref.c0[i, :3])
        cref.jrow = J
        so = oracle.step(CFG, scene, so, cref, Inputs(None, L, tau))["state"]
    traj_assert(ctx.get_state(), so, "closed-loop hand, 25 steps")


def test_device_count_mode_matches_host_count_mode():
    """comfree_collide with the count kept on the device (capacity-length
    streams, comfree_contacts.n_device) gives bitwise the same closed-loop
    trajectory as the host-count mode, and overflow is reported as
    COMFREE_ERR_CAPACITY at the next synchronising call."""
    import paper_2603_12185_b200 as cf
    import torch
    scene, st, _, inp = scenes.c3_hand(n_worlds=32)
    geo = scenes.hand_geometry(margin=0.002)
    outs = []
    for dev_count in (False, True):
        ctx = cf.Context(CFG)
        ctx.load_scene(scene, st.n_worlds, st)
        ctx.load_articulation(ART)
        ctx.load_geometry(geo)
        tL = torch.zeros((32, 4, 10), device="cuda")
        tt = torch.zeros((32, 16), device="cuda")
        te = torch.from_numpy(np.ascontiguousarray(inp.tree_tau, np.float32)).cuda()
        for _ in range(10):
            dc, link = ctx.collide(capacity=32 * 40, device_count=dev_count)
            ctx.articulation_update(tL, tt, dc, link, tau_ext=te)
            ctx.step(dc, Inputs(None, tL, tt), dt=CFG.dt)
        outs.append(ctx.get_state())
    for k in ("pos", "quat", "vel", "omega", "qpos", "qvel"):
        np.testing.assert_array_equal(outs[0][k], outs[1][k])
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_articulation(ART)
    ctx.load_geometry(scenes.hand_geometry(margin=10.0))   # 36 candidates per world emit
    ctx.collide(capacity=100, device_count=True)
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.get_state()
    assert ei.value.status == 3


def test_closed_loop_full_size_sampled_worlds():
    """Config-3 size (4096 hand worlds), the bench's closed-loop launch
    (device-side count): after 3 steps, sampled worlds against the oracle loop
    run on those worlds alone."""
    import paper_2603_12185_b200 as cf
    import torch
    scene, st, _, inp = scenes.c3_hand(n_worlds=4096)
    geo = scenes.hand_geometry(margin=0.005)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 4096, st)
    ctx.load_articulation(ART)
    ctx.load_geometry(geo)
    tL = torch.zeros((4096, 4, 10), device="cuda")
    tt = torch.zeros((4096, 16), device="cuda")
    te = torch.from_numpy(np.ascontiguousarray(inp.tree_tau, np.float32)).cuda()
    for _ in range(3):
        dc, link = ctx.collide(capacity=4096 * 40, device_count=True)
        ctx.articulation_update(tL, tt, dc, link, tau_ext=te)
        ctx.step(dc, Inputs(None, tL, tt), dt=CFG.dt)
    out = ctx.get_state()
    for w in (0, 1234, 4095):
        so = st.world_slice(w, w + 1).astype(np.float64)
        tau_w = inp.tree_tau[w:w + 1].astype(np.float64)
        for _ in range(3):
            cref = co.collide(geo, so, ART)
            J = np.zeros((cref.n, 2, 6, 4))
            for i in range(cref.n):
                for side, bid in enumerate((int(cref.body_a[i]), int(cref.body_b[i]))):
                    if bid < -1:
                        t = -2 - bid
                        J[i, side] = ar.point_rows(ART, t, so.qpos[0, 4 * t:4 * t + 4],
                                                   int(cref.meta["link"][i, side]), cref.c0[i, :3])
            cref.jrow = J
            L, tau = ar.upstream(ART, so.qpos, so.qvel, CFG.gravity, tau_w)
            so = oracle.step(CFG, scene, so, cref, Inputs(None, L, tau))["state"]
        for key in ("qvel", "qpos", "vel", "omega", "pos"):
            ref = getattr(so, key)
            err = np.abs(out[key][w:w + 1] - ref)
            assert np.all(err <= 1e-4 * np.abs(ref) + 1e-6), (w, key, float(err.max()))


@pytest.mark.parametrize("seed", range(3))
def test_random_capsules_boxes_spheres(seed):
    """Every supported pair kind including capsules and box-box, random poses."""
    import paper_2603_12185_b200 as cf
    from harness.types import Scene
    rng = np.random.default_rng(100 + seed)
    W, B = 24, 6
    kind = [2, 0, 1, 3, 1, 3, 0]
    body = [-1] + list(range(B))
    size = [(0, 0, 1.0), (0.02, 0, 0), (0.03, 0.025, 0.02), (0.015, 0.02, 0), (0.025, 0.02, 0.03),
            (0.012, 0.03, 0), (0.018, 0, 0)]
    pairs = [(0, g) for g in range(1, B + 1)] + [(1, 2), (2, 3), (3, 4), (4, 2), (3, 5), (5, 6), (6, 3),
                                                 (1, 3), (5, 4), (2, 6)]
    geo = Geometry(np.array(kind, np.int32), np.array(body, np.int32), np.zeros(B + 1, np.int32),
                   np.array(size), np.zeros((B + 1, 3)), np.array(pairs, np.int32), margin=0.01,
                   mu=(0.8, 0.01, 0.001), condim=3)
    pos = rng.uniform([-0.03, -0.03, 0.0], [0.03, 0.03, 0.05], (W, B, 3))
    quat = rng.normal(size=(W, B, 4))
    quat /= np.linalg.norm(quat, axis=2, keepdims=True)
    st = State(pos, quat, np.zeros((W, B, 3)), np.zeros((W, B, 3)), np.zeros((W, 0)), np.zeros((W, 0)))
    st32 = st.astype(np.float32)
    st64 = st32.astype(np.float64)
    skip = _tie_worlds(geo, st64, None)
    scene = Scene(np.full(B, 2.0, np.float32), np.full((B, 3), 500.0, np.float32))
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, W, st32)
    ctx.load_geometry(geo)
    dc, link = ctx.collide(capacity=W * 200)
    ref = co.collide(geo, st64, None)
    assert ref.n > W
    _compare(dc, link, ref, skip)


def test_closed_loop_pile_sampled_worlds():
    """The pile's full step at bench size (1024 worlds x 500 bodies, the
    config-4 geometry in broadphase mode, GPU collision then the step, as
    bench.py --collide runs it) for 10 steps; sampled worlds run the same loop in the oracle
    (oracle collision -> oracle step from its own state).  Contact counts
    agree each step up to candidates within 2e-5 of the emission threshold
    (where fp32 and fp64 may decide differently; such a contact's gap is
    ~the margin, so its impulse is 0 unless it approaches fast), and every
    state element is within the trajectory tolerance after 10 steps."""
    import paper_2603_12185_b200 as cf
    scene, st, _ = scenes.c4_pile(n_worlds=1024, contacts_per_world=2000)
    geo = scenes.pile_geometry((10, 10, 5), broadphase=True)     # bench.py --collide's geometry
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_geometry(geo)
    sample = (0, 517, 1023)
    so = st.astype(np.float64)
    so = State(*(getattr(so, k)[list(sample)] for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")))
    loose = Geometry(geo.kind, geo.body, geo.link, geo.size, geo.local, geo.pairs, margin=geo.margin + 4e-5,
                     mu=geo.mu, condim=geo.condim)
    for k in range(10):
        dc, _ = ctx.collide(capacity=1024 * 4000)
        wg = dc.world.cpu().numpy()
        cref = co.collide(geo, so, None)
        near = co.collide(loose, so, None)
        ties = np.bincount(near.world[np.abs(near.c0[:, 3] - geo.margin) < 2e-5], minlength=len(sample))
        for j, w in enumerate(sample):
            ng, no = int(np.count_nonzero(wg == w)), int(np.count_nonzero(cref.world == j))
            assert abs(ng - no) <= ties[j], f"step {k} world {w}: {ng} vs {no} contacts ({ties[j]} ties)"
        ctx.step(dc, None, dt=CFG.dt)
        so = oracle.step(CFG, scene, so, cref, None)["state"]
    out = ctx.get_state()
    sg = {key: out[key][list(sample)] for key in ("pos", "quat", "vel", "omega")}
    traj_assert(sg, so, "closed-loop pile, 10 steps", keys=("pos", "quat", "vel", "omega"))


def test_device_count_overflow_keeps_whole_pairs():
    """Overflow in device-count mode: the count is the offset of the first pair
    that does not fit (never a range with unwritten records), every record
    below it equals the unbounded run's, and the overflow surfaces at the next
    check (comfree_check)."""
    import paper_2603_12185_b200 as cf
    scene, st, _, _ = scenes.c3_hand(n_worlds=32)
    geo = scenes.hand_geometry(margin=0.01)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 32, st)
    ctx.load_articulation(ART)
    ctx.load_geometry(geo)
    full, _ = ctx.collide(capacity=32 * 40, device_count=True)
    nf = int(full.n_dev.item())
    ref = {k: getattr(full, k)[:nf].cpu().numpy().copy() for k in ("world", "c0", "c3")}
    cap = nf // 2 + 1
    full.c0.fill_(float("nan"))                         # stale records would show up as NaN / -7
    full.c3.fill_(-7)
    part, _ = ctx.collide(capacity=cap, device_count=True)
    n = int(part.n_dev.item())
    assert 0 < n <= cap
    for k in ("world", "c0", "c3"):
        np.testing.assert_array_equal(getattr(part, k)[:n].cpu().numpy(), ref[k][:n])
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.check()
    assert ei.value.status == 3


# ---------------------------------------------------------------- broadphase mode (reading R32)
def _compare_off_threshold(dc, link, ref, margin, band=2e-6):
    """Contact lists equal (ids exact, same order; records within fp32
    tolerance) once the records whose gap lies within `band` of the emission
    threshold are dropped from both (there fp32 and fp64 may decide
    differently; 2e-6 m is ~20x the fp32 error of a gap at these sizes)."""
    g_phi = dc.c0.cpu().numpy()[:, 3]
    gk = np.abs(g_phi - margin) >= band
    rk = np.abs(ref.c0[:, 3] - margin) >= band
    assert gk.sum() == rk.sum(), (gk.sum(), rk.sum())
    c3 = dc.c3.cpu().numpy()[gk]
    np.testing.assert_array_equal(dc.world.cpu().numpy()[gk], ref.world[rk])
    np.testing.assert_array_equal(c3[:, 0], ref.body_a[rk])
    np.testing.assert_array_equal(c3[:, 1], ref.body_b[rk])
    np.testing.assert_array_equal(link.cpu().numpy()[gk], ref.meta["link"][rk])
    assert_close(dc.c0.cpu().numpy()[gk, :3], ref.c0[rk, :3], rtol=0, atol=2e-6, what="contact point")
    assert_close(g_phi[gk], ref.c0[rk, 3], rtol=0, atol=1e-6, what="phi")
    assert_close(dc.c1.cpu().numpy()[gk], ref.c1[rk], rtol=0, atol=2e-5, what="normal, mu_t")
    assert_close(dc.c2.cpu().numpy()[gk], ref.c2[rk], rtol=0, atol=2e-5, what="t1, mu_tor")


def test_broadphase_pile_matches_oracle():
    """Config-4 pile geometry without a candidate list: the GPU's sort-and-
    sweep broadphase + narrowphase (one kernel, chained scan over worlds) gives
    the oracle's contact list -- ids exact and in the same order (candidate
    pairs in (g1, g2) order), records within fp32 tolerance -- including the
    diagonal neighbours and box-box edge-edge contacts the fixed lattice list
    missed."""
    import paper_2603_12185_b200 as cf
    scene, st, _ = scenes.c4_pile(n_worlds=6, contacts_per_world=2000)
    geo = scenes.pile_geometry((10, 10, 5), broadphase=True)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_geometry(geo)
    dc, link = ctx.collide(capacity=6 * 4000)
    st64 = st.astype(np.float64)
    ref = co.collide(geo, st64, None)
    assert ref.n > 6 * 1100
    lattice = co.collide(scenes.pile_geometry((10, 10, 5)), st64, None)
    assert ref.n > lattice.n                       # more than the fixed candidate list found
    _compare_off_threshold(dc, link, ref, geo.margin)


def test_broadphase_large_pile_one_cta_per_sm():
    """An 801-geom pile (16 x 10 x 5 lattice): the candidate list gets the
    one-CTA-per-SM shared-memory budget (two CTAs would leave room for fewer
    than 8 candidates per geom); same list as the oracle."""
    import paper_2603_12185_b200 as cf
    scene, st, _ = scenes.c4_pile(n_worlds=3, contacts_per_world=2000, lattice=(16, 10, 5))
    geo = scenes.pile_geometry((16, 10, 5), broadphase=True)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_geometry(geo)
    dc, link = ctx.collide(capacity=3 * 6000)
    ref = co.collide(geo, st.astype(np.float64), None)
    assert ref.n > 3 * 1800
    _compare_off_threshold(dc, link, ref, geo.margin)


def test_broadphase_sparse_1500_spheres():
    """1500 spheres scattered over a 1.5 m x 1.5 m x 0.3 m box above a plane
    (one CTA per SM, a 2048-entry sort, sparse candidates): same list as the
    oracle."""
    import paper_2603_12185_b200 as cf
    from harness.types import Scene
    rng = np.random.default_rng(7)
    W, B = 2, 1500
    geo = Geometry(np.array([2] + [0] * B, np.int32), np.array([-1] + list(range(B)), np.int32),
                   np.zeros(B + 1, np.int32), np.array([(0, 0, 1.0)] + [(0.02, 0, 0)] * B), np.zeros((B + 1, 3)),
                   None, margin=0.004, mu=(0.7, 0.01, 0.001), condim=3)
    pos = rng.uniform([0, 0, 0.01], [1.5, 1.5, 0.3], (W, B, 3))
    quat = np.zeros((W, B, 4))
    quat[..., 0] = 1
    st = State(pos, quat, np.zeros((W, B, 3)), np.zeros((W, B, 3)), np.zeros((W, 0)), np.zeros((W, 0))).astype(np.float32)
    scene = Scene(np.full(B, 2.0, np.float32), np.full((B, 3), 500.0, np.float32))
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, W, st)
    ctx.load_geometry(geo)
    dc, link = ctx.collide(capacity=W * 3000)
    ref = co.collide(geo, st.astype(np.float64), None)
    assert ref.n > W * 100
    _compare_off_threshold(dc, link, ref, geo.margin)


@pytest.mark.parametrize("seed", range(3))
def test_broadphase_random_scenes_match_oracle(seed):
    """Random spheres / boxes / capsules above a plane, random orientations
    (every pair kind, edge-edge included), broadphase mode."""
    import paper_2603_12185_b200 as cf
    from harness.types import Scene
    from test_oracle_collision import _random_geometry, _random_poses
    geo = _random_geometry(seed, n=14)
    stt = _random_poses(seed, 12, 14)
    st32 = stt.astype(np.float32)
    st64 = st32.astype(np.float64)
    scene = Scene(np.full(14, 2.0, np.float32), np.full((14, 3), 500.0, np.float32))
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 12, st32)
    ctx.load_geometry(geo)
    dc, link = ctx.collide(capacity=12 * 200)
    ref = co.collide(geo, st64, None)
    assert ref.n > 50
    _compare_off_threshold(dc, link, ref, geo.margin)


def test_broadphase_device_count_overflow_and_graph():
    """Device-count mode of the broadphase: the whole-pair count on overflow
    (records below it equal the unbounded run's), COMFREE_ERR_CAPACITY at the
    next check; and the launch replays in a CUDA graph (memsets + one kernel,
    the counters reset themselves) with the same records."""
    import torch
    import paper_2603_12185_b200 as cf
    scene, st, _ = scenes.c4_pile(n_worlds=5, contacts_per_world=2000)
    geo = scenes.pile_geometry((10, 10, 5), broadphase=True)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 5, st)
    ctx.load_geometry(geo)
    full, _ = ctx.collide(capacity=5 * 4000, device_count=True)
    nf = int(full.n_dev.item())
    ref = {k: getattr(full, k)[:nf].cpu().numpy().copy() for k in ("world", "c0", "c3")}
    ctx2 = cf.Context(CFG)
    ctx2.load_scene(scene, 5, st)
    ctx2.load_geometry(geo)
    part, _ = ctx2.collide(capacity=nf // 2, device_count=True)
    n = int(part.n_dev.item())
    assert 0 < n <= nf // 2
    for k in ("world", "c0", "c3"):
        np.testing.assert_array_equal(getattr(part, k)[:n].cpu().numpy(), ref[k][:n])
    with pytest.raises(cf.ComfreeError) as ei:
        ctx2.check()
    assert ei.value.status == 3
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ctx.collide(capacity=5 * 4000, device_count=True, stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    dc, _ = ctx.collide(capacity=5 * 4000, device_count=True)
    assert int(dc.n_dev.item()) == nf
    for k in ("world", "c0", "c3"):
        np.testing.assert_array_equal(getattr(dc, k)[:nf].cpu().numpy(), ref[k])


def test_broadphase_stage_fallback_identical(tmp_path):
    """The broadphase stages the records of its single narrowphase pass and
    places them once the world's base is known; a world with more records
    than the staging area evaluates the narrowphase again in place.  Both give
    bitwise the same contact list (host and device count, overflow cut):
    default staging vs a 600-record staging area (every pile world falls back)
    vs 1350 (some do: 1328-1362 records per world)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    outs = []
    for cap in ("0", "600", "1350"):
        out = str(tmp_path / f"bp_{cap}.npz")
        env = dict(os.environ)
        if cap != "0":
            env["COMFREE_BP_STAGE_CAP"] = cap
        subprocess.run([sys.executable, os.path.join(here, "_bp_stage_dump.py"), out], check=True, env=env,
                       cwd=os.path.dirname(here), timeout=300)
        outs.append(np.load(out))
    a = outs[0]
    assert a["0_world"].shape[0] > 7 * 1000 and 0 < int(a["cut_n"]) <= 3001
    for b in outs[1:]:
        assert set(a.files) == set(b.files)
        for k in a.files:
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_step_collided_bitwise(tmp_path):
    """comfree_step_collided (the step reading each world's staged records
    from the front-end, no emit pass, no public contact streams) gives the
    bit-identical state of comfree_collide + comfree_step over 6 pile steps:
    with the default staging area, with a 600-record area (every world written
    in place: the step reads the library-owned streams from the world's base)
    and with 1350 (some worlds each way); and with 8 tangent facets, which the
    call runs as collide + step on its own streams."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for cap in ("0", "600", "1350", "nt8"):
        out = str(tmp_path / f"fused_{cap}.npz")
        env = dict(os.environ)
        if cap == "nt8":                  # 8 tangent facets: comfree_step_collided's collide + step path
            env["FUSED_NT"] = "8"
        elif cap != "0":
            env["COMFREE_BP_STAGE_CAP"] = cap
        subprocess.run([sys.executable, os.path.join(here, "_bp_fused_run.py"), out], check=True, env=env,
                       cwd=os.path.dirname(here), timeout=300)
        r = np.load(out)
        keys = [k[len("split_"):] for k in r.files if k.startswith("split_")]
        assert "vel" in keys and "pos" in keys
        for k in keys:
            a, b = r["split_" + k], r["fused_" + k]
            assert np.all(np.isfinite(a))
            np.testing.assert_array_equal(a, b, err_msg=f"{k} (stage cap {cap})")
        assert np.abs(r["split_vel"]).max() > 0


def test_step_collided_refuses_list_geometry_and_chains():
    """comfree_step_collided needs the broadphase mode and a chain-free scene:
    a geometry with a candidate list, or the hand with chains, is refused with
    COMFREE_ERR_STATE and leaves the state untouched."""
    import paper_2603_12185_b200 as cf
    scene, st, _ = scenes.c4_pile(n_worlds=2, contacts_per_world=200, lattice=(5, 5, 2))
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_geometry(scenes.pile_geometry((5, 5, 2)))            # lattice candidate list
    before = ctx.get_state()
    with pytest.raises(cf.ComfreeError) as e:
        ctx.step_collided(2 * 2000)
    assert e.value.status == 6                       # COMFREE_ERR_STATE
    after = ctx.get_state()
    for k in before:
        np.testing.assert_array_equal(before[k], after[k])
    scene, st, _, _ = scenes.c3_hand(n_worlds=2)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 2, st)
    ctx.load_articulation(scenes.hand_articulation())
    ctx.load_geometry(scenes.hand_geometry(margin=0.002))
    with pytest.raises(cf.ComfreeError) as e:
        ctx.step_collided(2 * 40)
    assert e.value.status == 6                       # COMFREE_ERR_STATE
