"""GPU parity of the articulated upstream (comfree_load_articulation /
comfree_articulation_update) with the fp64 oracle
(oracle/articulation.py): chain Cholesky factors, tau - c and chain-side
contact J rows on the config-3 hand, then the full hand step (upstream +
contact resolution) and a multi-step trajectory with the upstream recomputed
every step."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import articulation as ar
from harness import scenes
from harness.types import Config, Inputs
from _gpu import assert_close, compare_step

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


def _oracle_rows(st, c, link):
    """J rows of every chain side, (C,2,6,4), from the oracle at the state's q."""
    T, nd = ART.n_trees, ART.tree_ndof
    J = np.zeros((c.n, 2, 6, 4))
    for k in range(c.n):
        for side, bid in enumerate((int(c.body_a[k]), int(c.body_b[k]))):
            if bid < -1:
                t = -2 - bid
                w = int(c.world[k])
                q = st.qpos[w, t * nd:(t + 1) * nd].astype(np.float64)
                J[k, side, :, :nd] = ar.point_rows(ART, t, q, int(link[k, side]), c.c0[k, :3].astype(np.float64))
    return J


def _gpu_upstream(ctx, st, c, link, tau_ext):
    import torch
    import paper_2603_12185_b200 as cf
    W, T, Q = st.n_worlds, ART.n_trees, ART.n_trees * ART.tree_ndof
    tL = torch.zeros((W, T, 10), device="cuda")
    tt = torch.zeros((W, Q), device="cuda")
    cz = c.take(np.arange(c.n))
    cz.jrow = np.zeros_like(c.jrow)                 # the rows must come from the kernel
    dc = cf.DeviceContacts.from_host(cz)
    lk = torch.from_numpy(np.ascontiguousarray(link, np.int32)).cuda()
    te = torch.from_numpy(np.ascontiguousarray(tau_ext, np.float32)).cuda()
    ctx.articulation_update(tL, tt, dc, lk, tau_ext=te)
    return tL, tt, dc


def test_upstream_factors_bias_and_rows():
    import paper_2603_12185_b200 as cf
    scene, st, c, inp = scenes.c3_hand(n_worlds=64)
    link = c.meta["link"]
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_articulation(ART)
    tL, tt, dc = _gpu_upstream(ctx, st, c, link, inp.tree_tau)
    L, tau = ar.upstream(ART, st.qpos.astype(np.float64), st.qvel.astype(np.float64), CFG.gravity,
                         inp.tree_tau.astype(np.float64))
    assert_close(tL.cpu().numpy(), L, rtol=2e-5, atol=2e-7, what="tree_L")
    assert_close(tt.cpu().numpy(), tau, rtol=1e-4, atol=1e-6, what="tau - c")
    from paper_2603_12185_b200 import pack_jrow
    J = _oracle_rows(st, c, link)
    got = dc.jrow.cpu().numpy()
    exp = pack_jrow(J)
    chain = np.zeros((2, c.n), bool)
    chain[0], chain[1] = c.body_a < -1, c.body_b < -1
    for side in range(2):
        m = chain[side]
        assert_close(got[side * 6:(side + 1) * 6, m], exp[side * 6:(side + 1) * 6, m], rtol=1e-5, atol=1e-7,
                     what=f"J rows side {side}")


def test_hand_step_with_gpu_upstream():
    """Upstream + contact resolution on the GPU vs oracle upstream + oracle step."""
    import paper_2603_12185_b200 as cf
    scene, st, c, inp = scenes.c3_hand(n_worlds=48)
    link = c.meta["link"]
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_articulation(ART)
    tL, tt, dc = _gpu_upstream(ctx, st, c, link, inp.tree_tau)
    ctx.step(dc, Inputs(None, tL, tt), dt=CFG.dt)
    out = ctx.get_state()
    L, tau = ar.upstream(ART, st.qpos.astype(np.float64), st.qvel.astype(np.float64), CFG.gravity,
                         inp.tree_tau.astype(np.float64))
    co = c.take(np.arange(c.n))
    co.jrow = _oracle_rows(st, c, link)
    o = oracle.step(CFG, scene, st, co, Inputs(None, L, tau))
    from harness.types import State
    g = dict(state=State(out["pos"], out["quat"], out["vel"], out["omega"], out["qpos"], out["qvel"]))
    compare_step(g, o)


def test_hand_trajectory_upstream_every_step():
    """20 steps, the upstream recomputed from the evolving q each step on both
    sides (fixed contact points), within 1e-3 relative at the end."""
    import paper_2603_12185_b200 as cf
    scene, st, c, inp = scenes.c3_hand(n_worlds=16)
    link = c.meta["link"]
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_articulation(ART)
    so = st.astype(np.float64)
    for _ in range(20):
        cur = ctx.get_state()
        from harness.types import State
        sg = State(cur["pos"], cur["quat"], cur["vel"], cur["omega"], cur["qpos"], cur["qvel"])
        tL, tt, dc = _gpu_upstream(ctx, sg, c, link, inp.tree_tau)
        ctx.step(dc, Inputs(None, tL, tt), dt=CFG.dt)
        L, tau = ar.upstream(ART, so.qpos, so.qvel, CFG.gravity, inp.tree_tau.astype(np.float64))
        co = c.take(np.arange(c.n))
        co.jrow = _oracle_rows(so, c, link)
        so = oracle.step(CFG, scene, so, co, Inputs(None, L, tau))["state"]
    out = ctx.get_state()
    for k in ("qvel", "qpos", "vel", "omega", "pos"):
        ref = getattr(so, k)
        err = np.abs(out[k] - ref)
        assert np.all(err <= 1e-3 * np.abs(ref) + 1e-5), (k, float(err.max()))


def test_bad_link_and_model_mismatch_rejected():
    import paper_2603_12185_b200 as cf
    scene, st, c, inp = scenes.c3_hand(n_worlds=4)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, st.n_worlds, st)
    bad = scenes.hand_articulation()
    bad.axis = bad.axis * 2.0                      # not unit
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.load_articulation(bad)
    assert ei.value.status == 2
    ctx.load_articulation(ART)
    link = c.meta["link"].copy()
    link[0, 0] = 7                                 # chain side with a link index beyond nd
    _gpu_upstream(ctx, st, c, link, inp.tree_tau)
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.get_state()
    assert ei.value.status == 2 and "articulation" in str(ei.value)
