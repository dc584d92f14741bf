"""Parity of the CUDA path (through the C ABI) with the fp64 oracle.

Tolerance (BASELINE.json north star): per step, from identical fp32 states,
|d| <= 1e-5 |ref| + 1e-6 on v+, omega+, chain qd+ and every facet impulse
Lambda_f; positions/orientations within fp32 rounding; integer outputs
(off, perm, foff) bit-exact; 100-step trajectories within 1e-3 relative.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from harness import scenes
from harness.types import Config, Contacts, Inputs, State
from _gpu import assert_close, compare_step, gpu_step, operand_scale, traj_assert
from _helpers import run_trajectory

pytestmark = pytest.mark.gpu

CFG = Config()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_12185_b200 as cf
    cf._lib.load()


# ---------------------------------------------------------------- random mixed instances
@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("cfg", [CFG, CFG.with_(n_t=8, n_rol=6), CFG.with_(n_t=6, n_rol=2, power=3.0)],
                         ids=["nt4", "nt8", "nt6p3"])
def test_random_mixed_step(seed, cfg):
    """Every condim, free/static sides, ragged worlds (incl. empty), unsorted ids."""
    cpw = [0, 3, 40, 257, 1, 70][seed % 6:] + [0, 3, 40, 257, 1, 70][:seed % 6]
    scene, st, c, inp = scenes.random_instance(500 + seed, n_worlds=6, n_bodies=9, contacts_per_world=cpw)
    c = scenes.shuffle_contacts(c, seed)
    o = oracle.step(cfg, scene, st, c, inp)
    g = gpu_step(cfg, scene, st, c, inp)
    compare_step(g, o)


def test_largest_world_that_fits_shared_memory():
    """2070 bodies per world: the step's per-world shared memory (28 words
    per body) just under the 227 KB a CTA may use, one world per SM, 8 warps;
    matches the oracle."""
    scene, st, c, inp = scenes.random_instance(777, n_worlds=3, n_bodies=2070, contacts_per_world=[4000, 17, 2500],
                                               condims=(3, 4, 6))
    compare_step(gpu_step(CFG, scene, st, c, inp), oracle.step(CFG, scene, st, c, inp))


@pytest.mark.parametrize("n_bodies,cpw", [(2100, [50, 3000]), (5000, [12000, 0, 7000])])
def test_large_worlds_global_scratch(n_bodies, cpw):
    """Worlds beyond shared memory (> ~2070 bodies): the step keeps the world's
    body records and fixed-point accumulators in a global, L2-resident scratch
    slab (global integer atomics) -- same arithmetic, parity with the oracle
    at 5000 bodies per world, every condim, ragged and empty worlds; and
    bitwise deterministic."""
    scene, st, c, inp = scenes.random_instance(778 + n_bodies, n_worlds=len(cpw), n_bodies=n_bodies,
                                               contacts_per_world=cpw, condims=(1, 3, 4, 6))
    g = gpu_step(CFG, scene, st, c, inp)
    compare_step(g, oracle.step(CFG, scene, st, c, inp))
    g2 = gpu_step(CFG, scene, st, c, inp)
    for k in ("pos", "quat", "vel", "omega"):
        np.testing.assert_array_equal(getattr(g["state"], k), getattr(g2["state"], k))


@pytest.mark.parametrize("seed", range(4))
def test_random_articulated_step(seed):
    """Chains (S8): tree sides with J rows, Cholesky M^-1, mixed with free bodies."""
    nd = [4, 3, 2, 1][seed]
    scene, st, c, inp = scenes.random_instance(600 + seed, n_worlds=5, n_bodies=3, contacts_per_world=[30, 0, 7, 64, 33],
                                               n_trees=4, tree_ndof=nd)
    o = oracle.step(CFG, scene, st, c, inp)
    g = gpu_step(CFG, scene, st, c, inp)
    compare_step(g, o)


def test_locked_dofs_and_no_fext():
    scene, st, c, inp = scenes.random_instance(700, n_worlds=4, n_bodies=6, contacts_per_world=25,
                                               with_fext=False, locked_frac=0.5)
    o = oracle.step(CFG, scene, st, c, inp)
    g = gpu_step(CFG, scene, st, c, inp)
    compare_step(g, o)


def test_max_facet_counts():
    """n_t = n_rol = 32 (66 facets per contact).  Friction that nearly stops a
    spin makes omega+ = omega_s + Iw^-1 p a cancellation of large terms, so
    the velocity bound is taken relative to the magnitude of the operands of
    Eq. (10) (reading R30, from the dense oracle B); impulses and positions
    keep the plain north-star bound."""
    cfg = CFG.with_(n_t=32, n_rol=32)
    scene, st, c, inp = scenes.random_instance(701, n_worlds=3, n_bodies=4, contacts_per_world=20,
                                               condims=(6,))
    g = gpu_step(cfg, scene, st, c, inp)
    o = oracle.step(cfg, scene, st, c, inp)
    compare_step(g, o, scale=operand_scale(cfg, scene, st, c, inp))


def test_no_contacts_and_empty_worlds():
    """No contacts at all (world[] may be empty/null): every world offset is 0.
    A context with contacts is stepped and destroyed first, so the empty step's
    buffers are likely recycled memory (a stale offset array once crashed it)."""
    scene, st, c, inp = scenes.random_instance(702, n_worlds=3, n_bodies=4, contacts_per_world=[0, 0, 0])
    assert c.n == 0
    s1, st1, c1, inp1 = scenes.random_instance(703, n_worlds=3, n_bodies=4, contacts_per_world=[500, 900, 700])
    g1 = gpu_step(CFG, s1, st1, c1, inp1)
    g1["ctx"].close()
    del g1
    compare_step(gpu_step(CFG, scene, st, c, inp, impulses=False), oracle.step(CFG, scene, st, c, inp))


# ---------------------------------------------------------------- paper-shaped workloads
def test_c4_pile_small_step():
    """Dense pile (config 4 shape) at a size the oracle finishes quickly:
    several 256-contact tiles per world plus a ragged tail."""
    scene, st, c = scenes.c4_pile(n_worlds=6, contacts_per_world=2000 + 77)
    o = oracle.step(CFG, scene, st, c, None)
    g = gpu_step(CFG, scene, st, c, None)
    compare_step(g, o)


def test_c3_hand_step():
    scene, st, c, inp = scenes.c3_hand(n_worlds=64)
    o = oracle.step(CFG, scene, st, c, inp)
    g = gpu_step(CFG, scene, st, c, inp)
    compare_step(g, o)


def test_c4_full_size_sampled_worlds():
    """BASELINE config 4 at full size (1024 worlds x 500 bodies x 2000
    contacts) in the bench's launch configuration; sampled worlds checked
    against the oracle one by one."""
    import torch
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=1024, contacts_per_world=2000)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 1024, st)
    dc = cf.DeviceContacts.from_host(c)
    ctx.step(dc, None, dt=CFG.dt)
    out = ctx.get_state()
    for w in (0, 1, 147, 511, 777, 1023):
        sel = np.nonzero(c.world == w)[0]
        cw = c.take(sel)
        cw.world = np.zeros(len(sel), np.int32)
        o = oracle.step(CFG, scene, st.world_slice(w, w + 1), cw, None)
        gst = State(*(out[k][w:w + 1] for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")))
        compare_step(dict(state=gst), o)


def test_c3_full_size_sampled_worlds():
    """BASELINE config 3 at full size (4096 hand worlds) in the bench's launch
    configuration (one warp per world); sampled worlds against the oracle."""
    import torch
    import paper_2603_12185_b200 as cf
    from harness.types import Inputs
    scene, st, c, inp = scenes.c3_hand(n_worlds=4096)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 4096, st)
    tin = Inputs(*(None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
                   for a in (inp.f_ext, inp.tree_L, inp.tree_tau)))
    ctx.step(cf.DeviceContacts.from_host(c), tin, dt=CFG.dt)
    out = ctx.get_state()
    for w in (0, 1, 1000, 2047, 4095):
        sel = np.nonzero(c.world == w)[0]
        cw = c.take(sel)
        cw.world = np.zeros(len(sel), np.int32)
        iw = Inputs(None, inp.tree_L[w:w + 1], inp.tree_tau[w:w + 1])
        o = oracle.step(CFG, scene, st.world_slice(w, w + 1), cw, iw)
        gst = State(*(out[k][w:w + 1] for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")))
        compare_step(dict(state=gst), o)


def test_c5_full_size_sampled_worlds():
    """BASELINE config 5 at full size on one GPU (65536 worlds: 32768 hand +
    32768 pile-lite as two contexts on two streams, as bench.py times it);
    sampled worlds of each part against the oracle."""
    import torch
    import paper_2603_12185_b200 as cf
    from harness.types import Inputs
    d = scenes.c5_mixed(n_worlds=65536)
    sh, sth, ch, ih = d["hand"]
    sp, stp, cp = d["pile"]
    s1 = torch.cuda.Stream()
    cpx, chx = cf.Context(CFG), cf.Context(CFG)
    cpx.load_scene(sp, stp.n_worlds, stp)
    chx.load_scene(sh, sth.n_worlds, sth)
    tin = Inputs(*(None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
                   for a in (ih.f_ext, ih.tree_L, ih.tree_tau)))
    dcp, dch = cf.DeviceContacts.from_host(cp), cf.DeviceContacts.from_host(ch)
    torch.cuda.synchronize()
    cpx.step(dcp, None, dt=CFG.dt)
    s1.wait_stream(torch.cuda.current_stream())
    chx.step(dch, tin, dt=CFG.dt, stream=s1)
    torch.cuda.synchronize()
    for ctx, scene, st, c, inp, ws in ((cpx, sp, stp, cp, None, (0, 4095, 4096, 32767)),
                                       (chx, sh, sth, ch, ih, (0, 1023, 1024, 32767))):
        out = ctx.get_state()
        for w in ws:
            sel = np.nonzero(c.world == w)[0]
            cw = c.take(sel)
            cw.world = np.zeros(len(sel), np.int32)
            iw = None if inp is None else Inputs(None, inp.tree_L[w:w + 1], inp.tree_tau[w:w + 1])
            o = oracle.step(CFG, scene, st.world_slice(w, w + 1), cw, iw)
            gst = State(*(out[k][w:w + 1] for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")))
            compare_step(dict(state=gst), o)
        ctx.close()


# ---------------------------------------------------------------- S0 integer outputs
@pytest.mark.parametrize("seed", range(3))
def test_segmentation_bit_exact(seed):
    import paper_2603_12185_b200 as cf
    scene, st, c, inp = scenes.random_instance(800 + seed, n_worlds=37, n_bodies=3,
                                               contacts_per_world=list(np.random.default_rng(seed).integers(0, 90, 37)))
    c = scenes.shuffle_contacts(c, seed)
    g = gpu_step(CFG, scene, st, c, inp, sorted_hint=False)
    off_g, perm_g = g["ctx"].segment_info(37, c.n)
    off_o, perm_o, foff_o = oracle.segment(c, 37, CFG)
    np.testing.assert_array_equal(off_g, off_o)
    np.testing.assert_array_equal(perm_g, perm_o)
    np.testing.assert_array_equal(g["foff"], foff_o)


def test_sorted_path_offsets_bit_exact():
    scene, st, c = scenes.c4_pile(n_worlds=5, contacts_per_world=300)
    keep = np.ones(c.n, bool)
    keep[(c.world == 2)] = False                 # an empty world in the middle
    c = c.take(np.nonzero(keep)[0])
    g = gpu_step(CFG, scene, st, c, None, sorted_hint=True)
    off_g, perm_g = g["ctx"].segment_info(5, c.n)
    off_o, perm_o, _ = oracle.segment(c, 5, CFG)
    np.testing.assert_array_equal(off_g, off_o)
    np.testing.assert_array_equal(perm_g, perm_o)


# ---------------------------------------------------------------- host-buffer (e2e) path
def test_host_buffers_match_device_path():
    scene, st, c, inp = scenes.random_instance(900, n_worlds=4, n_bodies=5, contacts_per_world=33)
    o = oracle.step(CFG, scene, st, c, inp)
    g = gpu_step(CFG, scene, st, c, inp, host=True)
    compare_step(g, o)


def test_sub_range_step_leaves_other_worlds():
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=6, contacts_per_world=200)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 6, st)
    sel = np.nonzero((c.world >= 2) & (c.world < 4))[0]
    cs = c.take(sel)
    cs.world = cs.world - 2
    ctx.step(cf.DeviceContacts.from_host(cs), None, first_world=2, n_worlds=2)
    out = ctx.get_state()
    for w in (0, 1, 4, 5):
        np.testing.assert_array_equal(out["vel"][w], st.vel[w])
        np.testing.assert_array_equal(out["pos"][w], st.pos[w])
    cw = cs.take(np.arange(cs.n))
    o = oracle.step(CFG, scene, st.world_slice(2, 4), cw, None)
    gst = State(*(out[k][2:4] for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")))
    compare_step(dict(state=gst), o)


# ---------------------------------------------------------------- errors surface
def test_nonfinite_state_reported_with_world():
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=4, contacts_per_world=50)
    st.vel[2, 7, 0] = np.nan
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 4, st)
    ctx.step(cf.DeviceContacts.from_host(c), None)
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.get_state()
    assert ei.value.status == 4 and "world 2" in str(ei.value)


def test_fixed_point_range_exceeded_is_reported():
    """S6 accumulates in 64-bit fixed point (~2^28 m/s of velocity change per
    step, include/comfree.h): an impulse beyond that range is reported as
    COMFREE_ERR_NONFINITE for its world instead of wrapping silently."""
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=4, contacts_per_world=50)
    i = int(np.nonzero((c.world == 1) & (c.body_b >= 0))[0][0])
    b = int(c.body_b[i])
    st.vel[1, b] = -1e12 * c.c1[i, :3]          # approach along the normal at 1e12 m/s
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 4, st)
    ctx.step(cf.DeviceContacts.from_host(c), None)
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.get_state()
    assert ei.value.status == 4 and "world 1" in str(ei.value)


def test_invalid_body_id_and_unsorted_lie_are_validation_errors():
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=3, contacts_per_world=40)
    bad = c.take(np.arange(c.n))
    bad.body_b[5] = 10_000
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 3, st)
    ctx.step(cf.DeviceContacts.from_host(bad), None)
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.get_state()
    assert ei.value.status == 2
    sh = scenes.shuffle_contacts(c, 1)
    ctx.step(cf.DeviceContacts.from_host(sh), None, sorted_hint=True)
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.get_state()
    assert ei.value.status == 2 and "sorted" in str(ei.value)


def test_stats_match_oracle():
    import paper_2603_12185_b200 as cf
    scene, st, c, inp = scenes.random_instance(901, n_worlds=5, n_bodies=6, contacts_per_world=[10, 0, 30, 5, 60])
    g = gpu_step(CFG, scene, st, c, inp, flags=cf.FLAG_STATS)
    ws = g["ctx"].get_world_stats()
    o = oracle.step(CFG, scene, st, c, inp)
    np.testing.assert_array_equal(ws["contacts"], o["stats"][:, 0].astype(np.int32))
    assert np.all(np.abs(ws["active_facets"] - o["stats"][:, 1]) <= 2)     # fp decides near the clamp
    assert_close(ws["max_penetration"], o["stats"][:, 2], what="max_pen")
    assert_close(ws["kinetic_energy"], o["stats"][:, 3], rtol=1e-4, atol=1e-6, what="KE")


# ---------------------------------------------------------------- trajectories (100 steps)
def _traj_compare(cfg, scene, st, geo, steps=100):
    import paper_2603_12185_b200 as cf
    ctx = cf.Context(cfg)
    ctx.load_scene(scene, st.n_worlds, st)

    def gstep(s, c):
        r = gpu_step(cfg, scene, s, c, None, impulses=False, ctx=ctx)
        return r["state"], None

    def ostep(s, c):
        o = oracle.step(cfg, scene, s, c, None)
        return o["state"], None
    sg, _ = run_trajectory(gstep, geo, st, steps)
    so, _ = run_trajectory(ostep, geo, st.astype(np.float64), steps)
    traj_assert(sg, so, f"{steps}-step trajectory")


def test_trajectory_c1_sphere_and_sliding_box():
    scene, st, geo = scenes.c1_scene(box_omega=(0.1, 0.1, 0.1))
    _traj_compare(CFG, scene, st, geo)


def test_trajectory_c2a_incline():
    scene, st, geos, th = scenes.c2a_incline(np.linspace(0.1, 1.5, 8))
    _traj_compare(CFG, scene, st, geos)


def test_trajectory_c2b_stack_6d():
    scene, st, geo = scenes.c2b_stack()
    _traj_compare(CFG.with_(n_t=8, n_rol=8), scene, st, geo)


# ---------------------------------------------------------------- per-contact impedance
def _kd(c, seed, lo=0.02, hi=0.6):
    rng = np.random.default_rng(seed)
    c2 = c.take(np.arange(c.n))
    c2.kd = np.stack([rng.uniform(lo, hi, c.n), rng.uniform(0.0, 0.01, c.n)], 1).astype(np.float32)
    return c2


@pytest.mark.parametrize("seed", range(3))
def test_per_contact_impedance_random(seed):
    """Per-contact (k_user, d_user) on mixed instances,
    unsorted ids (the pairs are permuted with the contacts), chains."""
    scene, st, c, inp = scenes.random_instance(1100 + seed, n_worlds=5, n_bodies=6, contacts_per_world=[9, 0, 33, 70, 2],
                                               n_trees=2 if seed else 0)
    c = _kd(scenes.shuffle_contacts(c, seed), seed)
    compare_step(gpu_step(CFG, scene, st, c, inp), oracle.step(CFG, scene, st, c, inp))


def test_per_contact_impedance_pile_and_identity():
    """C4-shaped pile with per-contact pairs (sorted ids, fused S0); pairs equal
    to the config's globals reproduce the plain step."""
    scene, st, c = scenes.c4_pile(n_worlds=6, contacts_per_world=700)
    ck = _kd(c, 7)
    compare_step(gpu_step(CFG, scene, st, ck, None), oracle.step(CFG, scene, st, ck, None))
    cg = c.take(np.arange(c.n))
    cg.kd = np.tile(np.array([CFG.k_user, CFG.d_user], np.float32), (c.n, 1))
    a, b = gpu_step(CFG, scene, st, cg, None), gpu_step(CFG, scene, st, c, None)
    for k in ("pos", "quat", "vel", "omega"):
        np.testing.assert_allclose(getattr(a["state"], k), getattr(b["state"], k), rtol=1e-6, atol=1e-7)


def test_per_contact_impedance_invalid_is_validation_error():
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=3, contacts_per_world=40)
    ck = _kd(c, 3)
    ck.kd[17] = (-0.1, 0.0)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 3, st)
    ctx.step(cf.DeviceContacts.from_host(ck), None)
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.get_state()
    assert ei.value.status == 2 and "impedance" in str(ei.value)


# ---------------------------------------------------------------- C5 mixed
def test_c5_mixed_two_contexts_concurrent_streams():
    """Config 5: hand and pile-lite worlds as two contexts stepped concurrently
    on two CUDA streams (as bench.py --workload mixed does); each part matches
    the oracle, and the concurrent result equals stepping each part alone."""
    import torch
    import paper_2603_12185_b200 as cf
    d = scenes.c5_mixed(n_worlds=48, unique_hand=6, unique_pile=5)
    sh, sth, ch, ih = d["hand"]
    sp, stp, cp = d["pile"]
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    cp_ctx, ch_ctx = cf.Context(CFG), cf.Context(CFG)
    cp_ctx.load_scene(sp, stp.n_worlds, stp)
    ch_ctx.load_scene(sh, sth.n_worlds, sth)
    dcp, dch = cf.DeviceContacts.from_host(cp), cf.DeviceContacts.from_host(ch)
    tin = type(ih)(*(None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
                     for a in (ih.f_ext, ih.tree_L, ih.tree_tau)))
    torch.cuda.synchronize()
    cp_ctx.step(dcp, None, stream=s0)
    ch_ctx.step(dch, tin, stream=s1)
    torch.cuda.synchronize()
    gp, gh = cp_ctx.get_state(), ch_ctx.get_state()
    op, oh = oracle.step(CFG, sp, stp, cp, None), oracle.step(CFG, sh, sth, ch, ih)
    compare_step({"state": type(stp)(**{k: gp[k] for k in gp})}, op)
    compare_step({"state": type(sth)(**{k: gh[k] for k in gh})}, oh)
    alone = gpu_step(CFG, sp, stp, cp, None, impulses=False)
    for k in ("pos", "quat", "vel", "omega"):
        np.testing.assert_array_equal(gp[k], getattr(alone["state"], k))
    cp_ctx.close(); ch_ctx.close()


# ---------------------------------------------------------------- determinism
def test_step_is_bitwise_deterministic_and_shard_invariant():
    """S6 accumulates in 64-bit fixed point with integer atomics (order-free),
    so repeated runs, the DETERMINISTIC flag (now a no-op) and different world
    batchings -- which change the grid and which CTA a world lands in -- give
    bit-identical states (worlds are independent); parity as usual.
    (Within a warp, runs of equal body ids are pre-summed in fp32 in a fixed
    lane order, so results depend on the contact order and on the warps per
    world, both of which are functions of the input alone.)"""
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=6, contacts_per_world=700)
    o = oracle.step(CFG, scene, st, c, None)
    runs = [gpu_step(CFG, scene, st, c, None, flags=f) for f in (0, 0, cf.FLAG_DETERMINISTIC)]
    for r in runs[1:]:
        for k in ("pos", "quat", "vel", "omega"):
            np.testing.assert_array_equal(getattr(r["state"], k), getattr(runs[0]["state"], k))
        np.testing.assert_array_equal(r["impulses"], runs[0]["impulses"])
    compare_step(runs[0], o)
    # worlds 2..3 stepped as their own batch
    sel = np.nonzero((c.world >= 2) & (c.world < 4))[0]
    cs = c.take(sel)
    cs.world = cs.world - 2
    part = gpu_step(CFG, scene, st.world_slice(2, 4), cs, None, impulses=False)
    for k in ("pos", "quat", "vel", "omega"):
        np.testing.assert_array_equal(getattr(part["state"], k), getattr(runs[0]["state"], k)[2:4])


def test_world_alone_equals_world_in_large_batch():
    """A world stepped inside a 600-world batch (many CTAs, graph of 75
    groups) and the same world stepped alone (one CTA) agree bit for bit."""
    scene, st, c = scenes.c4_pile(n_worlds=600, contacts_per_world=900)
    full = gpu_step(CFG, scene, st, c, None, impulses=False)
    for w in (0, 311, 599):
        sel = np.nonzero(c.world == w)[0]
        cs = c.take(sel)
        cs.world = cs.world - w
        one = gpu_step(CFG, scene, st.world_slice(w, w + 1), cs, None, impulses=False)
        for k in ("pos", "quat", "vel", "omega"):
            np.testing.assert_array_equal(getattr(one["state"], k), getattr(full["state"], k)[w:w + 1])


def test_deterministic_articulated():
    scene, st, c, inp = scenes.c3_hand(n_worlds=8)
    a = gpu_step(CFG, scene, st, c, inp)
    b = gpu_step(CFG, scene, st, c, inp)
    for k in ("pos", "quat", "vel", "omega", "qpos", "qvel"):
        np.testing.assert_array_equal(getattr(a["state"], k), getattr(b["state"], k))
    compare_step(a, oracle.step(CFG, scene, st, c, inp))


# ---------------------------------------------------------------- CUDA graphs
def test_step_is_cuda_graph_capturable():
    """A step (S0 + fused kernel) captured once in a CUDA graph and replayed
    gives the same states as direct launches, bit for bit."""
    import torch
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=8, contacts_per_world=500)
    outs = []
    for graph in (False, True):
        ctx = cf.Context(CFG)
        ctx.load_scene(scene, 8, st)
        dc = cf.DeviceContacts.from_host(c)
        ctx.step(dc, None)                       # allocates scratch outside capture
        if graph:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                ctx.step(dc, None)
            for _ in range(5):
                g.replay()
        else:
            for _ in range(5):
                ctx.step(dc, None)
        torch.cuda.synchronize()
        outs.append(ctx.get_state())
        ctx.close()
    for k in ("pos", "quat", "vel", "omega"):
        np.testing.assert_array_equal(outs[0][k], outs[1][k])


def test_fused_segmentation_uneven_worlds():
    """Sorted world ids with very uneven counts (the in-kernel range search
    starts from a uniform guess and must fall back): off bit-exact and parity."""
    cpw = [0, 0, 900, 1, 0, 3, 2500, 0, 17, 0]
    scene, st, c, inp = scenes.random_instance(950, n_worlds=len(cpw), n_bodies=4, contacts_per_world=cpw)
    g = gpu_step(CFG, scene, st, c, inp, sorted_hint=True)
    off_g, _ = g["ctx"].segment_info(len(cpw), c.n)
    off_o, _, _ = oracle.segment(c, len(cpw), CFG)
    np.testing.assert_array_equal(off_g, off_o)
    compare_step(g, oracle.step(CFG, scene, st, c, inp))


# ---------------------------------------------------------------- S6 range, off[] validation
def test_fixed_point_two_overflowing_adds_and_nan_normal():
    """Every S6 add is bounded so a sum cannot wrap: two contacts pushing one
    body far beyond the range (whose saturated adds would cancel if
    unchecked) are reported for their world, and so is a NaN normal (whose
    impulse the float-to-int conversion would turn into 0)."""
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=4, contacts_per_world=50)
    idx = np.nonzero((c.world == 1) & (c.body_b >= 0))[0]
    b = int(c.body_b[idx[0]])
    two = idx[c.body_b[idx] == b][:1].tolist()
    k2 = int(np.nonzero((c.world == 1) & (c.body_a >= 0) & (c.body_a != b))[0][0])
    c.body_a[k2] = b                                   # a second contact on body b, as side a
    st.vel[1, b] = -1e13 * c.c1[two[0], :3]
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 4, st)
    ctx.step(cf.DeviceContacts.from_host(c), None)
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.get_state()
    assert ei.value.status == 4 and "world 1" in str(ei.value)
    scene, st, c = scenes.c4_pile(n_worlds=4, contacts_per_world=50)
    i = int(np.nonzero(c.world == 2)[0][3])
    c.c1[i, :3] = np.nan
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 4, st)
    ctx.step(cf.DeviceContacts.from_host(c), None)
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.get_state()
    assert ei.value.status == 4 and "world 2" in str(ei.value)


def test_presegmented_off_matches_and_is_validated():
    """The benchmark's input form: off[W+1] from the caller (S0 skipped) gives
    the same bits as sorted world ids; an inconsistent off[] is a validation
    error."""
    import torch
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=7, contacts_per_world=400)
    off = np.searchsorted(c.world, np.arange(8)).astype(np.int64)
    a = gpu_step(CFG, scene, st, c, None, impulses=False)
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 7, st)
    ctx.step(cf.DeviceContacts.from_host(c), None, off=torch.from_numpy(off).cuda())
    out = ctx.get_state()
    for k in ("pos", "quat", "vel", "omega"):
        np.testing.assert_array_equal(out[k], getattr(a["state"], k))
    bad = off.copy()
    bad[-1] -= 1
    ctx.step(cf.DeviceContacts.from_host(c), None, off=torch.from_numpy(bad).cuda())
    with pytest.raises(cf.ComfreeError) as ei:
        ctx.get_state()
    assert ei.value.status == 2 and "off[]" in str(ei.value)


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_persistent_kernel_variants_bit_identical(mode, monkeypatch):
    """The opt-in persistent step kernel (COMFREE_PERSIST=1; mode 1: 8 warps,
    next world prefetched into L2; 2 / 3: 16 / 32 warps, next world's slab
    staged into shared memory by TMA bulk copies on an mbarrier) gives the
    same bits as the default kernel (per-world arithmetic is independent of
    the CTA that runs it), across more worlds than the grid holds at once."""
    scene, st, c = scenes.c4_pile(n_worlds=700, contacts_per_world=600)
    ref = gpu_step(CFG, scene, st, c, None, impulses=False)
    monkeypatch.setenv("COMFREE_PERSIST", "1")
    monkeypatch.setenv("COMFREE_PERSIST_MODE", str(mode))
    for _ in range(2):                              # the world queue resets itself between launches
        g = gpu_step(CFG, scene, st, c, None, impulses=False)
        for k in ("pos", "quat", "vel", "omega"):
            np.testing.assert_array_equal(getattr(g["state"], k), getattr(ref["state"], k))


def test_async_host_pipeline_matches_device_path():
    """COMFREE_MEM_HOST_ASYNC (pinned host buffers, the e2e pipeline): three
    steps, each state copied out asynchronously into its own pinned buffers,
    equal the device path's per-step states bit for bit; the copies of step
    k + 1 overlap step k (two staging slots, include/comfree.h)."""
    import torch
    import paper_2603_12185_b200 as cf
    scene, st, c = scenes.c4_pile(n_worlds=9, contacts_per_world=700)
    ref = cf.Context(CFG)
    ref.load_scene(scene, 9, st)
    dc = cf.DeviceContacts.from_host(c)
    want = []
    for _ in range(3):
        ref.step(dc, None)
        want.append(ref.get_state())
    ctx = cf.Context(CFG)
    ctx.load_scene(scene, 9, st)
    hca = cf.HostContacts.from_arrays(c, pin=True, asynchronous=True, n_worlds=9)
    outs = []
    s = torch.cuda.Stream()
    for _ in range(3):
        ctx.step(hca, None, stream=s)
        o = {k: torch.empty(v.shape, dtype=torch.float32).pin_memory().numpy() for k, v in want[0].items()}
        ctx.get_state_async(o, stream=s)
        outs.append(o)
    ctx.wait_async(s)
    s.synchronize()
    ctx.check(s)
    for o, w in zip(outs, want):
        for k in ("pos", "quat", "vel", "omega"):
            np.testing.assert_array_equal(o[k], w[k])
