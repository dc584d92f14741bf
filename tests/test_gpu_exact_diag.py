"""GPU parity of the per-facet impedance variants with the fp64 oracle, at the
north-star tolerance (|d| <= 1e-5 |ref| + 1e-6 per step on velocities and facet
impulses): Eq. (11) literally (reading R24, COMFREE_FLAG_EXACT_DIAGONAL,
Lambda_f = (-k phi - kappa s_f)_+ / (kappa A_f)) and Eq. (12) with the facet
diagonal (reading R28, COMFREE_FLAG_FACET_DIAGONAL)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from harness import scenes
from harness.types import Config
from _gpu import compare_step, gpu_step, operand_scale

pytestmark = pytest.mark.gpu

EX = Config(impedance="exact_diagonal")
FD = Config(impedance="facet_diagonal")
MODES = pytest.mark.parametrize("mode", ["exact_diagonal", "facet_diagonal"], ids=["eq11", "facet_diag"])


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_12185_b200 as cf
    cf._lib.load()


@MODES
@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("cfg", [EX, EX.with_(n_t=8, n_rol=6), EX.with_(n_t=6, n_rol=2, power=3.0)],
                         ids=["nt4", "nt8", "nt6p3"])
def test_exact_random_mixed_step(seed, cfg, mode):
    """Every condim, free/static sides, ragged worlds (incl. empty), unsorted ids."""
    cfg = cfg.with_(impedance=mode)
    cpw = [0, 3, 40, 257, 1, 70][seed % 6:] + [0, 3, 40, 257, 1, 70][:seed % 6]
    scene, st, c, inp = scenes.random_instance(1500 + seed, n_worlds=6, n_bodies=9, contacts_per_world=cpw)
    c = scenes.shuffle_contacts(c, seed)
    # Eq. (11) sizes every facet to cancel its own velocity alone, so a contact's
    # facets sum to far more than the net change: velocities by reading R30
    compare_step(gpu_step(cfg, scene, st, c, inp), oracle.step(cfg, scene, st, c, inp),
                 scale=operand_scale(cfg, scene, st, c, inp))


@MODES
@pytest.mark.parametrize("seed", range(3))
def test_exact_articulated_step(seed, mode):
    nd = [4, 3, 2][seed]
    cfg = EX.with_(impedance=mode)
    scene, st, c, inp = scenes.random_instance(1600 + seed, n_worlds=5, n_bodies=3,
                                               contacts_per_world=[30, 0, 7, 64, 33], n_trees=4, tree_ndof=nd)
    compare_step(gpu_step(cfg, scene, st, c, inp), oracle.step(cfg, scene, st, c, inp),
                 scale=operand_scale(cfg, scene, st, c, inp))


@MODES
def test_exact_pile_and_hand(mode):
    """C4-shaped pile (8 worlds x 2000 contacts) and the C3 hand (64 worlds)."""
    cfg = EX.with_(impedance=mode)
    scene, st, c = scenes.c4_pile(n_worlds=8, contacts_per_world=2000)
    compare_step(gpu_step(cfg, scene, st, c, None), oracle.step(cfg, scene, st, c, None),
                 scale=operand_scale(cfg, scene, st, c, None))
    scene, st, c, inp = scenes.c3_hand(n_worlds=64)
    compare_step(gpu_step(cfg, scene, st, c, inp), oracle.step(cfg, scene, st, c, inp),
                 scale=operand_scale(cfg, scene, st, c, inp))


@MODES
def test_exact_differs_from_heuristic_on_gpu(mode):
    scene, st, c, inp = scenes.random_instance(1700, n_worlds=2, n_bodies=4, contacts_per_world=[6, 9])
    a = gpu_step(EX.with_(impedance=mode), scene, st, c, inp)["impulses"]
    b = gpu_step(EX.with_(impedance="heuristic"), scene, st, c, inp)["impulses"]
    assert np.max(np.abs(a - b)) > 1e-3 * np.max(np.abs(b))


def test_eq11_single_facet_target_on_gpu():
    """Two point masses, one normal facet, no gravity: the GPU step drives the
    facet velocity to -(k dt/kappa) phi/dt (Eq. (9)-(11) closed form)."""
    from harness.types import Contacts, Scene
    scene = Scene(inv_mass=np.array([2.0, 0.5], np.float32), inv_inertia=np.zeros((2, 3), np.float32))
    st = scenes.empty_state(1, 2)
    st.pos[0, 1] = (0, 0, 0.1)
    st.vel[0, 1] = (0, 0, -0.3)
    phi = -0.0003
    c = Contacts(world=np.array([0], np.int32), c0=np.array([[0, 0, 0.05, phi]], np.float32),
                 c1=np.array([[0, 0, 1, 0.0]], np.float32), c2=np.array([[1, 0, 0, 0.0]], np.float32),
                 body_a=np.array([0], np.int32), body_b=np.array([1], np.int32),
                 mu_rol=np.zeros(1, np.float32), condim=np.array([1], np.int32))
    cfg = EX.with_(gravity=(0.0, 0.0, 0.0))
    g = gpu_step(cfg, scene, st, c, None)
    kappa = cfg.k_user * cfg.dt + cfg.d_user
    target = -(cfg.k_user / kappa) * np.float32(phi)
    un = float(g["state"].vel[0, 1, 2]) - float(g["state"].vel[0, 0, 2])
    assert abs(un - target) <= 1e-5 * abs(target) + 1e-6, (un, target)


@MODES
def test_exact_per_contact_impedance(mode):
    """Per-contact (k, d) pairs with the per-facet variants; a pair with
    k dt + d = 0 is a validation error under Eq. (11) (its split is undefined)."""
    import paper_2603_12185_b200 as cf
    cfg = EX.with_(impedance=mode)
    scene, st, c, inp = scenes.random_instance(1750, n_worlds=4, n_bodies=5, contacts_per_world=[9, 30, 0, 12])
    rng = np.random.default_rng(5)
    c.kd = np.stack([rng.uniform(0.02, 0.6, c.n), rng.uniform(0.0, 0.01, c.n)], 1).astype(np.float32)
    compare_step(gpu_step(cfg, scene, st, c, inp), oracle.step(cfg, scene, st, c, inp),
                 scale=operand_scale(cfg, scene, st, c, inp))
    if mode == "exact_diagonal":
        c.kd[3] = (0.0, 0.0)
        ctx = cf.Context(cfg)
        ctx.load_scene(scene, 4, st)
        ctx.step(cf.DeviceContacts.from_host(c), None)
        with pytest.raises(cf.ComfreeError) as ei:
            ctx.get_state()
        assert ei.value.status == 2 and "impedance" in str(ei.value)


def test_exact_c4_full_size_sampled_worlds():
    """The exact-diagonal variant at BASELINE config-4 size (1024 worlds x 500
    bodies x 2000 contacts, the bench's --impedance exact_diagonal launch);
    sampled worlds against the oracle one by one."""
    import paper_2603_12185_b200 as cf
    from harness.types import State
    scene, st, c = scenes.c4_pile(n_worlds=1024, contacts_per_world=2000)
    ctx = cf.Context(EX)
    ctx.load_scene(scene, 1024, st)
    ctx.step(cf.DeviceContacts.from_host(c), None, dt=EX.dt)
    out = ctx.get_state()
    for w in (0, 333, 1023):
        sel = np.nonzero(c.world == w)[0]
        cw = c.take(sel)
        cw.world = np.zeros(len(sel), np.int32)
        sw = st.world_slice(w, w + 1)
        o = oracle.step(EX, scene, sw, cw, None)
        gst = State(*(out[k][w:w + 1] for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")))
        compare_step(dict(state=gst), o, scale=operand_scale(EX, scene, sw, cw, None))
