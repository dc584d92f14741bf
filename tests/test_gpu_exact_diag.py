"""GPU parity of the exact-diagonal impedance variant (Eq. (11), reading R24,
COMFREE_FLAG_EXACT_DIAGONAL) with the fp64 oracle, at the north-star tolerance
(|d| <= 1e-5 |ref| + 1e-6 per step on velocities and facet impulses)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from harness import scenes
from harness.types import Config
from _gpu import compare_step, gpu_step

pytestmark = pytest.mark.gpu

EX = Config(impedance="exact_diagonal")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_12185_b200 as cf
    cf._lib.load()


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("cfg", [EX, EX.with_(n_t=8, n_rol=6), EX.with_(n_t=6, n_rol=2, power=3.0)],
                         ids=["nt4", "nt8", "nt6p3"])
def test_exact_random_mixed_step(seed, cfg):
    """Every condim, free/static sides, ragged worlds (incl. empty), unsorted ids."""
    cpw = [0, 3, 40, 257, 1, 70][seed % 6:] + [0, 3, 40, 257, 1, 70][:seed % 6]
    scene, st, c, inp = scenes.random_instance(1500 + seed, n_worlds=6, n_bodies=9, contacts_per_world=cpw)
    c = scenes.shuffle_contacts(c, seed)
    compare_step(gpu_step(cfg, scene, st, c, inp), oracle.step(cfg, scene, st, c, inp))


@pytest.mark.parametrize("seed", range(3))
def test_exact_articulated_step(seed):
    nd = [4, 3, 2][seed]
    scene, st, c, inp = scenes.random_instance(1600 + seed, n_worlds=5, n_bodies=3,
                                               contacts_per_world=[30, 0, 7, 64, 33], n_trees=4, tree_ndof=nd)
    compare_step(gpu_step(EX, scene, st, c, inp), oracle.step(EX, scene, st, c, inp))


def test_exact_pile_and_hand():
    """C4-shaped pile (8 worlds x 2000 contacts) and the C3 hand (64 worlds)."""
    scene, st, c = scenes.c4_pile(n_worlds=8, contacts_per_world=2000)
    compare_step(gpu_step(EX, scene, st, c, None), oracle.step(EX, scene, st, c, None))
    scene, st, c, inp = scenes.c3_hand(n_worlds=64)
    compare_step(gpu_step(EX, scene, st, c, inp), oracle.step(EX, scene, st, c, inp))


def test_exact_differs_from_heuristic_on_gpu():
    scene, st, c, inp = scenes.random_instance(1700, n_worlds=2, n_bodies=4, contacts_per_world=[6, 9])
    a = gpu_step(EX, scene, st, c, inp)["impulses"]
    b = gpu_step(EX.with_(impedance="heuristic"), scene, st, c, inp)["impulses"]
    assert np.max(np.abs(a - b)) > 1e-3 * np.max(np.abs(b))


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
        o = oracle.step(EX, scene, st.world_slice(w, w + 1), cw, None)
        gst = State(*(out[k][w:w + 1] for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")))
        compare_step(dict(state=gst), o)
