"""Host-side workload plumbing (no GPU): C5 tiling keeps world grouping and
copies every world's bytes exactly; C5 splits the batch half / half."""
import numpy as np

from harness import scenes


def test_tile_worlds_copies_and_regroups():
    scene, st, c, inp = scenes.c3_hand(n_worlds=3)
    st2, c2, inp2 = scenes.tile_worlds(st, c, inp, 8)
    assert st2.n_worlds == 8 and np.all(np.diff(c2.world) >= 0)
    assert np.array_equal(np.bincount(c2.world, minlength=8), np.bincount(c.world, minlength=3)[np.arange(8) % 3])
    for w in range(8):
        s = w % 3
        for k in ("pos", "quat", "vel", "omega", "qpos", "qvel"):
            assert np.array_equal(getattr(st2, k)[w], getattr(st, k)[s])
        a, b = c2.take(np.nonzero(c2.world == w)[0]), c.take(np.nonzero(c.world == s)[0])
        for k in ("c0", "c1", "c2", "body_a", "body_b", "mu_rol", "condim", "jrow"):
            assert np.array_equal(getattr(a, k), getattr(b, k))
        assert np.array_equal(inp2.tree_L[w], inp.tree_L[s]) and np.array_equal(inp2.tree_tau[w], inp.tree_tau[s])


def test_c5_mixed_split_and_shapes():
    d = scenes.c5_mixed(n_worlds=21, unique_hand=4, unique_pile=3)
    sh, sth, ch, ih = d["hand"]
    sp, stp, cp = d["pile"]
    assert sth.n_worlds == 10 and stp.n_worlds == 11
    assert sp.n_bodies == 100 and cp.n == 11 * 400
    assert sh.n_trees == 4 and ch.n == 10 * 20
    # world w is a copy of unique world w mod U
    assert np.array_equal(stp.pos[5], stp.pos[2]) and not np.array_equal(stp.pos[0], stp.pos[1])
