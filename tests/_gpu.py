"""GPU-side test helpers: run the CUDA path through the C ABI binding and
compare with the fp64 oracle on the same seeded inputs."""
from __future__ import annotations

import numpy as np

import oracle
from harness.types import Contacts, Inputs, State

# north star tolerance (BASELINE.json): per step |d| <= 1e-5 |ref| + 1e-6
RTOL, ATOL = 1e-5, 1e-6


def torch_inputs(inputs: Inputs | None):
    import torch
    if inputs is None:
        return None
    out = Inputs()
    for k in ("f_ext", "tree_L", "tree_tau"):
        a = getattr(inputs, k)
        setattr(out, k, None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda())
    return out


def gpu_step(cfg, scene, state: State, contacts: Contacts, inputs=None, flags=0, impulses=True,
             sorted_hint=None, ctx=None, host=False):
    import torch
    import paper_2603_12185_b200 as cf
    own = ctx is None
    if own:
        ctx = cf.Context(cfg, flags=flags)
        ctx.load_scene(scene, state.n_worlds, state)
    else:
        ctx.set_state(state)
    imp = foff = None
    F = 0
    if impulses:
        nf = np.array([ctx.facets_per_contact(int(c)) for c in contacts.condim], np.int64)
        F = int(nf.sum())
        if host:
            imp = np.zeros(max(F, 1), np.float32)
            foff = np.zeros(contacts.n + 1, np.int64)
        else:
            imp = torch.zeros(max(F, 1), dtype=torch.float32, device="cuda")
            foff = torch.zeros(contacts.n + 1, dtype=torch.int64, device="cuda")
    if host:
        dc = cf.HostContacts.from_arrays(contacts, pin=True)
        ctx.step(dc, inputs, dt=cfg.dt, impulses=imp, foff=foff, sorted_hint=sorted_hint)
    else:
        dc = cf.DeviceContacts.from_host(contacts)
        ctx.step(dc, torch_inputs(inputs), dt=cfg.dt, impulses=imp, foff=foff, sorted_hint=sorted_hint)
    out = ctx.get_state()
    res = dict(state=State(out["pos"], out["quat"], out["vel"], out["omega"], out["qpos"], out["qvel"]),
               ctx=ctx)
    if impulses:
        res["impulses"] = (imp if host else imp.cpu().numpy())[:F]
        res["foff"] = foff if host else foff.cpu().numpy()
    return res


def assert_close(got, ref, rtol=RTOL, atol=ATOL, what=""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    err = np.abs(got - ref)
    lim = atol + rtol * np.abs(ref)
    bad = err > lim
    if np.any(bad):
        i = np.argmax(err - lim)
        raise AssertionError(f"{what}: {bad.sum()}/{bad.size} elements exceed |d| <= {rtol}|ref| + {atol}; "
                             f"worst flat index {i}: got {got.flat[i]!r} ref {ref.flat[i]!r} |d| {err.flat[i]:.3g}")


def compare_step(g, o, pos_tol=1e-6, quat_tol=2e-6):
    gs, os_ = g["state"], o["state"]
    assert_close(gs.vel, os_.vel, what="v+")
    assert_close(gs.omega, os_.omega, what="omega+")
    assert_close(gs.qvel, os_.qvel, what="qd+")
    assert_close(gs.pos, os_.pos, rtol=pos_tol, atol=pos_tol, what="x+")
    assert_close(gs.qpos, os_.qpos, rtol=pos_tol, atol=pos_tol, what="q_chain+")
    assert_close(gs.quat, os_.quat, rtol=0, atol=quat_tol, what="quat+")
    if "impulses" in g and "impulses" in o:
        np.testing.assert_array_equal(g["foff"], o["foff"])
        assert_close(g["impulses"], o["impulses"], what="Lambda")


# Trajectories: per element, |d| <= 1e-3 |ref| + atol (north star: 1e-3
# relative over 100-step trajectories).  The absolute floors (DESIGN.md,
# "Trajectory tolerance") are 100 x the per-step floor of 1e-6 for velocities
# (m/s, rad/s): 1e-4; its time integral over a 0.2 s trajectory for positions:
# 2e-5 m (chain joint angles: 2e-5 rad); and for the unit quaternion the same
# 2e-5 rad of rotation (|dq| <= |d theta| / 2).
TRAJ_RTOL = 1e-3
TRAJ_ATOL = dict(pos=2e-5, quat=2e-5, vel=1e-4, omega=1e-4, qpos=2e-5, qvel=1e-4)


def traj_assert(sg, so, what="", keys=None):
    """sg / so: State-like objects or dicts of arrays."""
    get = (lambda o, k: o[k]) if isinstance(sg, dict) else getattr
    geto = (lambda o, k: o[k]) if isinstance(so, dict) else getattr
    for k, atol in TRAJ_ATOL.items():
        if keys is not None and k not in keys:
            continue
        a, b = np.asarray(get(sg, k), np.float64), np.asarray(geto(so, k), np.float64)
        if k == "quat":                               # q and -q are the same rotation
            sgn = np.sign(np.sum(a * b, axis=-1, keepdims=True))
            a = a * np.where(sgn == 0, 1.0, sgn)
        assert_close(a, b, rtol=TRAJ_RTOL, atol=atol, what=f"{what} {k}")
