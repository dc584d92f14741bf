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


def operand_scale(cfg, scene, st, c, inputs=None):
    """Magnitude of the operands of Eq. (10) per velocity element (DESIGN.md
    reading R30): |v_s| + sum_f |M^-1 J~_f^T Lambda_f| over every facet f,
    with the oracle's Lambda_f, the dense oracle B's Jacobians and facet rows
    (oracle/dense.py) and M^-1 per body / chain block (M is block diagonal).
    Returns dict(vel, omega, qvel) shaped like the state arrays."""
    import oracle as orc
    from oracle import dense
    W, B, T, nd = st.n_worlds, scene.n_bodies, scene.n_trees, scene.tree_ndof
    o = orc.step(cfg, scene, st, c, inputs)
    foff = o["foff"]
    out = dict(vel=np.zeros((W, B, 3)), omega=np.zeros((W, B, 3)), qvel=np.zeros((W, T * nd)))
    inputs = inputs or Inputs()
    for w in range(W):
        M, h, v = dense.world_system(cfg, scene, st, w, inputs) if B * 6 + T * nd <= 600 else (None, None, None)
        sc = np.zeros(6 * B + T * nd)
        minv = {}

        def block(side):                     # (columns, M^-1 block) of one side
            if side in minv:
                return minv[side]
            if side >= 0:
                q = np.asarray(st.quat[w, side], float)
                R = dense._quat_R(q)
                Iinv = R @ np.diag(np.asarray(scene.inv_inertia[side], float)) @ R.T
                blk = np.zeros((6, 6))
                blk[:3, :3] = float(scene.inv_mass[side]) * np.eye(3)
                blk[3:, 3:] = Iinv
                cols = np.arange(6 * side, 6 * side + 6)
            else:
                t = -2 - side
                L = dense._unpack_L(np.asarray(inputs.tree_L[w, t], float), nd)
                blk = np.linalg.inv(L @ L.T)
                cols = np.arange(6 * B + t * nd, 6 * B + (t + 1) * nd)
            minv[side] = (cols, blk)
            return minv[side]
        # |v_s|: v + M^-1 (tau - c) dt per block
        if M is None:
            M, h, v = dense.world_system(cfg, scene, st, w, inputs)
        for side in list(range(B)) + [-2 - t for t in range(T)]:
            cols, blk = block(side)
            sc[cols] += np.abs(v[cols] + blk @ h[cols] * cfg.dt)
        for k in np.nonzero(np.asarray(c.world) == w)[0]:
            p = np.asarray(c.c0[k, :3], float)
            jr = None if c.jrow is None else c.jrow[k]
            sides = [int(c.body_a[k]), int(c.body_b[k])]
            Jc = dense.side_jacobian(scene, st, w, sides[1], p, None if jr is None else jr[1]) - \
                dense.side_jacobian(scene, st, w, sides[0], p, None if jr is None else jr[0])
            rows = dense.facet_rows(cfg, np.asarray(c.c1[k, :3], float), np.asarray(c.c2[k, :3], float),
                                    float(c.c1[k, 3]), float(c.c2[k, 3]), float(c.mu_rol[k]), int(c.condim[k]), Jc)
            lam = o["impulses"][foff[k]:foff[k] + len(rows)]
            for side in sides:
                if side == -1:
                    continue
                cols, blk = block(side)
                for row, L_f in zip(rows, lam):
                    sc[cols] += np.abs(blk @ (row[cols] * L_f))
        body = sc[:6 * B].reshape(B, 6)
        out["vel"][w], out["omega"][w] = body[:, :3], body[:, 3:]
        out["qvel"][w] = sc[6 * B:]
    return out


def compare_step(g, o, pos_tol=1e-6, quat_tol=2e-6, scale=None):
    """Per-step parity.  With `scale` (operand_scale) the velocity bound is
    taken relative to max(|ref|, operand magnitude) -- reading R30, for steps
    whose contact terms nearly cancel; otherwise the plain north-star bound."""
    gs, os_ = g["state"], o["state"]
    for k, what in (("vel", "v+"), ("omega", "omega+"), ("qvel", "qd+")):
        a, b = getattr(gs, k), getattr(os_, k)
        if scale is not None:
            # |d| <= 1e-5 max(|ref|, S) + 1e-6  <=>  compare against a reference whose magnitude is max(|ref|, S)
            lim = ATOL + RTOL * np.maximum(np.abs(b), scale[k])
            err = np.abs(np.asarray(a, np.float64) - b)
            assert np.all(err <= lim), (what, int(np.sum(err > lim)), float(np.max(err - lim)))
        else:
            assert_close(a, b, what=what)
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
