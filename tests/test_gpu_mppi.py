"""GPU parity of MPPI on the batched step (reading R27)
with the fp64 oracle (oracle/mppi.py): sampling (counter-based noise),
incremental position control, Eq. (15) costs, the weighted update, and the
rollout costs J of a whole control step (collision -> upstream -> step for H
steps) against the same rollouts in the oracle."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import articulation as ar
from oracle import collision as co
from oracle import mppi as om
from harness import scenes
from harness.types import Config, Inputs, State
from _gpu import assert_close

pytestmark = pytest.mark.gpu

CFG = Config(dt=0.004)                 # the MPC's dt
ART = scenes.hand_articulation()
GEO = scenes.hand_geometry(margin=0.003)


def _task(P):
    rng = np.random.default_rng(5)
    tq = rng.normal(size=(P, 4))
    tq /= np.linalg.norm(tq, axis=1, keepdims=True)
    return dict(object_body=0, target_pos=rng.uniform([0.0, -0.01, 0.04], [0.03, 0.01, 0.06], (P, 3)),
                target_quat=tq, q_ref=np.tile([0.0, 0.6, 0.6, 0.6], 4), w=[1.0, 5.0, 5.0, 5.0, 2.0, 0.05],
                omega_fallen=10.0, z_fallen=0.03, phi1=50.0, phi2=2.0)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_12185_b200 as cf
    cf._lib.load()


def _mppi(P, N, H, **kw):
    from paper_2603_12185_b200.mppi import MPPI, MppiConfig
    scene, st, _, _ = scenes.c3_hand(n_worlds=P)
    mc = MppiConfig(n_problems=P, n_samples=N, horizon=H, task=_task(P), **kw)
    return MPPI(CFG, scene, ART, GEO, mc), scene, st


def test_sample_control_update_match_oracle():
    import torch
    m, scene, st = _mppi(3, 16, 5)
    rng = np.random.default_rng(1)
    m.plan.copy_(torch.as_tensor(rng.uniform(-0.08, 0.08, tuple(m.plan.shape)), dtype=torch.float32))
    m.iteration = 7
    m.rollout_costs(st, np.zeros((3, 16)))            # samples U (and runs the rollouts)
    U = m.U.cpu().numpy()
    eps = om.noise(m.mc.seed, 7, 3, 16, 5, 16, m.mc.sigma)
    assert_close(U, om.samples(m.plan.cpu().numpy().astype(np.float64), eps, -0.1, 0.1), rtol=0, atol=2e-6,
                 what="samples")
    J = rng.uniform(0, 0.05, 3 * 16).astype(np.float32)
    m.J.copy_(torch.as_tensor(J))
    m.update()
    plan, w = om.update(J.reshape(3, 16).astype(np.float64), U.astype(np.float64), m.mc.lam, -0.1, 0.1)
    assert_close(m.weights.cpu().numpy(), w, rtol=1e-4, atol=1e-7, what="weights")
    assert_close(m.plan.cpu().numpy(), plan, rtol=1e-4, atol=1e-7, what="plan")


def _oracle_J(m, scene, st, command, U, task, p, i, H):
    """The oracle rolling out sample i of problem p (the GPU-drawn U) through
    collision, upstream and step for H steps; returns J (Eq. (14))."""
    s = State(*(np.asarray(getattr(st, k)[p:p + 1], np.float64)
                for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")))
    cmd = command[p].astype(np.float64).copy()
    Jr = 0.0

    def c_of(s, terminal):
        tips = [ar.fk(ART, t, s.qpos[0, 4 * t:4 * t + 4])[3] for t in range(4)]
        return om.cost(task, s.pos[0, 0], s.quat[0, 0], tips, s.qpos[0], p, terminal)
    for t in range(H):
        Jr += c_of(s, False)
        cmd = cmd + U[p, i, t]
        tau_ext = om.pd_torque(cmd, s.qpos[0], s.qvel[0], m.mc.kp, m.mc.kd)[None]
        c = co.collide(GEO, s, ART)
        Jrow = np.zeros((c.n, 2, 6, 4))
        for k in range(c.n):
            for side, bid in enumerate((int(c.body_a[k]), int(c.body_b[k]))):
                if bid < -1:
                    tt = -2 - bid
                    Jrow[k, side] = ar.point_rows(ART, tt, s.qpos[0, 4 * tt:4 * tt + 4],
                                                  int(c.meta["link"][k, side]), c.c0[k, :3])
        c.jrow = Jrow
        L, tau = ar.upstream(ART, s.qpos, s.qvel, CFG.gravity, tau_ext)
        s = oracle.step(CFG, scene, s, c, Inputs(None, L, tau))["state"]
    return Jr + c_of(s, True)


def test_rollout_costs_match_oracle():
    """P=2 problems x N=4 samples x H=3 steps: J of every sample vs the oracle
    rolling out the same (GPU-drawn) samples through collision, upstream, step."""
    P, N, H = 2, 4, 3
    m, scene, st = _mppi(P, N, H)
    command = np.tile([0.0, 0.5, 0.5, 0.5], (P, 4))
    J = m.rollout_costs(st, command).cpu().numpy()
    U = m.U.cpu().numpy().astype(np.float64)
    task = _task(P)
    for p in range(P):
        for i in range(N):
            Jr = _oracle_J(m, scene, st, command, U, task, p, i, H)
            assert J[p * N + i] == pytest.approx(Jr, rel=2e-4, abs=1e-6), (p, i)


def test_rollout_costs_bench_shape_sampled():
    """The benchmarked shape (P = 16 problems x N = 256 samples x H = 48, the
    rollout as one CUDA-graph replay, as tools/mppi_bench.py times it):
    sampled rollouts' J against the oracle's 48-step rollouts of the same
    samples, and the weighted update of the whole batch against the oracle's.
    Tolerance: J sums 49 costs of states that went through 48 fp32 steps
    (per-step parity 1e-5 relative), so 1e-3 relative."""
    P, N, H = 16, 256, 48
    m, scene, st = _mppi(P, N, H)
    command = np.tile([0.0, 0.5, 0.5, 0.5], (P, 4))
    J = m.rollout_costs(st, command).cpu().numpy()
    U = m.U.cpu().numpy().astype(np.float64)
    task = _task(P)
    for p, i in ((0, 0), (3, 77), (9, 128), (15, 255)):
        Jr = _oracle_J(m, scene, st, command, U, task, p, i, H)
        assert J[p * N + i] == pytest.approx(Jr, rel=1e-3, abs=1e-5), (p, i, J[p * N + i], Jr)
    plan0 = m.plan.cpu().numpy().astype(np.float64)
    m.update()
    plan, w = om.update(J.reshape(P, N).astype(np.float64), U, m.mc.lam, -0.1, 0.1, plan_prev=plan0)
    assert_close(m.weights.cpu().numpy(), w, rtol=1e-4, atol=1e-7, what="weights")
    assert_close(m.plan.cpu().numpy(), plan, rtol=1e-4, atol=1e-7, what="plan")


def test_update_non_finite_costs():
    """Reading R29 on the GPU: NaN / inf costs get weight 0; a problem whose
    costs are all non-finite keeps its plan."""
    import torch
    m, scene, st = _mppi(3, 16, 5)
    rng = np.random.default_rng(2)
    m.plan.copy_(torch.as_tensor(rng.uniform(-0.08, 0.08, tuple(m.plan.shape)), dtype=torch.float32))
    m.rollout_costs(st, np.zeros((3, 16)))
    U = m.U.cpu().numpy().astype(np.float64)
    plan0 = m.plan.cpu().numpy().astype(np.float64)
    J = rng.uniform(0, 0.05, (3, 16)).astype(np.float32)
    J[0, 5] = np.nan
    J[1, 0] = np.inf
    J[2, :] = np.nan
    m.J.copy_(torch.as_tensor(J.reshape(-1)))
    m.update()
    plan, w = om.update(J.astype(np.float64), U, m.mc.lam, -0.1, 0.1, plan_prev=plan0)
    gw = m.weights.cpu().numpy()
    assert np.all(np.isfinite(gw)) and gw[0, 5] == 0.0 and gw[1, 0] == 0.0 and np.all(gw[2] == 0.0)
    assert_close(gw, w, rtol=1e-4, atol=1e-7, what="weights")
    assert_close(m.plan.cpu().numpy(), plan, rtol=1e-4, atol=1e-7, what="plan")
    np.testing.assert_array_equal(m.plan.cpu().numpy()[2], plan0[2].astype(np.float32))


def test_control_step_shifts_plan_and_is_reproducible():
    m1, _, st = _mppi(2, 8, 4)
    m2, _, _ = _mppi(2, 8, 4)
    u1 = m1.control_step(st, np.zeros((2, 16)))
    u2 = m2.control_step(st, np.zeros((2, 16)))
    np.testing.assert_array_equal(u1, u2)                 # counter-based noise, deterministic step
    assert np.all(np.abs(u1) <= 0.1 + 1e-7)
    assert np.all(m1.plan[:, -1].cpu().numpy() == 0.0)


def test_update_shift_and_state_broadcast():
    """comfree_mppi_update_shift: u0 = the new plan's first action and the plan
    advanced by one step (last step 0), against the oracle's update; a problem
    whose costs all diverged keeps its plan, advanced the same way.
    comfree_set_state_broadcast: the P live states replicated to the N rollout
    worlds of each problem on the device equal a host-side repeat."""
    import torch
    import paper_2603_12185_b200 as cf
    from paper_2603_12185_b200 import _lib
    m, scene, st = _mppi(3, 16, 5)
    rng = np.random.default_rng(4)
    m.plan.copy_(torch.as_tensor(rng.uniform(-0.08, 0.08, tuple(m.plan.shape)), dtype=torch.float32))
    m.rollout_costs(st, np.zeros((3, 16)))
    U = m.U.cpu().numpy().astype(np.float64)
    plan0 = m.plan.cpu().numpy().astype(np.float64)
    J = rng.uniform(0, 0.05, (3, 16)).astype(np.float32)
    J[2, :] = np.inf
    m.J.copy_(torch.as_tensor(J.reshape(-1)))
    u0 = torch.zeros((3, 16), device="cuda")
    m._chk(m._lib.comfree_mppi_update_shift(m.ctx.h, 3, 16, 5, cf._ptr(m.J), cf._ptr(m.U), m.mc.lam, -0.1, 0.1,
                                            cf._ptr(m.plan), cf._ptr(m.weights), cf._ptr(u0), None), "shift")
    plan, w = om.update(J.astype(np.float64), U, m.mc.lam, -0.1, 0.1, plan_prev=plan0)
    assert_close(u0.cpu().numpy(), plan[:, 0], rtol=1e-4, atol=1e-7, what="u0")
    g = m.plan.cpu().numpy()
    assert_close(g[:, :-1], plan[:, 1:], rtol=1e-4, atol=1e-7, what="shifted plan")
    assert np.all(g[:, -1] == 0.0)
    # broadcast of 3 live states to 3 x 16 rollout worlds
    live = State(*(np.asarray(getattr(st, k), np.float32) for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")))
    live.vel[:] = rng.normal(size=live.vel.shape).astype(np.float32)
    m.ctx.set_state_broadcast(live, 16)
    got = m.ctx.get_state()
    for k in ("pos", "quat", "vel", "omega", "qpos", "qvel"):
        np.testing.assert_array_equal(got[k], np.repeat(getattr(live, k), 16, axis=0))
