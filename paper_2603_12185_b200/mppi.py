"""MPPI on the batched step (§V, Eq. (14)-(15),
P:490-512; reading R27) — thin orchestration of C-ABI calls: every
arithmetic step (sampling, control, collision, articulated upstream, contact
resolution, costs, the weighted update) runs in libcomfree.so kernels.

One control step for P problems x N samples x horizon H (the H-step rollout
is captured once in a CUDA graph and replayed; the collision keeps its
contact count on the device, so nothing in it waits on the host):
  broadcast the live states to the P*N rollout worlds (comfree_set_state),
  U = clip(plan + eps)                                  comfree_mppi_sample
  for t < H:  J += c(x_t); command += u_t, tau = PD   comfree_mppi_cost_control (one launch)
              contacts, J rows, L, tau - c              comfree_collide / comfree_articulation_update
              x_{t+1}                                   comfree_step
  J += V(x_H); plan = clip(sum_i w_i U_i)              comfree_mppi_cost / comfree_mppi_update
then u_0 is returned and the plan is shifted (receding horizon).
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from . import Context, _ptr, _stream_handle


@dataclass
class MppiConfig:
    n_problems: int = 16
    n_samples: int = 256           # N
    horizon: int = 48              # H
    sigma: float = 0.02            # sampling standard deviation
    lam: float = 2e-3              # temperature lambda
    u_min: float = -0.1            # action clip
    u_max: float = 0.1
    kp: float = 0.5                # joint PD of the incremental position control (R27)
    kd: float = 0.005
    seed: int = 260312185
    contacts_per_world: int = 40   # collision output capacity per rollout world
    task: dict = field(default_factory=dict)


class MPPI:
    """Rollout context of P*N worlds plus the MPPI buffers (device)."""

    def __init__(self, cfg, scene, articulation, geometry, mc: MppiConfig, device: int = 0, use_graph: bool = True):
        import torch
        self.torch = torch
        self.mc = mc
        P, N, H = mc.n_problems, mc.n_samples, mc.horizon
        self.W = P * N
        self.Q = scene.n_tree_dofs
        self.ctx = Context(cfg, device=device)
        self.dt = cfg.dt
        self.ctx.load_scene(scene, self.W, None)
        self.ctx.load_articulation(articulation)
        self.ctx.load_geometry(geometry)
        dev = torch.device("cuda", device)
        f = dict(device=dev, dtype=torch.float32)
        self.plan = torch.zeros((P, H, self.Q), **f)
        self.U = torch.zeros((P, N, H, self.Q), **f)
        self.J = torch.zeros(self.W, **f)
        self.weights = torch.zeros((P, N), **f)
        self.command = torch.zeros((self.W, self.Q), **f)
        self.tau = torch.zeros((self.W, self.Q), **f)
        self.tL = torch.zeros((self.W, scene.n_trees, 10), **f)
        self.tt = torch.zeros((self.W, self.Q), **f)
        t = mc.task
        self._tp = torch.as_tensor(np.asarray(t["target_pos"], np.float32), device=dev)
        self._tq = torch.as_tensor(np.asarray(t["target_quat"], np.float32), device=dev)
        self._qr = torch.as_tensor(np.asarray(t["q_ref"], np.float32), device=dev)
        self.task_c = _lib.comfree_mppi_task(int(t.get("object_body", 0)), _ptr(self._tp), _ptr(self._tq),
                                             _ptr(self._qr), (ct.c_float * 6)(*[float(x) for x in t["w"]]),
                                             float(t["omega_fallen"]), float(t["z_fallen"]),
                                             float(t["phi1"]), float(t["phi2"]))
        self.iteration = 0
        self._lib = _lib.load()
        self.use_graph = use_graph
        self.graph = None

    def _chk(self, st, what):
        self.ctx._check(st, what)

    def _prepare(self, live_state, command, stream=None):
        """Broadcast the live states / commands to the rollout worlds, zero J, sample U."""
        from harness.types import State
        torch = self.torch
        mc, P, N, H = self.mc, self.mc.n_problems, self.mc.n_samples, self.mc.horizon
        # the P live states go up once; the device replicates them to the N
        # rollout worlds of each problem (comfree_set_state_broadcast)
        self.ctx.set_state_broadcast(live_state, N, stream=stream)
        self.command.copy_(torch.as_tensor(np.repeat(np.asarray(command, np.float32), N, axis=0),
                                           device=self.command.device))
        self.J.zero_()
        self._chk(self._lib.comfree_mppi_sample(self.ctx.h, P, N, H, _ptr(self.plan), mc.sigma, mc.u_min, mc.u_max,
                                                mc.seed, self.iteration, _ptr(self.U), _stream_handle(stream)),
                  "comfree_mppi_sample")

    def _rollout(self, stream=None):
        """H steps of (cost, control, collide, upstream, step), the terminal
        cost: launches only (device-side contact counts), CUDA-graph capturable."""
        from harness.types import Inputs
        mc, N, H = self.mc, self.mc.n_samples, self.mc.horizon
        s = _stream_handle(stream)
        for t in range(H):
            self._chk(self._lib.comfree_mppi_cost_control(self.ctx.h, 0, self.W, N, ct.byref(self.task_c),
                                                          _ptr(self.J), _ptr(self.U), t, H, mc.kp, mc.kd,
                                                          _ptr(self.command), _ptr(self.tau), s),
                      "comfree_mppi_cost_control")
            dc, link = self.ctx.collide(capacity=self.W * mc.contacts_per_world, stream=stream, device_count=True)
            self.ctx.articulation_update(self.tL, self.tt, dc, link, tau_ext=self.tau, stream=stream)
            self.ctx.step(dc, Inputs(None, self.tL, self.tt), dt=self.dt, stream=stream)
        self._chk(self._lib.comfree_mppi_cost(self.ctx.h, 0, self.W, N, ct.byref(self.task_c), 1, _ptr(self.J), s),
                  "comfree_mppi_cost")

    def rollout_costs(self, live_state, command, stream=None):
        """Broadcast, sample, roll out H steps; returns J (P*N) on the device.
        With use_graph the H-step rollout is one CUDA-graph replay (captured
        on the first call, after an eager warm-up that sizes every buffer)."""
        torch = self.torch
        self._prepare(live_state, command, stream)
        if not self.use_graph:
            self._rollout(stream)
            return self.J
        if self.graph is None:
            state0 = self.ctx.get_state()                     # warm-up run sizes the buffers, then restore
            cmd0, J0 = self.command.clone(), self.J.clone()
            self._rollout(stream)
            torch.cuda.synchronize()
            from harness.types import State
            self.ctx.set_state(State(*(state0[k] for k in ("pos", "quat", "vel", "omega", "qpos", "qvel"))))
            self.command.copy_(cmd0)
            self.J.copy_(J0)
            side = torch.cuda.Stream(device=self.J.device)
            side.wait_stream(torch.cuda.current_stream())
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=side):
                self._rollout(side)
            torch.cuda.current_stream().wait_stream(side)
        self.graph.replay()
        return self.J

    def update(self, stream=None):
        mc, P, N, H = self.mc, self.mc.n_problems, self.mc.n_samples, self.mc.horizon
        self._chk(self._lib.comfree_mppi_update(self.ctx.h, P, N, H, _ptr(self.J), _ptr(self.U), mc.lam, mc.u_min,
                                                mc.u_max, _ptr(self.plan), _ptr(self.weights),
                                                _stream_handle(stream)), "comfree_mppi_update")

    def control_step(self, live_state, command, stream=None):
        """One MPPI control step: returns u_0 (P, Q) as numpy; the update
        kernel also advances the plan (comfree_mppi_update_shift)."""
        mc, P, N, H = self.mc, self.mc.n_problems, self.mc.n_samples, self.mc.horizon
        self.rollout_costs(live_state, command, stream)
        if not hasattr(self, "u0"):
            self.u0 = self.torch.zeros((P, self.Q), dtype=self.torch.float32, device=self.plan.device)
        self._chk(self._lib.comfree_mppi_update_shift(self.ctx.h, P, N, H, _ptr(self.J), _ptr(self.U), mc.lam,
                                                      mc.u_min, mc.u_max, _ptr(self.plan), _ptr(self.weights),
                                                      _ptr(self.u0), _stream_handle(stream)),
                  "comfree_mppi_update_shift")
        self.ctx.check(stream)          # collision overflow / non-finite rollouts surface here
        self.iteration += 1
        return self.u0.cpu().numpy()
