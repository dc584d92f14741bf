#!/usr/bin/env python
"""MPPI control-step time on the batched closed-loop hand:
P problems x N samples rolled out H steps (collision -> upstream -> step per
step, all on the GPU) + the weighted update, at the paper's hyperparameters
(N = 256, H = 48, lambda = 2e-3, sigma = 0.02, clip 0.1, dt = 0.004).
Prints one JSON line: ms per control step (device events on the caller's
stream around the whole control step; includes the per-step contact-count
read-back of comfree_collide and the Python orchestration)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", type=int, default=16)
    ap.add_argument("--samples", type=int, default=256)
    ap.add_argument("--horizon", type=int, default=48)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    import torch
    from harness import scenes
    from harness.types import Config
    from paper_2603_12185_b200.mppi import MPPI, MppiConfig
    P = a.problems
    rng = np.random.default_rng(5)
    tq = rng.normal(size=(P, 4))
    tq /= np.linalg.norm(tq, axis=1, keepdims=True)
    task = dict(object_body=0, target_pos=np.tile([0.02, 0.0, 0.05], (P, 1)), target_quat=tq,
                q_ref=np.tile([0.0, 0.6, 0.6, 0.6], 4), w=[1.0, 5.0, 5.0, 5.0, 2.0, 0.05],
                omega_fallen=10.0, z_fallen=0.03, phi1=50.0, phi2=2.0)
    scene, st, _, _ = scenes.c3_hand(n_worlds=P)
    cfg = Config(dt=0.004)
    m = MPPI(cfg, scene, scenes.hand_articulation(), scenes.hand_geometry(margin=0.003),
             MppiConfig(n_problems=P, n_samples=a.samples, horizon=a.horizon, task=task))
    cmd = np.tile([0.0, 0.5, 0.5, 0.5], (P, 4))
    m.control_step(st, cmd)                       # warm-up
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    t0 = time.perf_counter()
    for e0, e1 in ev:
        e0.record()
        u0 = m.control_step(st, cmd)
        e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / a.steps * 1e3
    ms = float(np.median([e0.elapsed_time(e1) for e0, e1 in ev]))
    print(json.dumps({"metric": "MPPI time per control step (closed-loop hand, GPU rollouts)", "value": ms,
                      "unit": "ms", "higher_is_better": False, "wall_ms": wall,
                      "config": {"problems": P, "samples": a.samples, "horizon": a.horizon,
                                 "rollout_worlds": P * a.samples, "rollout_world_steps": P * a.samples * a.horizon,
                                 "dt": 0.004, "sigma": 0.02, "lambda": 2e-3, "clip": 0.1},
                      "rollout_world_steps_per_s": P * a.samples * a.horizon / (ms * 1e-3),
                      "context": "paper: 13.9-28.2 ms MPPI step on an RTX 4090 with its LEAP-hand model "
                                 "(PAPER.md Table, P:653); different model, hardware and per-problem setup",
                      "u0_finite": bool(np.isfinite(u0).all())}))


if __name__ == "__main__":
    main()
