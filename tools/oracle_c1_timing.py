#!/usr/bin/env python
"""Config C1 on the fp64 oracle (SURVEY §8(d) oracle timing): one sphere
resting on a plane plus one box sliding at 2 m/s with mu = 0.5, 4-facet cone,
dt = 2 ms, 1000 steps; contacts from the CPU collision helper every step.
Prints one JSON line: oracle seconds for the 1000 steps (the step calls only),
the whole loop's seconds (with the collision helper), the host CPU model and
core count.  Test infrastructure: it runs the oracle, never the product.

    python tools/oracle_c1_timing.py
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import oracle
    from harness import scenes
    from harness.collide import collide_batch
    from harness.types import Config
    cfg = Config()
    scene, st, geo = scenes.c1_scene()
    s = st.astype(np.float64)
    oracle.step(cfg, scene, s, collide_batch(geo, s.pos, s.quat, np.float64), None)   # load / warm
    t_or = 0.0
    t0 = time.perf_counter()
    for _ in range(1000):
        c = collide_batch(geo, s.pos, s.quat, np.float64)
        t1 = time.perf_counter()
        s = oracle.step(cfg, scene, s, c, None)["state"]
        t_or += time.perf_counter() - t1
    total = time.perf_counter() - t0
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    print(json.dumps({"config": "C1: sphere resting + box sliding (mu 0.5), 4-facet cone, dt 2 ms, 1000 steps",
                      "oracle_seconds": t_or, "loop_seconds_with_collision_helper": total,
                      "oracle_us_per_step": t_or * 1e3, "threads": 1, "cpu_model": model,
                      "host_cores": os.cpu_count(),
                      "box_final_speed": float(np.linalg.norm(s.vel[0, 1])),
                      "sphere_final_height": float(s.pos[0, 0, 2])}))


if __name__ == "__main__":
    main()
