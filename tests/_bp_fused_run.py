"""Helper of test_gpu_collide.test_step_collided_bitwise (run in a subprocess:
COMFREE_BP_STAGE_CAP is read once per process): the pile's full step for a few
steps through comfree_collide + comfree_step (device count) and through
comfree_step_collided (the step reading the staged records), states to an .npz."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import scenes  # noqa: E402
from harness.types import Config  # noqa: E402

import paper_2603_12185_b200 as cf  # noqa: E402


def main(out, n_worlds=40, steps=6):
    scene, st, _ = scenes.c4_pile(n_worlds=n_worlds, contacts_per_world=2000)
    geo = scenes.pile_geometry((10, 10, 5), broadphase=True)
    cfg = Config()
    if os.environ.get("FUSED_NT"):  # a facet set the staged kernel does not cover: the call's collide + step path
        cfg = cfg.with_(n_t=int(os.environ["FUSED_NT"]))
    cap = n_worlds * 6000
    res = {}
    for mode in ("split", "fused"):
        ctx = cf.Context(cfg)
        ctx.load_scene(scene, st.n_worlds, st)
        ctx.load_geometry(geo)
        for _ in range(steps):
            if mode == "split":
                dc, _ = ctx.collide(capacity=cap, device_count=True)
                ctx.step(dc, None, dt=cfg.dt)
            else:
                ctx.step_collided(cap, dt=cfg.dt)
        g = ctx.get_state()
        for k, v in g.items():
            res[f"{mode}_{k}"] = np.asarray(v).copy()
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
