"""Helper of test_gpu_collide.test_broadphase_stage_fallback_identical (run in
a subprocess: COMFREE_BP_STAGE_CAP is read once per process): the pile's
broadphase contacts (host and device count, an overflow cut) to an .npz."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import scenes  # noqa: E402
from harness.types import Config  # noqa: E402

import paper_2603_12185_b200 as cf  # noqa: E402


def main(out):
    scene, st, _ = scenes.c4_pile(n_worlds=7, contacts_per_world=2000)
    ctx = cf.Context(Config())
    ctx.load_scene(scene, st.n_worlds, st)
    ctx.load_geometry(scenes.pile_geometry((10, 10, 5), broadphase=True))
    res = {}
    for dev in (False, True):
        dc, link = ctx.collide(capacity=7 * 5000, device_count=dev)
        n = int(dc.n_dev.item()) if dev else dc.n
        for k in ("world", "c0", "c1", "c2", "c3"):
            res[f"{int(dev)}_{k}"] = getattr(dc, k)[:n].cpu().numpy().copy()
        res[f"{int(dev)}_link"] = link[:n].cpu().numpy().copy()
    dc, _ = ctx.collide(capacity=3001, device_count=True)
    n = int(dc.n_dev.item())
    res["cut_n"] = np.array(n)
    for k in ("world", "c0", "c1", "c2", "c3"):
        res[f"cut_{k}"] = getattr(dc, k)[:n].cpu().numpy().copy()
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
