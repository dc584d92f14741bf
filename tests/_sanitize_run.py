"""Small workload for compute-sanitizer runs (tests/test_sanitizer.py): every
kernel variant once on tiny inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402

import paper_2603_12185_b200 as cf  # noqa: E402
from _gpu import gpu_step  # noqa: E402
from harness import scenes  # noqa: E402
from harness.types import Config  # noqa: E402

cfg = Config()
scene, st, c, inp = scenes.random_instance(11, n_worlds=3, n_bodies=5, contacts_per_world=[7, 0, 40])
gpu_step(cfg, scene, st, scenes.shuffle_contacts(c, 1), inp)                     # unsorted S0 + impulses
gpu_step(cfg.with_(n_t=8, n_rol=6), scene, st, c, inp, impulses=False)          # sorted, fused S0, generic facets
gpu_step(cfg, scene, st, c, inp, flags=cf.FLAG_DETERMINISTIC | cf.FLAG_STATS)   # deterministic + stats
scene, st, c, inp = scenes.random_instance(12, n_worlds=2, n_bodies=3, contacts_per_world=[9, 33], n_trees=2, tree_ndof=3)
gpu_step(cfg, scene, st, c, inp)                                                 # articulated chains
scene, st, c = scenes.c4_pile(n_worlds=2, contacts_per_world=300, lattice=(5, 5, 2))
gpu_step(cfg, scene, st, c, None, host=True)                                     # host buffers, big-world CTA path
ck = c.take(np.arange(c.n))
ck.kd = np.tile(np.array([0.2, 0.001], np.float32), (c.n, 1))
gpu_step(cfg, scene, st, ck, None)                                               # per-contact impedance, fused S0
scene, st, c, inp = scenes.random_instance(13, n_worlds=3, n_bodies=4, contacts_per_world=[5, 20, 0])
c = scenes.shuffle_contacts(c, 2)
c.kd = np.tile(np.array([0.3, 0.002], np.float32), (c.n, 1))
gpu_step(cfg, scene, st, c, inp)                                                 # per-contact impedance, sort + gather
gpu_step(cfg.with_(impedance="exact_diagonal"), scene, st, c, inp)            # exact-diagonal impedance (Eq. (11))
gpu_step(cfg.with_(impedance="facet_diagonal"), scene, st, c, inp)            # facet-diagonal impedance (R28)
# a world beyond shared memory: the global-scratch step variant
scene_l, st_l, c_l, inp_l = scenes.random_instance(14, n_worlds=2, n_bodies=2100, contacts_per_world=[60, 11])
gpu_step(cfg, scene_l, st_l, c_l, inp_l)
# pipelined host buffers (COMFREE_MEM_HOST_ASYNC)
scene_p, st_p, c_p = scenes.c4_pile(n_worlds=3, contacts_per_world=200, lattice=(5, 5, 2))
ctx_p = cf.Context(cfg)
ctx_p.load_scene(scene_p, 3, st_p)
hca = cf.HostContacts.from_arrays(c_p, pin=True, asynchronous=True, n_worlds=3)
import torch as _t  # noqa: E402
outs = [{k: _t.empty(v.shape, dtype=_t.float32).pin_memory().numpy() for k, v in ctx_p.get_state().items()}
        for _ in range(3)]
for o in outs:
    ctx_p.step(hca, None)
    ctx_p.get_state_async(o)
ctx_p.wait_async()
ctx_p.check()
# broadphase collision (one CTA per world, chained scan) in both count modes
ctx_p.load_geometry(scenes.pile_geometry((5, 5, 2), broadphase=True))
ctx_p.collide(capacity=3 * 400)
dcb, _ = ctx_p.collide(capacity=3 * 400, device_count=True)
ctx_p.step(dcb, None)
ctx_p.step_collided(3 * 400)                     # fused: the step reads the staged records
ctx_p.check()
# articulated upstream + collision front-end + step (the closed-loop hand)
import torch  # noqa: E402
from harness.types import Inputs  # noqa: E402
scene, st, c, inp = scenes.c3_hand(n_worlds=3)
ctx = cf.Context(cfg)
ctx.load_scene(scene, 3, st)
ctx.load_articulation(scenes.hand_articulation())
ctx.load_geometry(scenes.hand_geometry(margin=0.01))
tL = torch.zeros((3, 4, 10), device="cuda")
tt = torch.zeros((3, 16), device="cuda")
for _ in range(2):
    dc, link = ctx.collide(capacity=3 * 40)
    ctx.articulation_update(tL, tt, dc, link)
    ctx.step(dc, Inputs(None, tL, tt), dt=cfg.dt)
ctx.get_state()
# MPPI kernels (sample, control, cost, update) on a tiny rollout batch
from paper_2603_12185_b200.mppi import MPPI, MppiConfig  # noqa: E402
task = dict(object_body=0, target_pos=np.tile([0.02, 0.0, 0.05], (2, 1)), target_quat=np.tile([1.0, 0, 0, 0], (2, 1)),
            q_ref=np.zeros(16), w=[1.0, 1.0, 1.0, 1.0, 1.0, 0.1], omega_fallen=10.0, z_fallen=0.03, phi1=1.0, phi2=1.0)
m = MPPI(Config(dt=0.004), scene, scenes.hand_articulation(), scenes.hand_geometry(margin=0.003),
         MppiConfig(n_problems=2, n_samples=4, horizon=2, task=task))
m.control_step(st.world_slice(0, 2), np.zeros((2, 16)))
print("sanitize run ok")
