import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from harness import scenes
from harness.types import Config
import paper_2603_12185_b200 as cf
scene, st, _ = scenes.c4_pile(n_worlds=1024, contacts_per_world=2000)
geo = scenes.pile_geometry((10, 10, 5), broadphase=True)
for rep in range(3):
    ctx = cf.Context(Config()); ctx.load_scene(scene, st.n_worlds, st); ctx.load_geometry(geo)
    dc, _ = ctx.collide(capacity=1024 * 4000)
    n = dc.n
    c3 = dc.c3[:n].cpu().numpy(); w = dc.world[:n].cpu().numpy()
    bad = np.nonzero((c3[:, 0] == -1) & (c3[:, 1] == -1))[0]
    print(rep, n, hash(c3.tobytes()), "empty records", len(bad), np.unique(w[bad]))
