"""Seeded synthetic workload generators (DESIGN.md §"Input recipe").

Shared by the oracle-side tests and the CUDA-side tests/bench: identical
bytes go to both.  This module holds no arithmetic of the method (no impulse,
impedance, facet or integration code) — only geometry, mass properties and
random draws shaped like the paper's workloads:

  C1  sphere resting + box sliding on a plane (BASELINE config 1)
  C2a incline stick/slip sweep; C2b 10-box stack, 6D friction (config 2)
  C3  LEAP-like hand: 4 chains x 4 DoF + free cube, ~20 contacts
  C4  dense pile of spheres/boxes/capsules, ~2000 contacts/world
  random_instance: mixed condim / side kinds for parity tests

Seeds: world w of a generator with base seed s draws from
np.random.default_rng([s, w]), so a world's bytes do not depend on how the
batch is sharded across ranks.
"""
from __future__ import annotations

import math

import numpy as np

from .collide import Friction, Geom, Plane, WorldGeometry, quat_R
from .types import Articulation, Config, Contacts, Inputs, Scene, State

BASE_SEED = 260312185


# ---------------------------------------------------------------- mass props
def mass_props(g: Geom, density: float = 1000.0):
    """(mass, principal inertia (3,)) of a primitive of uniform density."""
    if g.kind == "sphere":
        R = g.size[0]
        m = 4.0 / 3.0 * math.pi * R ** 3 * density
        I = 0.4 * m * R * R
        return m, np.array([I, I, I])
    if g.kind == "box":
        hx, hy, hz = g.size
        m = 8.0 * hx * hy * hz * density
        return m, np.array([m / 3 * (hy * hy + hz * hz), m / 3 * (hx * hx + hz * hz),
                            m / 3 * (hx * hx + hy * hy)])
    if g.kind == "capsule":
        R, L = g.size
        mc = math.pi * R * R * 2 * L * density
        ms = 4.0 / 3.0 * math.pi * R ** 3 * density
        Izz = mc * R * R / 2 + ms * 0.4 * R * R
        Ixx = mc * (3 * R * R + 4 * L * L) / 12 + ms * (0.4 * R * R + L * L + 0.375 * R * L)
        return mc + ms, np.array([Ixx, Ixx, Izz])
    raise ValueError(g.kind)


def scene_from_geoms(geoms, density=1000.0, masses=None, lock_rotation=False) -> Scene:
    B = len(geoms)
    inv_m = np.zeros(B, np.float32)
    inv_I = np.zeros((B, 3), np.float32)
    for i, g in enumerate(geoms):
        m, I = mass_props(g, density)
        if masses is not None and masses[i] is not None:
            I = I * (masses[i] / m)
            m = masses[i]
        inv_m[i] = 1.0 / m
        inv_I[i] = 0.0 if lock_rotation else 1.0 / I
    return Scene(inv_m, inv_I)


def _unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1
    return q


def empty_state(W, B, Q=0) -> State:
    quat = np.zeros((W, B, 4), np.float32)
    quat[..., 0] = 1
    z3 = np.zeros((W, B, 3), np.float32)
    return State(z3.copy(), quat, z3.copy(), z3.copy(), np.zeros((W, Q), np.float32),
                 np.zeros((W, Q), np.float32))


# ---------------------------------------------------------------- C1
def c1_scene(box_omega=(0.0, 0.0, 0.0)):
    """Config 1: sphere (R=0.05, rho=1000 -> m=0.5236) resting on a plane and
    a box (half 0.05, m=1) sliding at v=(2,0,0); mu_t=0.5, condim 3, n_t=4."""
    geoms = [Geom("sphere", (0.05,)), Geom("box", (0.05, 0.05, 0.05))]
    scene = scene_from_geoms(geoms)
    st = empty_state(1, 2)
    st.pos[0, 0] = (0.0, 0.0, 0.05)
    st.pos[0, 1] = (0.5, 0.0, 0.05)
    st.vel[0, 1] = (2.0, 0.0, 0.0)
    st.omega[0, 1] = box_omega
    geo = WorldGeometry(geoms, [Plane()], Friction(0.5, 0.0, 0.0), condim=3, margin=0.001)
    return scene, st, geo


# ---------------------------------------------------------------- C2a
def incline_plane(theta):
    """Plane through the origin tilted about y by theta; t1 points down-slope
    so facet j=0 is aligned with the slope."""
    n = (-math.sin(theta), 0.0, math.cos(theta))
    t1 = (math.cos(theta), 0.0, math.sin(theta))
    return Plane(n, 0.0, t1)


def c2a_incline(ratios=None, mu=0.5, half=0.05, mass=1.0, dt=0.002):
    """Config 2a: one world per tan(theta)/mu ratio; rotation-locked box of
    mass 1 resting on an incline whose facet axes align with the slope."""
    if ratios is None:
        ratios = np.linspace(0.1, 1.5, 16)
    thetas = [math.atan(r * mu) for r in ratios]
    geoms = [Geom("box", (half, half, half))]
    scene = scene_from_geoms(geoms, masses=[mass], lock_rotation=True)
    W = len(thetas)
    st = empty_state(W, 1)
    geos = []
    for w, th in enumerate(thetas):
        n = np.array([-math.sin(th), 0, math.cos(th)])
        st.pos[w, 0] = n * half
        st.quat[w, 0] = (math.cos(-th / 2), 0.0, math.sin(-th / 2), 0.0)
        # rotation about y by -theta maps local +z to n
        geos.append(WorldGeometry(geoms, [incline_plane(th)], Friction(mu, 0.0, 0.0), condim=3,
                                  margin=0.001))
    return scene, st, geos, np.asarray(thetas)


# ---------------------------------------------------------------- C2b
def c2b_stack(n_boxes=10, half=0.05, mu=(0.5, 0.005, 0.005)):
    """Config 2b: 10-box stack, 6D friction (condim 6; with Config n_t=8,
    n_rol=8: 18 facets per contact, reading A12)."""
    geoms = [Geom("box", (half, half, half)) for _ in range(n_boxes)]
    scene = scene_from_geoms(geoms)
    st = empty_state(1, n_boxes)
    for i in range(n_boxes):
        st.pos[0, i] = (0.002 * i, 0.0, half + 2 * half * i - 0.0004 * (i + 1))
    geo = WorldGeometry(geoms, [Plane()], Friction(*mu), condim=6, margin=0.001,
                        pairs=[(i, i + 1) for i in range(n_boxes - 1)])
    return scene, st, geo


# ---------------------------------------------------------------- random instances
def random_instance(seed, n_worlds=3, n_bodies=5, contacts_per_world=12, n_trees=0,
                    tree_ndof=4, condims=(1, 3, 4, 6), static_frac=0.25, tree_frac=0.3,
                    with_fext=True, locked_frac=0.0):
    """Mixed instance exercising every code path: free/static/articulated
    sides, all condims, ragged contact counts (contacts_per_world may be a
    list), unsorted world ids."""
    rng = np.random.default_rng([BASE_SEED, seed])
    B, T, nd = n_bodies, n_trees, tree_ndof
    W = n_worlds
    Q = T * nd
    mass = rng.uniform(0.05, 2.0, B)
    rad = rng.uniform(0.02, 0.08, B)                    # body size sets inertia and lever arms
    inertia = 0.4 * mass[:, None] * rad[:, None] ** 2 * rng.uniform(0.7, 1.3, (B, 3))
    inv_m = (1.0 / mass).astype(np.float32)
    inv_I = (1.0 / inertia).astype(np.float32)
    if locked_frac > 0:
        lk = rng.random(B) < locked_frac
        inv_I[lk] = 0
    scene = Scene(inv_m, inv_I, T, nd)
    st = State(rng.uniform(-0.2, 0.2, (W, B, 3)).astype(np.float32),
               _unit_quats(rng, W * B).reshape(W, B, 4).astype(np.float32),
               rng.normal(0, 0.3, (W, B, 3)).astype(np.float32),
               rng.normal(0, 2.0, (W, B, 3)).astype(np.float32),
               rng.uniform(-1, 1, (W, Q)).astype(np.float32),
               rng.normal(0, 0.5, (W, Q)).astype(np.float32))
    inputs = Inputs()
    if with_fext:                                       # ~0.5 g and ~5 rad/s^2 scale pushes
        fe = rng.normal(0, 1.0, (W, B, 6))
        fe[..., :3] *= 0.5 * 9.81 * mass[None, :, None]
        fe[..., 3:] *= 5.0 * inertia[None, :, :]
        inputs.f_ext = fe.astype(np.float32)
    if T:
        Ls = np.zeros((W, T, 10), np.float32)
        for w in range(W):
            for t in range(T):
                A = rng.normal(0, 0.02, (nd, nd))
                M = A @ A.T + np.diag(rng.uniform(2e-3, 1e-2, nd))
                L = np.linalg.cholesky(M)
                for i in range(nd):
                    for j in range(i + 1):
                        Ls[w, t, i * (i + 1) // 2 + j] = L[i, j]
                for i in range(nd, 4):          # unused DoFs: identity, never read
                    Ls[w, t, i * (i + 1) // 2 + i] = 1.0
        inputs.tree_L = Ls
        inputs.tree_tau = rng.normal(0, 0.05, (W, Q)).astype(np.float32)
    cpw = contacts_per_world if isinstance(contacts_per_world, (list, tuple, np.ndarray)) \
        else [contacts_per_world] * W
    parts = []
    for w in range(W):
        n = int(cpw[w])
        if n == 0:
            continue
        kinds = []
        tf = tree_frac if T else 0.0
        for _ in range(n):
            ids = []
            for s in range(2):
                u = rng.random()
                if u < tf:
                    ids.append(-2 - int(rng.integers(T)))
                elif u < tf + static_frac and s == 0:
                    ids.append(-1)
                else:
                    ids.append(int(rng.integers(B)))
            if ids[0] == ids[1] and ids[0] >= 0 and B > 1:      # no self contact
                ids[1] = (ids[0] + 1 + int(rng.integers(B - 1))) % B
            if ids[0] == -1 and ids[1] == -1:
                ids[1] = int(rng.integers(B))
            kinds.append(ids)
        kinds = np.asarray(kinds, np.int32)
        nrm = rng.normal(size=(n, 3))
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        t1 = np.cross(nrm, rng.normal(size=(n, 3)))
        t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
        # contact point on the surface of a free side (lever arm ~ body size)
        p = rng.uniform(-0.25, 0.25, (n, 3))
        u = rng.normal(size=(n, 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        for k in range(n):
            side = kinds[k, 1] if kinds[k, 1] >= 0 else kinds[k, 0]
            if side >= 0:
                p[k] = st.pos[w, side] + rad[side] * u[k]
        phi = rng.uniform(-3e-3, 5e-4, n)
        c0 = np.concatenate([p, phi[:, None]], 1).astype(np.float32)
        c1 = np.concatenate([nrm, rng.uniform(0.0, 1.2, (n, 1))], 1).astype(np.float32)
        c2 = np.concatenate([t1, rng.uniform(0.0, 0.02, (n, 1))], 1).astype(np.float32)
        jr = rng.normal(0, 0.05, (n, 2, 6, 4)).astype(np.float32) if T else None
        if T:
            jr[:, :, 3:, :] = rng.normal(0, 1.0, (n, 2, 3, 4))
            jr[:, :, :, nd:] = 0
        parts.append(Contacts(np.full(n, w, np.int32), c0, c1, c2, kinds[:, 0].copy(),
                              kinds[:, 1].copy(), rng.uniform(0, 0.02, n).astype(np.float32),
                              rng.choice(np.asarray(condims, np.int32), n), jr))
    contacts = Contacts.concat(parts) if parts else Contacts.empty(with_jrow=bool(T))
    if T and contacts.jrow is None:
        contacts.jrow = np.zeros((contacts.n, 2, 6, 4), np.float32)
    return scene, st, contacts, inputs


def shuffle_contacts(contacts: Contacts, seed: int) -> Contacts:
    rng = np.random.default_rng([BASE_SEED, 7, seed])
    return contacts.take(rng.permutation(contacts.n))


# ---------------------------------------------------------------- C4 pile
PILE_SHAPES = (Geom("sphere", (0.025,)), Geom("box", (0.025, 0.025, 0.025)),
               Geom("capsule", (0.015, 0.02)))


def _pile_template(nx, ny, nz):
    B = nx * ny * nz
    kinds = np.arange(B) % 3                    # 0 sphere, 1 box, 2 capsule
    idx = np.arange(B).reshape(nz, ny, nx)
    pairs = []
    for (da, db) in ((idx[:, :, :-1], idx[:, :, 1:]), (idx[:, :-1, :], idx[:, 1:, :]),
                     (idx[:-1, :, :], idx[1:, :, :])):
        pairs.append(np.stack([da.ravel(), db.ravel()], 1))
    pairs = np.concatenate(pairs)
    floor = np.stack([np.full(nx * ny, -1), idx[0].ravel()], 1)
    allp = np.concatenate([floor, pairs])

    def mult(a, b):
        ka = 1 if a < 0 else kinds[a]           # floor behaves like a box face
        kb = kinds[b]
        if a < 0:
            return {0: 1, 1: 4, 2: 2}[kb]
        if ka == 1 and kb == 1:
            return 4
        if ka == 2 or kb == 2:
            return 2
        return 1
    rows = []
    for a, b in allp:
        for k in range(mult(a, b)):
            rows.append((a, b, k, mult(a, b)))
    rows.sort(key=lambda r: (r[0], r[1], r[2]))
    return kinds, np.asarray(rows, np.int64)


def pile_geometry(lattice=(10, 10, 5), margin=0.001, mu=(1.0, 0.005, 0.0001), condim=3, broadphase=False):
    """Collision geometry of the config-4 pile for the GPU front-end: the floor
    plane z = 0, one geom per body (sphere R 2.5 cm / box half 2.5 cm / capsule
    R 1.5 cm, half-length 2 cm, as PILE_SHAPES), candidate pairs = the floor with
    the bottom layer and every lattice-neighbour pair (the generator's pairs);
    broadphase=True: no candidate list, the front-end's broadphase finds the
    pairs every step (reading R32)."""
    from .types import Geometry
    nx, ny, nz = lattice
    B = nx * ny * nz
    kinds, _ = _pile_template(nx, ny, nz)
    kmap = {"sphere": 0, "box": 1, "capsule": 3}
    kind, body, size = [2], [-1], [(0.0, 0.0, 1.0)]
    for i in range(B):
        g = PILE_SHAPES[kinds[i]]
        kind.append(kmap[g.kind])
        body.append(i)
        sz = tuple(g.size) + (0.0,) * (3 - len(g.size))
        size.append(sz)
    idx = np.arange(B).reshape(nz, ny, nx)
    pairs = [(0, 1 + int(i)) for i in idx[0].ravel()]
    for (da, db) in ((idx[:, :, :-1], idx[:, :, 1:]), (idx[:, :-1, :], idx[:, 1:, :]), (idx[:-1, :, :], idx[1:, :, :])):
        pairs += [(1 + int(a), 1 + int(b)) for a, b in zip(da.ravel(), db.ravel())]
    G = B + 1
    return Geometry(np.array(kind, np.int32), np.array(body, np.int32), np.zeros(G, np.int32),
                    np.array(size, np.float64), np.zeros((G, 3)), None if broadphase else np.array(pairs, np.int32),
                    margin=margin, mu=mu, condim=condim)


def c4_pile(n_worlds=1024, contacts_per_world=2000, lattice=(10, 10, 5), seed=0,
            world_offset=0, condim=3, mu=(1.0, 0.005, 0.0001)):
    """Config 4: per world a jittered nx*ny*nz lattice (5 cm pitch) of
    spheres (R 2.5 cm), boxes (half 2.5 cm) and capsules (R 1.5 cm, half-length
    2 cm), density 1000; contacts between lattice neighbours and the floor with
    shape-pair multiplicity (box 4, capsule 2, sphere 1), trimmed or
    replicated to exactly contacts_per_world, sorted by (world, a, b).
    phi ~ U(-3, 0.5) mm (P:297-305 depth scale); v ~ N(0, 1e-3) per axis
    (P:390); omega ~ N(0, 0.1^2); mu = (1, 0.005, 0.0001)."""
    nx, ny, nz = lattice
    B = nx * ny * nz
    kinds, rows = _pile_template(nx, ny, nz)
    geoms = [PILE_SHAPES[k] for k in kinds]
    scene = scene_from_geoms(geoms)
    R = len(rows)
    Cw = int(contacts_per_world)
    if Cw <= R:
        sel = np.floor(np.arange(Cw) * (R / Cw)).astype(np.int64)
    else:
        sel = np.arange(Cw) % R
        sel.sort(kind="stable")
    rows = rows[sel]
    a_idx, b_idx, k_idx, m_idx = rows[:, 0], rows[:, 1], rows[:, 2], rows[:, 3]
    W = n_worlds
    pitch = 0.05
    lat = np.zeros((B, 3))
    ii = np.arange(B)
    lat[:, 0] = (ii % nx) * pitch
    lat[:, 1] = ((ii // nx) % ny) * pitch
    lat[:, 2] = (ii // (nx * ny)) * pitch + 0.025
    pos = np.zeros((W, B, 3), np.float32)
    quat = np.zeros((W, B, 4), np.float32)
    vel = np.zeros((W, B, 3), np.float32)
    om = np.zeros((W, B, 3), np.float32)
    c0 = np.zeros((W, Cw, 4), np.float32)
    c1 = np.zeros((W, Cw, 4), np.float32)
    c2 = np.zeros((W, Cw, 4), np.float32)
    for wi in range(W):
        w = world_offset + wi
        rng = np.random.default_rng([BASE_SEED, seed, w])
        x = lat + rng.uniform(-0.002, 0.002, (B, 3))
        pos[wi] = x
        quat[wi] = _unit_quats(rng, B)
        vel[wi] = rng.normal(0, math.sqrt(1e-3), (B, 3))
        om[wi] = rng.normal(0, 0.1, (B, 3))
        xb = x[b_idx]
        xa = np.where(a_idx[:, None] < 0, xb * np.array([1, 1, 0]), x[np.maximum(a_idx, 0)])
        axis = np.where(a_idx[:, None] < 0, np.array([0.0, 0.0, 1.0]), xb - xa)
        axis /= np.linalg.norm(axis, axis=1, keepdims=True)
        # tilt by U(0, 5 deg) about a random perpendicular axis
        perp = np.cross(axis, rng.normal(size=(Cw, 3)))
        perp /= np.linalg.norm(perp, axis=1, keepdims=True)
        ang = np.deg2rad(rng.uniform(0, 5, Cw))[:, None]
        n = axis * np.cos(ang) + np.cross(perp, axis) * np.sin(ang)
        n /= np.linalg.norm(n, axis=1, keepdims=True)
        kmin = np.argmin(np.abs(n), axis=1)
        e = np.zeros((Cw, 3))
        e[np.arange(Cw), kmin] = 1.0
        t1 = e - np.sum(e * n, 1, keepdims=True) * n
        t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
        t2 = np.cross(n, t1)
        mid = 0.5 * (xa + xb)
        mid = np.where(a_idx[:, None] < 0, xb - n * 0.025, mid)
        # spread multiple contacts of one pair over the shared face
        angk = 2 * math.pi * k_idx / np.maximum(m_idx, 1)
        spread = np.where(m_idx[:, None] > 1, 0.015, 0.0)
        p = mid + spread * (np.cos(angk)[:, None] * t1 + np.sin(angk)[:, None] * t2)
        phi = rng.uniform(-3e-3, 5e-4, Cw)
        c0[wi] = np.concatenate([p, phi[:, None]], 1)
        c1[wi] = np.concatenate([n, np.full((Cw, 1), mu[0])], 1)
        c2[wi] = np.concatenate([t1, np.full((Cw, 1), mu[1])], 1)
    st = State(pos, quat, vel, om, np.zeros((W, 0), np.float32), np.zeros((W, 0), np.float32))
    C = W * Cw
    contacts = Contacts(np.repeat(np.arange(W, dtype=np.int32), Cw), c0.reshape(C, 4),
                        c1.reshape(C, 4), c2.reshape(C, 4),
                        np.tile(a_idx.astype(np.int32), W), np.tile(b_idx.astype(np.int32), W),
                        np.full(C, mu[2], np.float32), np.full(C, condim, np.int32))
    return scene, st, contacts


# ---------------------------------------------------------------- C3 hand
def hand_articulation() -> Articulation:
    """The synthetic LEAP-like hand of config 3 as an Articulation: 4 chains x
    4 hinges (first about the base z axis, then three about the link y axis),
    link lengths (0.045, 0.035, 0.03, 0.03) m, masses (0.04, 0.03, 0.02,
    0.015) kg, isotropic link inertia m l^2 / 12, armature 2e-4."""
    T, nd = 4, 4
    lens = np.array([0.045, 0.035, 0.03, 0.03])
    lmass = np.array([0.04, 0.03, 0.02, 0.015])
    bases = np.array([[0.04, -0.045, 0.0], [0.04, 0.0, 0.0], [0.04, 0.045, 0.0], [-0.02, -0.06, 0.0]])
    axis = np.zeros((T, nd, 3))
    axis[:, 0] = (0, 0, 1.0)
    axis[:, 1:] = (0, 1.0, 0)
    return Articulation(bases, axis, np.tile(lens, (T, 1)), np.tile(lmass, (T, 1)),
                        np.tile(lmass * lens ** 2 / 12, (T, 1)), np.full((T, nd), 2e-4))


def hand_geometry(margin=0.001, tip_radius=0.008, cube_half=0.03):
    """Collision geometry of the config-3 hand for the GPU front-end: the palm
    plane z = 0, the cube (free body 0, box), and a sphere at the far end of
    every finger link.  Candidate pairs: every link sphere with the cube
    (normal from the finger to the cube), the palm with every link sphere but
    the first of each finger, and the palm with the cube."""
    from .types import Geometry
    art = hand_articulation()
    T, nd = art.n_trees, art.tree_ndof
    kind, body, link, size, local = [2, 1], [-1, 0], [0, 0], [(0, 0, 1.0), (cube_half,) * 3], [(0.0, 0, 0), (0, 0, 0)]
    for t in range(T):
        for l in range(nd):
            kind.append(0)
            body.append(-2 - t)
            link.append(l)
            size.append((tip_radius, 0, 0))
            local.append((0, 0, float(art.length[t, l])))
    pairs = [(2 + t * nd + l, 1) for t in range(T) for l in range(nd)]
    pairs += [(0, 2 + t * nd + l) for t in range(T) for l in range(1, nd)]
    pairs += [(0, 1)]
    return Geometry(np.array(kind, np.int32), np.array(body, np.int32), np.array(link, np.int32),
                    np.array(size, np.float64), np.array(local, np.float64), np.array(pairs, np.int32),
                    margin=margin)


def c3_hand(n_worlds=4096, seed=0, world_offset=0):
    """Config 3: LEAP-like hand, 4 hinge chains x 4 DoF (nv = 16 + 6) plus a
    free cube (0.06 m, 0.1 kg).  Per world, from q ~ U(joint range): link
    Jacobians of a synthetic chain (link lengths ~ (0.045, 0.035, 0.03, 0.03) m,
    masses ~ (0.04, 0.03, 0.02, 0.015) kg), a CRBA-style M = sum J^T m J + J_w^T
    I J_w + armature and its Cholesky factor, 20 contacts: 12 finger-cube, 4
    cube-palm (static), 4 fingertip-palm; phi ~ U(-2, 0.5) mm; joint
    velocities N(0, 0.5^2); cube v N(0, 0.02^2), omega N(0, 0.2^2);
    mu = (1, 0.005, 0.0001), condim 3.  Synthetic, not the paper's model."""
    T, nd, B = 4, 4, 1
    W = n_worlds
    lens = np.array([0.045, 0.035, 0.03, 0.03])
    lmass = np.array([0.04, 0.03, 0.02, 0.015])
    cube_half = 0.03
    scene = Scene(np.array([1.0 / 0.1], np.float32),
                  np.full((1, 3), 1.0 / (0.1 / 3 * 2 * cube_half ** 2), np.float32), T, nd)
    Cw = 20
    pos = np.zeros((W, B, 3), np.float32)
    quat = np.zeros((W, B, 4), np.float32)
    vel = np.zeros((W, B, 3), np.float32)
    om = np.zeros((W, B, 3), np.float32)
    qpos = np.zeros((W, T * nd), np.float32)
    qvel = np.zeros((W, T * nd), np.float32)
    Ls = np.zeros((W, T, 10), np.float32)
    tau = np.zeros((W, T * nd), np.float32)
    c0 = np.zeros((W, Cw, 4), np.float32)
    c1 = np.zeros((W, Cw, 4), np.float32)
    c2 = np.zeros((W, Cw, 4), np.float32)
    ba = np.zeros((W, Cw), np.int32)
    bb = np.zeros((W, Cw), np.int32)
    jr = np.zeros((W, Cw, 2, 6, 4), np.float32)
    lk = np.zeros((W, Cw, 2), np.int32)       # link index of each chain side (articulated upstream)
    bases = np.array([[0.04, -0.045, 0.0], [0.04, 0.0, 0.0], [0.04, 0.045, 0.0],
                      [-0.02, -0.06, 0.0]])
    for wi in range(W):
        w = world_offset + wi
        rng = np.random.default_rng([BASE_SEED, 3, seed, w])
        cube = np.array([0.02, 0.0, 0.05]) + rng.uniform(-0.003, 0.003, 3)
        pos[wi, 0] = cube
        qc = np.array([1.0, 0, 0, 0]) + np.concatenate([[0], rng.normal(0, 0.02, 3)])
        quat[wi, 0] = qc / np.linalg.norm(qc)
        vel[wi, 0] = rng.normal(0, 0.02, 3)
        om[wi, 0] = rng.normal(0, 0.2, 3)
        q = rng.uniform([-0.3, 0.0, 0.0, 0.0], [0.3, 1.2, 1.2, 1.2], (T, nd))
        qpos[wi] = q.ravel()
        qvel[wi] = rng.normal(0, 0.5, T * nd)
        link_pts = []          # per tree: per link (origin, axes list, com) for Jacobians
        for t in range(T):
            o = bases[t].copy()
            R = np.eye(3)
            axes, origins, coms = [], [], []
            for j in range(nd):
                ax_local = np.array([0, 0, 1.0]) if j == 0 else np.array([0, 1.0, 0])
                ax = R @ ax_local
                c, s = math.cos(q[t, j]), math.sin(q[t, j])
                K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
                R = (np.eye(3) + s * K + (1 - c) * K @ K) @ R
                axes.append(ax)
                origins.append(o.copy())
                d = R @ np.array([0, 0, 1.0])
                coms.append(o + 0.5 * lens[j] * d)
                o = o + lens[j] * d
            link_pts.append((np.asarray(axes), np.asarray(origins), np.asarray(coms), o))
            # CRBA-style inertia from link Jacobians
            M = np.diag(np.full(nd, 2e-4))
            for l in range(nd):
                Jv = np.zeros((3, nd))
                Jw = np.zeros((3, nd))
                for j in range(l + 1):
                    Jw[:, j] = axes[j]
                    Jv[:, j] = np.cross(axes[j], coms[l] - origins[j])
                Il = lmass[l] * lens[l] ** 2 / 12
                M += lmass[l] * Jv.T @ Jv + Il * Jw.T @ Jw
            L = np.linalg.cholesky(M)
            for i in range(nd):
                for j in range(i + 1):
                    Ls[wi, t, i * (i + 1) // 2 + j] = L[i, j]
            tau[wi, t * nd:(t + 1) * nd] = rng.normal(0, 0.02, nd)

        def link_jac(t, l, p):
            axes, origins, _, _ = link_pts[t]
            J = np.zeros((6, 4))
            for j in range(l + 1):
                J[0:3, j] = np.cross(axes[j], p - origins[j])
                J[3:6, j] = axes[j]
            return J
        k = 0
        faces = [np.array([1.0, 0, 0]), np.array([0, 1.0, 0]), np.array([-1.0, 0, 0]),
                 np.array([0, -1.0, 0])]
        for t in range(T):                       # 12 finger-cube contacts (links 1..3)
            f = faces[t]
            for l in (1, 2, 3):
                p = cube + cube_half * f + rng.uniform(-0.02, 0.02, 3) * (1 - np.abs(f))
                n = -f + rng.normal(0, 0.03, 3)
                n /= np.linalg.norm(n)
                ba[wi, k], bb[wi, k] = -2 - t, 0
                jr[wi, k, 0] = link_jac(t, l, p)
                lk[wi, k, 0] = l
                c0[wi, k] = (*p, rng.uniform(-2e-3, 5e-4))
                c1[wi, k, :3] = n
                k += 1
        for s in range(4):                       # cube on palm
            sx, sy = (1 if s & 1 else -1), (1 if s & 2 else -1)
            p = cube + np.array([sx * cube_half, sy * cube_half, -cube_half])
            ba[wi, k], bb[wi, k] = -1, 0
            c0[wi, k] = (*p, rng.uniform(-2e-3, 5e-4))
            c1[wi, k, :3] = (0, 0, 1.0)
            k += 1
        for t in range(T):                       # fingertip on palm
            p = link_pts[t][3].copy()
            ba[wi, k], bb[wi, k] = -1, -2 - t
            jr[wi, k, 1] = link_jac(t, 3, p)
            lk[wi, k, 1] = 3
            c0[wi, k] = (*p, rng.uniform(-2e-3, 5e-4))
            c1[wi, k, :3] = (0, 0, 1.0)
            k += 1
        n_all = c1[wi, :, :3].astype(np.float64)
        kmin = np.argmin(np.abs(n_all), axis=1)
        e = np.zeros((Cw, 3))
        e[np.arange(Cw), kmin] = 1
        t1 = e - np.sum(e * n_all, 1, keepdims=True) * n_all
        t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
        c2[wi, :, :3] = t1
    c1[..., 3] = 1.0
    c2[..., 3] = 0.005
    st = State(pos, quat, vel, om, qpos, qvel)
    C = W * Cw
    contacts = Contacts(np.repeat(np.arange(W, dtype=np.int32), Cw), c0.reshape(C, 4),
                        c1.reshape(C, 4), c2.reshape(C, 4), ba.reshape(C), bb.reshape(C),
                        np.full(C, 1e-4, np.float32), np.full(C, 3, np.int32),
                        jr.reshape(C, 2, 6, 4))
    contacts.meta["link"] = lk.reshape(C, 2)
    return scene, st, contacts, Inputs(None, Ls, tau)


# ---------------------------------------------------------------- C5 mixed
def tile_worlds(st: State, c: Contacts, inp, n_worlds: int):
    """Repeat a batch of U worlds cyclically to n_worlds worlds (world w is a
    copy of world w mod U; contacts stay grouped and sorted by world).  Used
    to build large batches quickly: every copy is still stepped, the bytes are
    only not unique."""
    U = st.n_worlds
    src = np.arange(n_worlds) % U
    st2 = State(*(np.ascontiguousarray(a[src]) for a in (st.pos, st.quat, st.vel, st.omega, st.qpos, st.qvel)))
    off = np.zeros(U + 1, np.int64)
    np.cumsum(np.bincount(c.world, minlength=U), out=off[1:])
    counts = off[1:] - off[:-1]
    idx = np.concatenate([np.arange(off[s], off[s + 1]) for s in src]) if n_worlds else np.zeros(0, np.int64)
    c2 = c.take(idx)
    c2.world = np.repeat(np.arange(n_worlds, dtype=np.int32), counts[src])
    inp2 = None
    if inp is not None:
        inp2 = Inputs(*(None if a is None else np.ascontiguousarray(a[src]) for a in
                        (inp.f_ext, inp.tree_L, inp.tree_tau)))
    return st2, c2, inp2


def c5_mixed(n_worlds=65536, seed=0, world_offset=0, unique_hand=1024, unique_pile=4096):
    """Config 5: n_worlds // 2 C3 hand worlds plus n_worlds - n_worlds // 2
    "pile-lite" worlds (5x5x4 lattice = 100 bodies, 400 contacts), as two
    homogeneous batches (one library context each, stepped concurrently).
    At most unique_hand / unique_pile distinct worlds are generated per call
    (seeded by world_offset) and tiled to the requested counts.
    Returns {"hand": (scene, state, contacts, inputs), "pile": (scene, state, contacts)}."""
    nh = n_worlds // 2
    npl = n_worlds - nh
    uh, up = max(1, min(nh, unique_hand)), max(1, min(npl, unique_pile))
    sh, sth, ch, ih = c3_hand(n_worlds=uh, seed=seed + 5, world_offset=world_offset)
    sp, stp, cp = c4_pile(n_worlds=up, contacts_per_world=400, lattice=(5, 5, 4), seed=seed + 5,
                          world_offset=world_offset)
    sth, ch, ih = tile_worlds(sth, ch, ih, nh)
    stp, cp, _ = tile_worlds(stp, cp, None, npl)
    return {"hand": (sh, sth, ch, ih), "pile": (sp, stp, cp)}
