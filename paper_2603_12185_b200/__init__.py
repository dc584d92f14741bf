"""B200-native ComFree-Sim contact-resolution step (arXiv 2603.12185).

Thin Python binding over the C ABI in ``include/comfree.h`` (libcomfree.so,
hand-written CUDA for sm_100a).  The binding marshals numpy arrays / torch
tensors into the ABI's pointers and sizes; every step of the path runs in the
library's kernels.  PyTorch is used only for device memory and streams.

    ctx = Context(cfg)                       # comfree_create
    ctx.load_scene(scene, n_worlds, state)   # comfree_load_scene
    dc = DeviceContacts.from_host(contacts)  # contact-major SoA float4 streams on the GPU
    ctx.step(dc, inputs)                     # comfree_step (async on the current stream)
    st = ctx.get_state()                     # comfree_get_state
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (CONTACTS_SORTED, FLAG_DETERMINISTIC, FLAG_NO_FINITE_CHECK, FLAG_STATS,
                   MEM_DEVICE, MEM_HOST, MEM_HOST_ASYNC)

__all__ = ["Context", "DeviceContacts", "HostContacts", "ComfreeError", "make_config",
           "pack_c3", "pack_jrow", "FLAG_STATS", "FLAG_DETERMINISTIC", "FLAG_NO_FINITE_CHECK",
           "CONTACTS_SORTED", "build"]


def build(force: bool = False) -> str:
    from .build import build as _b
    return _b(force=force)


class ComfreeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_lib.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _torch():
    import torch
    return torch


def make_config(cfg=None, flags: int = 0, **kw) -> _lib.comfree_config:
    """comfree_config from the library defaults, overridden by the attributes
    of ``cfg`` (any object with k_user, d_user, ... fields) and ``kw``."""
    lib = _lib.load()
    c = _lib.comfree_config()
    lib.comfree_default_config(ct.byref(c))
    src = {}
    if cfg is not None:
        for name in ("k_user", "d_user", "r_min", "r_max", "width", "midpoint", "power",
                     "n_t", "n_rol", "gravity"):
            if hasattr(cfg, name):
                src[name] = getattr(cfg, name)
    src.update(kw)
    impedance = src.pop("impedance", getattr(cfg, "impedance", "heuristic"))
    if impedance == "exact_diagonal":      # Eq. (11) per facet (reading R24)
        flags |= _lib.FLAG_EXACT_DIAGONAL
    elif impedance == "facet_diagonal":    # Eq. (12) with the facet diagonal (reading R28)
        flags |= _lib.FLAG_FACET_DIAGONAL
    elif impedance != "heuristic":
        raise ValueError(f"impedance must be 'heuristic', 'exact_diagonal' or 'facet_diagonal', not {impedance!r}")
    for k, v in src.items():
        if k == "gravity":
            for i in range(3):
                c.gravity[i] = float(v[i])
        else:
            setattr(c, k, v)
    c.flags = flags
    return c


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        torch = _torch()
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def pack_c3(body_a, body_b, mu_rol, condim) -> np.ndarray:
    """(C,4) int32 stream c3 = (body_a, body_b, bits(mu_rol), condim)."""
    n = len(body_a)
    c3 = np.empty((n, 4), np.int32)
    c3[:, 0] = body_a
    c3[:, 1] = body_b
    c3[:, 2] = np.ascontiguousarray(mu_rol, np.float32).view(np.int32)
    c3[:, 3] = condim
    return c3


def pack_jrow(jrow) -> Optional[np.ndarray]:
    """(C,2,6,4) per-contact J rows -> (12, C, 4) streams (side*6 + row)."""
    if jrow is None:
        return None
    j = np.asarray(jrow, np.float32)
    return np.ascontiguousarray(j.reshape(j.shape[0], 12, 4).transpose(1, 0, 2))


@dataclass
class HostContacts:
    """Contact streams in host memory (pinned when possible): the e2e path."""
    n: int
    world: np.ndarray
    c0: object
    c1: object
    c2: object
    c3: object
    jrow: object
    sorted: bool
    kd: object = None
    asynchronous: bool = False             # COMFREE_MEM_HOST_ASYNC: pinned, copies overlap (comfree.h)
    off: object = None                     # pinned int64 off[W+1] (pre-segmented; world ids not copied)

    @staticmethod
    def from_arrays(contacts, pin: bool = True, asynchronous: bool = False, n_worlds=None) -> "HostContacts":
        """asynchronous (needs pin): the step's copies run on the context's own
        streams and overlap the previous step; with n_worlds, off[W+1] is
        passed instead of the world ids (the contacts must be sorted by world)."""
        torch = _torch()

        def host(a, dt):
            a = np.ascontiguousarray(a, dt)
            if pin and torch.cuda.is_available():
                t = torch.from_numpy(a).pin_memory()
                return t
            return a
        if asynchronous and not pin:
            raise ValueError("asynchronous host contacts must be pinned")
        w = np.ascontiguousarray(contacts.world, np.int32)
        srt = bool(np.all(np.diff(w) >= 0)) if len(w) else True
        off = None
        if n_worlds is not None:
            if not srt:
                raise ValueError("off[] needs contacts sorted by world")
            off = host(np.searchsorted(w, np.arange(n_worlds + 1)).astype(np.int64), np.int64)
        return HostContacts(contacts.n, None if off is not None else host(w, np.int32), host(contacts.c0, np.float32),
                            host(contacts.c1, np.float32), host(contacts.c2, np.float32),
                            host(pack_c3(contacts.body_a, contacts.body_b, contacts.mu_rol,
                                         contacts.condim), np.int32),
                            None if contacts.jrow is None else host(pack_jrow(contacts.jrow), np.float32),
                            srt,
                            None if getattr(contacts, "kd", None) is None else host(contacts.kd, np.float32),
                            asynchronous, off)

    def h2d_bytes(self) -> int:
        tot = 0
        for a in (self.world, self.off, self.c0, self.c1, self.c2, self.c3, self.jrow, self.kd):
            if a is not None:
                tot += a.nbytes if isinstance(a, np.ndarray) else a.numel() * a.element_size()
        return tot


@dataclass
class DeviceContacts:
    """Contact-major SoA float4 streams resident on the GPU (torch tensors)."""
    n: int
    world: object
    c0: object
    c1: object
    c2: object
    c3: object
    jrow: object
    sorted: bool
    kd: object = None                      # (C, 2) per-contact (k_user, d_user) or None
    n_dev: object = None                   # device int64 count of contacts in use (n = capacity), or None

    @staticmethod
    def from_host(contacts, device=None) -> "DeviceContacts":
        torch = _torch()
        dev = device or torch.device("cuda", torch.cuda.current_device())

        def d(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dt)).to(dev)
        w = np.ascontiguousarray(contacts.world, np.int32)
        srt = bool(np.all(np.diff(w) >= 0)) if len(w) else True
        return DeviceContacts(contacts.n, d(w, np.int32), d(contacts.c0, np.float32),
                              d(contacts.c1, np.float32), d(contacts.c2, np.float32),
                              d(pack_c3(contacts.body_a, contacts.body_b, contacts.mu_rol,
                                        contacts.condim), np.int32),
                              None if contacts.jrow is None else d(pack_jrow(contacts.jrow), np.float32),
                              srt,
                              None if getattr(contacts, "kd", None) is None else d(contacts.kd, np.float32))

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.c0, self.c1, self.c2, self.c3)) + \
            (0 if self.jrow is None else self.jrow.numel() * 4)


class Context:
    """One comfree_ctx (single owner)."""

    def __init__(self, cfg=None, device: int = 0, flags: int = 0, **kw):
        self._lib = _lib.load()
        self.cfg_c = make_config(cfg, flags, **kw)
        self.dt = float(getattr(cfg, "dt", 0.002)) if cfg is not None else 0.002
        h = ct.c_void_p()
        st = self._lib.comfree_create(ct.byref(self.cfg_c), device, ct.byref(h))
        if st != 0:
            raise ComfreeError(st, "comfree_create failed")
        self.h = h
        self.device = device
        self.n_worlds = 0
        self.scene = None
        self._col = None

    # ---------------------------------------------------------------- helpers
    def _check(self, st: int, what: str):
        if st != 0:
            msg = self._lib.comfree_last_error(self.h)
            raise ComfreeError(st, f"{what}: {msg.decode() if msg else ''}")

    def close(self):
        if getattr(self, "h", None):
            self._lib.comfree_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- API
    def load_scene(self, scene, n_worlds: int, state=None):
        inv_m = np.ascontiguousarray(scene.inv_mass, np.float32)
        inv_I = np.ascontiguousarray(scene.inv_inertia, np.float32)
        sc = _lib.comfree_scene(int(inv_m.shape[0]), inv_m.ctypes.data, inv_I.ctypes.data,
                                int(scene.n_trees), int(scene.tree_ndof))
        keep = []
        sp = None
        if state is not None:
            arrs = [np.ascontiguousarray(getattr(state, k), np.float32)
                    for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")]
            keep = arrs
            sp = _lib.comfree_state(*[a.ctypes.data if a.size else None for a in arrs], MEM_HOST)
        self._check(self._lib.comfree_load_scene(self.h, ct.byref(sc), int(n_worlds),
                                                 ct.byref(sp) if sp is not None else None),
                    "comfree_load_scene")
        del keep
        self.n_worlds = int(n_worlds)
        self.scene = scene
        return self

    def load_articulation(self, art):
        """comfree_load_articulation from a harness.types.Articulation (host arrays)."""
        arrs = [np.ascontiguousarray(getattr(art, k), np.float32)
                for k in ("base", "axis", "length", "mass", "inertia", "armature")]
        a = _lib.comfree_articulation(int(art.n_trees), int(art.tree_ndof), *[x.ctypes.data for x in arrs])
        self._check(self._lib.comfree_load_articulation(self.h, ct.byref(a)), "comfree_load_articulation")
        return self

    def load_geometry(self, geo):
        """comfree_load_geometry from a harness.types.Geometry (pairs None or
        empty: broadphase mode, candidates found every step, reading R32)."""
        pairs = np.zeros((0, 2), np.int32) if geo.pairs is None else np.ascontiguousarray(geo.pairs, np.int32).reshape(-1, 2)
        arrs = [np.ascontiguousarray(geo.kind, np.int32), np.ascontiguousarray(geo.body, np.int32),
                np.ascontiguousarray(geo.link, np.int32), np.ascontiguousarray(geo.size, np.float32),
                np.ascontiguousarray(geo.local, np.float32), pairs if pairs.size else np.zeros((1, 2), np.int32)]
        g = _lib.comfree_geometry(int(arrs[0].shape[0]), int(pairs.shape[0]), *[a.ctypes.data for a in arrs],
                                  float(geo.margin), (ct.c_float * 3)(*[float(m) for m in geo.mu]), int(geo.condim))
        self._check(self._lib.comfree_load_geometry(self.h, ct.byref(g)), "comfree_load_geometry")
        self._col = None
        return self

    def collide(self, capacity: int, first_world: int = 0, n_worlds: Optional[int] = None, stream=None,
                device_count: bool = False):
        """comfree_collide into device buffers of ``capacity`` records (kept by
        the context and reused).  Returns (DeviceContacts, link (n,2) int32);
        the contacts carry a zero J-row buffer when the scene has chains (for
        articulation_update).  device_count=True: asynchronous mode, the count
        stays on the device (contacts.n = capacity, contacts.n_dev = the count;
        no host round trip, CUDA-graph capturable)."""
        torch = _torch()
        nw = self.n_worlds - first_world if n_worlds is None else int(n_worlds)
        dev = torch.device("cuda", self.device)
        if self._col is None or self._col["cap"] != capacity:
            cap = max(int(capacity), 1)
            self._col = dict(cap=cap, world=torch.zeros(cap, dtype=torch.int32, device=dev),
                             c0=torch.zeros((cap, 4), device=dev), c1=torch.zeros((cap, 4), device=dev),
                             c2=torch.zeros((cap, 4), device=dev),
                             c3=torch.zeros((cap, 4), dtype=torch.int32, device=dev),
                             link=torch.zeros((cap, 2), dtype=torch.int32, device=dev),
                             n_dev=torch.zeros(1, dtype=torch.int64, device=dev),
                             jrow=torch.zeros((12, cap, 4), device=dev))
        b = self._col
        if device_count:
            st = self._lib.comfree_collide(self.h, int(first_world), nw, int(capacity), _ptr(b["world"]),
                                           _ptr(b["c0"]), _ptr(b["c1"]), _ptr(b["c2"]), _ptr(b["c3"]),
                                           _ptr(b["link"]), None, _ptr(b["n_dev"]), _stream_handle(stream))
            self._check(st, "comfree_collide")
            jrow = b["jrow"] if (self.scene is not None and self.scene.n_trees > 0) else None
            dc = DeviceContacts(int(capacity), b["world"], b["c0"], b["c1"], b["c2"], b["c3"], jrow, True,
                                n_dev=b["n_dev"])
            return dc, b["link"]
        n = ct.c_int64(0)
        st = self._lib.comfree_collide(self.h, int(first_world), nw, int(capacity), _ptr(b["world"]), _ptr(b["c0"]),
                                       _ptr(b["c1"]), _ptr(b["c2"]), _ptr(b["c3"]), _ptr(b["link"]), ct.byref(n),
                                       None, _stream_handle(stream))
        self._check(st, "comfree_collide")
        k = int(n.value)
        jrow = None
        if self.scene is not None and self.scene.n_trees > 0:
            jrow = torch.zeros((12, max(k, 1), 4), device=dev)[:, :k]
        dc = DeviceContacts(k, b["world"][:k], b["c0"][:k], b["c1"][:k], b["c2"][:k], b["c3"][:k],
                            None if jrow is None else jrow.contiguous(), True)
        return dc, b["link"][:k]

    def articulation_update(self, tree_L, tree_tau, contacts=None, link=None, tau_ext=None,
                            first_world: int = 0, n_worlds: Optional[int] = None, stream=None):
        """comfree_articulation_update: device tensors tree_L (W,T,10) and
        tree_tau (W,Q) receive the chain factors and tau - c; with
        ``contacts`` (DeviceContacts, jrow allocated) and ``link`` (device
        int32 (C,2)), the chain-side J rows are written into contacts.jrow."""
        nw = self.n_worlds - first_world if n_worlds is None else int(n_worlds)
        n = 0 if contacts is None else int(contacts.n)
        if n and (link is None or contacts.jrow is None):
            raise ValueError("articulation_update: contacts need link ids and a jrow buffer")
        s = _stream_handle(stream)
        st = self._lib.comfree_articulation_update(
            self.h, int(first_world), nw, _ptr(tau_ext), _ptr(tree_L), _ptr(tree_tau), n,
            _ptr(getattr(contacts, "n_dev", None)) if n else None, _ptr(contacts.world) if n else None, _ptr(contacts.c0) if n else None,
            _ptr(contacts.c3) if n else None, _ptr(link) if n else None, _ptr(contacts.jrow) if n else None, s)
        self._check(st, "comfree_articulation_update")

    def step(self, contacts, inputs=None, dt: Optional[float] = None, first_world: int = 0,
             n_worlds: Optional[int] = None, stream=None, impulses=None, foff=None,
             off=None, sorted_hint: Optional[bool] = None):
        """comfree_step.  ``contacts``: DeviceContacts (device path) or
        HostContacts (host buffers, copied inside the call).  ``impulses`` /
        ``foff``: optional output buffers of the same location."""
        nw = self.n_worlds - first_world if n_worlds is None else int(n_worlds)
        host = isinstance(contacts, HostContacts)
        asyn = host and contacts.asynchronous
        loc = MEM_HOST_ASYNC if asyn else (MEM_HOST if host else MEM_DEVICE)
        if host and off is None and contacts.off is not None:
            off = contacts.off
        srt = contacts.sorted if sorted_hint is None else sorted_hint
        cap = 0
        if impulses is not None:
            cap = impulses.size if isinstance(impulses, np.ndarray) else impulses.numel()
        c = _lib.comfree_contacts(int(contacts.n), _ptr(contacts.world) if contacts.n else None,
                                  _ptr(off), _ptr(contacts.c0), _ptr(contacts.c1), _ptr(contacts.c2),
                                  _ptr(contacts.c3), _ptr(contacts.jrow), _ptr(getattr(contacts, "kd", None)),
                                  _ptr(impulses), _ptr(foff),
                                  int(cap), CONTACTS_SORTED if srt else 0, loc,
                                  _ptr(getattr(contacts, "n_dev", None)))
        wloc = MEM_DEVICE
        fe = tl = tt = None
        if inputs is not None:
            arrs = [getattr(inputs, k, None) for k in ("f_ext", "tree_L", "tree_tau")]
            if any(isinstance(a, np.ndarray) for a in arrs):
                wloc = MEM_HOST_ASYNC if asyn else MEM_HOST
                arrs = [None if a is None else np.ascontiguousarray(a, np.float32) for a in arrs]
            fe, tl, tt = arrs
        w = _lib.comfree_worlds(int(first_world), nw, _ptr(fe), _ptr(tl), _ptr(tt), wloc)
        self._check(self._lib.comfree_step(self.h, ct.byref(w), ct.byref(c),
                                           float(self.dt if dt is None else dt),
                                           _stream_handle(stream)), "comfree_step")

    def step_collided(self, capacity: int, dt: Optional[float] = None, inputs=None, first_world: int = 0,
                      n_worlds: Optional[int] = None, stream=None):
        """comfree_step_collided: collision front-end (broadphase mode) and the
        contact step in one call, the contact records read by the step from the
        front-end's staging area (no public contact streams).  ``inputs``:
        optional device f_ext (no chains).  Asynchronous."""
        nw = self.n_worlds - first_world if n_worlds is None else int(n_worlds)
        fe = None if inputs is None else getattr(inputs, "f_ext", None)
        w = _lib.comfree_worlds(int(first_world), nw, _ptr(fe), None, None, MEM_DEVICE)
        self._check(self._lib.comfree_step_collided(self.h, ct.byref(w), int(capacity),
                                                    float(self.dt if dt is None else dt), _stream_handle(stream)),
                    "comfree_step_collided")

    def get_state(self, first_world: int = 0, n_worlds: Optional[int] = None, stream=None) -> dict:
        """comfree_get_state into host numpy arrays (synchronises)."""
        nw = self.n_worlds - first_world if n_worlds is None else int(n_worlds)
        B = int(np.asarray(self.scene.inv_mass).shape[0])
        Q = int(self.scene.n_trees * self.scene.tree_ndof)
        out = dict(pos=np.zeros((nw, B, 3), np.float32), quat=np.zeros((nw, B, 4), np.float32),
                   vel=np.zeros((nw, B, 3), np.float32), omega=np.zeros((nw, B, 3), np.float32),
                   qpos=np.zeros((nw, Q), np.float32), qvel=np.zeros((nw, Q), np.float32))
        st = _lib.comfree_state(*[out[k].ctypes.data if out[k].size else None
                                  for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")], MEM_HOST)
        self._check(self._lib.comfree_get_state(self.h, int(first_world), nw, ct.byref(st),
                                                _stream_handle(stream)), "comfree_get_state")
        return out

    def get_state_async(self, out: dict, first_world: int = 0, n_worlds: Optional[int] = None, stream=None):
        """comfree_get_state into caller-owned PINNED host arrays without
        synchronising (COMFREE_MEM_HOST_ASYNC): valid after wait_async(stream)
        and a synchronisation of `stream`."""
        nw = self.n_worlds - first_world if n_worlds is None else int(n_worlds)
        st = _lib.comfree_state(*[out[k].ctypes.data if out.get(k) is not None and out[k].size else None
                                  for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")], MEM_HOST_ASYNC)
        self._check(self._lib.comfree_get_state(self.h, int(first_world), nw, ct.byref(st),
                                                _stream_handle(stream)), "comfree_get_state")

    def wait_async(self, stream=None):
        """comfree_wait_async: `stream` waits for the asynchronous host copies."""
        self._check(self._lib.comfree_wait_async(self.h, _stream_handle(stream)), "comfree_wait_async")

    def get_state_device(self, out: dict, first_world: int = 0, n_worlds: Optional[int] = None, stream=None):
        """comfree_get_state into caller-owned device tensors (async)."""
        nw = self.n_worlds - first_world if n_worlds is None else int(n_worlds)
        st = _lib.comfree_state(*[_ptr(out.get(k)) if out.get(k) is not None and out[k].numel() else None
                                  for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")], MEM_DEVICE)
        self._check(self._lib.comfree_get_state(self.h, int(first_world), nw, ct.byref(st),
                                                _stream_handle(stream)), "comfree_get_state")

    def set_state(self, state, first_world: int = 0, stream=None):
        arrs = [np.ascontiguousarray(getattr(state, k), np.float32)
                for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")]
        nw = int(arrs[0].shape[0])
        st = _lib.comfree_state(*[a.ctypes.data if a.size else None for a in arrs], MEM_HOST)
        self._check(self._lib.comfree_set_state(self.h, int(first_world), nw, ct.byref(st),
                                                _stream_handle(stream)), "comfree_set_state")

    def set_state_device(self, state: dict, first_world: int = 0, stream=None):
        """comfree_set_state from caller-owned device tensors (async)."""
        nw = int(state["pos"].shape[0])
        st = _lib.comfree_state(*[_ptr(state.get(k)) if state.get(k) is not None and state[k].numel() else None
                                  for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")], MEM_DEVICE)
        self._check(self._lib.comfree_set_state(self.h, int(first_world), nw, ct.byref(st), _stream_handle(stream)),
                    "comfree_set_state")

    def set_state_broadcast(self, state, repeat: int, first_world: int = 0, stream=None):
        """comfree_set_state_broadcast: world first_world + i takes source
        state i // repeat (host numpy State of n_src worlds)."""
        arrs = [np.ascontiguousarray(getattr(state, k), np.float32)
                for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")]
        n_src = int(arrs[0].shape[0])
        st = _lib.comfree_state(*[a.ctypes.data if a.size else None for a in arrs], MEM_HOST)
        self._check(self._lib.comfree_set_state_broadcast(self.h, int(first_world), n_src, int(repeat), ct.byref(st),
                                                          _stream_handle(stream)), "comfree_set_state_broadcast")

    def get_stats(self, stream=None) -> dict:
        s = _lib.comfree_stats()
        self._check(self._lib.comfree_get_stats(self.h, ct.byref(s), _stream_handle(stream)),
                    "comfree_get_stats")
        return {k: getattr(s, k) for k, _ in s._fields_}

    def get_world_stats(self, first_world: int = 0, n_worlds: Optional[int] = None, stream=None):
        nw = self.n_worlds - first_world if n_worlds is None else int(n_worlds)
        arr = (_lib.comfree_world_stats * max(nw, 1))()
        self._check(self._lib.comfree_get_world_stats(self.h, int(first_world), nw, ct.cast(arr, ct.c_void_p),
                                                      MEM_HOST, _stream_handle(stream)),
                    "comfree_get_world_stats")
        return np.array([(a.contacts, a.active_facets, a.max_penetration, a.kinetic_energy)
                         for a in arr[:nw]], dtype=[("contacts", "i4"), ("active_facets", "i4"),
                                                    ("max_penetration", "f4"), ("kinetic_energy", "f4")])

    def segment_info(self, n_worlds: int, n_contacts: int, stream=None):
        off = np.zeros(n_worlds + 1, np.int64)
        perm = np.zeros(max(n_contacts, 1), np.int32)
        self._check(self._lib.comfree_segment_info(self.h, off.ctypes.data, perm.ctypes.data,
                                                   _stream_handle(stream)), "comfree_segment_info")
        return off, perm[:n_contacts]

    def check(self, stream=None):
        """Synchronise and raise the device errors latched by earlier
        asynchronous calls (comfree_check)."""
        self._check(self._lib.comfree_check(self.h, _stream_handle(stream)), "comfree_check")

    def set_timing(self, enable: bool = True):
        self._check(self._lib.comfree_set_timing(self.h, int(bool(enable))), "comfree_set_timing")

    def get_timing(self) -> dict:
        """Device ms of the fused step kernel / S0 kernels recorded since the
        last call (CUDA events on the step's stream)."""
        out = (ct.c_double * 3)()
        self._check(self._lib.comfree_get_timing(self.h, out), "comfree_get_timing")
        return dict(step_ms=out[0], segment_ms=out[1], step_launches=int(out[2]))

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.comfree_kernel_launches(self.h))

    def facets_per_contact(self, condim: int) -> int:
        return int(self._lib.comfree_facets_per_contact(ct.byref(self.cfg_c), int(condim)))
