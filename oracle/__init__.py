"""TEST INFRASTRUCTURE ONLY — the fp64 CPU oracle of the ComFree-Sim step.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2603_12185_b200``) never does, and the two share no code.

Contents
  oracle.c / oracle.h  plain fp64 C implementation of Algorithm 1
                       in the order of the paper (Kernel I-IV, Eq. (2)-(13)),
                       wrapped here with ctypes.
  dense.py             oracle B: generalized-coordinate dense assembly of
                       J~, M and Eq. (10) with numpy.linalg.solve, plus the
                       brute-force activation-pattern enumeration.

Parity pins: see tests/test_oracle_pins.py and DESIGN.md §"Oracle pins".
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

from harness.types import Config, Contacts, Inputs, Scene, State

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c (plain -O2, no fast-math, OpenMP only across worlds)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-fopenmp", "-shared",
                               "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


class _Cfg(ct.Structure):
    _fields_ = [("k_user", ct.c_double), ("d_user", ct.c_double),
                ("r_min", ct.c_double), ("r_max", ct.c_double), ("width", ct.c_double),
                ("midpoint", ct.c_double), ("power", ct.c_double),
                ("n_t", ct.c_int32), ("n_rol", ct.c_int32),
                ("gravity", ct.c_double * 3), ("dt", ct.c_double),
                ("exact_diagonal", ct.c_int32)]


class _Scene(ct.Structure):
    _fields_ = [("n_bodies", ct.c_int32), ("inv_mass", ct.POINTER(ct.c_double)),
                ("inv_inertia", ct.POINTER(ct.c_double)), ("n_trees", ct.c_int32),
                ("tree_ndof", ct.c_int32)]


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ct.CDLL(_LIB_PATH)
        P = ct.c_void_p
        lib.orc_step.restype = ct.c_int
        lib.orc_step.argtypes = [ct.POINTER(_Cfg), ct.POINTER(_Scene), ct.c_int64,
                                 P, P, P, P, P, P, P, P, P, ct.c_int64, P, P, P, P, P, P, P, P, P,
                                 P, P, P, P, ct.c_int]
        lib.orc_segment.restype = ct.c_int
        lib.orc_segment.argtypes = [ct.c_int64, P, ct.c_int64, P, ct.c_int32, ct.c_int32, P, P, P]
        lib.orc_gamma.restype = ct.c_double
        lib.orc_gamma.argtypes = [ct.c_double, ct.c_double, ct.c_double]
        lib.orc_r.restype = ct.c_double
        lib.orc_r.argtypes = [ct.c_double, ct.POINTER(_Cfg)]
        lib.orc_facet_lambda.restype = ct.c_double
        lib.orc_facet_lambda.argtypes = [ct.c_double] * 5
        lib.orc_facets_per_contact.restype = ct.c_int
        lib.orc_facets_per_contact.argtypes = [ct.c_int32] * 3
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    pass


def _cfg(cfg: Config) -> _Cfg:
    c = _Cfg()
    c.k_user, c.d_user = cfg.k_user, cfg.d_user
    c.r_min, c.r_max, c.width, c.midpoint, c.power = (cfg.r_min, cfg.r_max, cfg.width,
                                                     cfg.midpoint, cfg.power)
    c.n_t, c.n_rol = cfg.n_t, cfg.n_rol
    for i in range(3):
        c.gravity[i] = cfg.gravity[i]
    c.dt = cfg.dt
    c.exact_diagonal = {"heuristic": 0, "exact_diagonal": 1, "facet_diagonal": 2}[getattr(cfg, "impedance", "heuristic")]
    return c


def _d(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _p(a):
    return None if a is None else a.ctypes.data_as(ct.c_void_p)


def gamma(x: float, m: float, p: float) -> float:
    return _load().orc_gamma(x, m, p)


def r_of_phi(phi: float, cfg: Config) -> float:
    c = _cfg(cfg)
    return _load().orc_r(phi, ct.byref(c))


def facet_lambda(K: float, D: float, s: float, phi: float, dt: float) -> float:
    return _load().orc_facet_lambda(K, D, s, phi, dt)


def facets_per_contact(condim: int, n_t: int, n_rol: int) -> int:
    return _load().orc_facets_per_contact(condim, n_t, n_rol)


def segment(contacts: Contacts, n_worlds: int, cfg: Config):
    """S0 with plain loops: (off[W+1] int64, perm[C] int32, foff[C+1] int64)."""
    n = contacts.n
    off = np.zeros(n_worlds + 1, np.int64)
    perm = np.zeros(max(n, 1), np.int32)
    foff = np.zeros(n + 1, np.int64)
    w, cd = _i(contacts.world), _i(contacts.condim)
    rc = _load().orc_segment(n, _p(w), n_worlds, _p(cd), cfg.n_t, cfg.n_rol,
                             _p(off), _p(perm), _p(foff))
    if rc != 0:
        raise OracleError(f"orc_segment failed rc={rc}")
    return off, perm[:n], foff


def step(cfg: Config, scene: Scene, state: State, contacts: Contacts,
         inputs: Inputs | None = None, n_threads: int = 1, strict: bool = True) -> dict:
    """One oracle step from ``state`` (promoted to fp64; not modified).

    Returns dict(state=State fp64, impulses=(F,), wrench=(C,6), stats=(W,5),
    off, perm, foff, rc)."""
    inputs = inputs or Inputs()
    s = state.astype(np.float64).copy()
    W = s.n_worlds
    n = contacts.n
    inv_mass = _d(scene.inv_mass)
    inv_inertia = _d(scene.inv_inertia)
    sc = _Scene(scene.n_bodies, inv_mass.ctypes.data_as(ct.POINTER(ct.c_double)),
                inv_inertia.ctypes.data_as(ct.POINTER(ct.c_double)), scene.n_trees,
                scene.tree_ndof)
    c = _cfg(cfg)
    off, perm, foff = segment(contacts, W, cfg)
    F = int(foff[-1])
    imp = np.zeros(max(F, 1), np.float64)
    wr = np.zeros((max(n, 1), 6), np.float64)
    st = np.zeros((max(W, 1), 5), np.float64)
    c0, c1, c2 = _d(contacts.c0), _d(contacts.c1), _d(contacts.c2)
    ba, bb = _i(contacts.body_a), _i(contacts.body_b)
    mr, cd, wd = _d(contacts.mu_rol), _i(contacts.condim), _i(contacts.world)
    jr = _d(contacts.jrow)
    kd = _d(getattr(contacts, "kd", None))
    fe, tl, tt = _d(inputs.f_ext), _d(inputs.tree_L), _d(inputs.tree_tau)
    rc = _load().orc_step(ct.byref(c), ct.byref(sc), W,
                          _p(s.pos), _p(s.quat), _p(s.vel), _p(s.omega), _p(s.qpos), _p(s.qvel),
                          _p(fe), _p(tl), _p(tt), n, _p(wd), _p(c0), _p(c1), _p(c2),
                          _p(ba), _p(bb), _p(mr), _p(cd), _p(jr), _p(kd), _p(imp), _p(wr), _p(st),
                          int(n_threads))
    if rc == 1 or (strict and rc != 0):
        raise OracleError(f"orc_step failed rc={rc}")
    return dict(state=s, impulses=imp[:F], wrench=wr[:n], stats=st[:W], off=off, perm=perm,
                foff=foff, rc=rc)
