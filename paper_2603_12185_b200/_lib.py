"""ctypes binding of include/comfree.h (argument marshalling only).

Every step of the contact-resolution path runs in libcomfree.so's CUDA
kernels; this module only converts numpy arrays / torch tensors to the ABI's
pointers and sizes.  There is no CPU fallback: if the library is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes as ct
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcomfree.so")
# tuning experiments only: a variant build of the same sources (build.py --variant)
if os.environ.get("COMFREE_LIB"):
    LIB_PATH = os.path.abspath(os.environ["COMFREE_LIB"])

COMFREE_OK = 0
STATUS_NAMES = {0: "OK", 1: "ERR_INVALID_ARGUMENT", 2: "ERR_VALIDATION", 3: "ERR_CAPACITY",
                4: "ERR_NONFINITE", 5: "ERR_CUDA", 6: "ERR_STATE"}
MEM_DEVICE, MEM_HOST, MEM_HOST_ASYNC = 0, 1, 2
FLAG_STATS, FLAG_DETERMINISTIC, FLAG_NO_FINITE_CHECK, FLAG_EXACT_DIAGONAL, FLAG_FACET_DIAGONAL = 1, 2, 4, 8, 16
CONTACTS_SORTED = 1


class comfree_config(ct.Structure):
    _fields_ = [("k_user", ct.c_float), ("d_user", ct.c_float), ("r_min", ct.c_float),
                ("r_max", ct.c_float), ("width", ct.c_float), ("midpoint", ct.c_float),
                ("power", ct.c_float), ("n_t", ct.c_int32), ("n_rol", ct.c_int32),
                ("gravity", ct.c_float * 3), ("flags", ct.c_uint32)]


class comfree_scene(ct.Structure):
    _fields_ = [("n_bodies", ct.c_int32), ("inv_mass", ct.c_void_p), ("inv_inertia", ct.c_void_p),
                ("n_trees", ct.c_int32), ("tree_ndof", ct.c_int32)]


class comfree_state(ct.Structure):
    _fields_ = [("pos", ct.c_void_p), ("quat", ct.c_void_p), ("vel", ct.c_void_p),
                ("omega", ct.c_void_p), ("qpos", ct.c_void_p), ("qvel", ct.c_void_p),
                ("location", ct.c_int32)]


class comfree_articulation(ct.Structure):
    _fields_ = [("n_trees", ct.c_int32), ("tree_ndof", ct.c_int32), ("base", ct.c_void_p), ("axis", ct.c_void_p),
                ("length", ct.c_void_p), ("mass", ct.c_void_p), ("inertia", ct.c_void_p),
                ("armature", ct.c_void_p)]


class comfree_geometry(ct.Structure):
    _fields_ = [("n_geoms", ct.c_int32), ("n_pairs", ct.c_int32), ("kind", ct.c_void_p), ("body", ct.c_void_p),
                ("link", ct.c_void_p), ("size", ct.c_void_p), ("local", ct.c_void_p), ("pairs", ct.c_void_p),
                ("margin", ct.c_float), ("mu", ct.c_float * 3), ("condim", ct.c_int32)]


class comfree_mppi_task(ct.Structure):
    _fields_ = [("object_body", ct.c_int32), ("target_pos", ct.c_void_p), ("target_quat", ct.c_void_p),
                ("q_ref", ct.c_void_p), ("w", ct.c_float * 6), ("omega_fallen", ct.c_float), ("z_fallen", ct.c_float),
                ("phi1", ct.c_float), ("phi2", ct.c_float)]


class comfree_worlds(ct.Structure):
    _fields_ = [("first_world", ct.c_int64), ("n_worlds", ct.c_int64), ("f_ext", ct.c_void_p),
                ("tree_L", ct.c_void_p), ("tree_tau", ct.c_void_p), ("location", ct.c_int32)]


class comfree_contacts(ct.Structure):
    _fields_ = [("n_contacts", ct.c_int64), ("world", ct.c_void_p), ("off", ct.c_void_p),
                ("c0", ct.c_void_p), ("c1", ct.c_void_p), ("c2", ct.c_void_p), ("c3", ct.c_void_p),
                ("jrow", ct.c_void_p), ("kd", ct.c_void_p), ("impulses", ct.c_void_p), ("foff", ct.c_void_p),
                ("impulses_capacity", ct.c_int64), ("flags", ct.c_uint32), ("location", ct.c_int32),
                ("n_device", ct.c_void_p)]


class comfree_stats(ct.Structure):
    _fields_ = [("n_worlds", ct.c_int64), ("contacts", ct.c_int64), ("active_facets", ct.c_int64),
                ("max_penetration", ct.c_float), ("kinetic_energy", ct.c_double),
                ("first_nonfinite_world", ct.c_int64)]


class comfree_world_stats(ct.Structure):
    _fields_ = [("contacts", ct.c_int32), ("active_facets", ct.c_int32),
                ("max_penetration", ct.c_float), ("kinetic_energy", ct.c_float)]


# exported symbols and their signatures (kept in the order of comfree.h)
P = ct.c_void_p
SIGNATURES = {
    "comfree_abi_version": (ct.c_int, []),
    "comfree_status_string": (ct.c_char_p, [ct.c_int]),
    "comfree_default_config": (ct.c_int, [ct.POINTER(comfree_config)]),
    "comfree_validate_config": (ct.c_int, [ct.POINTER(comfree_config)]),
    "comfree_validate_scene": (ct.c_int, [ct.POINTER(comfree_scene)]),
    "comfree_facets_per_contact": (ct.c_int32, [ct.POINTER(comfree_config), ct.c_int32]),
    "comfree_create": (ct.c_int, [ct.POINTER(comfree_config), ct.c_int, ct.POINTER(P)]),
    "comfree_load_scene": (ct.c_int, [P, ct.POINTER(comfree_scene), ct.c_int64, ct.POINTER(comfree_state)]),
    "comfree_step": (ct.c_int, [P, ct.POINTER(comfree_worlds), ct.POINTER(comfree_contacts), ct.c_float, P]),
    "comfree_get_state": (ct.c_int, [P, ct.c_int64, ct.c_int64, ct.POINTER(comfree_state), P]),
    "comfree_set_state": (ct.c_int, [P, ct.c_int64, ct.c_int64, ct.POINTER(comfree_state), P]),
    "comfree_get_stats": (ct.c_int, [P, ct.POINTER(comfree_stats), P]),
    "comfree_load_articulation": (ct.c_int, [P, ct.POINTER(comfree_articulation)]),
    "comfree_load_geometry": (ct.c_int, [P, ct.POINTER(comfree_geometry)]),
    "comfree_mppi_sample": (ct.c_int, [P, ct.c_int32, ct.c_int32, ct.c_int32, P, ct.c_float, ct.c_float, ct.c_float,
                                       ct.c_uint64, ct.c_uint64, P, P]),
    "comfree_mppi_control": (ct.c_int, [P, ct.c_int64, ct.c_int64, P, ct.c_int32, ct.c_int32, ct.c_float, ct.c_float,
                                        P, P, P]),
    "comfree_mppi_cost": (ct.c_int, [P, ct.c_int64, ct.c_int64, ct.c_int32, ct.POINTER(comfree_mppi_task), ct.c_int32,
                                     P, P]),
    "comfree_mppi_cost_control": (ct.c_int, [P, ct.c_int64, ct.c_int64, ct.c_int32, ct.POINTER(comfree_mppi_task), P,
                                             P, ct.c_int32, ct.c_int32, ct.c_float, ct.c_float, P, P, P]),
    "comfree_mppi_update": (ct.c_int, [P, ct.c_int32, ct.c_int32, ct.c_int32, P, P, ct.c_float, ct.c_float, ct.c_float,
                                       P, P, P]),
    "comfree_mppi_update_shift": (ct.c_int, [P, ct.c_int32, ct.c_int32, ct.c_int32, P, P, ct.c_float, ct.c_float,
                                             ct.c_float, P, P, P, P]),
    "comfree_set_state_broadcast": (ct.c_int, [P, ct.c_int64, ct.c_int64, ct.c_int64, P, P]),
    "comfree_collide": (ct.c_int, [P, ct.c_int64, ct.c_int64, ct.c_int64, P, P, P, P, P, P, P, P, P]),
    "comfree_step_collided": (ct.c_int, [P, ct.POINTER(comfree_worlds), ct.c_int64, ct.c_float, P]),
    "comfree_articulation_update": (ct.c_int, [P, ct.c_int64, ct.c_int64, P, P, P, ct.c_int64, P, P, P, P, P, P, P]),
    "comfree_get_world_stats": (ct.c_int, [P, ct.c_int64, ct.c_int64, P, ct.c_int32, P]),
    "comfree_segment_info": (ct.c_int, [P, P, P, P]),
    "comfree_set_timing": (ct.c_int, [P, ct.c_int]),
    "comfree_get_timing": (ct.c_int, [P, ct.POINTER(ct.c_double)]),
    "comfree_check": (ct.c_int, [P, P]),
    "comfree_wait_async": (ct.c_int, [P, P]),
    "comfree_kernel_launches": (ct.c_int64, [P]),
    "comfree_destroy": (None, [P]),
    "comfree_last_error": (ct.c_char_p, [P]),
}

_lib = None


def load() -> ct.CDLL:
    """Load the in-tree libcomfree.so; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -m paper_2603_12185_b200.build` (there is no CPU fallback)")
        lib = ct.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
