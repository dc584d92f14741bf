"""C ABI checks that need no GPU: the library loads, exports every symbol
include/comfree.h declares, the ctypes structs match the C layout, and the
host-side validation answers as documented."""
from __future__ import annotations

import ctypes as ct
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "comfree.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2603_12185_b200 import build
    from paper_2603_12185_b200 import _lib
    build()
    return _lib.load()


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(comfree_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    from paper_2603_12185_b200 import _lib
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_lib.SIGNATURES) == names
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_struct_layouts_match_c(tmp_path):
    from paper_2603_12185_b200 import _lib
    src = tmp_path / "sz.c"
    structs = ["comfree_config", "comfree_scene", "comfree_state", "comfree_worlds", "comfree_contacts",
               "comfree_stats", "comfree_world_stats"]
    body = "".join(f'printf("%zu\\n", sizeof({s}));' for s in structs)
    src.write_text(f'#include <stdio.h>\n#include "comfree.h"\nint main(void){{{body} return 0;}}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    sizes = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    for s, n in zip(structs, sizes):
        assert ct.sizeof(getattr(_lib, s)) == n, s


def test_abi_version_and_status_strings(lib):
    assert lib.comfree_abi_version() == 2
    for s in range(7):
        assert lib.comfree_status_string(s)


def test_default_config_matches_paper(lib):
    from paper_2603_12185_b200 import _lib
    c = _lib.comfree_config()
    assert lib.comfree_default_config(ct.byref(c)) == 0
    assert (c.k_user, c.r_min, c.r_max, c.width, c.midpoint, c.power) == pytest.approx(
        (0.1, 0.9, 0.95, 0.001, 0.5, 2.0))
    assert c.n_t == 4 and c.n_rol == 4
    assert lib.comfree_validate_config(ct.byref(c)) == 0


@pytest.mark.parametrize("field,value", [("k_user", 0.0), ("d_user", -1.0), ("r_min", 0.0),
                                         ("r_max", 1.0), ("width", 0.0), ("midpoint", 1.0),
                                         ("power", 0.5), ("n_t", 5), ("n_t", 2), ("n_rol", 3),
                                         ("n_t", 34), ("k_user", float("nan"))])
def test_invalid_config_rejected(lib, field, value):
    from paper_2603_12185_b200 import _lib
    c = _lib.comfree_config()
    lib.comfree_default_config(ct.byref(c))
    setattr(c, field, value)
    if field == "r_min" and value == 0.0:
        pass
    assert lib.comfree_validate_config(ct.byref(c)) == 2


def test_r_min_above_r_max_rejected(lib):
    from paper_2603_12185_b200 import _lib
    c = _lib.comfree_config()
    lib.comfree_default_config(ct.byref(c))
    c.r_min, c.r_max = 0.96, 0.95
    assert lib.comfree_validate_config(ct.byref(c)) == 2


def test_facets_per_contact(lib):
    from paper_2603_12185_b200 import _lib
    c = _lib.comfree_config()
    lib.comfree_default_config(ct.byref(c))
    c.n_t, c.n_rol = 8, 6
    assert [lib.comfree_facets_per_contact(ct.byref(c), k) for k in (1, 3, 4, 6, 2, 5)] == [1, 8, 10, 16, -1, -1]


def test_validate_scene(lib):
    from paper_2603_12185_b200 import _lib
    im = np.array([1.0, 0.0], np.float32)
    iI = np.ones((2, 3), np.float32)
    s = _lib.comfree_scene(2, im.ctypes.data, iI.ctypes.data, 0, 4)
    assert lib.comfree_validate_scene(ct.byref(s)) == 0
    im[1] = -1.0
    assert lib.comfree_validate_scene(ct.byref(s)) == 2
    im[1] = 1.0
    s.n_trees, s.tree_ndof = 2, 5
    assert lib.comfree_validate_scene(ct.byref(s)) == 2
    s2 = _lib.comfree_scene(2, None, None, 0, 4)
    assert lib.comfree_validate_scene(ct.byref(s2)) == 1


def test_null_arguments_are_invalid(lib):
    assert lib.comfree_default_config(None) == 1
    assert lib.comfree_validate_config(None) == 1
    assert lib.comfree_step(None, None, None, 0.002, None) == 1
    assert lib.comfree_get_state(None, 0, 0, None, None) == 1
    assert lib.comfree_kernel_launches(None) == -1
    lib.comfree_destroy(None)


def test_create_fails_cleanly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_12185_b200 import _lib
    c = _lib.comfree_config()
    lib.comfree_default_config(ct.byref(c))
    h = ct.c_void_p()
    assert lib.comfree_create(ct.byref(c), 0, ct.byref(h)) == 5
    assert not h.value


def test_product_path_has_no_oracle_dependency():
    """The product package must not import, link or execute the oracle."""
    pkg = os.path.join(ROOT, "paper_2603_12185_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.lower() or f == "__init__.py" and "oracle" not in txt, f
