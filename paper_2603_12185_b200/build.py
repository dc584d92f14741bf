"""Build libcomfree.so in-tree (sm_100a) with nvcc; no JIT, no torch extension.

    python -m paper_2603_12185_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libcomfree.so")
OBJDIR = os.path.join(HERE, "_build")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["step.cu", "step_w1.cu", "step_w2.cu", "step_w4.cu", "step_w8.cu", "step_w16.cu", "step_p32.cu", "segment.cu", "state.cu", "articulation.cu", "collide.cu", "mppi.cu"]
CPP_SOURCES = ["capi.cpp"]
# collide.cu: no FMA contraction, so the narrowphase's count and emit
# specialisations compute bit-identical contacts (collide.cu, CF_NP_INLINE)
PER_FILE_FLAGS = {"collide.cu": ["-fmad=false"]}


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), tag: str = "") -> str:
    """Build libcomfree.so; with `tag`, a variant (extra -D `defines`) into
    _build_<tag>/libcomfree_<tag>.so for tuning experiments (COMFREE_LIB)."""
    objdir = OBJDIR + ("_" + tag if tag else "")
    lib = os.path.join(objdir, f"libcomfree_{tag}.so") if tag else LIB
    dflags = [f"-D{d}" for d in defines]
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, "internal.h"), os.path.join(CSRC, "step_impl.cuh"), os.path.join(CSRC, "chain.cuh"),
               os.path.join(INCLUDE, "comfree.h")]
    objs = []
    jobs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC, *ARCH, *dflags, *PER_FILE_FLAGS.get(src, []), "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                         "-Xptxas", "-v" if verbose else "-O3", "-I", INCLUDE, "-I", CSRC, "-c", s, "-o", o])
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for rc in ex.map(lambda c: subprocess.run(c).returncode, jobs):
            if rc != 0:
                raise subprocess.CalledProcessError(rc, "nvcc")
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [NVCC, "-x", "cu", *ARCH, *dflags, "-O2", "-std=c++17", "-Xcompiler", "-fPIC,-Wall",
                   "-I", INCLUDE, "-I", CSRC, "-c", s, "-o", o]
            subprocess.check_call(cmd)
    if force or _stale(lib, objs):
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"])
    return lib


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--variant", default="", help="tag of a tuning variant build")
    ap.add_argument("-D", action="append", default=[], help="extra preprocessor define (variant builds)")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, defines=a.D, tag=a.variant))
