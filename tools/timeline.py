#!/usr/bin/env python
"""Per-CTA phase timeline of one C4 step (tuning diagnostic, GPU box only).

Needs a variant build with -DCF_TIMELINE:
    python -m paper_2603_12185_b200.build --variant tl -D CF_TIMELINE
    COMFREE_LIB=paper_2603_12185_b200/_build_tl/libcomfree_tl.so python tools/timeline.py --worlds 1024

Prints the kernel span, the start-time waves, the mean prologue (S0+S1) /
contact loop (S2-S6) / epilogue (S7) durations per wave, and per-SM busy time.
"""
from __future__ import annotations

import argparse
import ctypes as ct
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", type=int, default=1024)
    ap.add_argument("--contacts", type=int, default=2000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import paper_2603_12185_b200 as cf
    from paper_2603_12185_b200 import _lib
    from harness import scenes
    from harness.types import Config

    lib = _lib.load()
    fn = lib.comfree_debug_timeline
    fn.restype = ct.c_int
    fn.argtypes = [ct.c_void_p, ct.c_int64]
    cfg = Config()
    scene, st, c = scenes.c4_pile(n_worlds=a.worlds, contacts_per_world=a.contacts)
    ctx = cf.Context(cfg, device=0)
    ctx.load_scene(scene, a.worlds, st)
    dc = cf.DeviceContacts.from_host(c, torch.device("cuda", 0))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(5):
        ctx.step(dc, None, dt=cfg.dt)
    rows = []
    for rep in range(5):
        flush.zero_()
        ctx.step(dc, None, dt=cfg.dt)
        torch.cuda.synchronize()
        n = a.worlds  # one CTA per world (WPW = 8)
        buf = np.zeros((n, 8), np.uint32)
        assert fn(buf.ctypes.data, n) == 0
        rows.append(buf.copy())
    buf = rows[-1]
    sm = buf[:, 0].astype(int)
    t = buf[:, 1:7].astype(np.int64)
    t -= t[:, 0].min()
    t = np.where(t < 0, t + (1 << 32), t)
    srch, s1 = t[:, 4] - t[:, 0], t[:, 5] - t[:, 0]
    span = t[:, 3].max()
    pro, loop, epi = t[:, 1] - t[:, 0], t[:, 2] - t[:, 1], t[:, 3] - t[:, 2]
    out = []
    out.append(f"worlds {a.worlds} x {a.contacts} contacts; kernel span (first start -> last end) {span/1e3:.1f} us")
    out.append(f"CTA duration mean {np.mean(t[:,3]-t[:,0])/1e3:.1f} us; prologue {pro.mean()/1e3:.2f}, loop {loop.mean()/1e3:.2f}, epilogue {epi.mean()/1e3:.2f} us")
    order = np.argsort(t[:, 0])
    starts = t[order, 0]
    # waves: CTAs starting within 2 us of the first start are wave 0, later ones are refills
    w0 = starts < 2000
    out.append(f"prologue detail (from CTA start, thread 0): search done {srch.mean()/1e3:.2f} us, S1 loop done {s1.mean()/1e3:.2f} us, sync passed {pro.mean()/1e3:.2f} us")
    out.append(f"CTAs started in the first 2 us: {w0.sum()}; last start at {starts[-1]/1e3:.1f} us")
    for lo, hi in ((0, 2e3), (2e3, 1e9)):
        m = (t[:, 0] >= lo) & (t[:, 0] < hi)
        if m.any():
            out.append(f"  start in [{lo/1e3:.0f},{min(hi,span)/1e3:.0f}) us: {m.sum():4d} CTAs, dur {np.mean(t[m,3]-t[m,0])/1e3:.1f} us "
                       f"(pro {pro[m].mean()/1e3:.2f} loop {loop[m].mean()/1e3:.2f} epi {epi[m].mean()/1e3:.2f}), "
                       f"end {t[m,3].min()/1e3:.1f}..{t[m,3].max()/1e3:.1f} us")
    # resident CTAs over time (all SMs), 1 us bins
    bins = np.arange(0, span + 1000, 1000)
    res = np.array([np.sum((t[:, 0] <= b) & (t[:, 3] > b)) for b in bins])
    out.append("resident CTAs per us bin: " + " ".join(str(x) for x in res))
    smend = np.array([t[sm == s, 3].max() if np.any(sm == s) else 0 for s in range(sm.max() + 1)])
    out.append(f"per-SM last end: min {smend.min()/1e3:.1f} median {np.median(smend)/1e3:.1f} max {smend.max()/1e3:.1f} us")
    cnt = np.bincount(sm)
    out.append(f"CTAs per SM: min {cnt.min()} max {cnt.max()} hist {np.bincount(cnt).tolist()}")
    txt = "\n".join(out)
    print(txt)
    if a.out:
        np.save(a.out, np.stack(rows))


if __name__ == "__main__":
    main()
