#!/usr/bin/env python
"""Throughput of the B200 ComFree-Sim contact-resolution step (one JSON line).

Workload (BASELINE.json metric, config 4 "dense pile"): per GPU 1024 worlds x
500 free bodies (spheres / boxes / capsules) x 2000 contacts, condim 3, 4-facet
cone, dt = 0.002, synthetic seeded inputs (harness/scenes.py c4_pile).  One
step = S0 (world offsets from the sorted world ids) + the fused S1-S7 kernel,
inputs resident in HBM; the per-step footprint (184 MB) exceeds the 126 MB L2
and L2 is additionally flushed between timed steps.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N   (weak scaling: 1024 worlds per GPU)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "world-steps/s (dense pile, 1024 worlds x 2000 contacts per GPU)"
BYTES_PER_CONTACT = 68      # c0..c3 float4 streams (64 B) + the world id read by fused S0
BYTES_PER_BODY = 104        # 52 B state read + 52 B written


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--worlds", type=int, default=None, help="worlds per GPU (pile 1024, hand 4096)")
    ap.add_argument("--contacts", type=int, default=2000, help="contacts per world")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="direct launches instead of CUDA-graph replay")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the multi-rank path on a single GPU")
    ap.add_argument("--workload", default="pile", choices=["pile", "hand"],
                    help="pile: config 4 (the BASELINE metric); hand: config 3")
    a = ap.parse_args()
    if a.worlds is None:
        a.worlds = 4096 if a.workload == "hand" else 1024
    return a


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) during the timed region."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {getattr(nv, k): k for k in dir(nv) if k.startswith("nvmlClocksEventReason")
                 and isinstance(getattr(nv, k), int)} if nv else {}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if bit and (r & bit) == bit and name not in ("nvmlClocksEventReasonNone",
                                                                 "nvmlClocksEventReasonAll",
                                                                 "nvmlClocksEventReasonGpuIdle"):
                        self.reasons.add(name.replace("nvmlClocksEventReason", ""))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per launch of the fused step kernel from the committed ncu
    --set full capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "step_kernel_traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


# ---------------------------------------------------------------- oracle (CPU) timing
def cpu_oracle_rate(scene, st, contacts, cfg, seconds: float, max_worlds: int, inputs=None):
    """The fp64 oracle as it stands, OpenMP across worlds on all host cores,
    repeated steps over a bounded sample of the workload's worlds."""
    import oracle
    W = min(max_worlds, st.n_worlds)
    sel = np.nonzero(contacts.world < W)[0]
    c = contacts.take(sel)
    s = st.world_slice(0, W)
    inp = None
    if inputs is not None:
        from harness.types import Inputs
        inp = Inputs(*(None if a is None else np.ascontiguousarray(a[:W]) for a in
                       (inputs.f_ext, inputs.tree_L, inputs.tree_tau)))
    cores = os.cpu_count() or 1
    oracle.step(cfg, scene, s, c, inp, n_threads=cores)   # warm
    n = 0
    t0 = time.perf_counter()
    while True:
        oracle.step(cfg, scene, s, c, inp, n_threads=cores)
        n += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    return dict(value=n * W / dt, unit="world-steps/s", cores=cores, kind="oracle",
                sample=f"{n} oracle steps x {W} worlds of the same workload ({c.n} contacts), fp64, "
                       f"{dt:.1f} s, OpenMP over worlds")


# ---------------------------------------------------------------- main arms
def run_reference(args, rank, world_size):
    from harness import scenes
    from harness.types import Config
    if rank != 0:
        return
    cfg = Config()
    W = args.worlds
    scene, st, c = scenes.c4_pile(n_worlds=W, contacts_per_world=args.contacts)
    import oracle
    cores = os.cpu_count() or 1
    # each step: a bounded sample of the workload (64 worlds) so K steps finish in minutes
    Ws = min(64, W)
    sel = np.nonzero(c.world < Ws)[0]
    cs = c.take(sel)
    ss = st.world_slice(0, Ws)
    for _ in range(args.warmup):
        ss = oracle.step(cfg, scene, ss, cs, None, n_threads=cores)["state"].astype(np.float32)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ss = oracle.step(cfg, scene, ss, cs, None, n_threads=cores)["state"].astype(np.float32)
    dt = time.perf_counter() - t0
    v = args.steps * Ws / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "world-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c4 dense pile", "worlds_per_gpu": W, "contacts_per_world": args.contacts,
                       "bodies_per_world": 500, "facets_per_contact": 4, "dt": cfg.dt,
                       "sample_worlds_per_step": Ws},
            "cpu_baseline": {"value": v, "unit": "world-steps/s", "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} steps x {Ws} of {W} worlds, fp64 oracle, OpenMP over worlds"},
            "e2e": {"value": v, "unit": "world-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def kernels_per_step(ctx, dc, tin, cfg):
    """Kernels one direct step launches (instrumentation counter of the library)."""
    n0 = ctx.kernel_launches
    ctx.step(dc, tin, dt=cfg.dt)
    import torch
    torch.cuda.synchronize()
    return ctx.kernel_launches - n0


def workload(args, rank):
    """(scene, state, contacts, inputs, name, algorithmic bytes per step per GPU)."""
    from harness import scenes
    W = args.worlds
    if args.workload == "hand":
        scene, st, c, inp = scenes.c3_hand(n_worlds=W, world_offset=rank * W)
        n_rows = int(np.count_nonzero(c.body_a < -1) + np.count_nonzero(c.body_b < -1))
        Q = scene.n_tree_dofs
        alg = (c.n * BYTES_PER_CONTACT + n_rows * 96 + W * scene.n_bodies * BYTES_PER_BODY
               + W * (Q * 16 + scene.n_trees * 40 + Q * 4))
        return scene, st, c, inp, "c3 LEAP-like hand + cube (4x4-DoF chains + free cube)", alg
    scene, st, c = scenes.c4_pile(n_worlds=W, contacts_per_world=args.contacts, world_offset=rank * W)
    alg = W * (args.contacts * BYTES_PER_CONTACT + scene.n_bodies * BYTES_PER_BODY)
    return scene, st, c, None, "c4 dense pile", alg


def run_ours(args, rank, world_size, local):
    import torch
    import torch.distributed as dist
    import paper_2603_12185_b200 as cf
    from paper_2603_12185_b200.dist import all_gather_worlds, reduce_max, uniform_ranges
    from harness.types import Config

    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world_size > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:                              # plumbing check with several ranks on one GPU
            dist.init_process_group(args.dist_backend)
    cfg = Config()
    W = args.worlds
    scene, st, c, inp, wname, alg_bytes = workload(args, rank)
    ctx = cf.Context(cfg, device=local)
    ctx.load_scene(scene, W, st)
    dc = cf.DeviceContacts.from_host(c, dev)
    assert dc.sorted
    tin = None
    if inp is not None:
        tin = type(inp)(*(None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                          for a in (inp.f_ext, inp.tree_L, inp.tree_tau)))
    stream = torch.cuda.current_stream()
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def one_step():
        ctx.step(dc, tin, dt=cfg.dt, stream=stream)

    for _ in range(max(args.warmup, 3)):
        one_step()
    torch.cuda.synchronize()
    # direct launches with the library's own event timing around the fused kernel
    ctx.get_timing()
    ctx.set_timing(True)
    for _ in range(min(args.steps, 20)):
        if flush is not None:
            flush.zero_()
        one_step()
    kt = ctx.get_timing()
    ctx.set_timing(False)
    k_ms_direct = kt["step_ms"] / max(kt["step_launches"], 1)
    # one step captured in a CUDA graph (no host launch path inside the timed region)
    graph = None
    if not args.no_graph:
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            ctx.step(dc, tin, dt=cfg.dt, stream=side)
        stream.wait_stream(side)
        torch.cuda.synchronize()
    launches0 = ctx.kernel_launches
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world_size > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clock = ClockSampler(local)
    with clock:
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()              # evict L2 between timed steps (untimed)
            evs[i][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                one_step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world_size > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))
    # kernels per step: one fused kernel (S0 fused for sorted ids); counted by the
    # library for direct launches, the same for each graph replay
    launches = (ctx.kernel_launches - launches0) if graph is None else args.steps * kernels_per_step(ctx, dc, tin, cfg)
    total_ms = reduce_max(total_ms, dev)   # the job is as slow as its slowest rank
    ms_per_step = total_ms / args.steps
    world_steps = W * world_size * args.steps
    value = world_steps / (total_ms * 1e-3)
    contacts_per_s = value * (c.n / W)

    # roofline of the dominant kernel: with one kernel per step the per-step CUDA
    # events around the graph replay bracket exactly that kernel
    k_ms = (total_ms / args.steps) if graph is not None else k_ms_direct
    peak, peak_kind = peaks()
    achieved = alg_bytes / (k_ms * 1e-3) / 1e9
    tr = ncu_traffic()
    traffic = None
    if tr and tr.get("workload") == args.workload and tr.get("worlds") == W and \
            tr.get("contacts_per_world") == c.n // W:
        traffic = tr.get("dram_bytes_per_launch")

    # after the timed region: final states all-gathered (NCCL) for verification
    final = ctx.get_state()
    finite = bool(np.isfinite(final["vel"]).all() and np.isfinite(final["pos"]).all())
    gathered_mb = None
    if world_size > 1:
        ranges = uniform_ranges(W * world_size, world_size)
        loc = {k: torch.from_numpy(final[k]).to(dev) for k in ("pos", "quat", "vel", "omega")}
        full = all_gather_worlds(loc, ranges)
        gathered_mb = sum(v.numel() * v.element_size() for v in full.values()) / 1e6
        finite = bool(reduce_max(0.0 if finite else 1.0, dev) == 0.0)

    # e2e: the same metric through the C ABI with HOST buffers (pinned), H2D of the
    # step's contacts and D2H of the resulting state inside the timed region
    hc = cf.HostContacts.from_arrays(c, pin=True)
    e2e_steps = max(1, args.e2e_steps)
    ctx.step(hc, inp, dt=cfg.dt)           # warm the staging buffers
    out_host = {k: torch.empty(v.shape, dtype=torch.float32).pin_memory().numpy() for k, v in final.items()}
    from paper_2603_12185_b200 import _lib
    import ctypes as ct
    st_h = _lib.comfree_state(*[out_host[k].ctypes.data if out_host[k].size else None
                                for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")], _lib.MEM_HOST)
    if world_size > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        ctx.step(hc, inp, dt=cfg.dt, stream=stream)
        rc = ctx._lib.comfree_get_state(ctx.h, 0, W, ct.byref(st_h), stream.cuda_stream)
        ctx._check(rc, "comfree_get_state")
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = reduce_max(e0.elapsed_time(e1), dev)
    e2e_value = W * world_size * e2e_steps / (e2e_ms * 1e-3)
    h2d = hc.h2d_bytes() + (0 if inp is None else sum(a.nbytes for a in (inp.f_ext, inp.tree_L, inp.tree_tau)
                                                      if a is not None))
    d2h = sum(v.nbytes for v in out_host.values())

    cpu = None
    if rank == 0 and world_size == 1:
        cpu = cpu_oracle_rate(scene, st, c, cfg, args.cpu_seconds, max_worlds=W, inputs=inp)
    if world_size > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC if args.workload == "pile" else "world-steps/s (LEAP-like hand + cube, 4096 worlds)",
            "value": value, "unit": "world-steps/s", "n_gpus": world_size,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": wname, "worlds_per_gpu": W, "contacts_per_world": c.n // W,
                       "bodies_per_world": scene.n_bodies, "chains_per_world": scene.n_trees,
                       "facets_per_contact": 4, "condim": 3, "dt": cfg.dt,
                       "l2": "flushed between timed steps (256 MB write)" if flush is not None else "not flushed",
                       "footprint_mb_per_step": alg_bytes / 1e6,
                       "parallelism": f"world-sharded x{world_size}"},
            "contacts_per_s": contacts_per_s,
            "gpu_launches": int(launches),
            "kernel_ms": {"fused_step": k_ms, "fused_step_direct_launch": k_ms_direct,
                          "segment_s0_separate": kt["segment_ms"] / max(kt["step_launches"], 1)},
            "cuda_graph": graph is not None,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "kernel": "k_step (S1-S7 fused)", "algorithmic_bytes_per_launch": alg_bytes},
            "clocks": clock.summary(),
            "e2e": {"value": e2e_value, "unit": "world-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps},
            "cpu_baseline": cpu,
            "allgather_final_state_mb": gathered_mb,
            "context": "paper: 2-3x MJWarp throughput in dense contact on one RTX 4090 (PAPER.md P:11, P:274); "
                       "full-step numbers, not this path alone",
            "final_state_finite": finite,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world_size > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world_size, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world_size)
        return
    run_ours(args, rank, world_size, local)


if __name__ == "__main__":
    main()
