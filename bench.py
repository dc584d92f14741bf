#!/usr/bin/env python
"""Throughput of the B200 ComFree-Sim contact-resolution step (one JSON line).

Workload (BASELINE.json metric, config 4 "dense pile"): per GPU 1024 worlds x
500 free bodies (spheres / boxes / capsules) x 2000 contacts, condim 3, 4-facet
cone, dt = 0.002, synthetic seeded inputs (harness/scenes.py c4_pile).  One
step = S0 (world offsets from the sorted world ids) + the fused S1-S7 kernel,
inputs resident in HBM and pre-segmented (the caller passes off[W+1], so S0 is
skipped); the per-step footprint (184.3 MB = 1024 x (2000 x 64 B
+ 500 x 104 B)) exceeds the 126 MB L2 and L2 is additionally
flushed between timed steps.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N   (weak scaling: 1024 worlds per GPU)

Other workloads (reported, not the BASELINE metric): --workload hand (config 3,
4096 worlds per GPU) and --workload mixed (config 5: 65536 worlds in total,
half hand / half pile-lite, sharded over the GPUs -- strong scaling; the two
world kinds are two library contexts stepped concurrently on two streams).
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
BYTES_PER_CONTACT = 64      # c0..c3 float4 streams; pre-segmented: no world-id stream
BYTES_PER_BODY = 104        # 52 B state read + 52 B written


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--worlds", type=int, default=None, help="worlds per GPU (pile 1024, hand 4096)")
    ap.add_argument("--contacts", type=int, default=2000, help="contacts per world")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--flush-mode", default="write+read", choices=["write", "write+read"],
                    help="L2 flush between timed steps: write 256 MB (leaves L2 full of dirty lines whose "
                         "write-back the next step pays), or write then read it back (cold, clean L2)")
    ap.add_argument("--no-graph", action="store_true", help="direct launches instead of CUDA-graph replay")
    ap.add_argument("--reset-state", action="store_true",
                    help="restore the initial state before every step (untimed, with the L2 flush): for variants "
                         "whose dynamics do not stay bounded over hundreds of steps of the same contact set "
                         "(e.g. --impedance exact_diagonal, Eq. (11) per facet, reading R24)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the multi-rank path on a single GPU")
    ap.add_argument("--condim", type=int, default=3, choices=[1, 3, 4, 6],
                    help="pile contact dimensionality (3: the BASELINE config; 6: the 6D variant, n_t = n_rol = 4)")
    ap.add_argument("--kd", action="store_true",
                    help="per-contact (k_user, d_user) impedance arrays (learned-impedance variant, P:206-208)")
    ap.add_argument("--impedance", default="heuristic", choices=["heuristic", "exact_diagonal", "facet_diagonal"],
                    help="exact_diagonal: Eq. (11) per facet (reading R24); facet_diagonal: Eq. (12) with the "
                         "facet diagonal (reading R28); default: the trace heuristic of Eq. (12)")
    ap.add_argument("--nt", type=int, default=4, help="tangential facets per contact (even, >= 4)")
    ap.add_argument("--nrol", type=int, default=4, help="rolling facets per contact at condim 6 (even)")
    ap.add_argument("--world-ids", action="store_true",
                    help="pass sorted world ids instead of off[W+1] (S0 fused into the step; +4 B per contact)")
    ap.add_argument("--upstream", action="store_true",
                    help="hand / mixed: run the articulated upstream (FK, M(q), Cholesky, c(q,v), chain J rows) "
                         "on the GPU every step before the contact resolution (SURVEY 8(f) rank 2)")
    ap.add_argument("--collide", action="store_true",
                    help="closed loop: the GPU collision front-end (SURVEY 8(f) rank 1) builds the contacts every "
                         "step (count kept on the device); hand: then the upstream and the step (implies --upstream); "
                         "pile: lattice-neighbour candidate pairs, then the step (the full-step metric, P:389-390)")
    ap.add_argument("--pair-list", action="store_true",
                    help="with --collide on the pile: the fixed lattice-neighbour candidate list instead of the "
                         "per-step broadphase")
    ap.add_argument("--split-collide", action="store_true",
                    help="with --collide on the pile (broadphase): comfree_collide + comfree_step (public contact "
                         "streams) instead of comfree_step_collided (the step reads the front-end's staged records)")
    ap.add_argument("--workload", default="pile", choices=["pile", "hand", "mixed"],
                    help="pile: config 4 (the BASELINE metric); hand: config 3; mixed: config 5")
    a = ap.parse_args(argv)
    if a.collide and a.workload != "pile":
        a.upstream = True              # closed-loop hands: collide -> upstream -> step
    if a.worlds is None:
        a.worlds = {"hand": 4096, "mixed": 65536}.get(a.workload, 1024)
    return a


METRICS = {"pile": METRIC,
           "hand": "world-steps/s (LEAP-like hand + cube, 4096 worlds per GPU)",
           "mixed": "world-steps/s (mixed hand + pile-lite, 65536 worlds in total)"}


def facets(args) -> int:
    """Facets per contact of the pile's condim (reading R11): 1, n_t, n_t + 2, n_t + 2 + n_rol."""
    return {1: 1, 3: args.nt, 4: args.nt + 2, 6: args.nt + 2 + args.nrol}[args.condim]


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


# ---------------------------------------------------------------- workloads
class Part:
    """One homogeneous batch of worlds (one library context)."""

    def __init__(self, name, scene, st, c, inp, alg_bytes):
        self.name, self.scene, self.st, self.c, self.inp, self.alg_bytes = name, scene, st, c, inp, alg_bytes
        self.W = st.n_worlds


def _hand_bytes(scene, c, W):
    n_rows = int(np.count_nonzero(c.body_a < -1) + np.count_nonzero(c.body_b < -1))
    Q = scene.n_tree_dofs
    return (c.n * BYTES_PER_CONTACT + n_rows * 96 + W * scene.n_bodies * BYTES_PER_BODY
            + W * (Q * 16 + scene.n_trees * 40 + Q * 4))


def workload(args, rank, world_size):
    """(parts, workload name, worlds per rank) -- parts are homogeneous batches."""
    parts, name, n = _workload(args, rank, world_size)
    if args.kd:                      # per-contact impedance: 8 more bytes per contact
        for p in parts:
            rng = np.random.default_rng([260312185, 11, rank])
            p.c.kd = np.stack([rng.uniform(0.05, 0.3, p.c.n), rng.uniform(0.0, 0.002, p.c.n)], 1).astype(np.float32)
            p.alg_bytes += 8 * p.c.n
        name += " + per-contact impedance"
    if args.impedance == "exact_diagonal":
        name += " + exact-diagonal impedance (Eq. 11)"
    elif args.impedance == "facet_diagonal":
        name += " + facet-diagonal impedance (Eq. 12 with the facet diagonal)"
    if args.upstream:
        name += " + articulated upstream on the GPU every step"
    if args.collide:
        name += " + GPU collision front-end every step (closed loop)"
        if args.workload == "pile":
            name += (" (fixed lattice-neighbour candidate list)" if args.pair_list else
                     " (sort-and-sweep broadphase + narrowphase, one kernel)") + \
                "; contacts from geometry, not the generator's"
            if not args.pair_list:
                name += ("; comfree_collide + comfree_step (public contact streams)" if args.split_collide else
                         "; comfree_step_collided (the step reads the front-end's staged records, no emit pass)")
    return parts, name, n


# World generators by global world id (harness/scenes.py seeds world g from
# (260312185, ..., g), so a world's bytes do not depend on the rank holding it).
# kind: "pile" (C4), "hand" (C3), and C5's "pile-lite" / "hand5" (seed 5).
UNIQUE = {"pile": 1 << 30, "hand": 1 << 30, "pile-lite": 4096, "hand5": 1024}


def gen_worlds(args, kind, first, count):
    """(scene, state, contacts, inputs) of global worlds [first, first + count)
    of one kind; at most UNIQUE[kind] distinct worlds are generated and tiled
    (local world k is a copy of global world first + k mod U)."""
    from harness import scenes
    U = max(1, min(count, UNIQUE[kind]))
    if kind in ("hand", "hand5"):
        scene, st, c, inp = scenes.c3_hand(n_worlds=U, seed=5 if kind == "hand5" else 0, world_offset=first)
    elif kind == "pile-lite":
        scene, st, c = scenes.c4_pile(n_worlds=U, contacts_per_world=400, lattice=(5, 5, 4), seed=5,
                                      world_offset=first)
        inp = None
    else:
        scene, st, c = scenes.c4_pile(n_worlds=U, contacts_per_world=args.contacts, world_offset=first,
                                      condim=args.condim)
        inp = None
    if count != U:
        st, c, inp = scenes.tile_worlds(st, c, inp, count)
    return scene, st, c, inp


def gen_copy_source(kind, first, local):
    """Global id of the generated world that local world `local` of a part
    starting at `first` copies (tiling, gen_worlds)."""
    return first + local % max(1, UNIQUE[kind])


def shard_plan(args, world_size):
    """Per rank, per part kind: (first global id, count).  Weak scaling (pile,
    hand): args.worlds per rank, rank r holding ids [r W, (r + 1) W).  C5
    (strong scaling): one global sequence of args.worlds worlds alternating
    pile-lite (even positions) and hand (odd), split into contiguous ranges
    balanced by per-world bytes 64 C_w + 104 B_w (+ chain rows for hands,
    SURVEY §8(e)) with dist.shard_ranges."""
    from paper_2603_12185_b200.dist import shard_ranges
    if args.workload != "mixed":
        kind = "hand" if args.workload == "hand" else "pile"
        W = args.worlds
        return [{kind: (r * W, W)} for r in range(world_size)]
    n = args.worlds
    cost_pile = 400 * BYTES_PER_CONTACT + 100 * BYTES_PER_BODY
    cost_hand = 20 * BYTES_PER_CONTACT + 16 * 96 + BYTES_PER_BODY + 16 * 16 + 4 * 40 + 16 * 4
    costs = np.where(np.arange(n) % 2 == 0, cost_pile, cost_hand).astype(np.float64)
    plan = []
    for lo, hi in shard_ranges(costs, world_size):
        pf, pl = (lo + 1) // 2, (hi + 1) // 2          # even positions -> pile-lite ids
        hf, hl = lo // 2, hi // 2                      # odd positions -> hand ids
        plan.append({"pile-lite": (pf, pl - pf), "hand5": (hf, hl - hf)})
    return plan


def _workload(args, rank, world_size):
    plan = shard_plan(args, world_size)[rank]
    parts = []
    for kind, (first, count) in plan.items():
        scene, st, c, inp = gen_worlds(args, kind, first, count)
        if kind in ("hand", "hand5"):
            ab = _hand_bytes(scene, c, count)
        else:
            ab = c.n * BYTES_PER_CONTACT + count * scene.n_bodies * BYTES_PER_BODY
        p = Part({"hand5": "hand"}.get(kind, kind), scene, st, c, inp, ab)
        p.kind, p.first = kind, first
        parts.append(p)
    n = sum(p.W for p in parts)
    if args.workload == "hand":
        return parts, "c3 LEAP-like hand + cube (4x4-DoF chains + free cube)", n
    if args.workload == "mixed":
        return parts, "c5 mixed: half c3 hand, half pile-lite (100 bodies, 400 contacts), cost-weighted shards", n
    return parts, "c4 dense pile" + ("" if args.condim == 3 else f" (condim {args.condim})") + \
        ("" if (args.nt, args.nrol) == (4, 4) else f" (n_t {args.nt}, n_rol {args.nrol}: {facets(args)} facets)"), n


# ---------------------------------------------------------------- multi-rank verification
def verify_shards(args, parts, finals, rank, world_size, n_steps, stepper, device=None, samples_per_rank=2):
    """After the timed region: all-gather every part's final states (NCCL, or
    gloo on CPU) into global world order, and on rank 0 re-run sampled worlds
    -- the first and last world of every rank's range -- alone (one world per
    call, `stepper(part, scene, st, c, inp, n_steps) -> dict of final arrays`)
    and compare bit for bit: per-world arithmetic does not depend on the
    sharding, and the step is deterministic (fixed-point S6).  Returns
    (gathered MB, report dict on rank 0 / None)."""
    import torch
    from paper_2603_12185_b200.dist import all_gather_worlds
    plan = shard_plan(args, world_size)
    keys = ("pos", "quat", "vel", "omega", "qpos", "qvel")
    mb = 0.0
    report = {"checked_worlds": 0, "bitwise_equal": True, "n_steps": int(n_steps), "mismatch": []}
    for p in parts:
        ranges = []
        for r in range(world_size):
            f, cnt = plan[r][p.kind]
            ranges.append((f - plan[0][p.kind][0], f - plan[0][p.kind][0] + cnt))
        loc = {k: torch.from_numpy(np.ascontiguousarray(finals[p.name][k])).to(device or "cpu") for k in keys}
        full = all_gather_worlds(loc, ranges)
        mb += sum(v.numel() * v.element_size() for v in full.values()) / 1e6
        if rank != 0:
            continue
        full = {k: v.cpu().numpy() for k, v in full.items()}
        for r in range(world_size):
            f, cnt = plan[r][p.kind]
            for local in (sorted({0, cnt - 1})[:samples_per_rank] if cnt and stepper is not None else []):
                src = gen_copy_source(p.kind, f, local)
                scene, st, c, inp = gen_worlds(args, p.kind, src, 1)
                one = stepper(p, scene, st, c, inp, n_steps)
                g = (f - plan[0][p.kind][0]) + local
                same = all(np.array_equal(np.asarray(one[k]).reshape(full[k][g].shape), full[k][g]) for k in keys)
                report["checked_worlds"] += 1
                if not same:
                    report["bitwise_equal"] = False
                    report["mismatch"].append({"part": p.name, "rank": r, "local": int(local)})
    return mb, (report if rank == 0 else None)


# ---------------------------------------------------------------- oracle (CPU) timing
def _sample(part, max_worlds):
    from harness.types import Inputs
    W = min(max_worlds, part.W)
    c = part.c.take(np.nonzero(part.c.world < W)[0])
    st = part.st.world_slice(0, W)
    inp = None
    if part.inp is not None:
        inp = Inputs(*(None if a is None else np.ascontiguousarray(a[:W]) for a in
                       (part.inp.f_ext, part.inp.tree_L, part.inp.tree_tau)))
    return W, st, c, inp


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_rate(parts, cfg, seconds, max_worlds, threads):
    import oracle
    samples = [(p, _sample(p, max_worlds)) for p in parts]
    for p, (W, st, c, inp) in samples:
        oracle.step(cfg, p.scene, st, c, inp, n_threads=threads)   # warm
    n = 0
    t0 = time.perf_counter()
    while True:
        for p, (W, st, c, inp) in samples:
            oracle.step(cfg, p.scene, st, c, inp, n_threads=threads)
        n += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    Ws = sum(x[1][0] for x in samples)
    nc = sum(x[1][2].n for x in samples)
    return n * Ws / dt, n, Ws, nc, dt


def cpu_oracle_rate(parts, cfg, seconds: float, max_worlds: int):
    """The fp64 oracle as it stands, timed twice on the host: OpenMP across
    worlds on all host cores (`value`, `cores`), and on one core, each over
    repeated steps of a bounded sample of each part's worlds."""
    cores = os.cpu_count() or 1
    v, n, Ws, nc, dt = _oracle_rate(parts, cfg, seconds, max_worlds, cores)
    v1, n1, Ws1, nc1, dt1 = _oracle_rate(parts, cfg, 0.5 * seconds, max(1, max_worlds // 8), 1)
    return dict(value=v, unit="world-steps/s", cores=cores, kind="oracle", cpu_model=cpu_model(),
                all_cores={"value": v, "threads": cores,
                           "sample": f"{n} oracle steps x {Ws} worlds ({nc} contacts), {dt:.1f} s"},
                single_core={"value": v1, "threads": 1,
                             "sample": f"{n1} oracle steps x {Ws1} worlds ({nc1} contacts), {dt1:.1f} s"},
                sample=f"{n} oracle steps x {Ws} worlds of the same workload ({nc} contacts), fp64, "
                       f"{dt:.1f} s, OpenMP over worlds on all {cores} host threads; single core: "
                       f"{v1:.4g} world-steps/s over {n1} x {Ws1} worlds")


# ---------------------------------------------------------------- main arms
def run_reference(args, rank, world_size):
    """--impl reference: the fp64 oracle as it stands on the host cores, each
    step a bounded sample of the same workload (rank 0 only)."""
    from harness.types import Config
    if rank != 0:
        return
    import oracle
    cfg = Config(impedance=args.impedance, n_t=args.nt, n_rol=args.nrol)
    parts, wname, n_local = workload(args, 0, world_size)
    cores = os.cpu_count() or 1
    Wcap = 64 if args.workload == "pile" else 256
    samples = [(p, _sample(p, Wcap)) for p in parts]
    states = [x[1][1] for x in samples]

    def one():
        for i, (p, (W, st, c, inp)) in enumerate(samples):
            states[i] = oracle.step(cfg, p.scene, states[i], c, inp, n_threads=cores)["state"].astype(np.float32)

    for _ in range(args.warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    dt = time.perf_counter() - t0
    Ws = sum(x[1][0] for x in samples)
    v = args.steps * Ws / dt
    line = {"impl": "reference", "metric": METRICS[args.workload], "value": v, "unit": "world-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.workload == "mixed" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wname, "worlds_per_gpu": n_local,
                       "contacts_per_world": sum(p.c.n for p in parts) // max(n_local, 1),
                       "facets_per_contact": facets(args), "dt": cfg.dt, "sample_worlds_per_step": Ws},
            "cpu_baseline": {"value": v, "unit": "world-steps/s", "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} steps x {Ws} of {n_local} worlds, fp64 oracle, OpenMP over worlds"},
            "e2e": {"value": v, "unit": "world-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world_size, local):
    import ctypes as ct
    import torch
    import torch.distributed as dist
    import paper_2603_12185_b200 as cf
    from paper_2603_12185_b200 import _lib
    from paper_2603_12185_b200.dist import all_gather_worlds, reduce_max, uniform_ranges
    from harness.types import Config

    n_dev = max(torch.cuda.device_count(), 1)
    shared = world_size > n_dev            # several ranks on one GPU: plumbing only, no throughput claim
    if shared and args.dist_backend == "nccl":
        raise SystemExit(f"bench.py: {world_size} ranks but {n_dev} visible GPU(s); one rank per GPU is required "
                         f"(--dist-backend gloo runs the multi-rank plumbing without a throughput value)")
    local = local % n_dev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world_size > 1:
        if args.dist_backend == "nccl":
            # communicator init (ranks, NVLink/NVLS paths) logged to a file per
            # process, so stdout keeps the one JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join("/tmp", "comfree_nccl.%h.%p.log"))
            dist.init_process_group("nccl", device_id=dev)
        else:                              # plumbing check with several ranks on one GPU
            dist.init_process_group(args.dist_backend)
    cfg = Config(impedance=args.impedance, n_t=args.nt, n_rol=args.nrol)
    parts, wname, n_local = workload(args, rank, world_size)
    stream = torch.cuda.current_stream()
    for i, p in enumerate(parts):
        p.ctx = cf.Context(cfg, device=local)
        p.ctx.load_scene(p.scene, p.W, p.st)
        p.dc = cf.DeviceContacts.from_host(p.c, dev)
        assert p.dc.sorted
        # pre-segmented input (the benchmark default): off[W+1]
        p.off = None if args.world_ids else torch.from_numpy(
            np.searchsorted(p.c.world, np.arange(p.W + 1)).astype(np.int64)).to(dev)
        p.tin = None
        if p.inp is not None:
            p.tin = type(p.inp)(*(None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                                  for a in (p.inp.f_ext, p.inp.tree_L, p.inp.tree_tau)))
        # part 0 on the caller's stream, the others on their own streams (fork / join)
        p.stream = stream if i == 0 else torch.cuda.Stream(device=dev)
        p.up = None
        p.col = None
        if args.collide and p.scene.n_trees == 0:    # pile: contacts from the GPU front-end every step
            from harness import scenes as _sc
            B = p.scene.n_bodies
            lat = {500: (10, 10, 5), 100: (5, 5, 4)}[B]
            # candidates every step (broadphase, reading R32), or the fixed lattice-neighbour list
            p.ctx.load_geometry(_sc.pile_geometry(lat, broadphase=not args.pair_list))
            p.col = p.W * 4 * args.contacts         # output capacity
        if args.upstream and p.scene.n_trees > 0:     # articulated upstream every step
            from harness import scenes as _sc
            p.ctx.load_articulation(_sc.hand_articulation())
            p.up = (torch.from_numpy(np.ascontiguousarray(p.c.meta["link"], np.int32)).to(dev),
                    p.tin.tree_tau.clone())          # applied joint torques; tree_tau receives tau - c
            if args.collide:
                p.ctx.load_geometry(_sc.hand_geometry(margin=0.005))
    alg_up = sum(p.W * p.scene.n_trees * (2 * 4 * p.scene.tree_ndof + 4 * 10 + 4 * p.scene.tree_ndof)
                 + int(np.count_nonzero(p.c.body_a < -1) + np.count_nonzero(p.c.body_b < -1)) * (16 + 4 + 96)
                 for p in parts if p.up is not None)
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_sink = torch.empty(1, dtype=torch.float32, device=dev)

    if args.reset_state:               # initial states kept on the device
        for p in parts:
            p.init_dev = {k: torch.from_numpy(np.ascontiguousarray(getattr(p.st, k), np.float32)).to(dev)
                          for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")}

    def reset():
        if args.reset_state:
            for p in parts:
                p.ctx.set_state_device(p.init_dev, stream=stream)

    def flush_l2():
        """Evict L2 between timed steps (untimed): write a 256 MB buffer (> the
        126 MB L2); in write+read mode read it back so the lines left in L2 are
        clean (the dirty lines' write-back happens here, not in the next step)."""
        reset()
        flush.zero_()
        if args.flush_mode == "write+read":
            torch.sum(flush, dim=0, keepdim=True, out=flush_sink)

    applied = [0]          # steps applied to the states (graph capture records, does not run)

    fused = args.collide and not args.pair_list and not args.split_collide

    def one_step(s0, capturing=False):
        """One step of every part: part 0 on s0, the rest forked from s0 and joined back."""
        applied[0] += 0 if capturing else 1
        for i, p in enumerate(parts):
            if i != 0:
                p.stream.wait_stream(s0)
            ps = s0 if i == 0 else p.stream
            if p.col is not None and fused:          # one call: collide, the step reads the staged records
                p.ctx.step_collided(p.col, dt=cfg.dt, stream=ps)
                continue
            if p.col is not None:
                p.dc, _ = p.ctx.collide(capacity=p.col, stream=ps, device_count=True)
            if p.up is not None:
                if args.collide:                     # contacts from the current state (closed loop)
                    p.dc, lk = p.ctx.collide(capacity=p.W * 40, stream=ps, device_count=True)
                    p.up = (lk, p.up[1])
                p.ctx.articulation_update(p.tin.tree_L, p.tin.tree_tau, p.dc, p.up[0], tau_ext=p.up[1], stream=ps)
            p.ctx.step(p.dc, p.tin, dt=cfg.dt, stream=ps, off=None if (p.col is not None or args.collide) else p.off)
        for p in parts[1:]:
            s0.wait_stream(p.stream)

    for _ in range(max(args.warmup, 3)):
        reset()
        one_step(stream)
    torch.cuda.synchronize()
    for p in parts:                                   # collision-built contacts: the step's real count
        if p.col is not None:
            if fused:                                 # the fused call keeps no public streams: count once
                p.dc, _ = p.ctx.collide(capacity=p.col, device_count=True)
            nc = int(p.dc.n_dev.item())
            p.alg_bytes = nc * BYTES_PER_CONTACT + p.W * p.scene.n_bodies * BYTES_PER_BODY
            p.c_count = nc
    # direct launches with the library's own event timing around each fused kernel
    for p in parts:
        p.ctx.get_timing()
        p.ctx.set_timing(True)
    for _ in range(min(args.steps, 20)):
        if flush is not None:
            flush_l2()
        one_step(stream)
    for p in parts:
        p.kt = p.ctx.get_timing()
        p.ctx.set_timing(False)
        p.k_ms_direct = p.kt["step_ms"] / max(p.kt["step_launches"], 1)
    # one step captured in a CUDA graph (no host launch path inside the timed region)
    graph = None
    if not args.no_graph:
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            one_step(side, capturing=True)
        stream.wait_stream(side)
        torch.cuda.synchronize()
    launches0 = sum(p.ctx.kernel_launches for p in parts)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world_size > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clock = ClockSampler(local)
    with clock:
        for i in range(args.steps):
            if flush is not None:
                flush_l2()                 # evict L2 between timed steps (untimed)
            evs[i][0].record(stream)
            if graph is not None:
                graph.replay()
                applied[0] += 1
            else:
                one_step(stream)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world_size > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))
    # kernels per step: one fused kernel per part (S0 fused for sorted ids); counted
    # by the library for direct launches, the same for each graph replay
    if graph is None:
        launches = sum(p.ctx.kernel_launches for p in parts) - launches0
    else:
        n0 = sum(p.ctx.kernel_launches for p in parts)
        one_step(stream)
        torch.cuda.synchronize()
        launches = args.steps * (sum(p.ctx.kernel_launches for p in parts) - n0)
    total_ms = reduce_max(total_ms, dev)   # the job is as slow as its slowest rank
    ms_per_step = total_ms / args.steps
    total_worlds = sum(c for pl in shard_plan(args, world_size) for _, c in pl.values())
    world_steps = total_worlds * args.steps
    value = world_steps / (total_ms * 1e-3)
    n_contacts = sum(getattr(p, "c_count", p.c.n) for p in parts)
    contacts_per_s = value * (n_contacts / n_local)

    # roofline of the dominant kernel (part 0: the pile / pile-lite k_step).  With
    # one part and one kernel per step the per-step CUDA events around the graph
    # replay bracket exactly that kernel; with several parts the kernel's own
    # events (library timing, direct launches, parts running concurrently) are used.
    dom = parts[0]
    k_ms = (total_ms / args.steps) if (graph is not None and len(parts) == 1 and dom.up is None
                                       and dom.col is None) else dom.k_ms_direct
    peak, peak_kind = peaks()
    achieved = dom.alg_bytes / (k_ms * 1e-3) / 1e9
    tr = ncu_traffic()
    traffic = None
    if tr and tr.get("workload") == args.workload and tr.get("worlds") == dom.W and \
            tr.get("contacts_per_world") == dom.c.n // dom.W and dom.col is None:
        traffic = tr.get("dram_bytes_per_launch")

    # after the timed region: final states all-gathered (NCCL) and, on rank 0,
    # sampled worlds re-run alone on this GPU and compared bit for bit
    finite = True
    gathered_mb = verification = None
    for p in parts:
        p.final = p.ctx.get_state()
        finite &= bool(np.isfinite(p.final["vel"]).all() and np.isfinite(p.final["pos"]).all())
    if world_size > 1:
        plain = not (args.upstream or args.collide or args.kd)   # inputs constant over the steps

        def gpu_stepper(p, scene, st, c, inp, n):
            ctx = cf.Context(cfg, device=local)
            ctx.load_scene(scene, 1, st)
            dc = cf.DeviceContacts.from_host(c, dev)
            off = torch.tensor([0, c.n], dtype=torch.int64, device=dev)
            tin = None if inp is None else type(inp)(*(None if a is None else torch.from_numpy(
                np.ascontiguousarray(a)).to(dev) for a in (inp.f_ext, inp.tree_L, inp.tree_tau)))
            for _ in range(n):
                ctx.step(dc, tin, dt=cfg.dt, off=None if args.world_ids else off)
            out = ctx.get_state()
            ctx.close()
            return out
        gathered_mb, verification = verify_shards(args, parts, {p.name: p.final for p in parts}, rank, world_size,
                                                  applied[0], gpu_stepper if plain else None, device=dev,
                                                  samples_per_rank=2 if plain else 0)
        finite = bool(reduce_max(0.0 if finite else 1.0, dev) == 0.0)

    # e2e: the same metric through the C ABI with HOST buffers (pinned), H2D of the
    # step's contacts (and inputs) and D2H of the resulting state inside the
    # timed region, every step.  Pipelined (COMFREE_MEM_HOST_ASYNC, the value
    # reported): step k + 1's upload runs on the context's copy-in stream while
    # step k's kernel and download run; serial (COMFREE_MEM_HOST, context): each
    # call copies, steps and synchronises in turn.
    from harness.types import Inputs
    e2e_steps = max(1, args.e2e_steps)
    h2d = d2h = 0

    def pinned(a):
        return None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float32)).pin_memory().numpy()
    for p in parts:
        if args.collide:                 # closed loop: contacts come from the GPU front-end, no host inputs
            p.out_host = {k: torch.empty(v.shape, dtype=torch.float32).pin_memory().numpy() for k, v in p.final.items()}
            d2h += sum(v.nbytes for v in p.out_host.values())
            continue
        p.hc = cf.HostContacts.from_arrays(p.c, pin=True, n_worlds=None if args.world_ids else p.W)
        p.hca = cf.HostContacts.from_arrays(p.c, pin=True, asynchronous=True, n_worlds=None if args.world_ids else p.W)
        p.inp_h = None if p.inp is None else Inputs(*(pinned(a) for a in (p.inp.f_ext, p.inp.tree_L, p.inp.tree_tau)))
        reset()
        p.ctx.step(p.hc, p.inp_h, dt=cfg.dt)          # warm the staging buffers
        p.ctx.step(p.hca, p.inp_h, dt=cfg.dt)
        p.ctx.step(p.hca, p.inp_h, dt=cfg.dt)
        p.out_host = {k: torch.empty(v.shape, dtype=torch.float32).pin_memory().numpy() for k, v in p.final.items()}
        p.ctx.get_state_async(p.out_host)
        p.ctx.get_state_async(p.out_host)
        p.ctx.wait_async()
        p.ctx.check()
        p.st_h = _lib.comfree_state(*[p.out_host[k].ctypes.data if p.out_host[k].size else None
                                      for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")], _lib.MEM_HOST)
        h2d += p.hc.h2d_bytes() + (0 if p.inp_h is None else sum(a.nbytes for a in (p.inp_h.f_ext, p.inp_h.tree_L,
                                                                                    p.inp_h.tree_tau) if a is not None))
        d2h += sum(v.nbytes for v in p.out_host.values())

    def e2e_run(asynchronous):
        if world_size > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            if args.collide:             # the closed-loop step on the device, the state read back
                one_step(stream)
                for p in parts:
                    p.ctx.get_state_async(p.out_host, stream=stream)
                continue
            reset()                      # --reset-state only: a device-side state copy (~10 us)
            for p in parts:
                if asynchronous:
                    p.ctx.step(p.hca, p.inp_h, dt=cfg.dt, stream=stream)
                    p.ctx.get_state_async(p.out_host, stream=stream)
                else:
                    p.ctx.step(p.hc, p.inp_h, dt=cfg.dt, stream=stream)
                    rc = p.ctx._lib.comfree_get_state(p.ctx.h, 0, p.W, ct.byref(p.st_h), stream.cuda_stream)
                    p.ctx._check(rc, "comfree_get_state")
        if asynchronous:
            for p in parts:
                p.ctx.wait_async(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        for p in parts:
            p.ctx.check(stream)                       # latched errors of the asynchronous calls
        return reduce_max(e0.elapsed_time(e1), dev)
    e2e_serial_ms = e2e_run(False) if not args.collide else float("nan")
    e2e_ms = e2e_run(True)
    e2e_value = total_worlds * e2e_steps / (e2e_ms * 1e-3)
    e2e_serial_value = total_worlds * e2e_steps / (e2e_serial_ms * 1e-3) if not args.collide else None

    cpu = None
    if rank == 0:                      # rank 0 only (the other ranks wait at the barrier)
        cpu = cpu_oracle_rate(parts, cfg, args.cpu_seconds, max_worlds=(parts[0].W if args.workload != "mixed" else 256))
    if world_size > 1:
        dist.barrier()
    if rank == 0:
        alg_total = sum(p.alg_bytes for p in parts)
        line = {
            "metric": METRICS[args.workload],
            "value": value, "unit": "world-steps/s", "n_gpus": world_size,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if args.workload == "mixed" else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wname, "worlds_per_gpu": n_local,
                       "contacts_per_world": n_contacts // n_local,
                       "parts": {p.name: {"worlds": p.W, "contacts_per_world": p.c.n // p.W,
                                          "bodies_per_world": p.scene.n_bodies, "chains_per_world": p.scene.n_trees}
                                 for p in parts},
                       "facets_per_contact": facets(args), "condim": args.condim, "n_t": args.nt, "n_rol": args.nrol,
                       "dt": cfg.dt,
                       "l2": (("flushed between timed steps (256 MB write, then read back: cold clean L2)"
                               if args.flush_mode == "write+read" else "flushed between timed steps (256 MB write)")
                              if flush is not None else "not flushed"),
                       "footprint_mb_per_step": alg_total / 1e6,
                       "state": "reset to the initial state before every step (untimed)" if args.reset_state
                                else "evolving",
                       "articulated_upstream": bool(args.upstream),
                       "upstream_mb_per_step": alg_up / 1e6,
                       "parallelism": f"world-sharded x{world_size}"},
            "contacts_per_s": contacts_per_s,
            "gpu_launches": int(launches),
            "kernel_ms": {**{f"k_step[{p.name}]_events_direct_launch": p.k_ms_direct for p in parts},
                          "step_graph_replay_events": total_ms / args.steps,
                          "segment_s0_separate": sum(p.kt["segment_ms"] / max(p.kt["step_launches"], 1) for p in parts)},
            "segmentation": ("world ids (S0 fused into the step)" if args.world_ids or args.collide
                             else "pre-segmented off[W+1] from the caller (S0 skipped, SURVEY 8(a))"),
            "cuda_graph": graph is not None,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "kernel": f"k_step (S1-S7 fused) [{dom.name}]", "algorithmic_bytes_per_launch": dom.alg_bytes},
            "clocks": clock.summary(),
            "e2e": {"value": e2e_value, "unit": "world-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "mode": ("closed loop on the device (collision front-end every step), the state downloaded "
                             "every step into pinned host memory (COMFREE_MEM_HOST_ASYNC); no per-step host inputs"
                             if args.collide else
                             "pinned host buffers through comfree_step / comfree_get_state (COMFREE_MEM_HOST_ASYNC): "
                             "step k+1's upload overlaps step k's kernel and download"),
                    "ms_per_step": e2e_ms / e2e_steps,
                    "pcie_gbs": (h2d + d2h) / (e2e_ms / e2e_steps * 1e-3) / 1e9,
                    "serial_value": e2e_serial_value,
                    "serial_ms_per_step": None if args.collide else e2e_serial_ms / e2e_steps},
            "cpu_baseline": cpu,
            "allgather_final_state_mb": gathered_mb,
            "sharded_verification": verification,
            "nccl_debug_file": os.environ.get("NCCL_DEBUG_FILE") if (world_size > 1 and args.dist_backend == "nccl")
                               else None,
            "context": "paper: 2-3x MJWarp throughput in dense contact on one RTX 4090 (PAPER.md P:11, P:274); "
                       "full-step numbers, not this path alone",
            "final_state_finite": finite,
        }
        if shared:                     # ranks share a GPU: the multi-rank plumbing ran, no throughput claim
            line.update(value=None, contacts_per_s=None, plumbing_only=True,
                        note=f"{world_size} ranks on {n_dev} GPU(s) ({args.dist_backend}): plumbing check only")
        print(json.dumps(line), flush=True)
    for p in parts:
        p.ctx.close()
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
