"""bench.py's multi-rank plumbing on CPU (gloo, world_size 2): the shard plan
(C5 split by per-world bytes with dist.shard_ranges; C4 weak scaling), the
per-rank workload generation by global world id, the NCCL-path all-gather of
final states and rank 0's bitwise re-run of sampled worlds (verify_shards).
The stepping function is the fp64 oracle here (tests may use it); bench.py
passes a one-world CUDA context instead."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_stepper(p, scene, st, c, inp, n):
    import oracle
    from harness.types import Config
    s = st
    for _ in range(n):
        s = oracle.step(Config(), scene, s, c, inp)["state"]
    return {k: getattr(s, k) for k in ("pos", "quat", "vel", "omega", "qpos", "qvel")}


def _worker(rank, ws, port, argv, n_steps, out_path, corrupt):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    args = bench.parse(argv)
    parts, name, n_local = bench.workload(args, rank, ws)
    finals = {}
    for p in parts:
        finals[p.name] = _oracle_stepper(p, p.scene, p.st, p.c, p.inp, n_steps)
        if corrupt and rank == 1:                     # a wrong shard must be caught
            finals[p.name]["vel"][-1, 0, 0] += 1e-9
    mb, rep = bench.verify_shards(args, parts, finals, rank, ws, n_steps, _oracle_stepper)
    if rank == 0:
        torch.save({"rep": rep, "mb": mb, "plan": bench.shard_plan(args, ws), "n_local": n_local}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, argv, n_steps=2, corrupt=False):
    out = str(tmp_path / "r0.pt")
    mp.start_processes(_worker, args=(2, _free_port(), argv, n_steps, out, corrupt), nprocs=2, join=True,
                       start_method="spawn")
    return torch.load(out, weights_only=False)


def test_shard_plan_mixed_cost_weighted():
    sys.path.insert(0, ROOT)
    import bench
    args = bench.parse(["--workload", "mixed", "--worlds", "65536"])
    for ws in (1, 2, 4, 8):
        plan = bench.shard_plan(args, ws)
        for kind in ("pile-lite", "hand5"):
            firsts = [pl[kind][0] for pl in plan]
            counts = [pl[kind][1] for pl in plan]
            assert sum(counts) == 32768 and firsts[0] == 0          # every world exactly once, in order
            assert all(f + c == g for f, c, g in zip(firsts, counts, firsts[1:]))
        cost = [pl["pile-lite"][1] * (400 * 64 + 100 * 104) + pl["hand5"][1] * (20 * 64 + 16 * 96 + 104 + 256 + 160 + 64)
                for pl in plan]
        assert max(cost) - min(cost) <= 2 * (400 * 64 + 100 * 104)  # balanced to one world's bytes


def test_two_rank_mixed_gather_and_bitwise_rerun(tmp_path):
    res = _run(tmp_path, ["--workload", "mixed", "--worlds", "24"])
    rep = res["rep"]
    assert rep["bitwise_equal"] and rep["checked_worlds"] == 8 and rep["n_steps"] == 2, rep
    assert res["mb"] > 0


def test_two_rank_pile_weak_and_a_wrong_shard_is_caught(tmp_path):
    rep = _run(tmp_path, ["--worlds", "3", "--contacts", "300"])["rep"]
    assert rep["bitwise_equal"] and rep["checked_worlds"] == 4, rep
    rep = _run(tmp_path, ["--worlds", "3", "--contacts", "300"], corrupt=True)["rep"]
    assert not rep["bitwise_equal"] and rep["mismatch"][0]["rank"] == 1, rep
