"""World-sharded multi-process path on CPU (gloo, world_size 2).

The stepping function here is the fp64 oracle (tests may use it); the product
runs the same sharding / gather / max-reduce plumbing with the CUDA step over
NCCL.  Sharded results must equal the single-process result bit for bit,
because worlds are independent and each world's inputs are seeded by
its global id.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2603_12185_b200.dist import shard_ranges, uniform_ranges


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_cover_and_balance():
    rng = np.random.default_rng(0)
    for n, ws in ((1024, 8), (10, 3), (3, 8), (0, 2), (65536, 8)):
        costs = rng.uniform(1, 3, n)
        r = shard_ranges(costs, ws)
        assert len(r) == ws and r[0][0] == 0 and r[-1][1] == n
        for (a, b), (c, d) in zip(r, r[1:]):
            assert b == c and a <= b
        if n >= ws * 10:
            loads = [costs[a:b].sum() for a, b in r]
            assert max(loads) - min(loads) <= 2 * costs.max() + 1e-9
    assert uniform_ranges(10, 2) == [(0, 5), (5, 10)]


def _worker(rank, ws, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    import torch.distributed as dist
    import oracle
    from harness import scenes
    from harness.types import Config
    from paper_2603_12185_b200.dist import all_gather_worlds, reduce_max, uniform_ranges
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    W = 10
    ranges = uniform_ranges(W, ws)
    lo, hi = ranges[rank]
    scene, st, c = scenes.c4_pile(n_worlds=hi - lo, contacts_per_world=60, lattice=(4, 4, 2), world_offset=lo)
    o = oracle.step(Config(), scene, st, c, None)
    local = {k: torch.from_numpy(np.ascontiguousarray(getattr(o["state"], k))) for k in ("pos", "quat", "vel", "omega")}
    full = all_gather_worlds(local, ranges)
    tmax = reduce_max(float(rank + 1))
    if rank == 0:
        torch.save({"full": full, "tmax": tmax}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shard_gather_matches_single_process(tmp_path):
    import oracle
    from harness import scenes
    from harness.types import Config
    out = str(tmp_path / "r0.pt")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    res = torch.load(out)
    assert res["tmax"] == 2.0                      # max over ranks
    scene, st, c = scenes.c4_pile(n_worlds=10, contacts_per_world=60, lattice=(4, 4, 2))
    o = oracle.step(Config(), scene, st, c, None)
    for k in ("pos", "quat", "vel", "omega"):
        np.testing.assert_array_equal(res["full"][k].numpy(), getattr(o["state"], k))
