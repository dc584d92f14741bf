"""World sharding across ranks (one process per GPU, torch.distributed).

Worlds are independent (the update decouples across contact
pairs, hence across worlds), so the multi-GPU path partitions worlds into
contiguous ranges and steps each range with no per-step communication.  NCCL
is used only around the timed region: a max-reduction of the per-rank device
time and an all-gather of final states for verification.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np


def shard_ranges(costs: Sequence[float], world_size: int) -> List[Tuple[int, int]]:
    """Contiguous [lo, hi) world ranges, one per rank, balancing the prefix sum
    of per-world costs (e.g. 64 B x contacts + 104 B x bodies).  Every world
    belongs to exactly one range; ranges are in rank order."""
    costs = np.asarray(costs, dtype=np.float64)
    n = len(costs)
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    if n == 0:
        return [(0, 0)] * world_size
    csum = np.concatenate([[0.0], np.cumsum(np.maximum(costs, 0.0))])
    total = csum[-1]
    bounds = [0]
    for r in range(1, world_size):
        target = total * r / world_size
        b = int(np.searchsorted(csum, target, side="left"))
        b = min(max(b, bounds[-1]), n)
        bounds.append(b)
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world_size)]


def uniform_ranges(n_worlds: int, world_size: int) -> List[Tuple[int, int]]:
    return shard_ranges(np.ones(n_worlds), world_size)


def reduce_max(value: float, device=None) -> float:
    """Max over ranks (device timing rule: the job is as slow as its slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_gather_worlds(local: Dict[str, "torch.Tensor"], ranges: List[Tuple[int, int]]) -> Dict[str, "torch.Tensor"]:
    """All-gather per-world arrays (leading dim = local worlds) from every rank
    into full arrays in global world order.  Shards are padded to the largest
    range so one all_gather_into_tensor moves each array."""
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size()
    rank = dist.get_rank()
    maxw = max(hi - lo for lo, hi in ranges)
    cpu = dist.get_backend() == "gloo"
    out = {}
    for k, t in local.items():
        if cpu:
            t = t.cpu()
        n_local = ranges[rank][1] - ranges[rank][0]
        assert t.shape[0] == n_local, (k, t.shape, n_local)
        pad = torch.zeros((maxw,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:n_local] = t
        full = torch.empty((ws * maxw,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(full, pad)
        parts = [full[r * maxw:r * maxw + (hi - lo)] for r, (lo, hi) in enumerate(ranges)]
        out[k] = torch.cat(parts, 0)
    return out
