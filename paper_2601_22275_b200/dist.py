"""Multi-GPU plumbing for the VMonarch forward.

Batch*head units are independent (video.hpp:115-148; bitwise identical regardless of
partitioning, test_video.cpp:197-216), so N GPUs shard the units with no data-path
collective: rank r owns a contiguous block of units.  The only collective here is the
optional gather of the outputs for callers that want the full tensor on every rank.
"""
from __future__ import annotations

from typing import List, Tuple


def unit_shards(units: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous [start, stop) unit ranges per rank; sizes differ by at most one."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    base, extra = divmod(units, world)
    out, start = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((start, start + n))
        start += n
    return out


def gather_units(local, units: int, group=None):
    """all_gather the per-rank (units_r, N, d) outputs into (units, N, d) on every rank.

    Uneven shards are padded to the largest shard for the collective and trimmed after.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    shards = unit_shards(units, world)
    width = max(b - a for a, b in shards)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([buf[: b - a] for buf, (a, b) in zip(bufs, shards)], dim=0)
