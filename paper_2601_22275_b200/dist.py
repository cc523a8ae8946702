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


# ----------------------------------------------------------------------------- sequence sharding
def slab_partition(positions: int, world: int) -> List[Tuple[int, int]]:
    """(begin, count) of each rank's spatial slab: contiguous, sizes differ by at most one."""
    return [(a, b - a) for a, b in unit_shards(positions, world)]


def local_slab(x, grid, begin: int, count: int):
    """Rank-local slab of a full (units, N, d) tensor: (units, T * count, d), token t*count + i."""
    U, n, d = x.shape
    hw = grid.h * grid.w
    return x.view(U, grid.t_frames, hw, d)[:, :, begin:begin + count].reshape(U, grid.t_frames * count, d)


def gather_slabs(x_local, grid, group=None):
    """all_gather the ranks' (units, T*count_r, d) slabs into (world, units, T, slab_max, d)
    (slabs zero-padded to the largest): the one collective of the sequence-sharded mode."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    parts = slab_partition(grid.h * grid.w, world)
    smax = max(c for _, c in parts)
    U, nl, d = x_local.shape
    cnt = nl // grid.t_frames
    send = x_local.new_zeros((U, grid.t_frames, smax, d))
    send[:, :, :cnt] = x_local.view(U, grid.t_frames, cnt, d)
    recv = x_local.new_empty((world * U, grid.t_frames, smax, d))
    dist.all_gather_into_tensor(recv, send, group=group)
    return recv.view(world, U, grid.t_frames, smax, d), parts, smax


_SIDE_STREAMS: dict = {}


def _side_stream(device):
    """One V-gather stream per device, reused by every call (streams are not free to create)."""
    import torch

    key = device.index
    st = _SIDE_STREAMS.get(key)
    if st is None:
        st = _SIDE_STREAMS[key] = torch.cuda.Stream(device=device)
    return st


def vmonarch_attention_seq(q_local, k_local, v_local, grid, cfg=None, group=None):
    """Sequence-sharded VMonarch forward: every rank holds the slab
    slab_partition(h*w, world)[rank] of all frames for Q, K, V; K and V are all-gathered over
    NCCL (one exchange per call) and assembled into frame-major order by a libvmb kernel; the
    forward then runs on the local query slab.  Returns the local output slab."""
    import torch.distributed as dist

    import paper_2601_22275_b200 as vm

    import torch

    cfg = cfg or vm.VMonarchConfig()
    rank = dist.get_rank(group)
    main = torch.cuda.current_stream(q_local.device)
    # K first, on the caller's stream: the first R half-step needs it
    kg, parts, _ = gather_slabs(k_local, grid, group)
    begins = [a for a, _ in parts]
    counts = [c for _, c in parts]
    k_full = vm.seq_assemble(kg, grid, begins, counts)
    # V on a side stream: first read by the last R half-step, so its all-gather overlaps the
    # first R and L half-steps (every rank issues K then V: the same collective order)
    side = _side_stream(q_local.device)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        vg, _, _ = gather_slabs(v_local, grid, group)
        v_full = vm.seq_assemble(vg, grid, begins, counts)
        v_ready = torch.cuda.Event()
        v_ready.record(side)
    b0, cnt = parts[rank]
    out = vm.vmonarch_attention_slab(q_local, k_full, v_full, grid, b0, cnt, cfg, check=False, v_ready=v_ready)
    main.wait_stream(side)
    v_full.record_stream(main)  # allocated on the side stream, read on the main one
    return out
