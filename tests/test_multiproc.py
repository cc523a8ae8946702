"""Host-side multi-GPU logic on CPU: head/unit sharding over world_size 2 with gloo.
Each rank computes its unit shard (here with the CPU oracle standing in for the device),
gathers, and the result must equal the single-process computation bitwise (units are
independent, test_video.cpp:197-216)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_22275_b200.dist import gather_units, unit_shards


def test_unit_shards_cover_exactly():
    for units in (1, 5, 12, 40):
        for world in (1, 2, 3, 4, 8):
            sh = unit_shards(units, world)
            assert len(sh) == world and sh[0][0] == 0 and sh[-1][1] == units
            assert all(a <= b for a, b in sh) and all(sh[i][1] == sh[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in sh]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle, workload
    orc = Oracle("port")
    units, grid = 5, (3, 4, 4)
    q, k, v = workload(units, 48, 16, seed=3)
    a, b = unit_shards(units, world)[rank]
    local = orc.vmonarch_attention(q[a:b], k[a:b], v[a:b], grid) if b > a else np.zeros((0, 48, 16), np.float32)
    full = gather_units(torch.from_numpy(np.ascontiguousarray(local)), units)
    if rank == 0:
        ref = orc.vmonarch_attention(q, k, v, grid)
        out_q.put(bool(np.array_equal(full.numpy(), ref)))
    dist.destroy_process_group()


def test_gloo_world2_sharded_equals_single():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


# ----------------------------------------------------------------------------- sequence sharding
def _assemble_reference(gathered, parts, grid):
    """Host restatement of vmb_seq_assemble (csrc/kernels/seq_gather.cu) for the CPU test."""
    world, U, T, smax, d = gathered.shape
    hw = grid.h * grid.w
    full = torch.zeros((U, T, hw, d), dtype=gathered.dtype)
    for r, (a, c) in enumerate(parts):
        full[:, :, a:a + c] = gathered[r, :, :, :c]
    return full.reshape(U, T * hw, d)


def _seq_worker(rank, world, port, hw_shape, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2601_22275_b200 as vm
    from paper_2601_22275_b200.dist import gather_slabs, local_slab, slab_partition
    T, h, w = hw_shape
    grid = vm.TokenGrid(T, h, w, 16, 3, 1)
    g = torch.Generator().manual_seed(11)
    k_full = torch.randn((3, grid.tokens(), 16), generator=g)
    parts = slab_partition(h * w, world)
    a, c = parts[rank]
    k_loc = local_slab(k_full, grid, a, c)
    gathered, parts2, smax = gather_slabs(k_loc, grid)
    ok = parts2 == parts and smax == max(cc for _, cc in parts)
    ok = ok and torch.equal(_assemble_reference(gathered, parts, grid), k_full)
    # every query row of the full problem belongs to exactly one rank's slab
    seen = torch.zeros(grid.tokens(), dtype=torch.int32)
    for aa, cc in parts:
        idx = torch.arange(grid.tokens()).view(T, h * w)[:, aa:aa + cc].reshape(-1)
        seen[idx] += 1
    ok = ok and bool((seen == 1).all())
    out_q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,hw_shape", [(2, (3, 4, 5)), (3, (2, 5, 7))])
def test_gloo_sequence_sharded_gather(world, hw_shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world * 10 + (os.getpid() % 500)
    procs = [ctx.Process(target=_seq_worker, args=(r, world, port, hw_shape, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(res.values()), res


def test_slab_partition_and_local_slab():
    import paper_2601_22275_b200 as vm
    from paper_2601_22275_b200.dist import local_slab, slab_partition
    for hw, world in [(1456, 8), (1560, 8), (11648, 8), (10, 3), (7, 7)]:
        parts = slab_partition(hw, world)
        assert parts[0][0] == 0 and sum(c for _, c in parts) == hw
        assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(world - 1))
    grid = vm.TokenGrid(3, 2, 5, 4, 2, 1)
    x = torch.arange(2 * 30 * 4, dtype=torch.float32).view(2, 30, 4)
    s = local_slab(x, grid, 3, 4)
    assert s.shape == (2, 12, 4)
    # local token t*4 + i is global token t*10 + 3 + i
    for t in range(3):
        for i in range(4):
            assert torch.equal(s[:, t * 4 + i], x[:, t * 10 + 3 + i])
