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
