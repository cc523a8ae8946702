"""GPU: the process-per-GPU sequence-sharded path (dist.vmonarch_attention_seq: K/V slab
all-gather, vmb_seq_assemble, the slab forward with V arriving on a side stream) with 2 and 3
real ranks.  The box this suite runs on has one GPU, and NCCL refuses two ranks on one device,
so the ranks share cuda:0 over a gloo group (CUDA tensors); everything but the transport of
the all-gather is the code path the NCCL run takes.  Each rank's output slab must equal the
unsharded forward's rows of that slab bitwise on frames >= 1 (the first frame is the
recompute, exact attention over all keys, also compared)."""
import os

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, out_q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2601_22275_b200 as vm
    from paper_2601_22275_b200.dist import local_slab, slab_partition, vmonarch_attention_seq

    grid = vm.TokenGrid(4, 8, 16, 128, 2, 1)
    g = torch.Generator(device="cuda").manual_seed(9)
    q, k, v = (torch.randn((2, grid.tokens(), 128), device="cuda", generator=g).bfloat16() for _ in range(3))
    b0, cnt = slab_partition(grid.h * grid.w, world)[rank]
    ql, kl, vl = (local_slab(x, grid, b0, cnt).contiguous() for x in (q, k, v))
    out = vmonarch_attention_seq(ql, kl, vl, grid)
    torch.cuda.synchronize()
    full = vm.vmonarch_attention(q, k, v, grid)
    want = local_slab(full, grid, b0, cnt)
    T = grid.t_frames
    o4, w4 = out.view(2, T, cnt, 128), want.view(2, T, cnt, 128)
    later = bool(torch.equal(o4[:, 1:], w4[:, 1:]))
    first = float((o4[:, 0].float() - w4[:, 0].float()).abs().max().item())
    out_q.put((rank, later, first))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_seq_sharded_multirank_equals_unsharded(cuda, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31000 + world * 17 + (os.getpid() % 500)
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, later, first in res:
        assert later, f"rank {rank}: frames >= 1 differ from the unsharded forward"
        assert first <= 2e-2, f"rank {rank}: first-frame rows differ by {first}"
