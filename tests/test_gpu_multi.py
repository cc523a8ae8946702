"""GPU: the single-process multi-GPU entry vmb_vmonarch_fwd_multi.

The gpurun box has one B200, so the n "devices" of the call are the same ordinal with
separate buffers and workspaces: the partition, the peer-memory K/V gather kernel (here a
same-device read), the cross-stream joins and the per-part forwards all run exactly as on n
GPUs; only the NVLink transport itself is not exercised.  Parts must reproduce the
unsharded forward: head blocks bitwise, sequence slabs bitwise on frames >= 1 and to
fp32-combine rounding on the first-frame recompute rows (split count depends on the slab)."""
import pytest
import torch

from oracle.oracle import bf16_round, workload
from vmb_testutil import relfro

pytestmark = pytest.mark.gpu


def _inputs(vm, cuda, grid, seed):
    q, k, v = workload(grid.units(), grid.tokens(), grid.head_dim, seed=seed)
    return [torch.from_numpy(bf16_round(x)).to(cuda, torch.bfloat16) for x in (q, k, v)]


def test_shard_range_matches_dist_partitions(vm):
    from paper_2601_22275_b200.dist import slab_partition, unit_shards
    for n, parts in [(40, 8), (40, 3), (1456, 8), (5, 8), (7, 1)]:
        assert [vm.shard_range(n, parts, r) for r in range(parts)] == slab_partition(n, parts)
        assert [(a, a + c) for a, c in (vm.shard_range(n, parts, r) for r in range(parts))] == unit_shards(n, parts)


@pytest.mark.parametrize("gridt,heads,ndev", [((4, 8, 16), 5, 2), ((21, 30, 52), 4, 3), ((4, 8, 16), 2, 3)])
def test_multi_heads_equals_single_call_bitwise(vm, cuda, gridt, heads, ndev):
    grid = vm.TokenGrid(*gridt, 128, heads, 1)
    q, k, v = _inputs(vm, cuda, grid, 31)
    full = vm.vmonarch_attention(q, k, v, grid)
    blocks = [vm.shard_range(heads, ndev, r) for r in range(ndev)]
    sl = lambda x: [x[a:a + c] for a, c in blocks]  # noqa: E731
    outs = vm.vmonarch_attention_multi(sl(q), sl(k), sl(v), grid, mode="heads")
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs, 0), full)


@pytest.mark.parametrize("gridt,heads,ndev", [((4, 8, 16), 2, 2), ((6, 10, 26), 2, 3), ((21, 30, 52), 1, 8)])
def test_multi_seq_equals_unsharded(vm, cuda, gridt, heads, ndev):
    from paper_2601_22275_b200.dist import local_slab
    grid = vm.TokenGrid(*gridt, 128, heads, 1)
    q, k, v = _inputs(vm, cuda, grid, 37)
    full = vm.vmonarch_attention(q, k, v, grid)
    parts = [vm.shard_range(grid.h * grid.w, ndev, r) for r in range(ndev)]
    outs = vm.vmonarch_attention_multi([local_slab(q, grid, a, c) for a, c in parts],
                                       [local_slab(k, grid, a, c).contiguous() for a, c in parts],
                                       [local_slab(v, grid, a, c).contiguous() for a, c in parts], grid, mode="seq")
    torch.cuda.synchronize()
    T, hw = grid.t_frames, grid.h * grid.w
    stitched = torch.empty_like(full).view(heads, T, hw, 128)
    for (a, c), o in zip(parts, outs):
        stitched[:, :, a:a + c] = o.view(heads, T, c, 128)
    f = full.float().view(heads, T, hw, 128)
    s = stitched.float()
    assert torch.equal(f[:, 1:], s[:, 1:])
    # frame 0: split-KV recompute with a slab-dependent split count -> bf16-ulp level differences
    assert relfro(s[:, 0].cpu().numpy(), f[:, 0].cpu().numpy()) <= 5e-3


def test_multi_fp32_heads_parity_and_errors(vm, orc, cuda):
    grid = vm.TokenGrid(3, 4, 4, 16, 3, 1)
    q, k, v = workload(3, grid.tokens(), 16, seed=41)
    tq, tk, tv = (torch.from_numpy(x).to(cuda) for x in (q, k, v))
    outs = vm.vmonarch_attention_multi([tq[:2], tq[2:]], [tk[:2], tk[2:]], [tv[:2], tv[2:]], grid, mode="heads")
    ref = orc.vmonarch_attention(q, k, v, (grid.t_frames, grid.h, grid.w), iters=2)
    assert relfro(torch.cat(outs).cpu().numpy(), ref) <= 1e-4
    with pytest.raises(vm.DimensionError):  # seq mode is bf16-only
        vm.vmonarch_attention_multi([tq], [tk], [tv], grid, mode="seq")
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention_multi([tq], [tk], [tv], grid, mode="frames")
    bad = tq.clone()
    bad[2, 3, 2] = float("nan")
    with pytest.raises(vm.DomainError):  # finite check of Q (monarch.hpp:44) on the part that holds it
        vm.vmonarch_attention_multi([tq[:2], bad[2:]], [tk[:2], tk[2:]], [tv[:2], tv[2:]], grid, mode="heads")
