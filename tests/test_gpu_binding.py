"""GPU: the Python binding's argument checks and stream/workspace discipline."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _inputs(vm, cuda, heads=2, dtype=torch.bfloat16, seed=0):
    grid = vm.TokenGrid(4, 8, 16, 128, heads, 1)
    g = torch.Generator(device=cuda).manual_seed(seed)
    q, k, v = (torch.randn((heads, grid.tokens(), 128), device=cuda, generator=g).to(dtype) for _ in range(3))
    return grid, q, k, v


def test_out_dtype_and_device_are_checked(vm, cuda):
    grid, q, k, v = _inputs(vm, cuda)
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention(q, k, v, grid, out=torch.empty(q.shape, dtype=torch.float32, device=cuda))
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention(q, k, v, grid, out=torch.empty((1,) + tuple(q.shape[1:]), dtype=q.dtype, device=cuda))
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention(q, k.float(), v, grid)


def test_slab_out_is_checked(vm, cuda):
    grid, q, k, v = _inputs(vm, cuda)
    hw = grid.h * grid.w
    ql = q.view(2, grid.t_frames, hw, 128)[:, :, :64].reshape(2, grid.t_frames * 64, 128)
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention_slab(ql, k, v, grid, 0, 64, out=torch.empty((2, grid.t_frames * 32, 128), dtype=q.dtype,
                                                                          device=cuda))
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention_slab(ql, k, v, grid, 0, 64, out=torch.empty(ql.shape, dtype=torch.float32, device=cuda))


def test_multi_parts_are_checked(vm, cuda):
    grid, q, k, v = _inputs(vm, cuda, heads=3)
    # heads mode, 2 parts: shard_range(3, 2, r) = 2 / 1 units
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention_multi([q[:1], q[1:]], [k[:1], k[1:]], [v[:1], v[1:]], grid)
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention_multi([q[:2], q[2:]], [k[:2], k[2:]], [v[:2], v[2:].float()], grid)


def test_two_streams_two_shapes_do_not_share_a_workspace(vm, cuda):
    # CFG-style: two differently shaped calls in flight on two streams, repeatedly; each must
    # equal its solo result bitwise (one workspace per (device, stream), vmb.h)
    grid_a, qa, ka, va = _inputs(vm, cuda, heads=2, seed=1)
    grid_b = vm.TokenGrid(3, 10, 20, 128, 3, 1)
    g = torch.Generator(device=cuda).manual_seed(2)
    qb, kb, vb = (torch.randn((3, grid_b.tokens(), 128), device=cuda, generator=g).bfloat16() for _ in range(3))
    ref_a = vm.vmonarch_attention(qa, ka, va, grid_a)
    ref_b = vm.vmonarch_attention(qb, kb, vb, grid_b)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    outs = []
    for _ in range(4):
        with torch.cuda.stream(s1):
            oa = vm.vmonarch_attention(qa, ka, va, grid_a, check=False)
        with torch.cuda.stream(s2):
            ob = vm.vmonarch_attention(qb, kb, vb, grid_b, check=False)
        outs.append((oa, ob))
    torch.cuda.synchronize()
    for oa, ob in outs:
        assert torch.equal(oa, ref_a)
        assert torch.equal(ob, ref_b)


def test_caller_workspace(vm, cuda):
    grid, q, k, v = _inputs(vm, cuda)
    ws = torch.empty(vm.workspace_size(grid), dtype=torch.uint8, device=cuda)
    a = vm.vmonarch_attention(q, k, v, grid, workspace=ws)
    b = vm.vmonarch_attention(q, k, v, grid)
    assert torch.equal(a, b)
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention(q, k, v, grid, workspace=ws[:1024])


def test_host_call_returns_finished_results(vm, cuda):
    grid, q, k, v = _inputs(vm, cuda)
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
    ref = vm.vmonarch_attention(q, k, v, grid).cpu()
    out = vm.vmonarch_attention_host(hq, hk, hv, grid, chunk_units=1)
    # no synchronize: the call itself waits for its last D2H copy
    assert torch.equal(out, ref)


def test_call_on_the_tensors_device_stream(vm, cuda):
    # the ABI call is ordered on q.device's current stream even when another stream is current
    grid, q, k, v = _inputs(vm, cuda)
    ref = vm.vmonarch_attention(q, k, v, grid)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = vm.vmonarch_attention(q, k, v, grid)
    s.synchronize()
    assert torch.equal(out, ref)
