"""CPU-side checks of the C ABI (no device work): every symbol declared in include/vmb.h is
exported by libvmb.so, the host bookkeeping is bit-exact with the reference (factorize,
make_perm, flops_estimate), and host-detectable errors map to the reference's error classes."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "vmb.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(vmb_[a-z0-9_]+)\s*\(", txt)))


def test_every_declared_symbol_is_exported(vm):
    syms = declared_symbols()
    assert len(syms) >= 18
    missing = [s for s in syms if not hasattr(vm.lib, s)]
    assert not missing, missing


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2601_22275_b200", "libvmb.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


@pytest.mark.parametrize("grid,override", [((81, 28, 52), None), ((21, 30, 52), None), ((16, 28, 52), (4, 5824)),
                                           ((4, 3, 3), (6, 6)), ((1, 8, 8), None)])
def test_factorize_and_flops_bit_exact(vm, orc, grid, override):
    g = vm.TokenGrid(*grid, head_dim=64)
    cfg = vm.VMonarchConfig(override_m_b=override)
    m, b = vm.factorize(g, cfg)
    if override:
        assert (m, b) == override
    else:
        assert (m, b) == (grid[0], grid[1] * grid[2])
    for d in (8, 64, 128):
        for recompute in (True, False):
            for iters in (1, 2, 3):
                c = vm.VMonarchConfig(iters=iters, recompute_first_frame=recompute, override_m_b=override)
                a = vm.flops_estimate(g, c, d)
                r = orc.flops_estimate(grid, d, iters=iters, recompute=recompute, override=override or (0, 0))
                assert (a.monarch_flops, a.full_attn_flops, a.recompute_flops) == \
                    (r["monarch_flops"], r["full_attn_flops"], r["recompute_flops"])
                assert a.reduction_ratio == r["reduction_ratio"]
                assert a.sparsity == r["sparsity"] and a.sparsity_approx == r["sparsity_approx"]


def test_flops_golden_values(vm):
    # test_video.cpp:156-168 (wan-321f at d=64)
    rep = vm.flops_estimate(vm.TokenGrid(*vm.preset_grid("wan-321f"), head_dim=64), vm.VMonarchConfig(), 64)
    assert rep.full_attn_flops == 3560678424576
    assert rep.monarch_flops == 116011284480
    assert rep.recompute_flops == 43958992896
    assert abs(rep.reduction_ratio - 22.258) < 22.258e-3


def test_sparsity_table(vm):
    # acceptance.cpp:139-156 / test_video.cpp:109-116
    cfg = vm.VMonarchConfig()
    r61 = vm.flops_estimate(vm.TokenGrid(16, 28, 52, 64), cfg, 64)
    assert abs(r61.sparsity - 0.873626) < 1e-4 and r61.sparsity_approx == 0.875
    r141 = vm.flops_estimate(vm.TokenGrid(36, 28, 52, 64), cfg, 64)
    assert abs(r141.sparsity - 0.943070) < 1e-4


@pytest.mark.parametrize("b,n", [(3, 6), (1, 12), (12, 12), (4, 12), (1456, 1456 * 3)])
def test_make_perm_bit_exact(vm, orc, b, n):
    assert vm.make_perm(b, n) == orc.make_perm(b, n).tolist()


def test_make_perm_properties(vm):
    assert vm.make_perm(3, 6) == [0, 3, 1, 4, 2, 5]          # test_tensor_core.cpp:14-18
    for m in range(1, 7):
        for b in range(1, 7):
            n = m * b
            p = vm.make_perm(b, n)
            assert sorted(p) == list(range(n))                 # bijection
            q = vm.make_perm(n // b, n)
            assert [p[q[i]] for i in range(n)] == list(range(n))  # dual permutation is the inverse


def test_errors_map_to_reference_classes(vm):
    with pytest.raises(vm.DimensionError, match="dimension error"):
        vm.make_perm(3, 10)                                   # test_tensor_core.cpp:26-29
    with pytest.raises(vm.DimensionError, match="override factor sizes"):
        vm.factorize(vm.TokenGrid(4, 3, 3, 8), vm.VMonarchConfig(override_m_b=(5, 7)))
    with pytest.raises(vm.DimensionError):
        vm.factorize(vm.TokenGrid(0, 3, 3, 8))


def test_fwd_host_validation_without_device(vm):
    g = vm.TokenGrid(4, 8, 8, 64, 2, 1)._c()
    c = vm.VMonarchConfig(iters=0)._c()
    st = vm.lib.vmb_vmonarch_fwd(C.byref(g), C.byref(c), 0, None, None, None, None, None, None, None, 0, None)
    assert st == 1 and vm.lib.vmb_last_error().startswith(b"dimension error: iteration count")
    c = vm.VMonarchConfig()._c()
    st = vm.lib.vmb_vmonarch_fwd(C.byref(g), C.byref(c), 0, None, None, None, None, None, None, None, 0, None)
    assert st == 1 and b"workspace" in vm.lib.vmb_last_error()


def test_workspace_size(vm):
    g = vm.TokenGrid(81, 28, 52, 128, 40, 1)
    c = vm.VMonarchConfig()
    n = g.tokens() * 40
    ws = vm._vmb_ws_size(C.byref(g._c()), C.byref(c._c()), 1)
    base = 4 * n * 128 * 2 + 2 * n * 4  # aR, aL, aL_lo, y (bf16) + cR, cL (f32)
    split_kv = 40 * 16 * (28 * 52) * 129 * 4  # recompute split-KV partials, at most 16 splits
    assert base <= ws <= base + split_kv + 8 * 256


def test_cpu_tensors_are_refused(vm):
    import torch
    x = torch.zeros(2, 256, 64)
    with pytest.raises(vm.DimensionError, match="CUDA"):
        vm.vmonarch_attention(x, x, x, vm.TokenGrid(4, 8, 8, 64, 2, 1))


def test_shard_range_and_multi_workspace_sizes(vm):
    """vmb_shard_range is the partition of dist.unit_shards / slab_partition; the multi-GPU
    workspace of part r is the forward's workspace for that part (+ the gathered K/V in seq mode)."""
    import ctypes as C
    from paper_2601_22275_b200 import _vmb_ws_size_multi, _vmb_ws_size, _vmb_ws_size_seq
    from paper_2601_22275_b200.dist import slab_partition
    for n, parts in [(40, 8), (1456, 3), (3, 8)]:
        assert [vm.shard_range(n, parts, r) for r in range(parts)] == slab_partition(n, parts)
    assert vm.shard_range(10, 0, 0) == (0, 0)
    grid = vm.TokenGrid(81, 28, 52, 128, 40, 1)
    g, c = grid._c(), vm.VMonarchConfig()._c()
    for r in range(3):
        u = vm.shard_range(40, 3, r)[1]
        gp = vm.TokenGrid(81, 28, 52, 128, u, 1)._c()
        assert _vmb_ws_size_multi(3, r, 0, C.byref(g), C.byref(c), 1) == _vmb_ws_size(C.byref(gp), C.byref(c), 1)
        cnt = vm.shard_range(28 * 52, 3, r)[1]
        kv = 40 * grid.tokens() * 128 * 2
        seq = _vmb_ws_size_multi(3, r, 1, C.byref(g), C.byref(c), 1)
        assert seq >= _vmb_ws_size_seq(C.byref(g), C.byref(c), 1, cnt) + 2 * kv
    assert _vmb_ws_size_multi(3, 3, 0, C.byref(g), C.byref(c), 1) == 0        # rank out of range
    assert _vmb_ws_size_multi(3, 0, 1, C.byref(g), C.byref(c), 0) == 0        # seq mode is bf16-only
    assert "bf16" in vm._vmb_last_error().decode()


def test_torch_op_fake_kernel_on_cpu(vm):
    """The DiT op's fake kernel (shape propagation) works without a GPU."""
    import torch
    from torch._subclasses.fake_tensor import FakeTensorMode
    import paper_2601_22275_b200.torch_op  # noqa: F401  (registers vmb::vmonarch_attention)
    with FakeTensorMode():
        qkv = torch.empty((2, 4 * 8 * 16, 3, 2, 128), dtype=torch.bfloat16)
        q, k, v = qkv.unbind(2)
        o = torch.ops.vmb.vmonarch_attention(q, k, v, 4, 8, 16)
        assert o.shape == (2, 512, 2, 128) and o.dtype == torch.bfloat16


def test_plain_c_caller(tmp_path):
    """include/vmb.h is a plain C ABI: a C11 program (-Wall -Werror) links libvmb and calls it."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2601_22275_b200")
    exe = str(tmp_path / "c_abi_example")
    cc = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                         os.path.join(root, "tests", "c_abi_example.c"), "-L", libdir, "-lvmb", f"-Wl,-rpath,{libdir}",
                         "-L/usr/local/cuda/lib64", "-lcudart", "-o", exe], capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and r.stdout.startswith("ok"), (r.returncode, r.stdout, r.stderr)
