"""GPU: the fp32 parity mode on tensor cores (d = 128, m <= 128).  Q, K, V and each aR are
split into bf16 hi/lo halves and every product runs as three bf16 tcgen05 MMA groups with
fp32 accumulation (csrc/kernels/fa2_tc.cu, hilo instantiation); the L half-steps stay on the
CUDA cores.  The north-star fp32 tolerance is <= 1e-4 relative Frobenius against the reference
CPU path (monarch.hpp:81-98 precision policy: exp in T = float, sums in double).

Also: the plan really is the tensor-core one (the per-kernel profile sees fa2 launches and
CUDA-core time only for the L-steps and the split), and fp32 shapes outside it (d != 128)
still take the CUDA-core kernels."""
import numpy as np
import pytest
import torch

from oracle.oracle import workload
from test_gpu_parity import oracle_fwd, run_gpu
from vmb_testutil import relfro

pytestmark = pytest.mark.gpu
F32_TOL = 1e-4

CASES = [
    # (T, h, w), heads, batch, config, sigma
    ((4, 8, 16), 2, 1, dict(), 1.0),
    ((4, 8, 16), 1, 2, dict(iters=3), 1.0),
    ((3, 10, 20), 2, 1, dict(iters=1), 1.0),                        # ragged tiles (b = 200)
    ((5, 6, 6), 1, 1, dict(iters=3, clamp_enabled=False), 1.0),
    ((4, 7, 7), 2, 1, dict(iters=3, recompute_first_frame=False, override_m_b=(49, 4)), 3.0),
    ((21, 6, 7), 1, 1, dict(), 2.5),
    ((8, 12, 16), 1, 1, dict(clamp_min=0.5), 3.0),
    ((2, 16, 40), 1, 1, dict(override_m_b=(40, 32)), 1.0),
]


@pytest.mark.parametrize("gridt,heads,batch,kw,sigma", CASES)
def test_fp32_tensor_core_path_matches_oracle(vm, orc, cuda, gridt, heads, batch, kw, sigma):
    grid = vm.TokenGrid(*gridt, head_dim=128, heads=heads, batch=batch)
    cfg = vm.VMonarchConfig(**kw)
    q, k, v = workload(grid.units(), grid.tokens(), 128, seed=sum(gridt) + heads, sigma=sigma)
    ref = oracle_fwd(orc, q, k, v, grid, cfg)
    got = run_gpu(vm, q, k, v, grid, cfg, torch.float32, cuda)
    err = relfro(got, ref)
    print(f"fp32 tensor-core {gridt} {kw} sigma={sigma}: rel-Fro {err:.2e}")
    assert err <= F32_TOL


def _profile(vm, fn):
    """Per-kernel-family launch counts of fn() (vmb_profile_read ids, vmb.h)."""
    import ctypes as C
    vm.lib.vmb_profile_enable.argtypes = [C.c_int32]
    vm.lib.vmb_profile_read.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
    ms, cnt = (C.c_double * 7)(), (C.c_uint64 * 7)()
    vm.lib.vmb_profile_read(C.addressof(ms), C.addressof(cnt), 1)
    vm.lib.vmb_profile_enable(1)
    fn()
    torch.cuda.synchronize()
    vm.lib.vmb_profile_enable(0)
    vm.lib.vmb_profile_read(C.addressof(ms), C.addressof(cnt), 1)
    return list(cnt)


def test_fp32_tensor_core_plan_is_used(vm, cuda):
    grid = vm.TokenGrid(4, 8, 16, 128, 2, 1)
    x = [torch.randn((2, grid.tokens(), 128), device=cuda) for _ in range(3)]
    vm.vmonarch_attention(*x, grid)
    cnt = _profile(vm, lambda: vm.vmonarch_attention(*x, grid, check=False))
    # ids (vmb.h): 0 R half-steps (fa2, value = K: t = 2), 2 attention with a separate V (fa2 hilo:
    # the y pass and the recompute), 5 CUDA cores (the hi/lo splits and the L-steps)
    assert cnt[0] == 2 and cnt[2] == 2 and cnt[5] > 0
    # d = 64 in fp32 stays on the CUDA cores
    g64 = vm.TokenGrid(4, 8, 16, 64, 2, 1)
    y = [torch.randn((2, g64.tokens(), 64), device=cuda) for _ in range(3)]
    cnt = _profile(vm, lambda: vm.vmonarch_attention(*y, g64, check=False))
    assert cnt[0] == 0 and cnt[5] > 0


def test_fp32_bhsd_views_equal_contiguous(vm, cuda):
    # BSHD activations (a strided view) go through the hi/lo split, not a contiguous copy
    grid = vm.TokenGrid(4, 8, 16, 128, 2, 1)
    g = torch.Generator(device=cuda).manual_seed(4)
    qkv = torch.randn((1, grid.tokens(), 3, 2, 128), device=cuda, generator=g)
    q, k, v = (qkv[:, :, i].transpose(1, 2) for i in range(3))
    a = vm.vmonarch_attention(q, k, v, grid)
    b = vm.vmonarch_attention(q.contiguous(), k.contiguous(), v.contiguous(), grid)
    assert torch.equal(a, b)


@pytest.mark.slow
def test_fp32_c2_one_head(vm, orc, cuda):
    # C2 grid (21x30x52, N = 32 760), one head, fp32 vs the oracle (~15 s of CPU)
    grid = vm.TokenGrid(21, 30, 52, 128, 1, 1)
    cfg = vm.VMonarchConfig()
    q, k, v = workload(1, grid.tokens(), 128, seed=11)
    ref = oracle_fwd(orc, q, k, v, grid, cfg)
    got = run_gpu(vm, q, k, v, grid, cfg, torch.float32, cuda)
    err = relfro(got, ref)
    print(f"fp32 tensor-core C2 one head: rel-Fro {err:.2e}")
    assert err <= F32_TOL


def test_fp32_tensor_core_factor_export(vm, orc, cuda):
    # MonarchFactors after the tensor-core plan: the export rebuilds fp32 aR / aL from their
    # hi/lo pairs (vmb_export_factors), so L and R match the oracle's f32 factors
    import ctypes as C
    grid = vm.TokenGrid(3, 4, 10, 128, 1, 1)
    cfg = vm.VMonarchConfig(iters=2, recompute_first_frame=False)
    q, k, v = workload(1, grid.tokens(), 128, seed=21)
    f = []
    vm.vmonarch_attention(*(torch.from_numpy(x).to(cuda) for x in (q, k, v)), grid, cfg, factors_out=f)
    L, R = (t.cpu().numpy() for t in f[0])
    m, b = 3, 40
    rL = np.zeros((b, m, m), np.float32)
    rR = np.zeros((m, b, b), np.float32)
    out = np.zeros((grid.tokens(), 128), np.float32)
    fn = orc.lib.vmo_vmonarch_unit_f32
    fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 5 + [C.c_double, C.c_int, C.c_int] + [C.c_int64] * 4 + \
        [C.c_void_p] * 3
    ptr = lambda a: np.ascontiguousarray(a).ctypes.data_as(C.c_void_p)  # noqa: E731
    qq, kk, vv = (np.ascontiguousarray(x[0]) for x in (q, k, v))
    assert fn(ptr(qq), ptr(kk), ptr(vv), 3, 4, 10, 128, 2, 0.1, 1, 0, 0, 0, 64, 64, ptr(out), ptr(rL), ptr(rR)) == 0
    assert np.abs(L - rL).max() <= 1e-4
    assert np.abs(R - rR).max() <= 1e-4
