"""GPU properties the reference tests pin, restated on the CUDA path, plus size-independent
properties checked at the full BASELINE sizes (C2 / C4) where the CPU oracle is too slow."""
import numpy as np
import pytest
import torch

from oracle.oracle import bf16_round, randn, workload
from vmb_testutil import relfro

pytestmark = pytest.mark.gpu


def dev_inputs(vm, grid, dtype, cuda, seed=0, sigma=1.0):
    q, k, v = workload(grid.units(), grid.tokens(), grid.head_dim, seed=seed, sigma=sigma)
    if dtype == torch.bfloat16:
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    return [torch.from_numpy(x).to(cuda, dtype) for x in (q, k, v)]


@pytest.mark.parametrize("dtype,d", [(torch.float32, 8), (torch.bfloat16, 128)])
def test_single_frame_reduces_to_dense(vm, orc, cuda, dtype, d):
    # test_video.cpp:60-71: T = 1 grids are dense attention (with and without recompute)
    grid = vm.TokenGrid(1, 4, 8, d, 1, 1)
    q, k, v = dev_inputs(vm, grid, dtype, cuda)
    ref, _, _ = orc.dense_attention_f64(q[0].double().cpu().numpy(), k[0].double().cpu().numpy(),
                                        v[0].double().cpu().numpy())
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    for rc in (True, False):
        out = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig(recompute_first_frame=rc))
        assert relfro(out[0].double().cpu().numpy(), ref) <= tol


@pytest.mark.parametrize("n,m,b", [(48, 48, 1), (48, 1, 48), (256, 256, 1), (200, 1, 200)])
def test_degenerate_factorizations_equal_dense_fp32(vm, orc, cuda, n, m, b):
    # test_monarch_core.cpp:285-309 / acceptance #1: b = 1 or m = 1 is dense attention
    grid = vm.TokenGrid(1, 1, n, 16, 1, 1)
    cfg = vm.VMonarchConfig(iters=3, recompute_first_frame=False, override_m_b=(m, b))
    q, k, v = dev_inputs(vm, grid, torch.float32, cuda, seed=21)
    out = vm.vmonarch_attention(q, k, v, grid, cfg)
    ref, _, _ = orc.dense_attention_f64(*(x[0].double().cpu().numpy() for x in (q, k, v)))
    assert np.abs(out[0].double().cpu().numpy() - ref).max() < 1e-4


@pytest.mark.parametrize("dtype,d,gridt", [(torch.float32, 8, (4, 4, 4)), (torch.bfloat16, 128, (4, 8, 16)),
                                           (torch.bfloat16, 128, (3, 10, 20))])
def test_recompute_touches_only_first_frame_rows(vm, cuda, dtype, d, gridt):
    # test_video.cpp:73-91 / acceptance #8: rows >= hw are bitwise identical to a recompute-off run
    grid = vm.TokenGrid(*gridt, head_dim=d, heads=2, batch=1)
    q, k, v = dev_inputs(vm, grid, dtype, cuda, seed=2)
    on = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig())
    off = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig(recompute_first_frame=False))
    hw = grid.frame_tokens()
    assert torch.equal(on[:, hw:], off[:, hw:])
    assert not torch.equal(on[:, :hw], off[:, :hw])


@pytest.mark.parametrize("dtype,d,gridt", [(torch.float32, 8, (4, 4, 4)), (torch.bfloat16, 128, (3, 10, 20))])
def test_recomputed_rows_equal_dense(vm, orc, cuda, dtype, d, gridt):
    # test_video.cpp:93-107
    grid = vm.TokenGrid(*gridt, head_dim=d, heads=1, batch=1)
    q, k, v = dev_inputs(vm, grid, dtype, cuda, seed=3)
    out = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig())
    hw = grid.frame_tokens()
    ref, _, _ = orc.dense_attention_f64(q[0, :hw].double().cpu().numpy(), k[0].double().cpu().numpy(),
                                        v[0].double().cpu().numpy())
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    assert relfro(out[0, :hw].double().cpu().numpy(), ref) <= tol


@pytest.mark.parametrize("dtype,d", [(torch.float32, 6), (torch.bfloat16, 128)])
def test_units_independent_bitwise(vm, cuda, dtype, d):
    # test_video.cpp:197-216: each unit equals its own single-unit run, bitwise
    grid = vm.TokenGrid(3, 4, 8, d, 3, 2)
    q, k, v = dev_inputs(vm, grid, dtype, cuda, seed=4)
    full = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig())
    g1 = vm.TokenGrid(3, 4, 8, d, 1, 1)
    for u in range(grid.units()):
        solo = vm.vmonarch_attention(q[u:u + 1].contiguous(), k[u:u + 1].contiguous(), v[u:u + 1].contiguous(),
                                     g1, vm.VMonarchConfig())
        assert torch.equal(solo[0], full[u])


@pytest.mark.parametrize("dtype,d", [(torch.float32, 16), (torch.bfloat16, 128)])
def test_deterministic(vm, cuda, dtype, d):
    grid = vm.TokenGrid(5, 8, 16, d, 2, 1)
    q, k, v = dev_inputs(vm, grid, dtype, cuda, seed=5)
    a = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig())
    b = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig())
    assert torch.equal(a, b)


@pytest.mark.parametrize("dtype,d", [(torch.float32, 16), (torch.bfloat16, 128)])
def test_bhsd_strided_views_equal_contiguous(vm, cuda, dtype, d):
    # BSHD activations passed as a (B, H, N, d) view
    grid = vm.TokenGrid(4, 8, 16, d, 2, 2)
    n = grid.tokens()
    x = torch.randn(3, 2, n, 2, d, device=cuda).to(dtype)   # (qkv, B, N, H, d)
    q, k, v = (x[i].transpose(1, 2) for i in range(3))      # (B, H, N, d) strided views
    out = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig())
    ref = vm.vmonarch_attention(*(t.reshape(4, n, d).contiguous() if False else
                                  t.contiguous().reshape(4, n, d) for t in (q, k, v)), grid, vm.VMonarchConfig())
    assert torch.equal(out.reshape(4, n, d), ref)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_nonfinite_q_is_domain_error(vm, cuda, dtype):
    # test_monarch_core.cpp:60-66 (init_state rejects non-finite Q)
    d = 128 if dtype == torch.bfloat16 else 8
    grid = vm.TokenGrid(2, 4, 8, d, 1, 1)
    q, k, v = dev_inputs(vm, grid, dtype, cuda)
    q[0, 17, 3] = float("nan")
    with pytest.raises(vm.DomainError):
        vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig())
    q[0, 17, 3] = float("inf")
    with pytest.raises(vm.DomainError):
        vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig())


def test_shape_validation(vm, cuda):
    # test_video.cpp:238-244
    grid = vm.TokenGrid(2, 2, 2, 4)
    q = torch.randn(1, 8, 4, device=cuda)
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention(q, torch.randn(1, 7, 4, device=cuda), q, grid)
    with pytest.raises(vm.DimensionError):
        vm.vmonarch_attention(q, q, q, grid, vm.VMonarchConfig(iters=0))


def test_factors_out_row_stochastic_and_identity(vm, orc, cuda):
    # test_video.cpp:218-236 and test_monarch_core.cpp:323-356 / acceptance #7: O == M(F) V
    grid = vm.TokenGrid(3, 2, 2, 4, 2, 1)
    q, k, v = dev_inputs(vm, grid, torch.float32, cuda, seed=5)
    cfg = vm.VMonarchConfig(recompute_first_frame=False)
    facs = []
    out = vm.vmonarch_attention(q, k, v, grid, cfg, factors_out=facs)
    assert len(facs) == 2
    m, b = 3, 4
    for u, (L, R) in enumerate(facs):
        assert torch.allclose(R.sum(-1), torch.ones_like(R.sum(-1)), atol=1e-5)
        assert torch.allclose(L.sum(-1), torch.ones_like(L.sum(-1)), atol=1e-5)
        M = orc.materialize_monarch(L.double().cpu().numpy(), R.double().cpu().numpy(), b, m * b)
        assert np.abs(M @ v[u].double().cpu().numpy() - out[u].double().cpu().numpy()).max() < 1e-4
        _, rL, rR = orc.monarch_attention(q[u].cpu().numpy(), k[u].cpu().numpy(), v[u].cpu().numpy(), m, b,
                                          iters=2, want_factors=True)
        assert np.abs(L.cpu().numpy() - rL).max() < 1e-5 and np.abs(R.cpu().numpy() - rR).max() < 1e-5


def test_objective_monotone_without_clamp(vm, orc, cuda):
    # acceptance #2 on the device path: the variational objective never decreases over t
    for seed in range(5):
        m, b, d = 3 + seed % 3, 4 + seed, 4
        grid = vm.TokenGrid(m, 1, b, d, 1, 1)
        q, k, v = dev_inputs(vm, grid, torch.float32, cuda, seed=100 + seed)
        prev = -np.inf
        for t in range(1, 5):
            facs = []
            cfg = vm.VMonarchConfig(iters=t, clamp_enabled=False, recompute_first_frame=False)
            vm.vmonarch_attention(q, k, v, grid, cfg, factors_out=facs)
            L, R = facs[0]
            j = orc.monarch_objective(L.double().cpu().numpy(), R.double().cpu().numpy(),
                                      q[0].double().cpu().numpy(), k[0].double().cpu().numpy(), m, b)
            assert j >= prev - 1e-5 * abs(j)
            prev = j


# ------------------------------------------------------------------ full-size properties (BASELINE shapes)
@pytest.mark.parametrize("gridt,heads", [((21, 30, 52), 2), ((81, 28, 52), 2)])
def test_full_size_constant_values_give_constant_output(vm, cuda, gridt, heads):
    # R and L are row-stochastic, so V == c gives O == c for any Q, K (size-independent)
    grid = vm.TokenGrid(*gridt, head_dim=128, heads=heads, batch=1)
    n = grid.tokens()
    g = torch.Generator(device=cuda).manual_seed(0)
    q = torch.randn(heads, n, 128, device=cuda, generator=g).bfloat16()
    k = torch.randn(heads, n, 128, device=cuda, generator=g).bfloat16()
    v = torch.full((heads, n, 128), 0.75, device=cuda, dtype=torch.bfloat16)
    out = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig())
    assert (out.float() - 0.75).abs().max().item() <= 0.75 * 2e-2


@pytest.mark.parametrize("gridt", [(21, 30, 52), (81, 28, 52)])
def test_full_size_linearity_in_v(vm, cuda, gridt):
    # O is linear in V for fixed Q, K (the factors do not depend on V)
    grid = vm.TokenGrid(*gridt, head_dim=128, heads=1, batch=1)
    n = grid.tokens()
    g = torch.Generator(device=cuda).manual_seed(1)
    q, k, v1, v2 = (torch.randn(1, n, 128, device=cuda, generator=g).bfloat16() for _ in range(4))
    cfg = vm.VMonarchConfig()
    o1 = vm.vmonarch_attention(q, k, v1, grid, cfg).float()
    o2 = vm.vmonarch_attention(q, k, v2, grid, cfg).float()
    o12 = vm.vmonarch_attention(q, k, (v1.float() + v2.float()).bfloat16(), grid, cfg).float()
    assert relfro((o1 + o2).cpu().numpy(), o12.cpu().numpy()) <= 2e-2


def test_full_size_c4_first_frame_rows_match_dense_kernel(vm, cuda):
    # the recomputed rows [0, hw) equal dense attention of Q[0:hw] against all keys
    grid = vm.TokenGrid(81, 28, 52, 128, 1, 1)
    n, hw = grid.tokens(), grid.frame_tokens()
    g = torch.Generator(device=cuda).manual_seed(2)
    q, k, v = (torch.randn(1, n, 128, device=cuda, generator=g).bfloat16() for _ in range(3))
    out = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig())
    ref = torch.nn.functional.scaled_dot_product_attention(q[:, :hw].float(), k.float(), v.float())
    assert relfro(out[:, :hw].float().cpu().numpy(), ref.cpu().numpy()) <= 2e-2
    assert torch.isfinite(out).all()


@pytest.mark.parametrize("chunk", [1, 3, 8])
def test_host_pipeline_equals_device_call(vm, cuda, chunk):
    """vmonarch_attention_host (chunked H2D / forward / D2H streams) == the device call."""
    grid = vm.TokenGrid(6, 10, 26, 128, 5, 1)
    g = torch.Generator().manual_seed(3)
    q, k, v = (torch.randn((5, grid.tokens(), 128), generator=g).to(torch.bfloat16).pin_memory() for _ in range(3))
    ref = vm.vmonarch_attention(q.to(cuda), k.to(cuda), v.to(cuda), grid).cpu()
    got = vm.vmonarch_attention_host(q, k, v, grid, chunk_units=chunk)
    torch.cuda.synchronize()
    T, hw = grid.t_frames, grid.h * grid.w
    a, b = got.float().view(5, T, hw, 128), ref.float().view(5, T, hw, 128)
    assert torch.equal(a[:, 1:], b[:, 1:])                   # R/L half-steps: per-unit, bitwise
    assert float((a[:, 0] - b[:, 0]).norm() / b[:, 0].norm()) <= 2e-3  # recompute: split plan may differ


def test_c4_unit_equals_its_solo_run_bitwise(vm, cuda):
    # test_video.cpp:197-216 at the C4 shape: the split-KV recompute plan depends on the
    # per-unit shape only, so a head's output does not depend on the other heads in the call
    grid = vm.TokenGrid(81, 28, 52, 128, 6, 1)
    g = torch.Generator(device=cuda).manual_seed(11)
    q, k, v = (torch.randn((6, grid.tokens(), 128), generator=g, device=cuda).to(torch.bfloat16) for _ in range(3))
    full = vm.vmonarch_attention(q, k, v, grid)
    g1 = vm.TokenGrid(81, 28, 52, 128, 1, 1)
    for u in (0, 5):
        solo = vm.vmonarch_attention(q[u:u + 1].contiguous(), k[u:u + 1].contiguous(), v[u:u + 1].contiguous(), g1)
        assert torch.equal(solo[0], full[u])
