"""GPU parity: the CUDA path (through libvmb.so) against the CPU oracle on identical inputs.

Tolerances (north_star): fp32 parity mode <= 1e-4 relative, bf16 <= 2e-2 relative, both
norm-wise (relative Frobenius, as the reference bench reports, bench_main.cpp:64-76).
bf16 inputs are bf16-rounded once and the oracle runs in fp32 on the same values."""
import numpy as np
import pytest
import torch

from oracle.oracle import bf16_round, randn, workload
from vmb_testutil import relfro

pytestmark = pytest.mark.gpu

F32_TOL = 1e-4
BF16_TOL = 2e-2


def run_gpu(vm, q, k, v, grid, cfg, dtype, cuda):
    tq, tk, tv = (torch.from_numpy(np.ascontiguousarray(x)).to(cuda, dtype) for x in (q, k, v))
    out = vm.vmonarch_attention(tq, tk, tv, grid, cfg)
    torch.cuda.synchronize()
    return out.float().cpu().numpy()


def oracle_fwd(orc, q, k, v, grid, cfg):
    return orc.vmonarch_attention(q, k, v, (grid.t_frames, grid.h, grid.w), iters=cfg.iters,
                                  clamp_min=cfg.clamp_min, clamp_enabled=cfg.clamp_enabled,
                                  recompute=cfg.recompute_first_frame, override=cfg.override_m_b or (0, 0))


# ------------------------------------------------------------------ C1 (BASELINE configs[0]), fp32
def test_c1_fp32_matches_reference_golden(vm, golden, cuda):
    grid = vm.TokenGrid(4, 8, 8, 64, 2, 1)
    cfg = vm.VMonarchConfig(iters=3)
    got = run_gpu(vm, golden["c1_q"], golden["c1_k"], golden["c1_v"], grid, cfg, torch.float32, cuda)
    assert relfro(got, golden["c1_out"]) <= F32_TOL
    assert np.abs(got - golden["c1_out"]).max() <= 1e-4


FP32_CASES = [
    ((3, 4, 5), 16, 2, 1, dict()),
    ((4, 4, 4), 8, 1, 1, dict(recompute_first_frame=False)),
    ((4, 8, 8), 32, 1, 2, dict(override_m_b=(16, 16))),
    ((2, 3, 7), 12, 3, 1, dict(iters=1)),
    ((5, 6, 6), 128, 1, 1, dict(iters=3, clamp_enabled=False)),
    ((6, 10, 10), 96, 1, 2, dict()),
    ((3, 8, 8), 256, 1, 1, dict()),
]


@pytest.mark.parametrize("gridt,d,heads,batch,kw", FP32_CASES)
def test_fp32_forward_parity(vm, orc, cuda, gridt, d, heads, batch, kw):
    grid = vm.TokenGrid(*gridt, head_dim=d, heads=heads, batch=batch)
    cfg = vm.VMonarchConfig(**kw)
    q, k, v = workload(grid.units(), grid.tokens(), d, seed=5, sigma=1.5)
    ref = oracle_fwd(orc, q, k, v, grid, cfg)
    got = run_gpu(vm, q, k, v, grid, cfg, torch.float32, cuda)
    assert relfro(got, ref) <= F32_TOL


BF16_CASES = [
    # (T, h, w), heads, batch, sigma, cfg kwargs   — d = 128 (tcgen05 path)
    ((4, 8, 16), 2, 1, 1.0, dict()),                 # b = 128 (one tile)
    ((3, 10, 20), 2, 1, 1.0, dict()),                # b = 200 (tail tile 72)
    ((5, 12, 13), 1, 2, 1.0, dict(iters=3)),         # b = 156, batch > 1
    ((4, 8, 16), 1, 1, 1.0, dict(recompute_first_frame=False)),
    ((21, 6, 7), 1, 1, 1.0, dict()),                 # m = 21 (Wan temporal size), b = 42
    ((81, 3, 4), 1, 1, 1.0, dict()),                 # m = 81 (321-frame temporal size)
    ((100, 2, 3), 1, 1, 1.0, dict()),                # m = 100 > 96: L-step column sums on the tensor core
    ((49, 3, 5), 2, 1, 1.0, dict()),                 # m = 49: two positions per L-step CTA, b = 15 odd
    ((21, 5, 3), 1, 1, 2.0, dict(iters=3)),          # m = 21: four positions per L-step CTA, b = 15
    ((6, 9, 11), 2, 1, 3.0, dict()),                 # peaky attention, sigma 3
    ((4, 8, 16), 1, 1, 2.0, dict(iters=1)),
    ((4, 8, 16), 1, 1, 2.0, dict(clamp_min=0.9)),    # clamp-forcing
    ((4, 8, 8), 1, 1, 1.0, dict(override_m_b=(8, 32))),  # override factorization (recompute after apply)
]


@pytest.mark.parametrize("gridt,heads,batch,sigma,kw", BF16_CASES)
def test_bf16_forward_parity(vm, orc, cuda, gridt, heads, batch, sigma, kw):
    grid = vm.TokenGrid(*gridt, head_dim=128, heads=heads, batch=batch)
    cfg = vm.VMonarchConfig(**kw)
    q, k, v = workload(grid.units(), grid.tokens(), 128, seed=9, sigma=sigma)
    q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    ref = oracle_fwd(orc, q, k, v, grid, cfg)
    got = run_gpu(vm, q, k, v, grid, cfg, torch.bfloat16, cuda)
    assert relfro(got, ref) <= BF16_TOL


@pytest.mark.slow
def test_bf16_c2_one_head_parity(vm, orc, cuda):
    # C2 shape (21x30x52, N = 32760, b = 1560 = 12*128 + 24), one head: oracle ~15 s
    grid = vm.TokenGrid(21, 30, 52, 128, 1, 1)
    cfg = vm.VMonarchConfig()
    q, k, v = workload(1, grid.tokens(), 128, seed=1)
    q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    ref = oracle_fwd(orc, q, k, v, grid, cfg)
    got = run_gpu(vm, q, k, v, grid, cfg, torch.bfloat16, cuda)
    assert relfro(got, ref) <= BF16_TOL


# ------------------------------------------------------------------ half steps
@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.bfloat16, BF16_TOL)])
@pytest.mark.parametrize("m,b,d", [(3, 150, 128), (2, 128, 128), (4, 37, 32), (1, 256, 64)])
def test_rstep_parity(vm, orc, cuda, dtype, tol, m, b, d):
    qs = bf16_round(randn((2, m, b, d), 11, dtype=np.float32) / np.sqrt(d))
    kk = bf16_round(randn((2, m, b, d), 12, dtype=np.float32))
    cR = (0.05 + np.abs(randn((2, m, b), 13, dtype=np.float32))).astype(np.float32)
    aL, cL, _ = vm.r_update(torch.from_numpy(qs).to(cuda, dtype), torch.from_numpy(cR).to(cuda),
                            torch.from_numpy(kk).to(cuda, dtype))
    for u in range(2):
        raL, rcL, _ = orc.rstep(qs[u], cR[u], kk[u], want_R=False)
        assert relfro(aL[u].float().cpu().numpy(), raL) <= tol
        assert relfro(cL[u].cpu().numpy(), rcL) <= tol


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.bfloat16, BF16_TOL)])
@pytest.mark.parametrize("m,b,d", [(4, 16, 128), (5, 2, 128), (21, 40, 128), (21, 7, 128), (33, 6, 128), (49, 5, 128),
                                   (64, 3, 128), (81, 8, 128), (96, 5, 128), (100, 4, 128), (128, 3, 128),
                                   (5, 7, 32)])
def test_lstep_parity(vm, orc, cuda, dtype, tol, m, b, d):
    rng = np.random.default_rng(2)
    Qb = bf16_round(rng.standard_normal((2, b, m, d)).astype(np.float32) / np.sqrt(d))
    aL = bf16_round(rng.standard_normal((2, b, m, d)).astype(np.float32))
    cL = (-np.log(max(b, 2)) + 0.3 * rng.standard_normal((2, b, m))).astype(np.float32)
    aR, cR, _ = vm.l_update(torch.from_numpy(Qb).to(cuda, dtype), torch.from_numpy(aL).to(cuda, dtype),
                            torch.from_numpy(cL).to(cuda))
    for u in range(2):
        raR, rcR, _ = orc.lstep(Qb[u], aL[u], cL[u], want_L=False)
        assert relfro(aR[u].float().cpu().numpy(), raR) <= tol
        assert relfro(cR[u].cpu().numpy(), rcR) <= tol


def test_half_step_factor_export_fp32(vm, orc, cuda):
    m, b, d = 3, 20, 16
    qs = randn((1, m, b, d), 3, dtype=np.float32)
    kk = randn((1, m, b, d), 4, dtype=np.float32)
    cR = np.ones((1, m, b), np.float32)
    aL, cL, R = vm.r_update(torch.from_numpy(qs).to(cuda), torch.from_numpy(cR).to(cuda),
                            torch.from_numpy(kk).to(cuda), want_R=True)
    _, _, rR = orc.rstep(qs[0], cR[0], kk[0])
    assert np.abs(R[0].cpu().numpy() - rR).max() <= 1e-5
    Qb = np.ascontiguousarray(qs[0].transpose(1, 0, 2))[None]
    aR, cRo, L = vm.l_update(torch.from_numpy(Qb).to(cuda), aL, cL, want_L=True)
    _, _, rL = orc.lstep(Qb[0], aL[0].cpu().numpy(), cL[0].cpu().numpy())
    assert np.abs(L[0].cpu().numpy() - rL).max() <= 1e-5


def test_clamp_disabled_nonpositive_cR_is_domain_error(vm, cuda):
    # test_monarch_core.cpp:229-238
    aR = torch.randn(1, 2, 3, 2, device=cuda)
    cR = torch.ones(1, 2, 3, device=cuda)
    cR[0, 1, 1] = 0.0
    with pytest.raises(vm.DomainError):
        vm.r_update(aR, cR, torch.randn(1, 2, 3, 2, device=cuda), clamp_enabled=False)


# ------------------------------------------------------------------ online-entropy attention
@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.bfloat16, BF16_TOL)])
@pytest.mark.parametrize("nq,nk,d", [(128, 128, 128), (100, 300, 128), (300, 1000, 128), (40, 256, 16),
                                    (64, 5000, 64)])  # last: 19-way split-KV on CUDA cores in fp32
def test_flash_entropy_parity(vm, orc, cuda, dtype, tol, nq, nk, d):
    q = bf16_round(randn((2, nq, d), 1, dtype=np.float32) / np.sqrt(d))
    k = bf16_round(randn((2, nk, d), 2, dtype=np.float32))
    v = bf16_round(randn((2, nk, d), 3, dtype=np.float32))
    o, lse, ent = vm.flash_entropy_fwd(*(torch.from_numpy(x).to(cuda, dtype) for x in (q, k, v)),
                                       want_entropy=dtype == torch.float32)
    for u in range(2):
        ro, rl, re = orc.flash_entropy_fwd(q[u], k[u], v[u])
        assert relfro(o[u].float().cpu().numpy(), ro) <= tol
        assert np.abs(lse[u].cpu().numpy() - rl).max() <= 1e-4
        if ent is not None:
            assert np.abs(ent[u].cpu().numpy() - re).max() <= 1e-4


def test_flash_constant_keys_entropy_is_log_n(vm, cuda):
    # test_flash_entropy.cpp:15-25
    n, d = 37, 8
    q = torch.randn(1, 5, d, device=cuda)
    k = (0.25 * torch.arange(1, d + 1, device=cuda, dtype=torch.float32)).expand(1, n, d).contiguous()
    v = torch.randn(1, n, d, device=cuda)
    _, _, ent = vm.flash_entropy_fwd(q, k, v)
    assert (ent - np.log(n)).abs().max().item() < 1e-5


def test_dense_forward_parity(vm, orc, cuda):
    n, d = 384, 128
    q, k, v = (bf16_round(randn((1, n, d), s, dtype=np.float32)) for s in (4, 5, 6))
    got = vm.dense_forward(*(torch.from_numpy(x).to(cuda, torch.bfloat16) for x in (q, k, v)))
    ref = orc.dense_forward(q[0], k[0], v[0])
    assert relfro(got[0].float().cpu().numpy(), ref) <= BF16_TOL


@pytest.mark.parametrize("U,nq,nk", [(2, 300, 1000), (1, 100, 20000), (3, 257, 4100)])
def test_flash_entropy_bf16_tcgen05(vm, orc, cuda, U, nq, nk):
    """bf16 / d = 128 flash_entropy_fwd with entropy on the tcgen05 kernel (fa3): the row
    entropy accumulates sum p x' beside the row sum; split-KV partial entropies combine as
    H = sum_s w_s (H_s - ln w_s).  (1, 100, 20000) takes the split path."""
    d = 128
    q = bf16_round(randn((U, nq, d), 41, dtype=np.float32) / np.sqrt(d))
    k = bf16_round(randn((U, nk, d), 42, dtype=np.float32))
    v = bf16_round(randn((U, nk, d), 43, dtype=np.float32))
    launches = vm.kernel_launch_count()
    o, lse, ent = vm.flash_entropy_fwd(*(torch.from_numpy(x).to(cuda, torch.bfloat16) for x in (q, k, v)))
    torch.cuda.synchronize()
    assert vm.kernel_launch_count() > launches
    for u in range(U):
        ro, rl, re = orc.flash_entropy_fwd(q[u], k[u], v[u])
        assert relfro(o[u].float().cpu().numpy(), ro) <= BF16_TOL
        assert np.abs(lse[u].cpu().numpy() - rl).max() <= 1e-3
        assert np.abs(ent[u].cpu().numpy() - re).max() <= 1e-3
