"""GPU: factorizations with more than 128 row blocks on the tcgen05 path:
the multi-pass L-step (kernels/lstep_big.cu: row statistics, then the ITER or FINAL pass)
against the CPU oracle, and the degenerate b = 1 factorization against dense attention
(test_monarch_core.cpp:285-309: b = 1 reduces VMonarch to dense softmax attention)."""
import numpy as np
import pytest
import torch

from oracle.oracle import bf16_round, workload
from test_gpu_parity import oracle_fwd, run_gpu
from vmb_testutil import relfro

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gridt,mb,heads,kw", [
    ((8, 16, 16), (256, 8), 2, dict()),
    ((8, 16, 16), (512, 4), 1, dict(iters=3)),
    ((10, 13, 12), (195, 8), 2, dict()),                       # m not a multiple of 64
    ((10, 13, 12), (130, 12), 1, dict(iters=1)),
    ((4, 8, 16), (512, 1), 1, dict()),                         # b = 1: dense attention
    ((6, 10, 26), (260, 6), 1, dict(clamp_min=0.9)),
    ((8, 16, 16), (256, 8), 1, dict(recompute_first_frame=False)),
])
def test_large_m_bf16_parity(vm, orc, cuda, gridt, mb, heads, kw):
    grid = vm.TokenGrid(*gridt, head_dim=128, heads=heads, batch=1)
    cfg = vm.VMonarchConfig(override_m_b=mb, **kw)
    q, k, v = workload(heads, grid.tokens(), 128, seed=17, sigma=1.5)
    q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    ref = oracle_fwd(orc, q, k, v, grid, cfg)
    launches = vm.kernel_launch_count()
    got = run_gpu(vm, q, k, v, grid, cfg, torch.bfloat16, cuda)
    assert vm.kernel_launch_count() > launches
    assert relfro(got, ref) <= 2e-2


def test_b1_factorization_equals_dense_at_8k(vm, cuda):
    # N = 8192, (m, b) = (N, 1): every half-step is dense attention over all tokens
    grid = vm.TokenGrid(8, 32, 32, 128, 2, 1)
    g = torch.Generator(device=cuda).manual_seed(4)
    q, k, v = (torch.randn((2, grid.tokens(), 128), generator=g, device=cuda).to(torch.bfloat16) for _ in range(3))
    out = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig(override_m_b=(grid.tokens(), 1)))
    dense = vm.dense_forward(q, k, v)
    torch.cuda.synchronize()
    assert relfro(out.float().cpu().numpy(), dense.float().cpu().numpy()) <= 2e-2


@pytest.mark.parametrize("m,b", [(200, 3), (256, 2)])
def test_large_m_lstep_half_step_parity(vm, orc, cuda, m, b):
    # vmb_lstep with m > 128 (bf16, d = 128) runs the multi-pass L-step; the oracle l_update
    rng = np.random.default_rng(3)
    Qb = bf16_round(rng.standard_normal((2, b, m, 128)).astype(np.float32) / np.sqrt(128))
    aL = bf16_round(rng.standard_normal((2, b, m, 128)).astype(np.float32))
    cL = (-np.log(m) + 0.3 * rng.standard_normal((2, b, m))).astype(np.float32)
    aR, cR, _ = vm.l_update(torch.from_numpy(Qb).to(cuda, torch.bfloat16), torch.from_numpy(aL).to(cuda, torch.bfloat16),
                            torch.from_numpy(cL).to(cuda))
    torch.cuda.synchronize()
    for u in range(2):
        raR, rcR, _ = orc.lstep(Qb[u], aL[u], cL[u], want_L=False)
        assert relfro(aR[u].float().cpu().numpy(), raR) <= 2e-2
        assert relfro(cR[u].cpu().numpy(), rcR) <= 2e-2


def test_b1_factorization_many_row_blocks_on_tensor_cores(vm, cuda):
    # (m, b) = (N, 1) with units x m > 65535: the 1-D R-step grid and the multi-pass L-step;
    # b = 1 reduces VMonarch to dense attention (test_monarch_core.cpp:285-309)
    grid = vm.TokenGrid(8, 32, 64, 128, 5, 1)  # N = 16384, 5 units -> 81920 (unit, row block) pairs
    g = torch.Generator(device=cuda).manual_seed(8)
    q, k, v = (torch.randn((5, grid.tokens(), 128), generator=g, device=cuda).to(torch.bfloat16) for _ in range(3))
    out = vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig(override_m_b=(grid.tokens(), 1)))
    dense = vm.dense_forward(q, k, v)
    torch.cuda.synchronize()
    assert relfro(out.float().cpu().numpy(), dense.float().cpu().numpy()) <= 2e-2
