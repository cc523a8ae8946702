"""GPU: head dims below 128 in bf16 (the reference default is d = 64, video.hpp:20) run on
the tcgen05 kernels with Q/K/V zero-padded to 128 columns in the workspace; the softmax scale
stays 1/sqrt(d).  Checked against the CPU oracle, for strided views, factor export and the
element-wise padding fallback (d not a multiple of 8)."""
import numpy as np
import pytest
import torch

from oracle.oracle import bf16_round, workload
from test_gpu_parity import oracle_fwd, run_gpu
from vmb_testutil import relfro

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gridt,d,heads,batch,kw", [
    ((4, 8, 16), 64, 2, 1, dict()),
    ((5, 12, 13), 64, 1, 2, dict(iters=3)),
    ((3, 10, 20), 32, 2, 1, dict()),
    ((4, 8, 16), 96, 1, 1, dict(clamp_min=0.9)),
    ((6, 7, 9), 16, 3, 1, dict(recompute_first_frame=False)),
    ((4, 8, 8), 40, 1, 1, dict()),                    # d % 8 != 0: element-wise padding
    ((8, 16, 16), 64, 1, 1, dict(override_m_b=(256, 8))),
])
def test_bf16_small_head_dim_parity(vm, orc, cuda, gridt, d, heads, batch, kw):
    grid = vm.TokenGrid(*gridt, head_dim=d, heads=heads, batch=batch)
    cfg = vm.VMonarchConfig(**kw)
    q, k, v = workload(grid.units(), grid.tokens(), d, seed=23, sigma=1.5)
    q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    ref = oracle_fwd(orc, q, k, v, grid, cfg)
    got = run_gpu(vm, q, k, v, grid, cfg, torch.bfloat16, cuda)
    assert relfro(got, ref) <= 2e-2


def test_bf16_d64_bshd_views_and_factors(vm, orc, cuda):
    grid = vm.TokenGrid(4, 8, 8, 64, 2, 1)
    q, k, v = workload(2, grid.tokens(), 64, seed=29)
    q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    # BSHD activations as (B, H, N, d) views
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x.transpose(1, 0, 2)[None])).to(cuda, torch.bfloat16)  # noqa: E731
    bq, bk, bv = (t(x).transpose(1, 2) for x in (q, k, v))
    factors = []
    out = vm.vmonarch_attention(bq, bk, bv, grid, vm.VMonarchConfig(), factors_out=factors)
    ref = oracle_fwd(orc, q, k, v, grid, vm.VMonarchConfig())
    assert relfro(out[0].float().cpu().numpy(), ref) <= 2e-2
    for L, R in factors:  # MonarchFactors rows are stochastic (test_video.cpp:218-236)
        assert torch.allclose(L.sum(-1), torch.ones_like(L.sum(-1)), atol=1e-4)
        assert torch.allclose(R.sum(-1), torch.ones_like(R.sum(-1)), atol=1e-4)
