"""GPU: the C5 long-video stress shape (81x112x104 latent, N = 943 488, d = 128, bf16) on one
B200, one head (VERDICT r1 "what's missing" #4).

The reference cannot run C5 end to end (it materialises R: 44 GB per unit),
so correctness is pinned two ways:
* the first-frame rows are exact streaming attention over all N keys (video.hpp:117-126):
  64 of them are checked against the UNMODIFIED reference flash_entropy_fwd
  (flash_entropy.hpp:85-139, oracle/_ref), which streams and needs no N x N memory;
* size-independent properties of the whole output: constant V gives a constant output (every
  row of M(F) is stochastic) and the forward is linear in V."""
import numpy as np
import pytest
import torch

from vmb_testutil import relfro

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

T, H, W, D = 81, 112, 104, 128


def _c5_inputs(vm, cuda, seed=7):
    grid = vm.TokenGrid(T, H, W, D, 1, 1)
    g = torch.Generator(device=cuda).manual_seed(seed)
    q, k, v = (torch.randn((1, grid.tokens(), D), device=cuda, generator=g).bfloat16() for _ in range(3))
    return grid, q, k, v


def test_c5_first_frame_rows_match_reference_flash(vm, ref, cuda):
    grid, q, k, v = _c5_inputs(vm, cuda)
    out = vm.vmonarch_attention(q, k, v, grid)
    torch.cuda.synchronize()
    hw = H * W
    rows = torch.linspace(0, hw - 1, 64).round().long().to(cuda)  # spread over the first frame
    q0 = (q[0, rows].float() * (1.0 / np.sqrt(D))).cpu().numpy()
    kk, vv = k[0].float().cpu().numpy(), v[0].float().cpu().numpy()
    ro, _, _ = ref.flash_entropy_fwd(q0, kk, vv)
    got = out[0, rows].float().cpu().numpy()
    err = relfro(got, ro)
    print(f"C5 first-frame rows vs reference flash_entropy_fwd: rel-Fro {err:.3e}")
    assert err <= 2e-2


def test_c5_constant_values_and_linearity(vm, cuda):
    grid, q, k, v = _c5_inputs(vm, cuda, seed=8)
    c = torch.linspace(-1, 1, D, device=cuda).bfloat16()
    vc = c.expand(1, grid.tokens(), D).contiguous()
    out = vm.vmonarch_attention(q, k, vc, grid)
    assert (out.float() - c.float()).abs().max().item() <= 2e-2
    o1 = vm.vmonarch_attention(q, k, v, grid).float()
    o2 = vm.vmonarch_attention(q, k, (2 * v.float()).bfloat16(), grid).float()
    assert relfro(o2.cpu().numpy(), (2 * o1).cpu().numpy()) <= 1e-2
