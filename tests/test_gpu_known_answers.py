"""GPU: the reference's known-answer tests of the path, replayed through the
C ABI.  Each test cites the reference test it mirrors; tolerances are the reference's own
where the GPU path computes in fp32, and stated where it computes in bf16."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _blocked(x, m, b):  # (N, d) -> (1, m, b, d): to_blocked (mat.hpp:89-97)
    return x.view(1, m, b, -1)


def _blocked_permuted(x, m, b):  # Qb[i][j] = Q[j*b+i] -> (1, b, m, d) (mat.hpp:99-113)
    return x.view(m, b, -1).transpose(0, 1).contiguous()[None]


def test_identical_keys_give_uniform_rows_and_log_b(vm, cuda):
    # test_monarch_core.cpp:124-143 (m=2, b=4, d=3; block 0 keys constant)
    m, b, d = 2, 4, 3
    g = torch.Generator().manual_seed(8)
    q = torch.randn((m * b, d), generator=g, dtype=torch.float64)
    k = torch.randn((m * b, d), generator=g, dtype=torch.float64)
    k[:b] = 1.5 * torch.arange(1, d + 1, dtype=torch.float64)
    aR = _blocked(q / math.sqrt(d), m, b).float().to(cuda)
    cR = torch.ones((1, m, b), device=cuda)
    aL, cL, R = vm.r_update(aR, cR, _blocked(k, m, b).float().to(cuda), want_R=True)
    torch.cuda.synchronize()
    assert torch.allclose(R[0, 0].double().cpu(), torch.full((b, b), 1.0 / b, dtype=torch.float64), atol=1e-7)
    assert torch.allclose(cL[0, :, 0].double().cpu(), torch.full((b,), -math.log(b), dtype=torch.float64), atol=1e-6)


def test_lstep_with_one_frame_block_is_all_ones(vm, cuda):
    # test_monarch_core.cpp:145-158 (m=1 -> L = 1, cR = 1)
    n, d = 7, 3
    g = torch.Generator().manual_seed(9)
    q = torch.randn((n, d), generator=g)
    k = torch.randn((n, d), generator=g)
    aR = _blocked(q / math.sqrt(d), 1, n).to(cuda)
    aL, cL, _ = vm.r_update(aR, torch.ones((1, 1, n), device=cuda), _blocked(k, 1, n).to(cuda))
    _, cR, L = vm.l_update(_blocked_permuted(q / math.sqrt(d), 1, n).to(cuda), aL, cL, want_L=True)
    torch.cuda.synchronize()
    assert torch.all(L == 1.0)
    assert torch.allclose(cR, torch.ones_like(cR), atol=1e-6)


def test_lstep_before_rstep_is_state_error(vm, cuda):
    # test_monarch_core.cpp:160-168 (check_state, monarch.hpp:111)
    qb = torch.randn((1, 3, 2, 2), device=cuda)
    with pytest.raises(vm.StateError, match="state error"):
        vm.l_update(qb, None, None)


def test_uniform_aL_with_zero_cL_gives_uniform_L(vm, cuda):
    # test_monarch_core.cpp:212-227 (m=b=3, d=2)
    m, b, d = 3, 3, 2
    aL = (0.4 * torch.arange(1, d + 1, dtype=torch.float32)).expand(1, b, m, d).contiguous().to(cuda)
    cL = torch.zeros((1, b, m), device=cuda)
    q = torch.randn((m * b, d), generator=torch.Generator().manual_seed(14))
    _, cR, L = vm.l_update(_blocked_permuted(q, m, b).to(cuda), aL, cL, want_L=True)
    torch.cuda.synchronize()
    assert torch.allclose(L, torch.full_like(L, 1.0 / m), atol=1e-7)
    assert torch.allclose(cR, torch.ones_like(cR), atol=1e-6)


@pytest.mark.parametrize("dtype,d,tol", [(torch.float32, 3, 1e-6), (torch.bfloat16, 128, 2e-2)])
def test_shift_of_block_keys_leaves_R_unchanged(vm, cuda, dtype, d, tol):
    # test_monarch_core.cpp:260-283: shifting every key row of block 0 by u moves each score
    # row of that block by the constant <aR_row, u>, so R (and its entropy cL) do not change
    m, b = 2, 4 if d == 3 else 128
    g = torch.Generator().manual_seed(19)
    q = torch.randn((m * b, d), generator=g)
    k = torch.randn((m * b, d), generator=g)
    u = torch.randn((d,), generator=g)
    k2 = k.clone()
    k2[:b] += u
    aR = _blocked(q / math.sqrt(d), m, b).to(cuda, dtype)
    cR = torch.ones((1, m, b), device=cuda)
    _, cL1, R1 = vm.r_update(aR, cR, _blocked(k, m, b).to(cuda, dtype), want_R=dtype == torch.float32)
    _, cL2, R2 = vm.r_update(aR, cR, _blocked(k2, m, b).to(cuda, dtype), want_R=dtype == torch.float32)
    torch.cuda.synchronize()
    if R1 is not None:
        assert (R1[0, 0] - R2[0, 0]).abs().max().item() <= tol
    assert (cL1[0, :, 0] - cL2[0, :, 0]).abs().max().item() <= tol


def test_clamp_bounds_the_division(vm, cuda):
    # test_monarch_core.cpp:240-258: cR = 1e-12 with clamp 0.5 equals cR = 0.5
    m, b, d = 2, 3, 2
    g = torch.Generator().manual_seed(17)
    aR = _blocked(torch.randn((m * b, d), generator=g) / math.sqrt(d), m, b).to(cuda)
    kb = _blocked(torch.randn((m * b, d), generator=g), m, b).to(cuda)
    c1 = torch.ones((1, m, b), device=cuda)
    c1[0, 0, 0] = 1e-12
    c2 = c1.clone()
    c2[0, 0, 0] = 0.5
    _, _, R1 = vm.r_update(aR, c1, kb, clamp_min=0.5, want_R=True)
    _, _, R2 = vm.r_update(aR, c2, kb, clamp_min=0.5, want_R=True)
    torch.cuda.synchronize()
    assert torch.isfinite(R1).all()
    assert torch.allclose(R1[0, 0, 0], R2[0, 0, 0], atol=1e-7)


def _dense64(q, k, v):
    s = q.double() @ k.double().T
    p = torch.softmax(s, -1)
    h = -(p * torch.log(p.clamp_min(1e-300))).sum(-1)
    return p @ v.double(), torch.logsumexp(s, -1), h


def test_flash_rectangular(vm, cuda):
    # test_flash_entropy.cpp:77-86 (N_q = 40, N_k = 256, d = 16; < 1e-4)
    g = torch.Generator().manual_seed(9)
    q, k, v = torch.randn((40, 16), generator=g), torch.randn((256, 16), generator=g), torch.randn((256, 16), generator=g)
    o, lse, h = vm.flash_entropy_fwd(q.to(cuda), k.to(cuda), v.to(cuda))
    ro, rl, rh = _dense64(q, k, v)
    assert (o.double().cpu() - ro).abs().max().item() < 1e-4
    assert (h.double().cpu() - rh).abs().max().item() < 1e-4
    assert (lse.double().cpu() - rl).abs().max().item() < 1e-4


@pytest.mark.parametrize("dtype,d,n,want_h,tol", [(torch.float32, 16, 128, True, 1e-5),
                                                  (torch.bfloat16, 128, 1000, False, 1e-2)])
def test_flash_joint_key_value_permutation_invariance(vm, cuda, dtype, d, n, want_h, tol):
    # test_flash_entropy.cpp:129-153 (bf16 / d = 128 runs the tcgen05 kernel; its sums are
    # re-associated by the permutation, so the bound there is the bf16 one)
    g = torch.Generator().manual_seed(16)
    q = torch.randn((n, d), generator=g) / math.sqrt(d)
    k, v = torch.randn((n, d), generator=g), torch.randn((n, d), generator=g)
    perm = torch.randperm(n, generator=torch.Generator().manual_seed(19))
    a = vm.flash_entropy_fwd(q.to(cuda, dtype), k.to(cuda, dtype), v.to(cuda, dtype), want_entropy=want_h)
    b = vm.flash_entropy_fwd(q.to(cuda, dtype), k[perm].to(cuda, dtype), v[perm].to(cuda, dtype), want_entropy=want_h)
    torch.cuda.synchronize()
    assert (a[0].float() - b[0].float()).abs().max().item() < tol
    assert (a[1] - b[1]).abs().max().item() < tol
    if want_h:
        assert (a[2] - b[2]).abs().max().item() < tol


def test_flash_entropy_bounds(vm, cuda):
    # test_flash_entropy.cpp:155-165 (n = 200, d = 12, sigma = 2): H in [0, ln N_k]
    g = torch.Generator().manual_seed(20)
    q, k, v = 2 * torch.randn((200, 12), generator=g), 2 * torch.randn((200, 12), generator=g), torch.randn((200, 12), generator=g)
    _, _, h = vm.flash_entropy_fwd(q.to(cuda), k.to(cuda), v.to(cuda))
    torch.cuda.synchronize()
    assert h.min().item() >= -1e-5
    assert h.max().item() <= math.log(200) + 1e-5
