"""tcgen05 / TMA building blocks (descriptor encodings, SW128 swizzle, TMEM A operand)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_umma_selftest(vm, cuda, mode):
    torch.manual_seed(mode)
    A = torch.randn(128, 128, device=cuda).bfloat16()
    B = torch.randn(128, 128, device=cuda).bfloat16()
    Af, Bf = A.float(), B.float()
    ref = {0: Af @ Bf.T, 1: Af @ Bf, 2: Af @ Bf, 3: Af.T @ Bf}[mode]
    C = vm.selftest_umma(mode, A, B)
    assert (C - ref).abs().max().item() < 1e-2


def test_smoke_entry(cuda):
    import __graft_entry__
    __graft_entry__.smoke()
