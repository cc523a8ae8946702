"""GPU: the DiT-side torch op vmb::vmonarch_attention and VMonarchSelfAttention (SURVEY §8f
row 3).  Strided BSHD views from a fused QKV projection must give exactly the result of the
contiguous unit-major call (the kernels read through vmb_strides; no copies are made)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _unit_major(x):  # (B, S, H, D) -> (B*H, S, D)
    B, S, H, D = x.shape
    return x.permute(0, 2, 1, 3).reshape(B * H, S, D).contiguous()


@pytest.mark.parametrize("gridt,B,H", [((4, 8, 16), 2, 3), ((21, 30, 52), 1, 2)])
def test_op_on_fused_qkv_views_equals_unit_major_call(vm, cuda, gridt, B, H):
    from paper_2601_22275_b200.torch_op import vmonarch_attention_op
    S = gridt[0] * gridt[1] * gridt[2]
    g = torch.Generator(device=cuda).manual_seed(3)
    qkv = torch.randn((B, S, 3, H, 128), device=cuda, generator=g).to(torch.bfloat16)
    q, k, v = qkv.unbind(2)
    launches = vm.kernel_launch_count()
    o = torch.ops.vmb.vmonarch_attention(q, k, v, *gridt)
    assert vm.kernel_launch_count() > launches  # the CUDA path ran
    assert o.shape == (B, S, H, 128) and o.is_contiguous()
    grid = vm.TokenGrid(*gridt, 128, H, B)
    ref = vm.vmonarch_attention(_unit_major(q), _unit_major(k), _unit_major(v), grid)
    torch.cuda.synchronize()
    assert torch.equal(_unit_major(o), ref)
    assert torch.equal(vmonarch_attention_op(q, k, v, *gridt), o)


def test_op_opcheck_schema_and_fake(vm, cuda):
    S = 4 * 8 * 16
    q = torch.randn((1, S, 2, 128), device=cuda).to(torch.bfloat16)
    torch.library.opcheck(torch.ops.vmb.vmonarch_attention.default, (q, q, q, 4, 8, 16),
                          test_utils=("test_schema", "test_faketensor"))


def test_op_check_flag_raises_domain_error(vm, cuda):
    S = 4 * 8 * 16
    q = torch.randn((1, S, 2, 128), device=cuda).to(torch.bfloat16)
    q[0, 5, 1, 7] = float("inf")
    with pytest.raises(vm.DomainError):
        torch.ops.vmb.vmonarch_attention(q, q, q, 4, 8, 16, check=True)


def test_self_attention_module(vm, cuda):
    from paper_2601_22275_b200.torch_op import VMonarchSelfAttention
    torch.manual_seed(0)
    gridt, H, dim = (4, 8, 16), 2, 256
    S = 4 * 8 * 16
    blk = VMonarchSelfAttention(dim, H, gridt, device=cuda, dtype=torch.bfloat16)
    x = torch.randn((2, S, dim), device=cuda, dtype=torch.bfloat16)
    with torch.no_grad():
        y = blk(x)
        qkv = blk.qkv(x).view(2, S, 3, H, 128)
        grid = vm.TokenGrid(*gridt, 128, H, 2)
        o = vm.vmonarch_attention(*(_unit_major(t) for t in qkv.unbind(2)), grid)
        o = o.view(2, H, S, 128).permute(0, 2, 1, 3).reshape(2, S, dim)
        ref = blk.proj(o)
    torch.cuda.synchronize()
    assert y.shape == (2, S, dim)
    assert torch.equal(y, ref)
