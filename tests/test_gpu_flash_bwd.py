"""GPU: backward of the online-entropy attention (flash_entropy.hpp:146-221, Alg. 2 of the
paper) against the CPU oracle (pinned bit-exact to the reference's flash_entropy_bwd in
tests/test_oracle_pin.py) and against torch autograd of <dO, O> + <dH, H> in fp64.
Mirrors tests/test_flash_bwd.cpp of the reference."""
import numpy as np
import pytest
import torch

from oracle.oracle import bf16_round, randn
from vmb_testutil import relfro

pytestmark = pytest.mark.gpu


def _fwd_inputs(nq, nk, d, seed, sigma=1.0):
    q = randn((nq, d), seed, sigma) / np.sqrt(d)  # pre-scaled, as the reference's callers do
    k = randn((nk, d), seed + 1, sigma)
    v = randn((nk, d), seed + 2, sigma)
    g = randn((nq, d), seed + 3)
    dh = randn((nq,), seed + 4)
    return q.astype(np.float32), k, v, g, dh


@pytest.mark.parametrize("nq,nk,d,eg", [(24, 24, 6, False), (64, 64, 8, False), (32, 32, 5, True), (40, 130, 64, True),
                                        (128, 300, 128, True), (7, 1, 16, True)])
def test_bwd_matches_oracle_fp32(vm, orc, cuda, nq, nk, d, eg):
    q, k, v, g, dh = _fwd_inputs(nq, nk, d, 11)
    o, lse, ent = orc.flash_entropy_fwd(q, k, v, br=16, bc=16)
    ref = orc.flash_entropy_bwd(q, k, v, o, g, lse, ent, dh, eg, br=16, bc=16)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(cuda)  # noqa: E731
    got = vm.flash_entropy_bwd(t(q), t(k), t(v), t(o), t(g), t(lse), t(ent), t(dh), entropy_grad=eg)
    torch.cuda.synchronize()
    for name, a, b in zip(("dq", "dk", "dv"), got, ref):
        a = a.cpu().numpy()
        # rel-Fro, or absolute for gradients that vanish analytically (nk = 1: dS = P (dP - D) = 0
        # up to rounding, both sides are pure rounding noise)
        assert relfro(a, b) <= 1e-4 or np.abs(a - b).max() <= 1e-5, name
        assert np.abs(a - b).max() <= 1e-4 * max(1.0, np.abs(b).max()), name


def test_bwd_bf16_storage(vm, orc, cuda):
    q, k, v, g, dh = _fwd_inputs(100, 256, 128, 21)
    q, k, v, g = bf16_round(q), bf16_round(k), bf16_round(v), bf16_round(g)
    o, lse, ent = orc.flash_entropy_fwd(q, k, v)
    o = bf16_round(o)
    ref = orc.flash_entropy_bwd(q, k, v, o, g, lse, ent, dh, True)
    tb = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(cuda, torch.bfloat16)  # noqa: E731
    tf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(cuda)  # noqa: E731
    got = vm.flash_entropy_bwd(tb(q), tb(k), tb(v), tb(o), tb(g), tf(lse), tf(ent), tf(dh), entropy_grad=True)
    for a, b in zip(got, ref):
        assert relfro(a.float().cpu().numpy(), b) <= 2e-2


def test_zero_upstream_gradients_give_exactly_zero(vm, orc, cuda):
    q, k, v, _, _ = _fwd_inputs(24, 24, 6, 1)
    o, lse, ent = orc.flash_entropy_fwd(q, k, v, br=8, bc=8)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(cuda)  # noqa: E731
    z = torch.zeros((24, 6), device=cuda)
    dq, dk, dv = vm.flash_entropy_bwd(t(q), t(k), t(v), t(o), z, t(lse), t(ent), torch.zeros(24, device=cuda),
                                      entropy_grad=True)
    assert not dq.any() and not dk.any() and not dv.any()


def test_bwd_matches_torch_autograd_with_entropy_term(vm, cuda):
    """<dO, O> + <dH, H> with H = -sum_l P ln P = lse - sum_l P S (flash_entropy.hpp:137)."""
    torch.manual_seed(0)
    U, nq, nk, d = 3, 50, 70, 32
    q = (torch.randn(U, nq, d, dtype=torch.float64, device=cuda) / d ** 0.5).requires_grad_()
    k = torch.randn(U, nk, d, dtype=torch.float64, device=cuda).requires_grad_()
    v = torch.randn(U, nk, d, dtype=torch.float64, device=cuda).requires_grad_()
    s = q @ k.transpose(1, 2)
    lse = torch.logsumexp(s, -1)
    p = torch.exp(s - lse[..., None])
    o = p @ v
    h = lse - (p * s).sum(-1)
    g = torch.randn_like(o)
    dh = torch.randn_like(h)
    ((o * g).sum() + (h * dh).sum()).backward()
    f = lambda x: x.detach().float()  # noqa: E731
    dq, dk, dv = vm.flash_entropy_bwd(f(q), f(k), f(v), f(o), f(g), f(lse), f(h), f(dh), entropy_grad=True)
    for a, b in ((dq, q.grad), (dk, k.grad), (dv, v.grad)):
        assert float((a.double() - b).norm() / b.norm()) <= 1e-4


def test_bwd_rejects_bad_statistics(vm, cuda):
    x = torch.zeros((8, 4), device=cuda)
    l8 = torch.zeros(8, device=cuda)
    with pytest.raises(vm.DimensionError):
        vm.flash_entropy_bwd(x, x, x, x, x, torch.zeros(7, device=cuda))
    with pytest.raises(vm.DimensionError):
        vm.flash_entropy_bwd(x, x, x, x, x, l8, entropy_grad=True)
    with pytest.raises(vm.DomainError):
        vm.flash_entropy_bwd(x, x[:0], x[:0], x, x, l8)


def _torch_ref(U, nq, nk, d, cuda, seed, sigma=1.0):
    """bf16-rounded inputs, fp64 autograd of <dO, O> + <dH, H> (the entropy-gradient loss)."""
    g = torch.Generator(device=cuda).manual_seed(seed)
    mk = lambda *s: torch.randn(*s, generator=g, device=cuda).to(torch.bfloat16).double()  # noqa: E731
    q = (sigma * mk(U, nq, d) / d ** 0.5).to(torch.bfloat16).double().requires_grad_()
    k = (sigma * mk(U, nk, d)).to(torch.bfloat16).double().requires_grad_()
    v = mk(U, nk, d).requires_grad_()
    s = q @ k.transpose(1, 2)
    lse = torch.logsumexp(s, -1)
    p = torch.exp(s - lse[..., None])
    o = p @ v
    h = lse - (p * s).sum(-1)
    gr = mk(U, nq, d)
    dh = torch.randn(U, nq, generator=g, device=cuda, dtype=torch.float64)
    return q, k, v, o, h, lse, gr, dh


@pytest.mark.parametrize("U,nq,nk,eg", [(1, 128, 128, True), (3, 300, 1000, True), (2, 1000, 300, False),
                                        (2, 4096, 4096, True), (1, 65, 1, True), (1, 1, 200, True)])
def test_tcgen05_bwd_bf16_matches_fp64_autograd(vm, cuda, U, nq, nk, eg):
    """bf16 / d = 128 runs the tcgen05 kernels (flash_bwd_tc.cu): ragged tiles on both axes,
    several units, with and without the entropy-gradient term; bf16 tolerance (north star)."""
    d = 128
    q, k, v, o, h, lse, gr, dh = _torch_ref(U, nq, nk, d, cuda, 7 + nq + nk)
    loss = (o * gr).sum() + ((h * dh).sum() if eg else 0.0)
    loss.backward()
    b = lambda x: x.detach().to(torch.bfloat16)  # noqa: E731
    f = lambda x: x.detach().float()  # noqa: E731
    launches = vm.kernel_launch_count()
    dq, dk, dv = vm.flash_entropy_bwd(b(q), b(k), b(v), b(o), b(gr), f(lse), f(h), f(dh), entropy_grad=eg)
    torch.cuda.synchronize()
    assert vm.kernel_launch_count() - launches == 3  # rowstat + dQ + dK/dV: the tcgen05 path ran
    for name, a, ref in (("dq", dq, q.grad), ("dk", dk, k.grad), ("dv", dv, v.grad)):
        err = float((a.double() - ref).norm() / ref.norm().clamp_min(1e-30))
        # nk = 1: dS = P (dP - D) - dH P (S - lse + H) = 0 analytically, dQ and dK are rounding noise
        assert err <= 2e-2 or float((a.double() - ref).abs().max()) <= 2e-3, (name, err)


def test_tcgen05_bwd_is_deterministic(vm, cuda):
    q, k, v, o, h, lse, gr, dh = _torch_ref(2, 700, 900, 128, cuda, 3)
    b = lambda x: x.detach().to(torch.bfloat16)  # noqa: E731
    f = lambda x: x.detach().float()  # noqa: E731
    args = (b(q), b(k), b(v), b(o), b(gr), f(lse), f(h), f(dh))
    r1 = vm.flash_entropy_bwd(*args, entropy_grad=True)
    r2 = vm.flash_entropy_bwd(*args, entropy_grad=True)
    torch.cuda.synchronize()
    for a, c in zip(r1, r2):
        assert torch.equal(a, c)
