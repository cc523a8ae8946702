"""GPU: the f64 mode (VMB_F64) -- the reference operator is a template over T
(video.hpp:84) and its own tests run in double.  The forward runs the CUDA-core kernels in
double (exp / log / fma in f64, row sums and entropy in double as monarch.hpp:87-98) and must
agree with the reference CPU path in double to round-off, not to a bf16/fp32 tolerance.

Checked against the UNMODIFIED reference (oracle/_ref, vmonarch_attention<double>) when it is
built, else the C restatement (pinned to it by tests/test_oracle_pin.py)."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

from oracle.oracle import REF_SO, Oracle
from test_gpu_parity import oracle_fwd
from vmb_testutil import relfro

pytestmark = pytest.mark.gpu
F64_TOL = 1e-11


@pytest.fixture(scope="module")
def checker():
    return Oracle("reference") if os.path.exists(REF_SO) else Oracle("port")


def _inputs(units, n, d, seed, sigma=1.0):
    rng = np.random.default_rng(seed)
    return [sigma * rng.standard_normal((units, n, d)) for _ in range(3)]


CASES = [
    ((4, 8, 8), 64, 2, 1, dict(iters=3)),                      # C1 shape
    ((3, 4, 5), 16, 2, 1, dict()),
    ((5, 6, 6), 128, 1, 1, dict(iters=3, clamp_enabled=False)),
    ((4, 8, 8), 32, 1, 2, dict(override_m_b=(16, 16))),
    ((2, 3, 7), 12, 3, 1, dict(iters=1, recompute_first_frame=False)),
    ((6, 10, 10), 96, 1, 1, dict(clamp_min=0.5)),
]


@pytest.mark.parametrize("gridt,d,heads,batch,kw", CASES)
def test_f64_forward_matches_reference_double(vm, checker, cuda, gridt, d, heads, batch, kw):
    grid = vm.TokenGrid(*gridt, head_dim=d, heads=heads, batch=batch)
    cfg = vm.VMonarchConfig(**kw)
    q, k, v = _inputs(grid.units(), grid.tokens(), d, seed=sum(gridt) + d)
    ref = oracle_fwd(checker, q, k, v, grid, cfg)
    out = vm.vmonarch_attention(*(torch.from_numpy(x).to(cuda) for x in (q, k, v)), grid, cfg)
    assert out.dtype == torch.float64
    got = out.cpu().numpy()
    assert relfro(got, ref) <= F64_TOL
    assert np.abs(got - ref).max() <= 1e-10


def test_f64_sharp_inputs(vm, checker, cuda):
    # sigma = 3: peaky rows, the regime where bf16 state is most exposed
    grid = vm.TokenGrid(4, 7, 7, 128, 2, 1)
    cfg = vm.VMonarchConfig(iters=3, recompute_first_frame=False, override_m_b=(49, 4))
    q, k, v = _inputs(2, grid.tokens(), 128, seed=638, sigma=3.0)
    ref = oracle_fwd(checker, q, k, v, grid, cfg)
    got = vm.vmonarch_attention(*(torch.from_numpy(x).to(cuda) for x in (q, k, v)), grid, cfg).cpu().numpy()
    assert relfro(got, ref) <= F64_TOL


def test_f64_single_frame_equals_dense(vm, orc, cuda):
    # test_video.cpp:60-71: one frame -> exact attention; against the oracle's f64 dense map
    grid = vm.TokenGrid(1, 6, 7, 32, 1, 1)
    q, k, v = _inputs(1, grid.tokens(), 32, seed=5)
    got = vm.vmonarch_attention(*(torch.from_numpy(x).to(cuda) for x in (q, k, v)), grid).cpu().numpy()
    dense = orc.dense_attention_f64(q[0], k[0], v[0])
    dense = dense[0] if isinstance(dense, tuple) else dense
    assert np.abs(got[0] - dense).max() <= 1e-12


def test_f64_factor_export_matches_reference(vm, orc, cuda):
    grid = vm.TokenGrid(3, 4, 5, 16, 1, 1)
    cfg = vm.VMonarchConfig(iters=2, recompute_first_frame=False)
    q, k, v = _inputs(1, grid.tokens(), 16, seed=9)
    f = []
    vm.vmonarch_attention(*(torch.from_numpy(x).to(cuda) for x in (q, k, v)), grid, cfg, factors_out=f)
    L, R = (t.cpu().numpy() for t in f[0])
    assert L.dtype == np.float64 and R.dtype == np.float64
    m, b = 3, 20
    rL = np.zeros((b, m, m))
    rR = np.zeros((m, b, b))
    out = np.zeros((grid.tokens(), 16))
    fn = orc.lib.vmo_vmonarch_unit_f64
    fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 5 + [C.c_double, C.c_int, C.c_int] + [C.c_int64] * 4 + \
        [C.c_void_p] * 3
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    assert fn(ptr(q[0]), ptr(k[0]), ptr(v[0]), 3, 4, 5, 16, 2, 0.1, 1, 0, 0, 0, 64, 64, ptr(out), ptr(rL),
              ptr(rR)) == 0
    assert np.abs(L - rL).max() <= 1e-12
    assert np.abs(R - rR).max() <= 1e-12


def test_f64_nonfinite_q_is_domain_error(vm, cuda):
    grid = vm.TokenGrid(2, 4, 4, 16, 1, 1)
    q, k, v = (torch.from_numpy(x).to(cuda) for x in _inputs(1, grid.tokens(), 16, seed=2))
    q[0, 5, 3] = float("nan")
    with pytest.raises(vm.DomainError):
        vm.vmonarch_attention(q, k, v, grid)


def test_f64_half_steps_are_refused(vm, cuda):
    # the f64 mode covers the operator and its factor export; the half-step ABI stays f32/bf16
    aR = torch.zeros((1, 2, 3, 8), dtype=torch.float64, device=cuda)
    with pytest.raises(vm.DimensionError):
        vm.r_update(aR, torch.ones((1, 2, 3), device=cuda), aR)
