"""The CPU restatement (oracle/vmonarch_oracle.c) is pinned two ways:
(1) against the committed fixtures generated from the reference itself (tests/golden/), and
(2) against the reference library compiled from /root/reference (oracle/_ref), when present.
Both comparisons are bit-exact (same operation order, no FMA contraction)."""
import numpy as np
import pytest

from oracle.oracle import bf16_round, randn, workload


def test_golden_c1_forward(orc, golden):
    q, k, v = golden["c1_q"], golden["c1_k"], golden["c1_v"]
    out = orc.vmonarch_attention(q, k, v, (4, 8, 8), iters=3)
    assert np.array_equal(out, golden["c1_out"])
    out2 = orc.vmonarch_attention(q, k, v, (4, 8, 8), iters=3, recompute=False)
    assert np.array_equal(out2, golden["c1_out_norecompute"])


def test_golden_generator(golden):
    # the libstdc++ mt19937_64 + normal_distribution convention of the reference tests
    q, k, v = workload(2, 256, 64, seed=0)
    assert np.array_equal(q, golden["c1_q"]) and np.array_equal(v, golden["c1_v"])


@pytest.mark.parametrize("b,n", [(3, 6), (4, 12), (5, 20), (1, 7), (7, 7), (1456, 5824)])
def test_golden_perm(orc, golden, b, n):
    assert np.array_equal(orc.make_perm(b, n), golden[f"perm_{b}_{n}"])


def test_golden_blocked(orc, golden):
    assert np.array_equal(orc.to_blocked_permuted(golden["blocked_x"], 3, 4), golden["blocked_qb"])


@pytest.mark.parametrize("name,grid,d", [("wan321_d64", (81, 28, 52), 64), ("wan61_d64", (16, 28, 52), 64),
                                         ("c4_d128", (81, 28, 52), 128), ("c2_d128", (21, 30, 52), 128)])
def test_golden_flops(orc, golden, name, grid, d):
    rep = orc.flops_estimate(grid, d)
    assert [rep["monarch_flops"], rep["full_attn_flops"], rep["recompute_flops"]] == \
        golden[f"flops_{name}"].tolist()
    assert rep["reduction_ratio"] == golden[f"ratio_{name}"][0]


def test_golden_half_steps_f64(orc, golden):
    m, b, d = 3, 5, 4
    qs, kk = golden["rs_qs"], golden["rs_k"]
    aL, cL, R = orc.rstep(qs.reshape(m, b, d), np.ones((m, b)), kk.reshape(m, b, d))
    assert np.array_equal(aL, golden["rs_aL"]) and np.array_equal(cL, golden["rs_cL"])
    assert np.array_equal(R, golden["rs_R"])
    aR, cR, L = orc.lstep(golden["ls_qb"], aL, cL)
    assert np.array_equal(aR, golden["ls_aR"]) and np.array_equal(cR, golden["ls_cR"])
    assert np.array_equal(L, golden["ls_L"])


def test_golden_half_steps_f32(orc, golden):
    m, b, d = 3, 150, 128
    qs, k, cR = golden["rs32_qs"], golden["rs32_k"], golden["rs32_cR"]
    aL, cL, _ = orc.rstep(qs.reshape(m, b, d), cR, k.reshape(m, b, d), want_R=False)
    assert np.array_equal(aL, golden["rs32_aL"]) and np.array_equal(cL, golden["rs32_cL"])
    qb = np.ascontiguousarray(qs.reshape(m, b, d).transpose(1, 0, 2))
    aR, cRo, _ = orc.lstep(qb, aL, cL, want_L=False)
    assert np.array_equal(aR, golden["ls32_aR"]) and np.array_equal(cRo, golden["ls32_cR"])


def test_golden_flash(orc, golden):
    o, l, e = orc.flash_entropy_fwd(golden["fl_q"], golden["fl_k"], golden["fl_v"], 32, 48)
    assert np.array_equal(o, golden["fl_out"]) and np.array_equal(l, golden["fl_lse"])
    assert np.array_equal(e, golden["fl_ent"])


def test_golden_monarch_factors(orc, golden):
    o, L, R = orc.monarch_attention(golden["mo_q"], golden["mo_k"], golden["mo_v"], 4, 12, iters=2,
                                    clamp_enabled=False, want_factors=True)
    assert np.array_equal(o, golden["mo_out"])
    assert np.array_equal(L, golden["mo_L"]) and np.array_equal(R, golden["mo_R"])


# ---- live comparison with the compiled reference (skipped when oracle/_ref is absent)
@pytest.mark.parametrize("grid,d,units,iters,sigma,clamp,recompute,override", [
    ((4, 8, 8), 64, 2, 3, 1.0, True, True, (0, 0)),
    ((3, 4, 5), 16, 2, 2, 3.0, True, True, (0, 0)),
    ((4, 4, 4), 8, 1, 2, 1.0, False, False, (0, 0)),
    ((4, 8, 8), 32, 1, 2, 2.0, True, True, (16, 16)),
    ((2, 3, 7), 12, 3, 1, 1.0, True, True, (0, 0)),
    ((5, 6, 6), 128, 1, 2, 1.0, True, True, (0, 0)),
])
def test_port_equals_reference(orc, ref, grid, d, units, iters, sigma, clamp, recompute, override):
    n = grid[0] * grid[1] * grid[2]
    q, k, v = workload(units, n, d, seed=11, sigma=sigma)
    kw = dict(iters=iters, clamp_enabled=clamp, recompute=recompute, override=override)
    a = orc.vmonarch_attention(q, k, v, grid, **kw)
    b = ref.vmonarch_attention(q, k, v, grid, **kw)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("n,m,b", [(48, 48, 1), (48, 1, 48), (256, 256, 1)])
def test_port_equals_reference_degenerate(orc, ref, n, m, b):
    q, k, v = (randn((n, 8), s, dtype=np.float64) for s in (21, 22, 23))
    a = orc.monarch_attention(q, k, v, m, b, iters=3, want_factors=True)
    r = ref.monarch_attention(q, k, v, m, b, iters=3, want_factors=True)
    for x, y in zip(a, r):
        assert np.array_equal(x, y)


def test_port_equals_reference_errors(orc, ref):
    q = randn((6, 2), 2, dtype=np.float64)
    q[3, 1] = np.nan
    from oracle.oracle import OracleError
    for o in (orc, ref):
        with pytest.raises(OracleError) as e:
            o.monarch_attention(q, q, q, 2, 3)
        assert e.value.status == 2  # domain error (monarch.hpp:44)
    aR = randn((2, 3, 2), 15, dtype=np.float64)
    cR = np.ones((2, 3))
    cR[1, 1] = 0.0
    for o in (orc, ref):
        with pytest.raises(OracleError) as e:
            o.rstep(aR, cR, randn((2, 3, 2), 16, dtype=np.float64), clamp_enabled=False)
        assert e.value.status == 2  # monarch.hpp:78


def test_bf16_round_matches_torch():
    import torch
    x = randn((1000,), 5, sigma=3.0, dtype=np.float32)
    assert np.array_equal(bf16_round(x), torch.from_numpy(x).bfloat16().float().numpy())


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("eg", [False, True])
def test_port_flash_bwd_equals_reference(orc, ref, dtype, eg):
    """flash_entropy.hpp:146-221: the C restatement of the backward is bit-exact."""
    q = randn((24, 6), 1, dtype=dtype)
    k = randn((30, 6), 2, dtype=dtype)
    v = randn((30, 6), 3, dtype=dtype)
    g = randn((24, 6), 4, dtype=dtype)
    dh = randn((24,), 5, dtype=dtype)
    o, lse, ent = ref.flash_entropy_fwd(q, k, v, br=8, bc=8)
    a = orc.flash_entropy_bwd(q, k, v, o, g, lse, ent, dh, eg, br=8, bc=8)
    b = ref.flash_entropy_bwd(q, k, v, o, g, lse, ent, dh, eg, br=8, bc=8)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
