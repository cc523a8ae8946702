"""GPU: seeded random sweep of forward configurations against the CPU oracle.

Draws grids (T, h, w), heads, batch, head dim, iterations, clamp, recompute, override
factorizations and input scale at random (fixed seed, so the cases are reproducible and the
ids name them), and checks the device forward against the oracle with the north-star
tolerances: fp32 <= 1e-4, bf16 <= 2e-2 (rel-Fro).  bf16 cases use d = 128 (tcgen05 path),
fp32 cases any d (CUDA-core parity mode)."""
import random

import pytest
import torch

from oracle.oracle import bf16_round, workload
from test_gpu_parity import oracle_fwd, run_gpu
from vmb_testutil import relfro

pytestmark = pytest.mark.gpu


def _divisors(n):
    return [x for x in range(1, n + 1) if n % x == 0]


def _cases(count=40, seed=2601):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        bf16 = rng.random() < 0.5
        T, h, w = rng.randint(1, 9), rng.randint(1, 12), rng.randint(1, 24)
        n = T * h * w
        if n < 2 or n > 2000:
            continue
        d = 128 if bf16 else rng.choice([4, 16, 32, 64, 128])
        kw = dict(iters=rng.randint(1, 3), clamp_enabled=rng.random() < 0.85,
                  recompute_first_frame=rng.random() < 0.8)
        if kw["clamp_enabled"]:
            kw["clamp_min"] = rng.choice([0.1, 0.1, 0.5, 0.9])
        if rng.random() < 0.2:
            m = rng.choice(_divisors(n))
            if m <= 128 or not bf16:
                kw["override_m_b"] = (m, n // m)
        sigma = rng.choice([0.5, 1.0, 1.0, 2.0, 3.0]) if kw["clamp_enabled"] else 1.0
        out.append(((T, h, w), d, rng.randint(1, 3), rng.randint(1, 2), bf16, sigma, kw))
    return out


CASES = _cases()


@pytest.mark.parametrize("gridt,d,heads,batch,bf16,sigma,kw", CASES,
                         ids=[f"{'bf16' if c[4] else 'f32'}-{c[0][0]}x{c[0][1]}x{c[0][2]}-d{c[1]}-h{c[2]}b{c[3]}"
                              f"-s{c[5]}-{'-'.join(f'{k}{v}' for k, v in sorted(c[6].items()))}" for c in CASES])
def test_random_forward_parity(vm, orc, cuda, gridt, d, heads, batch, bf16, sigma, kw):
    grid = vm.TokenGrid(*gridt, head_dim=d, heads=heads, batch=batch)
    cfg = vm.VMonarchConfig(**kw)
    q, k, v = workload(grid.units(), grid.tokens(), d, seed=hash((gridt, d, heads)) % 1000, sigma=sigma)
    if bf16:
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    ref = oracle_fwd(orc, q, k, v, grid, cfg)
    got = run_gpu(vm, q, k, v, grid, cfg, torch.bfloat16 if bf16 else torch.float32, cuda)
    assert relfro(got, ref) <= (2e-2 if bf16 else 1e-4)
