"""Staged GPU diagnostics (run one stage per process under `timeout`).

    python scripts/gpu_diag.py <stage>

Stages: selftest, rstep, lstep, flash, fwd_f32, fwd_bf16, fwd_big.  Prints max / rel-Fro errors
against torch or the CPU oracle.  Used while bringing up kernels; the pytest suite holds the
asserted versions.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22275_b200 as vm  # noqa: E402
from oracle.oracle import Oracle, bf16_round, workload  # noqa: E402

dev = "cuda"


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)), float(np.abs(a - b).max())


def stage_selftest():
    torch.manual_seed(0)
    A = torch.randn(128, 128, device=dev).bfloat16()
    B = torch.randn(128, 128, device=dev).bfloat16()
    Af, Bf = A.float(), B.float()
    refs = {0: Af @ Bf.T, 1: Af @ Bf, 2: Af @ Bf, 3: Af.T @ Bf}
    for mode in range(4):
        C = vm.selftest_umma(mode, A, B)
        torch.cuda.synchronize()
        err = (C - refs[mode]).abs().max().item()
        print(f"selftest mode {mode}: max err {err:.3e}  (ref max {refs[mode].abs().max().item():.2f})")
        if err > 1e-2:
            # diagnose: which rows/cols are wrong
            bad = (C - refs[mode]).abs() > 1e-2
            print("   bad rows", bad.any(1).nonzero().flatten()[:16].tolist(), "bad cols",
                  bad.any(0).nonzero().flatten()[:16].tolist())
            print("   C[0,:8]", C[0, :8].tolist())
            print("   R[0,:8]", refs[mode][0, :8].tolist())


def _state(m, b, d, seed, U=1):
    rng = np.random.default_rng(seed)
    aR = bf16_round(rng.standard_normal((U, m, b, d)).astype(np.float32) / np.sqrt(d))
    cR = (0.5 + rng.random((U, m, b))).astype(np.float32)
    Kb = bf16_round(rng.standard_normal((U, m, b, d)).astype(np.float32))
    return aR, cR, Kb


def stage_rstep():
    P = Oracle("port")
    for (m, b, d) in [(2, 128, 128), (3, 200, 128), (2, 64, 64), (3, 37, 16)]:
        aR, cR, Kb = _state(m, b, d, 1, U=2)
        for dtn, dt in [("f32", torch.float32), ("bf16", torch.bfloat16)]:
            ta = torch.from_numpy(aR).to(dev, dt)
            tk = torch.from_numpy(Kb).to(dev, dt)
            tc = torch.from_numpy(cR).to(dev)
            aL, cL, _ = vm.r_update(ta, tc, tk)
            torch.cuda.synchronize()
            for u in range(2):
                raL, rcL, _ = P.rstep(aR[u], cR[u], Kb[u])
                e1 = rel(aL[u].float().cpu().numpy(), raL)
                e2 = rel(cL[u].cpu().numpy(), rcL)
                print(f"rstep m={m} b={b} d={d} {dtn} u={u}: aL relfro {e1[0]:.2e} max {e1[1]:.2e} | "
                      f"cL relfro {e2[0]:.2e} max {e2[1]:.2e}")


def stage_lstep():
    P = Oracle("port")
    for (m, b, d) in [(4, 16, 128), (21, 40, 128), (81, 8, 128), (5, 7, 32)]:
        rng = np.random.default_rng(2)
        U = 2
        Qb = bf16_round(rng.standard_normal((U, b, m, d)).astype(np.float32) / np.sqrt(d))
        aL = bf16_round(rng.standard_normal((U, b, m, d)).astype(np.float32))
        cL = (-np.log(b) + 0.3 * rng.standard_normal((U, b, m))).astype(np.float32)
        for dtn, dt in [("f32", torch.float32), ("bf16", torch.bfloat16)]:
            aR, cR, _ = vm.l_update(torch.from_numpy(Qb).to(dev, dt), torch.from_numpy(aL).to(dev, dt),
                                    torch.from_numpy(cL).to(dev))
            torch.cuda.synchronize()
            for u in range(U):
                raR, rcR, _ = P.lstep(Qb[u], aL[u], cL[u])
                e1 = rel(aR[u].float().cpu().numpy(), raR)
                e2 = rel(cR[u].cpu().numpy(), rcR)
                print(f"lstep m={m} b={b} d={d} {dtn} u={u}: aR relfro {e1[0]:.2e} max {e1[1]:.2e} | "
                      f"cR relfro {e2[0]:.2e} max {e2[1]:.2e}")


def stage_flash():
    P = Oracle("port")
    for (nq, nk, d) in [(128, 128, 128), (100, 300, 128), (300, 1000, 128), (77, 129, 32)]:
        rng = np.random.default_rng(3)
        q = bf16_round(rng.standard_normal((2, nq, d)).astype(np.float32) / np.sqrt(d))
        k = bf16_round(rng.standard_normal((2, nk, d)).astype(np.float32))
        v = bf16_round(rng.standard_normal((2, nk, d)).astype(np.float32))
        for dtn, dt in [("f32", torch.float32), ("bf16", torch.bfloat16)]:
            o, lse, ent = vm.flash_entropy_fwd(*(torch.from_numpy(x).to(dev, dt) for x in (q, k, v)),
                                               want_entropy=(dtn == "f32"))
            torch.cuda.synchronize()
            ro, rl, re = P.flash_entropy_fwd(q[0], k[0], v[0])
            e1 = rel(o[0].float().cpu().numpy(), ro)
            e2 = rel(lse[0].cpu().numpy(), rl)
            print(f"flash nq={nq} nk={nk} d={d} {dtn}: O relfro {e1[0]:.2e} max {e1[1]:.2e} | lse max {e2[1]:.2e}")


def _fwd(grid, cfg, dt, seed=0, sigma=1.0):
    P = Oracle("port")
    q, k, v = workload(grid.units(), grid.tokens(), grid.head_dim, seed=seed, sigma=sigma)
    q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    t0 = time.time()
    ref = P.vmonarch_attention(q, k, v, (grid.t_frames, grid.h, grid.w), iters=cfg.iters,
                               clamp_min=cfg.clamp_min, clamp_enabled=cfg.clamp_enabled,
                               recompute=cfg.recompute_first_frame,
                               override=cfg.override_m_b or (0, 0))
    t_cpu = time.time() - t0
    tq, tk, tv = (torch.from_numpy(x).to(dev, dt) for x in (q, k, v))
    o = vm.vmonarch_attention(tq, tk, tv, grid, cfg)
    torch.cuda.synchronize()
    e = rel(o.float().cpu().numpy(), ref)
    return e, t_cpu


def stage_fwd_f32():
    for grid, cfg in [(vm.TokenGrid(4, 8, 8, 64, 2, 1), vm.VMonarchConfig(iters=3)),
                      (vm.TokenGrid(3, 4, 5, 16, 2, 1), vm.VMonarchConfig()),
                      (vm.TokenGrid(4, 4, 4, 8, 1, 1), vm.VMonarchConfig(recompute_first_frame=False)),
                      (vm.TokenGrid(4, 8, 8, 32, 1, 1), vm.VMonarchConfig(override_m_b=(16, 16)))]:
        e, t = _fwd(grid, cfg, torch.float32)
        print(f"fwd f32 {grid} iters={cfg.iters}: relfro {e[0]:.2e} max {e[1]:.2e} (cpu {t:.2f}s)")


def stage_fwd_bf16():
    for grid, cfg in [(vm.TokenGrid(4, 8, 16, 128, 2, 1), vm.VMonarchConfig()),
                      (vm.TokenGrid(3, 10, 20, 128, 2, 1), vm.VMonarchConfig()),
                      (vm.TokenGrid(5, 12, 13, 128, 1, 2), vm.VMonarchConfig(iters=3)),
                      (vm.TokenGrid(4, 8, 16, 128, 1, 1), vm.VMonarchConfig(recompute_first_frame=False))]:
        e, t = _fwd(grid, cfg, torch.bfloat16)
        print(f"fwd bf16 {grid} iters={cfg.iters}: relfro {e[0]:.2e} max {e[1]:.2e} (cpu {t:.2f}s)")


def stage_fwd_big():
    grid = vm.TokenGrid(21, 30, 52, 128, 12, 1)
    cfg = vm.VMonarchConfig()
    q = torch.randn(grid.units(), grid.tokens(), 128, device=dev, dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    o = vm.vmonarch_attention(q, k, v, grid, cfg)
    torch.cuda.synchronize()
    for _ in range(3):
        vm.vmonarch_attention(q, k, v, grid, cfg, out=o, check=False)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(5):
        vm.vmonarch_attention(q, k, v, grid, cfg, out=o, check=False)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 5
    F = vm.flops_estimate(grid, cfg, 128)
    tot = (F.monarch_flops + F.recompute_flops) * grid.units()
    print(f"C2 bf16: {ms:.3f} ms/call, {tot / ms / 1e9:.1f} TFLOP/s, finite={bool(torch.isfinite(o).all())}")
    grid = vm.TokenGrid(81, 28, 52, 128, 40, 1)
    q = torch.randn(grid.units(), grid.tokens(), 128, device=dev, dtype=torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    o = vm.vmonarch_attention(q, k, v, grid, cfg)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(3):
        vm.vmonarch_attention(q, k, v, grid, cfg, out=o, check=False)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 3
    F = vm.flops_estimate(grid, cfg, 128)
    tot = (F.monarch_flops + F.recompute_flops) * grid.units()
    print(f"C4 bf16: {ms:.3f} ms/call, {tot / ms / 1e9:.1f} TFLOP/s, finite={bool(torch.isfinite(o).all())}")


if __name__ == "__main__":
    globals()["stage_" + sys.argv[1]]()
