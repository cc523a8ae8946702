"""Generate tests/golden/golden.npz from the REFERENCE itself (oracle/_ref/libvmref.so, compiled
from /root/reference/proj by oracle/Makefile).  Run in the container that has /root/reference:

    python tests/golden/make_golden.py

The fixtures pin the CPU restatement (oracle/vmonarch_oracle.c) and, through it, the GPU
parity tests.  Inputs follow the reference's generator convention (std::mt19937_64 +
std::normal_distribution<double>, test_support.hpp:17-24; per-unit seeds s+3u, s+3u+1, s+3u+2,
bench_main.cpp:169-173).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle, randn, workload  # noqa: E402


def main():
    R = Oracle("reference")
    g = {}
    # C1 (BASELINE configs[0]): B=1 H=2 d=64, 4 frames x 8x8 latent, fp32, t=3
    q, k, v = workload(2, 256, 64, seed=0)
    g["c1_q"], g["c1_k"], g["c1_v"] = q, k, v
    g["c1_out"] = R.vmonarch_attention(q, k, v, (4, 8, 8), iters=3)
    g["c1_out_norecompute"] = R.vmonarch_attention(q, k, v, (4, 8, 8), iters=3, recompute=False)
    # permutation / layout (perm.hpp:19-30, mat.hpp:99-113)
    for b, n in [(3, 6), (4, 12), (5, 20), (1, 7), (7, 7), (1456, 1456 * 4)]:
        g[f"perm_{b}_{n}"] = R.make_perm(b, n)
    x = randn((12, 5), 9, dtype=np.float32)
    g["blocked_x"] = x
    g["blocked_qb"] = R.to_blocked_permuted(x, 3, 4)
    # FLOP / sparsity accounting (video.cpp:24-59)
    for name, (tf, h, w, d) in {"wan321_d64": (81, 28, 52, 64), "wan61_d64": (16, 28, 52, 64),
                                 "c4_d128": (81, 28, 52, 128), "c2_d128": (21, 30, 52, 128)}.items():
        rep = R.flops_estimate((tf, h, w), d)
        g[f"flops_{name}"] = np.array([rep["monarch_flops"], rep["full_attn_flops"], rep["recompute_flops"]],
                                      dtype=np.uint64)
        g[f"ratio_{name}"] = np.array([rep["reduction_ratio"], rep["sparsity"], rep["sparsity_approx"]])
    # half steps in f64 (monarch.hpp:53-147)
    m, b, d = 3, 5, 4
    qs = randn((m * b, d), 3, dtype=np.float64) / np.sqrt(d)
    kk = randn((m * b, d), 4, dtype=np.float64)
    aR, cR = qs.reshape(m, b, d), np.ones((m, b))
    aL, cL, Rf = R.rstep(aR, cR, kk.reshape(m, b, d))
    qb = R.to_blocked_permuted(qs.astype(np.float32), m, b).astype(np.float64)
    qb = np.ascontiguousarray(qs.reshape(m, b, d).transpose(1, 0, 2))
    aR2, cR2, Lf = R.lstep(qb, aL, cL)
    g.update(rs_qs=qs, rs_k=kk, rs_aL=aL, rs_cL=cL, rs_R=Rf, ls_qb=qb, ls_aR=aR2, ls_cR=cR2, ls_L=Lf)
    # f32 half steps at a d=128 tile-straddling size
    m, b, d = 3, 150, 128
    qs32 = (randn((m * b, d), 11, dtype=np.float32) * np.float32(1 / np.sqrt(d))).astype(np.float32)
    k32 = randn((m * b, d), 12, dtype=np.float32)
    cR32 = (0.5 + np.abs(randn((m, b), 13, dtype=np.float32))).astype(np.float32)
    aL32, cL32, _ = R.rstep(qs32.reshape(m, b, d), cR32, k32.reshape(m, b, d), want_R=False)
    qb32 = np.ascontiguousarray(qs32.reshape(m, b, d).transpose(1, 0, 2))
    aR32, cRo32, _ = R.lstep(qb32, aL32, cL32, want_L=False)
    g.update(rs32_qs=qs32, rs32_k=k32, rs32_cR=cR32, rs32_aL=aL32, rs32_cL=cL32, ls32_aR=aR32, ls32_cR=cRo32)
    # online-entropy attention (flash_entropy.hpp:85-139), rectangular, tail tiles
    fq = randn((40, 16), 9, dtype=np.float32)
    fk = randn((256, 16), 10, dtype=np.float32)
    fv = randn((256, 16), 11, dtype=np.float32)
    fo, fl, fe = R.flash_entropy_fwd(fq, fk, fv, 32, 48)
    g.update(fl_q=fq, fl_k=fk, fl_v=fv, fl_out=fo, fl_lse=fl, fl_ent=fe)
    # monarch_attention f64 with factors, clamp off (test_monarch_core.cpp:323-356)
    q64, k64, v64 = (randn((48, 5), s, dtype=np.float64) for s in (27, 28, 29))
    mo, mL, mR = R.monarch_attention(q64, k64, v64, 4, 12, iters=2, clamp_enabled=False, want_factors=True)
    g.update(mo_q=q64, mo_k=k64, mo_v=v64, mo_out=mo, mo_L=mL, mo_R=mR)
    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **g)
    print("wrote", out, os.path.getsize(out), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
