"""Where the bf16 error of the sigma=3 / t=3 / (49, 4) corner comes from: each GPU half-step
fed the oracle's own (bf16-rounded) state, against the oracle's next state."""
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import torch
from oracle.oracle import Oracle, bf16_round, workload
from vmb_testutil import relfro
import paper_2601_22275_b200 as vm

orc = Oracle("port")
dev = "cuda"
T, h, w, d = 4, 7, 7, 128
m, b = 49, 4
N = m * b
for sigma, iters in ((3.0, 3), (2.0, 3), (3.0, 2)):
    worst = []
    for seed in range(6):
        q, k, v = workload(2, N, d, seed=seed, sigma=sigma)
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
        grid = vm.TokenGrid(T, h, w, d, 2, 1)
        cfg = vm.VMonarchConfig(iters=iters, recompute_first_frame=False, override_m_b=(m, b))
        ref = orc.vmonarch_attention(q, k, v, (T, h, w), iters=iters, recompute=False, override=(m, b))
        got = vm.vmonarch_attention(*(torch.from_numpy(x).to(dev, torch.bfloat16) for x in (q, k, v)), grid, cfg)
        got = got.float().cpu().numpy()
        per_head = [relfro(got[u], ref[u]) for u in range(2)]
        line = [f"s{seed} fwd " + " ".join(f"{e:.4f}" for e in per_head)]
        for u in range(2):
            qs = (q[u] / np.sqrt(d)).astype(np.float32)
            Kb = k[u].reshape(m, b, d)
            Qb = np.ascontiguousarray(qs.reshape(m, b, d).transpose(1, 0, 2))
            aR = qs.reshape(m, b, d).copy(); cR = np.ones((m, b), np.float32)
            errs = []
            for t in range(iters):
                aL, cL, _ = orc.rstep(aR, cR, Kb, want_R=False)
                gaL, gcL, _ = vm.r_update(torch.from_numpy(bf16_round(aR)[None]).to(dev, torch.bfloat16),
                                          torch.from_numpy(cR[None]).to(dev),
                                          torch.from_numpy(Kb[None].copy()).to(dev, torch.bfloat16))
                errs.append(("R", relfro(gaL[0].float().cpu().numpy(), aL),
                             float(np.abs(gcL[0].cpu().numpy() - cL).max())))
                aR, cR, _ = orc.lstep(Qb, aL, cL, want_L=False)
                gaR, gcR, _ = vm.l_update(torch.from_numpy(bf16_round(Qb)[None]).to(dev, torch.bfloat16),
                                          torch.from_numpy(bf16_round(aL)[None]).to(dev, torch.bfloat16),
                                          torch.from_numpy(cL[None].copy()).to(dev))
                errs.append(("L", relfro(gaR[0].float().cpu().numpy(), aR),
                             relfro(gcR[0].cpu().numpy(), cR)))
            line.append(f"u{u} " + " ".join(f"{n}:{a:.4f}/{c:.4f}" for n, a, c in errs))
        print(f"sigma {sigma} iters {iters} " + " | ".join(line), flush=True)
