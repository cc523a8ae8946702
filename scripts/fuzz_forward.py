import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
import torch
import test_gpu_fuzz as tf
from oracle.oracle import Oracle, bf16_round, workload
from test_gpu_parity import oracle_fwd, run_gpu
from vmb_testutil import relfro
import paper_2601_22275_b200 as vm
orc = Oracle("port")
bad = 0
cases = tf._cases(count=int(sys.argv[1]), seed=int(sys.argv[2]))
for (gridt, d, heads, batch, bf16, sigma, kw) in cases:
    grid = vm.TokenGrid(*gridt, head_dim=d, heads=heads, batch=batch)
    cfg = vm.VMonarchConfig(**kw)
    q, k, v = workload(grid.units(), grid.tokens(), d, seed=hash((gridt, d, heads)) % 1000, sigma=sigma)
    if bf16: q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    try:
        ref = oracle_fwd(orc, q, k, v, grid, cfg)
        got = run_gpu(vm, q, k, v, grid, cfg, torch.bfloat16 if bf16 else torch.float32, "cuda")
        e = relfro(got, ref)
        tol = 2e-2 if bf16 else 1e-4
        if not e <= tol:
            bad += 1; print("FAIL", gridt, d, heads, batch, bf16, sigma, kw, e)
    except Exception as ex:
        print("ERR", gridt, d, heads, batch, bf16, sigma, kw, repr(ex)[:200]); bad += 1
print("cases", len(cases), "bad", bad)
