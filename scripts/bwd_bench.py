"""Time flash_entropy_bwd (the tcgen05 kernels, or the CUDA-core ones with VMB_BWD=simt).
    python scripts/bwd_bench.py [U] [n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2601_22275_b200 as vm

U = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
d = 128
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, generator=g, device="cuda").to(torch.bfloat16)  # noqa: E731
q, k, v, gr = mk(U, n, d) / d ** 0.5, mk(U, n, d), mk(U, n, d), mk(U, n, d)
o, lse, h = vm.flash_entropy_fwd(q, k, v, want_entropy=True) if n <= 4096 else (mk(U, n, d), torch.zeros(U, n, device="cuda"), torch.zeros(U, n, device="cuda"))
dh = torch.randn(U, n, device="cuda")
for _ in range(2):
    vm.flash_entropy_bwd(q, k, v, o, gr, lse, h, dh, entropy_grad=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    vm.flash_entropy_bwd(q, k, v, o, gr, lse, h, dh, entropy_grad=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
flops = 5 * 2 * n * n * d * U  # the 5 GEMMs of the standard backward (convention)
print(f'{{"U": {U}, "n": {n}, "ms": {ms:.3f}, "tflops_5gemm": {flops / ms / 1e9:.1f}}}')
