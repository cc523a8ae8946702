"""One call each of the §8(f) kernels for ncu: the m > 128 L-step passes (lstep_big) at the C2
grid with (m, b) = (210, 156), 12 heads, and the tcgen05 flash backward at 8 x 8192."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22275_b200 as vm  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
r = lambda *s: torch.randn(*s, generator=g, device="cuda").to(torch.bfloat16)  # noqa: E731
grid = vm.TokenGrid(21, 30, 52, 128, 12, 1)
q, k, v = (r(12, grid.tokens(), 128) for _ in range(3))
vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig(override_m_b=(210, 156)), check=False)
U, n = 8, 8192
qb, kb, vb, gb, ob = (r(U, n, 128) for _ in range(5))
lse = torch.zeros(U, n, device="cuda")
vm.flash_entropy_bwd(qb, kb, vb, ob, gb, lse, torch.zeros(U, n, device="cuda"), torch.randn(U, n, device="cuda"),
                     entropy_grad=True)
torch.cuda.synchronize()
