"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck):
    compute-sanitizer --tool memcheck python scripts/sanitize_small.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22275_b200 as vm  # noqa: E402
from paper_2601_22275_b200.torch_op import vmonarch_attention_op  # noqa: E402,F401

dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
r = lambda *s: torch.randn(*s, generator=g, device=dev).to(torch.bfloat16)  # noqa: E731
# forward: default factorization (fa2, lstep, fa4, lstep apply, fa3 + combine)
grid = vm.TokenGrid(3, 10, 20, 128, 2, 1)
q, k, v = r(2, grid.tokens(), 128), r(2, grid.tokens(), 128), r(2, grid.tokens(), 128)
vm.vmonarch_attention(q, k, v, grid)
# L-step with two positions per CTA (m = 49, ragged b = 15) and one position (m = 81)
for tg in ((49, 3, 5), (81, 3, 4)):
    gg = vm.TokenGrid(*tg, 128, 1, 1)
    z = r(1, gg.tokens(), 128)
    vm.vmonarch_attention(z, z, z, gg)
# m > 128 (lstep_big), d < 128 (padding)
g2 = vm.TokenGrid(8, 8, 8, 128, 1, 1)
x = r(1, g2.tokens(), 128)
vm.vmonarch_attention(x, x, x, g2, vm.VMonarchConfig(override_m_b=(256, 2)))
g3 = vm.TokenGrid(4, 8, 8, 64, 1, 1)
y = r(1, g3.tokens(), 64)
vm.vmonarch_attention(y, y, y, g3)
# flash with entropy (fa3 ENT, split path), dense, backward (tcgen05)
qf, kf = r(1, 100, 128), r(1, 4000, 128)
o, lse, h = vm.flash_entropy_fwd(qf, kf, kf)
vm.dense_forward(r(1, 300, 128), r(1, 300, 128), r(1, 300, 128))
vm.flash_entropy_bwd(qf, kf, kf, o, r(1, 100, 128), lse, h, torch.randn(1, 100, device=dev), entropy_grad=True)
# multi (heads, seq) on one device
vm.vmonarch_attention_multi([q[:1], q[1:]], [k[:1], k[1:]], [v[:1], v[1:]], grid, mode="heads")
torch.cuda.synchronize()
print("sanitize_small: done")
