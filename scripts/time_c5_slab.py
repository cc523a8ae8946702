"""Per-GPU device time of the C5 sequence-sharded forward (81x112x104, H=40, d=128) on one
B200: rank r of W owns slab_partition(h*w, W)[r] of every frame; K/V are the full tensors
(what the all-gather delivers).  python scripts/time_c5_slab.py [W] [rank]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22275_b200 as vm  # noqa: E402
from paper_2601_22275_b200.dist import slab_partition  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
r = int(sys.argv[2]) if len(sys.argv) > 2 else 0
grid = vm.TokenGrid(81, 112, 104, 128, 40, 1)
a, c = slab_partition(112 * 104, W)[r]
g = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn((40, grid.tokens(), 128), generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn((40, grid.tokens(), 128), generator=g, device="cuda").to(torch.bfloat16)
q = torch.randn((40, 81 * c, 128), generator=g, device="cuda").to(torch.bfloat16)
out = vm.vmonarch_attention_slab(q, k, v, grid, a, c)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    vm.vmonarch_attention_slab(q, k, v, grid, a, c, out=out, check=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
rep = vm.flops_estimate(grid, vm.VMonarchConfig(), 128)
job = (rep.monarch_flops + rep.recompute_flops) * grid.units()  # per-unit estimate x 40 units
print(json.dumps({"world": W, "rank": r, "slab_positions": c, "ms_per_rank": round(ms, 2), "job_flops": job,
                  "job_tflops_if_ranks_equal": round(job / (ms * 1e-3) / 1e12, 1)}))
