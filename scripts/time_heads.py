"""Device time of one vmonarch_attention call with H heads (the per-GPU load of a heads-sharded
run): python scripts/time_heads.py H [reps] [T h w]   (default grid: C4, 81 28 52)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22275_b200 as vm  # noqa: E402

H = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
T, h, w = (int(x) for x in sys.argv[3:6]) if len(sys.argv) > 5 else (81, 28, 52)
grid = vm.TokenGrid(T, h, w, 128, H, 1)
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = (torch.randn((H, grid.tokens(), 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
for _ in range(3):
    vm.vmonarch_attention(q, k, v, grid, check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    vm.vmonarch_attention(q, k, v, grid, check=False)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"grid": [T, h, w], "heads": H, "ms": round(e0.elapsed_time(e1) / reps, 4)}))
