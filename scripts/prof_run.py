"""Minimal driver for ncu captures: one (or a few) VMonarch forward calls at a BASELINE shape."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22275_b200 as vm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--calls", type=int, default=1)
ap.add_argument("--heads", type=int, default=40)
ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
args = ap.parse_args()
T, h, w = {"c4": (81, 28, 52), "c2": (21, 30, 52)}[args.config]
grid = vm.TokenGrid(T, h, w, 128, args.heads, 1)
n = grid.tokens()
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(args.heads, n, 128, device="cuda", generator=g, dtype=torch.float32 if args.dtype == "f32" else torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
for _ in range(args.calls):
    vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig(), out=o, check=False)
torch.cuda.synchronize()
print("done", bool(torch.isfinite(o).all()))
