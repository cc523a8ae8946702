"""Diagnostic: is the forward bitwise deterministic alone, and next to other work on a second
stream?  Prints, per configuration, how many of R repeated calls differ from the first."""
import sys

import torch

import os; sys.path.insert(0, os.environ.get("VMB_PKG_ROOT", "."))
import paper_2601_22275_b200 as vm  # noqa: E402

dev = torch.device("cuda:0")
R = int(sys.argv[1]) if len(sys.argv) > 1 else 8


def inputs(grid, seed):
    g = torch.Generator(device=dev).manual_seed(seed)
    return [torch.randn((grid.units(), grid.tokens(), grid.head_dim), device=dev, generator=g).bfloat16()
            for _ in range(3)]


def run(grid, cfg, qkv, noise):
    ref = vm.vmonarch_attention(*qkv, grid, cfg)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    outs = []
    for _ in range(R):
        with torch.cuda.stream(s1):
            outs.append(vm.vmonarch_attention(*qkv, grid, cfg, check=False))
        if noise == "mm":
            with torch.cuda.stream(s2):
                for _ in range(3):
                    a = (a @ a).clamp_(-1, 1)
        elif noise == "vm":
            with torch.cuda.stream(s2):
                g2 = vm.TokenGrid(3, 10, 20, 128, 3, 1)
                vm.vmonarch_attention(*inputs(g2, 5), g2, check=False)
    torch.cuda.synchronize()
    bad = [o for o in outs if not torch.equal(o, ref)]
    rows = set()
    for o in bad:
        diff = (o != ref).any(-1)
        rows |= set(torch.nonzero(diff)[:, 1].tolist())
    n = grid.tokens()
    hw = grid.h * grid.w
    return len(bad), (min(rows) if rows else None, max(rows) if rows else None, len(rows), n, hw)


grid = vm.TokenGrid(4, 8, 16, 128, 2, 1)
qkv = inputs(grid, 1)
for iters in (1, 2):
    for rec in (False, True):
        cfg = vm.VMonarchConfig(iters=iters, recompute_first_frame=rec)
        for noise in ("none", "mm", "vm"):
            print(f"iters={iters} recompute={rec} noise={noise}: bad/rows {run(grid, cfg, qkv, noise)}", flush=True)
