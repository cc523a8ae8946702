"""Host enqueue time per vmonarch_attention call against its device time (is the GPU ever
starved by the host?).  python scripts/host_overhead.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22275_b200 as vm  # noqa: E402

for gridt, H in [((21, 30, 52), 12), ((81, 28, 52), 40), ((4, 8, 16), 2)]:
    g = vm.TokenGrid(*gridt, 128, H, 1)
    x = [torch.randn((H, g.tokens(), 128), device="cuda").bfloat16() for _ in range(3)]
    o = torch.empty_like(x[0])
    for _ in range(3):
        vm.vmonarch_attention(*x, g, out=o, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    t0 = time.perf_counter()
    for _ in range(n):
        vm.vmonarch_attention(*x, g, out=o, check=False)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"{gridt} H={H}: host enqueue {1e3 * (t1 - t0) / n:.3f} ms/call, device {e0.elapsed_time(e1) / n:.3f} ms/call")
