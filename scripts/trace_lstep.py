"""Debug per-CTA timeline of the L-step kernels (unit 0 of a C4 call).
Build: make -C paper_2601_22275_b200/csrc EXTRA=-DVMB_TRACE=1 OUT=../libvmb_trace.so BUILD=build_trace
Run:   VMB_LIB=$PWD/paper_2601_22275_b200/libvmb_trace.so python scripts/trace_lstep.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_22275_b200 as vm  # noqa: E402

grid = vm.TokenGrid(81, 28, 52, 128, 40, 1)
n = grid.tokens()
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(40, n, 128, device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
for _ in range(2):
    vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig(), out=o, check=False)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (2 * 1456 * 8))()
vm.lib.vmb_debug_tracel_read.argtypes = [C.c_void_p]
vm.lib.vmb_debug_tracel_read(C.addressof(buf))
t = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1456, 8).astype(np.float64) / 1000.0  # us
lo = (C.c_int * (2 * 1456))()
vm.lib.vmb_debug_tracel_lo_read.argtypes = [C.c_void_p]
vm.lib.vmb_debug_tracel_lo_read(C.addressof(lo))
lo = np.frombuffer(lo, dtype=np.int32).reshape(2, 1456)
names = ["start", "prologue", "S ready", "L written", "colsum", "O ready", "staged", "stored"]
for f, kname in enumerate(["lstep (ITER)", "lstep_apply (FINAL)"]):
    x = t[f, 600:1456]  # steady state: past the first wave of 592 CTAs
    print(f"{kname}: CTA phases (us, mean / p10 / p90 over positions 600..1455)")
    for ev in range(1, 8):
        d = x[:, ev] - x[:, ev - 1]
        print(f"  {names[ev - 1]:>10} -> {names[ev]:<10}: {d.mean():6.2f}  {np.percentile(d, 10):6.2f}  {np.percentile(d, 90):6.2f}")
    print(f"  CTAs that read aL's low half: {lo[f].mean():.3f}")
    life = x[:, 7] - x[:, 0]
    print(f"  lifetime: {life.mean():.2f} us; CTA start rate {len(x) / (x[:, 0].max() - x[:, 0].min()):.1f} per us")
