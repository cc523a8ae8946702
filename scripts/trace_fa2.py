"""Debug per-CTA timeline of the R half-step kernel (fa2_kernel<1>) at C4.
Build: make -C paper_2601_22275_b200/csrc EXTRA=-DVMB_TRACE=1 OUT=../libvmb_trace.so BUILD=build_trace
Run:   VMB_LIB=$PWD/paper_2601_22275_b200/libvmb_trace.so python scripts/trace_fa2.py"""
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
buf = (C.c_ulonglong * (4096 * 8))()
vm.lib.vmb_debug_trace2_read.argtypes = [C.c_void_p]
vm.lib.vmb_debug_trace2_read(C.addressof(buf))
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.float64) / 1000.0  # us
x = t[600:4096]
names = ["start", "Q in (softmax warps)", "S0 ready", "last P", "O full", "epilogue done", "exit barrier"]
print("fa2 R half-step: CTA phases (us, mean / p10 / p90 over CTAs 600..4095; 23 key tiles of 64 per CTA)")
for ev in range(1, 7):
    d = x[:, ev] - x[:, ev - 1]
    print(f"  {names[ev - 1]:>20} -> {names[ev]:<20}: {d.mean():6.2f}  {np.percentile(d, 10):6.2f}  {np.percentile(d, 90):6.2f}")
life = x[:, 6] - x[:, 0]
print(f"  lifetime {life.mean():.2f} us; main loop per tile {((x[:, 3] - x[:, 2]) / 22).mean() * 1000:.0f} ns")
starts = np.sort(x[:, 0])
print(f"  CTA start rate {len(starts) / (starts[-1] - starts[0]):.2f} per us (2 per SM x 148 SMs / lifetime = "
      f"{296 / life.mean():.2f})")
