"""Debug timeline of the last R-step kernel (fa_tc_kernel<2,2>): per-CTA globaltimer stamps.
Build: make -C paper_2601_22275_b200/csrc EXTRA=-DVMB_TRACE=1 OUT=../libvmb_trace.so BUILD=build_trace
Run:   VMB_LIB=$PWD/paper_2601_22275_b200/libvmb_trace.so python scripts/trace_fa.py"""
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
for _ in range(3):
    vm.vmonarch_attention(q, k, v, grid, vm.VMonarchConfig(), out=o, check=False)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (4096 * 8))()
vm.lib.vmb_debug_trace_read.argtypes = [C.c_void_p, C.c_int]
got = vm.lib.vmb_debug_trace_read(C.addressof(buf), 4096)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8)[:got].astype(np.float64)
t0 = t[:, 0].min()
names = ["start", "tmem+bars", "S0 ready", "S_last ready", "last P", "O done", "O staged", "exit"]
d = np.diff(t[:, :8], axis=1) / 1000.0
print("per-CTA phase durations (us): mean / p50 / p90")
for i in range(7):
    print(f"  {names[i]:>12} -> {names[i + 1]:<12} {d[:, i].mean():7.2f} {np.median(d[:, i]):7.2f} {np.percentile(d[:, i], 90):7.2f}")
life = (t[:, 7] - t[:, 0]) / 1000.0
print(f"CTA lifetime mean {life.mean():.2f} us; launch span of these CTAs {(t[:, 7].max() - t0) / 1e3:.1f} us")
# concurrency: how many CTAs alive on average (should be ~148)
ev = sorted([(a, 1) for a in t[:, 0]] + [(b, -1) for b in t[:, 7]])
alive, acc, last, span = 0, 0.0, ev[0][0], ev[-1][0] - ev[0][0]
for x, dlt in ev:
    acc += alive * (x - last)
    alive += dlt
    last = x
print(f"mean CTAs in flight {acc / span:.1f}")
