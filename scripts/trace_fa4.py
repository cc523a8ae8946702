"""Debug per-item timeline of the persistent fa4 kernel (last R-step, VMB_RSTEP=4).
Build: make -C paper_2601_22275_b200/csrc EXTRA=-DVMB_TRACE=1 OUT=../libvmb_trace.so BUILD=build_trace
Run:   VMB_RSTEP=4 VMB_LIB=$PWD/paper_2601_22275_b200/libvmb_trace.so python scripts/trace_fa4.py"""
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
buf = (C.c_ulonglong * (64 * 16 * 8))()
vm.lib.vmb_debug_trace4_read.argtypes = [C.c_void_p]
vm.lib.vmb_debug_trace4_read(C.addressof(buf))
t = np.frombuffer(buf, dtype=np.uint64).reshape(64, 16, 8).astype(np.float64) / 1000.0  # us
names = ["item start", "S0 ready", "last P", "stats in", "O full", "O drained", "stored"]
print("item 1..14, mean over 64 CTAs (us, relative to the item's start):")
for ev in range(1, 7):
    d = t[:, 1:15, ev] - t[:, 1:15, 0]
    print(f"  {names[ev]:>10}: {d.mean():7.2f}")
gap = t[:, 2:15, 0] - t[:, 1:14, 2]
print(f"  softmax gap between items (next item start - last P): {gap.mean():.2f} us")
per_item = np.diff(t[:, 1:15, 0], axis=1)
print(f"  item period (start to next start): {per_item.mean():.2f} us")
wait_s0 = t[:, 1:15, 1] - t[:, 1:15, 0]
print(f"  wait for S0 at item start: {wait_s0.mean():.2f} us")

# fine-grained softmax tile phases (clock64 cycles), warp 4 lane 0, items 1-2, tiles 0-11
tb = (C.c_longlong * (16 * 2 * 12 * 6))()
vm.lib.vmb_debug_trace4t_read.argtypes = [C.c_void_p]
vm.lib.vmb_debug_trace4t_read(C.addressof(tb))
tt = np.frombuffer(tb, dtype=np.int64).reshape(16, 2, 12, 6).astype(np.float64)
ph = ["wait S", "TMEM ld", "max", "exp/P st", "st wait+arrive"]
d = np.diff(tt, axis=3)[:, :, 1:11]  # tiles 1..10
print("softmax tile phases (cycles, mean over CTAs/items/tiles):", {ph[i]: round(float(d[..., i].mean())) for i in range(5)})
per = np.diff(tt[:, :, :, 0], axis=2)[:, :, 1:10]
print("softmax tile period (cycles):", round(float(per.mean())))

# MMA issuer waits (clock64 cycles), tiles 24..47 of the first 16 CTAs
tm = (C.c_longlong * (16 * 24 * 4))()
vm.lib.vmb_debug_trace4m_read.argtypes = [C.c_void_p]
vm.lib.vmb_debug_trace4m_read(C.addressof(tm))
m = np.frombuffer(tm, dtype=np.int64).reshape(16, 24, 4).astype(np.float64)
print("MMA issuer per tile (cycles): kv_full wait", round(float((m[:, :, 1] - m[:, :, 0]).mean())),
      " p_full wait", round(float((m[:, :, 3] - m[:, :, 2]).mean())),
      " tile period", round(float(np.diff(m[:, :, 0], axis=1).mean())))
print("MMA issuer per tile (cycles): S issue+commit", round(float((m[:, :, 2] - m[:, :, 1]).mean())),
      " PV issue+commit", round(float((m[:, 1:, 0] - m[:, :-1, 3]).mean())))
print("per-tile samples CTA0:", [(int(m[0, i, 1] - m[0, i, 0]), int(m[0, i, 2] - m[0, i, 1]), int(m[0, i, 3] - m[0, i, 2]),
                                  int(m[0, i + 1, 0] - m[0, i, 3])) for i in range(12)])
