"""Debug tile timeline of the persistent fa5 kernel (R-step, VMB_RSTEP=5).
Build: make -C paper_2601_22275_b200/csrc EXTRA=-DVMB_TRACE=1 OUT=../libvmb_trace.so BUILD=build_trace"""
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
cfg = vm.VMonarchConfig(recompute_first_frame=False)  # R-step 0 runs on fa5 (the last on fa4)
for _ in range(2):
    vm.vmonarch_attention(q, k, v, grid, cfg, out=o, check=False)
torch.cuda.synchronize()
tb = (C.c_longlong * (16 * 2 * 12 * 4))()
vm.lib.vmb_debug_trace5_read.argtypes = [C.c_void_p]
vm.lib.vmb_debug_trace5_read(C.addressof(tb))
tt = np.frombuffer(tb, dtype=np.int64).reshape(16, 2, 12, 4).astype(np.float64)
d = np.diff(tt, axis=3)[:, :, 1:11]
print("fa5 softmax A tile phases (cycles): wait S %.0f, compute %.0f, st-wait+arrive %.0f" %
      tuple(float(d[..., i].mean()) for i in range(3)))
per = np.diff(tt[:, :, :, 0], axis=2)[:, :, 1:10]
print("tile period (cycles): %.0f" % per.mean())
gap = tt[:, 1, 0, 0] - tt[:, 0, 11, 3]
print("item boundary gap, last P of item 1 -> start of item 2 tile 0 (cycles): %.0f" % gap.mean())
