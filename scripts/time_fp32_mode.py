"""Per-head time of the fp32 parity mode (tensor cores for d = 128: hi/lo bf16 operands) next
to the bf16 mode, with the per-kernel-family split of the fp32 call (vmb_profile ids)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, '/root/repo')
import paper_2601_22275_b200 as vm  # noqa: E402

NAMES = ["rstep (fa2)", "rstep_y", "attention V (fa2 y pass + recompute)", "lstep_tc", "lstep_final", "cuda cores", "combine"]
vm.lib.vmb_profile_enable.argtypes = [C.c_int32]
vm.lib.vmb_profile_read.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
for gridt, H in [((21, 30, 52), 1), ((81, 28, 52), 1), ((81, 28, 52), 8)]:
    g = vm.TokenGrid(*gridt, 128, H, 1)
    x = [torch.randn((H, g.tokens(), 128), device='cuda') for _ in range(3)]
    vm.vmonarch_attention(*x, g); torch.cuda.synchronize()
    ms, cnt = (C.c_double * 7)(), (C.c_uint64 * 7)()
    vm.lib.vmb_profile_read(C.addressof(ms), C.addressof(cnt), 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); vm.vmonarch_attention(*x, g, check=False); e1.record(); torch.cuda.synchronize()
    t32 = e0.elapsed_time(e1)
    vm.lib.vmb_profile_enable(1)
    vm.vmonarch_attention(*x, g, check=False); torch.cuda.synchronize()
    vm.lib.vmb_profile_enable(0)
    vm.lib.vmb_profile_read(C.addressof(ms), C.addressof(cnt), 1)
    split = {NAMES[i]: round(ms[i], 3) for i in range(7) if cnt[i]}
    xb = [t.bfloat16() for t in x]
    vm.vmonarch_attention(*xb, g); torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(); vm.vmonarch_attention(*xb, g, check=False); e3.record(); torch.cuda.synchronize()
    print(gridt, f"{H} head(s): fp32 {t32:.2f} ms ({t32 / H:.2f} ms/head); bf16 {e2.elapsed_time(e3):.3f} ms;",
          "fp32 split (ms):", split, flush=True)
