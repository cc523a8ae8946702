import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2601_22275_b200 as vm
for gridt, H in [((21, 30, 52), 1), ((81, 28, 52), 1)]:
    g = vm.TokenGrid(*gridt, 128, H, 1)
    x = [torch.randn((H, g.tokens(), 128), device='cuda') for _ in range(3)]
    vm.vmonarch_attention(*x, g); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); vm.vmonarch_attention(*x, g, check=False); e1.record(); torch.cuda.synchronize()
    xb = [t.bfloat16() for t in x]
    vm.vmonarch_attention(*xb, g); torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(); vm.vmonarch_attention(*xb, g, check=False); e3.record(); torch.cuda.synchronize()
    print(gridt, "1 head fp32 (CUDA cores):", round(e0.elapsed_time(e1), 2), "ms; bf16 (tcgen05):", round(e2.elapsed_time(e3), 3), "ms")
