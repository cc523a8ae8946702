import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_2601_22275_b200 as vm
def t(grid, cfg, reps=3):
    g = torch.Generator(device='cuda').manual_seed(0)
    q, k, v = (torch.randn((grid.units(), grid.tokens(), 128), generator=g, device='cuda').to(torch.bfloat16) for _ in range(3))
    vm.vmonarch_attention(q, k, v, grid, cfg); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): vm.vmonarch_attention(q, k, v, grid, cfg, check=False)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
G = vm.TokenGrid(21, 30, 52, 128, 1, 1)
print("C2 1 head default (21,1560):", t(G, vm.VMonarchConfig()))
print("C2 1 head override (4, 8190):", t(G, vm.VMonarchConfig(override_m_b=(4, 8190))))
print("C2 1 head override (210, 156):", t(G, vm.VMonarchConfig(override_m_b=(210, 156))))
G2 = vm.TokenGrid(8, 32, 32, 128, 1, 1)
print("8192 tok b=1 (m=8192):", t(G2, vm.VMonarchConfig(override_m_b=(8192, 1)), 1))
print("8192 tok default:", t(G2, vm.VMonarchConfig()))
