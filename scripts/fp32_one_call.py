import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2601_22275_b200 as vm
g = vm.TokenGrid(21, 30, 52, 128, 1, 1)
x = [torch.randn((1, g.tokens(), 128), device='cuda') for _ in range(3)]
vm.vmonarch_attention(*x, g); torch.cuda.synchronize()
