"""Host <-> device copy bandwidth on this box (pinned memory): the e2e path's ceiling."""
import torch

n = 1 << 30  # 1 GiB
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
for name, fn in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))]:
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    print(f"{name}: {n / e0.elapsed_time(e1) / 1e6:.1f} GB/s", flush=True)
# concurrent H2D + D2H on two streams
torch.cuda.synchronize()
e0.record()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize()
print(f"H2D + D2H concurrent: {2 * n / e0.elapsed_time(e1) / 1e6:.1f} GB/s total", flush=True)
# two concurrent H2D streams
e0.record()
with torch.cuda.stream(s1):
    d[: n // 2].copy_(h[: n // 2], non_blocking=True)
with torch.cuda.stream(s2):
    d[n // 2:].copy_(h[n // 2:], non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize()
print(f"H2D on two streams: {n / e0.elapsed_time(e1) / 1e6:.1f} GB/s", flush=True)
