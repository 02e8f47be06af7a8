"""Measure pinned host<->device copy bandwidth alone and overlapped (the e2e ceiling)."""
import time
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); a = time.perf_counter() - t
t = time.perf_counter(); h2.copy_(d2, non_blocking=True); torch.cuda.synchronize(); b = time.perf_counter() - t
t = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); c = time.perf_counter() - t
print({"h2d_GBps": n / a / 1e9, "d2h_GBps": n / b / 1e9, "duplex_each_GBps": n / c / 1e9})
