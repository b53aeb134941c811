"""Pinned host -> device copy bandwidth (one and two concurrent streams)."""
import torch
n = 218 * (1 << 20)
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print("one stream GB/s", 10 * n / (e0.elapsed_time(e1) * 1e6))
half = n // 2
import time
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        d[half:].copy_(h[half:], non_blocking=True)
torch.cuda.synchronize()
print("two streams GB/s", 10 * n / ((time.perf_counter() - t) * 1e9))
