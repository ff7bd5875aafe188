"""Probe host<->device copy bandwidth on the box: H2D, D2H, both at once,
pinned vs pageable, whole vs 64 MB chunks."""
import time
import torch
n = 1 << 28  # 1 GiB of float32
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - a)
    return best
gb = n * 4 / 1e9
x = t(lambda: d.copy_(h, non_blocking=True)); print(f"H2D 1GiB pinned: {x*1e3:.1f} ms {gb/x:.1f} GB/s")
x = t(lambda: h.copy_(d, non_blocking=True)); print(f"D2H 1GiB pinned: {x*1e3:.1f} ms {gb/x:.1f} GB/s")
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
x = t(both); print(f"H2D+D2H concurrent: {x*1e3:.1f} ms {2*gb/x:.1f} GB/s aggregate")
c = 1 << 24
def chunked():
    for i in range(0, n, c):
        d[i:i+c].copy_(h[i:i+c], non_blocking=True)
x = t(chunked); print(f"H2D 64MB chunks: {x*1e3:.1f} ms {gb/x:.1f} GB/s")
hp = torch.empty(n, dtype=torch.float32)
x = t(lambda: d.copy_(hp), reps=2); print(f"H2D pageable: {x*1e3:.1f} ms {gb/x:.1f} GB/s")
a = time.perf_counter(); p = torch.cuda.caching_allocator_alloc(2 << 30) if False else None
import ctypes
