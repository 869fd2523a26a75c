"""Host<->device copy bandwidth with pinned buffers (sequential and concurrent)."""
import time
import torch

n = 120 * 1024 * 1024 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(fn, k=10):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / k
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bt = t(both)
mb = n * 4 / 1e9
print(f"H2D {mb / h2d:.1f} GB/s  D2H {mb / d2h:.1f} GB/s  concurrent {2 * mb / bt:.1f} GB/s total")
x = torch.empty(n, dtype=torch.float32, pin_memory=True)
a = time.perf_counter(); y = torch.empty(n, dtype=torch.float32, pin_memory=True); print("pinned alloc (cached?)", time.perf_counter() - a)
