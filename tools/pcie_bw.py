"""PCIe bandwidth of the box: 1 GiB pinned H2D, D2H, and both at once (e2e bound)."""
import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
for _ in range(2):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
t = time.perf_counter()
for _ in range(5):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("H2D GB/s", 5 * n / dt / 1e9)
t = time.perf_counter()
for _ in range(5):
    h2.copy_(d, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("D2H GB/s", 5 * n / dt / 1e9)
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("bidir GB/s each", 5 * n / dt / 1e9)
