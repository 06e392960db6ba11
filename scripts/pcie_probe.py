"""H2D / D2H pinned bandwidth alone and concurrently (the e2e ceiling)."""
import torch, time
n = 2 * 1024**3 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True); h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn):
    torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - t
for _ in range(2):
    a = timed(lambda: d.copy_(h, non_blocking=True))
    b = timed(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    c = timed(both)
gb = n * 8 / 1e9
print(f"H2D {gb/a:.1f} GB/s  D2H {gb/b:.1f} GB/s  concurrent {2*gb/c:.1f} GB/s total")
