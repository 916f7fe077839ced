"""PCIe probe: H2D, D2H alone and concurrently (two streams), pinned memory."""
import time, torch
h = torch.empty(60_000_000 // 4, dtype=torch.float32).pin_memory()
d = torch.empty_like(h, device="cuda")
ho = torch.empty(105_000_000 // 4, dtype=torch.float32).pin_memory()
do = torch.empty_like(ho, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, n=10):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3
def h2d():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
def both():
    h2d(); d2h()
def d2h_chunks():
    with torch.cuda.stream(s2):
        for c in range(72):
            n = ho.numel() // 72
            ho[c*n:(c+1)*n].copy_(do[c*n:(c+1)*n], non_blocking=True)
a, b, c, e = t(h2d), t(d2h), t(both), t(d2h_chunks)
print(f"h2d 60MB {a:.3f} ms ({60/a:.1f} GB/s); d2h 105MB {b:.3f} ms ({105/b:.1f} GB/s); both {c:.3f} ms; d2h 72 chunks {e:.3f} ms")
