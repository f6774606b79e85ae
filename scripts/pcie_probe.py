"""Measure PCIe copy rates on the box: H2D, D2H, both at once (1 GiB pinned)."""
import time, torch
n = 1 << 28
h1 = torch.empty(n, dtype=torch.uint32, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint32, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint32, device="cuda"); d2 = torch.empty(n, dtype=torch.uint32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - a)
    return best * 1e3
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
def seq6():
    for i in range(6):
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
print(f"H2D 1GiB {t(h2d):.2f} ms  D2H {t(d2h):.2f} ms  both {t(both):.2f} ms  6xH2D {t(seq6,1):.2f} ms")
