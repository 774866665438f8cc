"""Host<->device copy rates for 16.8 MB (C2's x / y) pinned buffers: H2D alone,
D2H alone, both concurrently on two streams."""
import sys, time
import torch
n = 2097152
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True); h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def h2d():
    d1.copy_(h1, non_blocking=True)
def d2h():
    h2.copy_(d2, non_blocking=True)
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    el = t(fn)
    gb = (2 if name == "both" else 1) * n * 8 / el / 1e9
    print(f"{name}: {el*1e3:.3f} ms, {gb:.1f} GB/s")
