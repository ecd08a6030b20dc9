"""Measure H2D / D2H / bidirectional pinned-copy bandwidth on the box."""
import time, torch
torch.cuda.set_device(0)
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def bw(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return reps * n / (time.perf_counter() - t) / 1e9
print("H2D GB/s", round(bw(lambda: d.copy_(h, non_blocking=True)), 1))
print("D2H GB/s", round(bw(lambda: h.copy_(d, non_blocking=True)), 1))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print("bidir GB/s (each way)", round(bw(both), 1))
