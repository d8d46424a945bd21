"""Developer probe: pinned H2D / D2H bandwidth alone and concurrently (two streams)."""
import torch
import sys
n = int(sys.argv[1]) << 20 if len(sys.argv) > 1 else 64 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both(): h2d(); d2h()
a = t(h2d); b = t(d2h); c = t(both)
print(f"H2D {n/a/1e6:.1f} GB/s, D2H {n/b/1e6:.1f} GB/s, concurrent {2*n/c/1e6:.1f} GB/s total")
