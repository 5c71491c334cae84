#!/usr/bin/env python3
"""Host<->device and write-only bandwidth probe (pinned memory, CUDA events):
the floors that bound bench.py's e2e leg and the zero-fill pass."""
import torch

dev = torch.device("cuda", 0)
nb = 2 << 30
h1 = torch.empty(nb // 8, dtype=torch.float64).pin_memory()
h2 = torch.empty(nb // 8, dtype=torch.float64).pin_memory()
d1 = torch.empty(nb // 8, dtype=torch.float64, device=dev)
d2 = torch.empty(nb // 8, dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


t = timed(lambda: d1.copy_(h1, non_blocking=True))
print(f"H2D pinned {nb / t / 1e6:.1f} GB/s")
t = timed(lambda: h1.copy_(d1, non_blocking=True))
print(f"D2H pinned {nb / t / 1e6:.1f} GB/s")


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t = timed(both)
print(f"H2D+D2H concurrent {2 * nb / t / 1e6:.1f} GB/s total ({nb / t / 1e6:.1f} each)")
big = torch.empty(2500 << 20, dtype=torch.uint8, device=dev)
t = timed(lambda: big.zero_(), 5)
print(f"device memset 2.5 GB: {t:.3f} ms = {big.numel() / t / 1e6:.0f} GB/s")
src = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
dst = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
t = timed(lambda: dst.copy_(src), 5)
print(f"device copy 1 GiB: {2 * src.numel() / t / 1e6:.0f} GB/s (read+write)")
