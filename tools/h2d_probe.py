#!/usr/bin/env python3
"""H2D link probe: one stream vs two concurrent streams vs an SM-driven copy
(kernel loads from mapped pinned memory)."""
import torch

n = 512 << 20
src = torch.empty(n, dtype=torch.uint8).pin_memory()
src.random_(0, 255)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
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


def one():
    dst.copy_(src, non_blocking=True)


def two():
    h = n // 2
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        dst[:h].copy_(src[:h], non_blocking=True)
    with torch.cuda.stream(s2):
        dst[h:].copy_(src[h:], non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def chunks(k):
    def f():
        step = n // k
        for i in range(k):
            dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
    return f


for name, fn in (("one stream", one), ("two streams", two), ("16 chunks", chunks(16)), ("64 chunks", chunks(64))):
    ms = timed(fn)
    print(f"{name}: {n / ms / 1e6:.2f} GB/s ({ms:.3f} ms)", flush=True)
# SM-driven copy from mapped pinned memory
try:
    import ctypes
    cudart = ctypes.CDLL("libcudart.so")
except OSError:
    cudart = None
import cupy  # noqa: F401  (absent -> skip)
