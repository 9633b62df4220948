#!/usr/bin/env python3
"""M<=128 weight-streaming GEMM sweep over tile width and split-K count."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402

cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4,
                    dtype=K.KRUL_BF16, max_tokens=64)
ctx = K.Context(cfg, 0)
lib = K.lib()
for M, N, Kd, epi in ((128, 6144, 4096, 0), (128, 4096, 4096, 2), (128, 28672, 4096, 4),
                      (128, 4096, 14336, 2)):
    wb = N * Kd * 2
    res = []
    for var in (1, 2):
        for sp in (1, 2, 3, 4, 6, 8):
            ms = C.c_float(0)
            rc = lib.krul_debug_gemm_bench(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), epi, var, sp,
                                           20, C.byref(ms))
            if rc == 0:
                res.append((round(ms.value * 1e3, 1), var, sp, round(wb / (ms.value * 1e-3) / 1e9)))
    ms = C.c_float(0)
    lib.krul_debug_gemm_bench(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), epi, 0, 0, 20, C.byref(ms))
    res.sort()
    print(f"M={M} N={N} K={Kd}: auto {ms.value * 1e3:.1f} us; best (us, var, splits, GB/s):", res[:6], flush=True)
