#!/usr/bin/env python3
"""Fixed vs streaming cost of a weight-streaming GEMM launch: M=128, N=4096,
K swept, automatic plan, back-to-back launches (weights rotated through HBM).
The intercept of time vs weight bytes is the per-launch fixed cost."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402

cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4, dtype=K.KRUL_BF16, max_tokens=64)
ctx = K.Context(cfg, 0)
lib = K.lib()
for N in (4096, 16384):
    for Kd in (256, 512, 1024, 2048, 4096, 8192, 16384):
        for force, sp in ((0, 0), (2, 1)):
            ms = C.c_float(0)
            rc = lib.krul_debug_gemm_bench(ctx.h, C.c_int64(128), C.c_int64(N), C.c_int64(Kd), 2, force, sp, 40,
                                           C.byref(ms))
            mb = N * Kd * 2 / 1e6
            print(f"N={N} K={Kd:6d} f{force}s{sp} weights {mb:7.1f} MB: {ms.value * 1e3:7.2f} us", flush=True)
