#!/usr/bin/env python3
"""One weight-streaming GEMM shape through krul_debug_gemm_bench (graph replay): ncu target.
usage: gemm_one.py N K [epi] [force] [splits] [iters]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402

a = [int(x) for x in sys.argv[1:]] + [2, 0, 0, 10][len(sys.argv) - 3:]
N, Kd, epi, force, sp, iters = a[:6]
cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4, dtype=K.KRUL_BF16, max_tokens=64)
ctx = K.Context(cfg, 0)
ms = C.c_float(0)
rc = K.lib().krul_debug_gemm_bench(ctx.h, C.c_int64(128), C.c_int64(N), C.c_int64(Kd), epi, force, sp, iters,
                                   C.byref(ms))
print(f"N={N} K={Kd} epi={epi} f{force}s{sp}: {ms.value * 1e3:.2f} us/launch (graph replay)")
