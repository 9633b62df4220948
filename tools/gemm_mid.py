#!/usr/bin/env python3
"""Mid-M GEMM sweep (the pyramid recompute's shapes): auto plan vs forced variants."""
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
V = {0: "auto", 1: "1sm256", 2: "1sm128", 3: "pair"}
for M in (160, 300, 500, 700, 1000):
    for N, Kd, epi, name in ((6144, 4096, 10 if False else 0, "qkv"), (4096, 4096, 2, "o"),
                             (28672, 4096, 4, "ffn1"), (4096, 14336, 2, "ffn2")):
        row = []
        for var in (0, 1, 2, 3):
            for sp in ((0,) if var == 0 else (0, 2)):
                ms = C.c_float(0)
                rc = lib.krul_debug_gemm_bench(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), epi, var,
                                               sp, 20, C.byref(ms))
                if rc == 0:
                    row.append((round(2 * M * N * Kd / (ms.value * 1e-3) / 1e12), V[var], sp))
        best = max(row)
        auto = [r for r in row if r[1] == "auto"][0]
        print(f"M={M} {name}: auto {auto[0]} TF/s; best {best}; all {sorted(row, reverse=True)[:4]}", flush=True)
