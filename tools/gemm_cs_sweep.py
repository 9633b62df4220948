#!/usr/bin/env python3
"""Weight-streaming GEMM plans (M <= 128): the automatic plan, the automatic
plan without cluster split-K (force 9: split-K through a reduce kernel), and
cluster split-K forced at cs = 2 / 3 / 4 with 256- / 128-wide tiles (force
11 / 12: cs CTAs per tile, fp32 partials reduced over DSMEM inside the GEMM). Back-to-back launches, weights
rotated over >= 320 MB (streamed from HBM)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402

cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4, dtype=K.KRUL_BF16, max_tokens=64)
ctx = K.Context(cfg, 0)
lib = K.lib()
shapes = {"8b": ((6144, 4096, 0, "qkv"), (4096, 4096, 2, "o"), (28672, 4096, 4, "ffn1"), (4096, 14336, 2, "ffn2")),
          "70b": ((10240, 8192, 0, "qkv"), (8192, 8192, 2, "o"), (57344, 8192, 4, "ffn1"), (8192, 28672, 2, "ffn2"))}
for model in os.environ.get("MODELS", "8b,70b").split(","):
    for M in [int(x) for x in os.environ.get("MS", "128,1").split(",")]:
        tot = {}
        for N, Kd, epi, name in shapes[model]:
            row = []
            for force, sp in ((0, 0), (9, 0), (11, 2), (11, 3), (11, 4), (12, 2), (12, 3), (12, 4)):
                ms = C.c_float(0)
                rc = lib.krul_debug_gemm_bench(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), epi, force, sp, 40,
                                               C.byref(ms))
                us = ms.value * 1e3 if rc == 0 else float("nan")
                gbs = (N * Kd * 2 + M * Kd * 2 + M * N * 4) / (us * 1e-6) / 1e9
                key = f"f{force}s{sp}"
                row.append(f"{key}: {us:6.1f}")
                tot[key] = tot.get(key, 0.0) + us
            print(f"{model} M={M:4d} {name:5s} N={N:6d} K={Kd:6d} | " + " | ".join(row), flush=True)
        print(f"{model} M={M:4d} layer sum: " + " ".join(f"{k}={v:.1f}" for k, v in tot.items()), flush=True)
