#!/usr/bin/env python3
"""Back-to-back weight-streaming GEMMs (automatic plan) with and without
programmatic dependent launch: how much of a launch's fixed cost (launch gap,
prologue, pipeline fill) PDL hides. Run twice: KRUL_PDL=0 / KRUL_PDL=1."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402

cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4, dtype=K.KRUL_BF16, max_tokens=64)
ctx = K.Context(cfg, 0)
lib = K.lib()
tag = "pdl" if os.environ.get("KRUL_PDL") == "1" else "nopdl"
for N, Kd, epi, name in ((6144, 4096, 0, "qkv"), (4096, 4096, 2, "o"), (28672, 4096, 4, "ffn1"), (4096, 14336, 2, "ffn2")):
    for force, sp in ((0, 0), (2, 1), (2, 2), (2, 3), (1, 1), (1, 2)):
        ms = C.c_float(0)
        rc = lib.krul_debug_gemm_bench(ctx.h, C.c_int64(128), C.c_int64(N), C.c_int64(Kd), epi, force, sp, 40, C.byref(ms))
        print(f"{tag} {name:5s} f{force}s{sp}: {ms.value * 1e3 if rc == 0 else float('nan'):7.2f} us", flush=True)
