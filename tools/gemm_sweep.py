#!/usr/bin/env python3
"""GEMM plan sweep over the pyramid-recompute shapes: every (variant, split-K)
at each M, weights streamed from HBM. Writes CSV rows for fitting plan_gemm."""
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
out = open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gemm_sweep.csv", "w")
out.write("M,N,K,epi,variant,splits,us\n")
Ms = [int(x) for x in os.environ.get("MS", "64,128,130,200,256,300,400,500,600,700,800,1000,1200,1600").split(",")]
for M in Ms:
    shapes = ((6144, 4096, 0), (4096, 4096, 2), (28672, 4096, 4), (4096, 14336, 2))
    if os.environ.get("SHAPES") == "70b":  # Llama-3-70B: QKV, O, FFN1 (gate+up), FFN2
        shapes = ((10240, 8192, 0), (8192, 8192, 2), (57344, 8192, 4), (8192, 28672, 2))
    for N, Kd, epi in shapes:
        nk = (Kd + 63) // 64
        for var in (0, 1, 2, 3, 5, 6):
            for sp in ((0,) if var in (0, 5, 6) else (1, 2, 3, 4, 6, 8)):
                if sp:
                    kb = (nk + sp - 1) // sp
                    if (nk + kb - 1) // kb != sp or (sp > 1 and M * N * sp * 4 > (256 << 20)):
                        continue
                    if var == 3 and M <= 128:
                        continue
                if var in (5, 6) and M > 128:
                    continue
                ms = C.c_float(0)
                rc = lib.krul_debug_gemm_bench(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), epi, var,
                                               sp, 30, C.byref(ms))
                if rc == 0:
                    out.write(f"{M},{N},{Kd},{epi},{var},{sp},{ms.value * 1e3:.2f}\n")
        out.flush()
    print("done M", M, flush=True)
