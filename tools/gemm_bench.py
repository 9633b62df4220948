#!/usr/bin/env python3
"""GEMM tuning sweep on the device (krul_debug_gemm_bench): shapes of the
Llama-3-8B recompute/new-input layers x kernel variants x epilogues."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402

VAR = {0: "auto", 1: "1sm256", 2: "1sm128", 3: "pair", 4: "pairBK128"}
EPI = {0: "f32", 2: "resid", 4: "swiglu", 5: "none", 6: "stage", 7: "direct"}


def main():
    cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4,
                        dtype=K.KRUL_BF16, max_tokens=64)
    ctx = K.Context(cfg, 0)
    lib = K.lib()
    if len(sys.argv) > 1 and sys.argv[1] == "epi":
        for M, N, Kd in ((983, 6144, 4096), (4096, 4096, 4096)):
            for var in (1, 3):
                for e in (5, 6, 7, 0):
                    ms = C.c_float(0)
                    lib.krul_debug_gemm_bench(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd),
                                              e, var, 0, 10, C.byref(ms))
                    print(M, N, Kd, VAR[var], EPI[e], round(ms.value * 1e3, 1), "us", flush=True)
        return
    shapes = [(983, 6144, 4096, 0), (951, 4096, 4096, 2), (951, 28672, 4096, 4),
              (951, 4096, 14336, 2), (128, 6144, 4096, 0), (128, 28672, 4096, 4),
              (128, 4096, 14336, 2), (4096, 4096, 4096, 5), (8192, 8192, 8192, 5)]
    out = []
    for M, N, Kd, epi in shapes:
        for var in (0, 1, 2, 3, 4):
            for e in ((epi, 5) if epi != 5 else (5,)):
                ms = C.c_float(0)
                rc = lib.krul_debug_gemm_bench(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd),
                                               e, var, 0, 10, C.byref(ms))
                if rc != 0:
                    print("err", M, N, Kd, var, e, K.last_error() if hasattr(K, "last_error") else rc)
                    continue
                tf = 2.0 * M * N * Kd / (ms.value * 1e-3) / 1e12
                r = dict(M=M, N=N, K=Kd, variant=VAR[var], epi=EPI[e], us=round(ms.value * 1e3, 1),
                         tflops=round(tf, 1))
                out.append(r)
                print(json.dumps(r), flush=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "gemm_bench.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
