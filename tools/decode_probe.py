#!/usr/bin/env python3
"""One decode step at the bench shape inside cuProfilerStart/Stop (ncu launch list)."""
import ctypes
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2507_08045_b200 import native as K  # noqa: E402

spec = CONFIGS["llama3-8b-8k"]
L = int(sys.argv[1]) if len(sys.argv) > 1 else spec["L"]
cfg = K.ModelConfig(n_layers=spec["n_layers"], n_heads=spec["n_heads"], n_kv_heads=spec["n_kv_heads"],
                    head_dim=spec["head_dim"], d_model=spec["d_model"], vocab_size=spec["vocab_size"],
                    ffn_mult=spec["ffn_mult"], ffn_kind=spec["ffn_kind"], rope_theta=spec["rope_theta"],
                    seed=1234, dtype=K.KRUL_BF16, max_tokens=L + 64)
ctx = K.Context(cfg, 0)
ctx.init_weights(1234)
hist = np.random.default_rng(1).integers(0, cfg.vocab_size, L, dtype=np.int32)
conv = ctx.conversation(L + 64)
ctx.prefill(conv, hist)
for _ in range(3):
    ctx.decode_step(conv, 5)
t0 = time.perf_counter()
for _ in range(5):
    ctx.decode_step(conv, 5)
print(f"decode step {1e3 * (time.perf_counter() - t0) / 5:.3f} ms at W={len(conv)}", flush=True)
cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuProfilerStart()
ctx.decode_step(conv, 5)
ctx.sync()
cuda.cuProfilerStop()
