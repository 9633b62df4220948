#!/usr/bin/env python3
"""Host cost of an eager restore DAG enqueue (KRUL_GRAPHS=0) vs graph replay
on the configs[1] shape: wall clock of restore_and_prefill, device TTFT."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, model_kwargs  # noqa: E402
from paper_2507_08045_b200 import native as K  # noqa: E402

spec = CONFIGS["llama3-8b-8k"]
L, n_new = spec["L"], spec["n_new"]
cfg = K.ModelConfig(**model_kwargs(spec), seed=1234, dtype=K.KRUL_BF16, max_tokens=L + n_new + 64)
ctx = K.Context(cfg, 0)
ctx.init_weights(1234)
rng = np.random.default_rng(1)
hist = rng.integers(0, cfg.vocab_size, L, dtype=np.int32)
new = rng.integers(0, cfg.vocab_size, n_new, dtype=np.int32)
prev = ctx.conversation(L + n_new + 64)
ctx.prefill(prev, hist)
pairs = [(a, b, 0.0) for a, b in spec["pairs"]]
snap = K.KVSnapshot.compress(ctx, prev, pairs, K.build_plan(L, cfg.n_layers, 0.02, pairs), L, K.MERGE_MEAN)
conv = ctx.conversation(L + n_new + 64)
ctx.set_capture(False)
for i in range(6):
    t0 = time.perf_counter()
    _, st, ttft = ctx.restore_and_prefill(conv, hist, snap, new)
    w = (time.perf_counter() - t0) * 1e3
    print(f"call {i}: wall {w:.2f} ms, device TTFT {ttft:.3f} ms, launches so far {K.launch_count()}", flush=True)
