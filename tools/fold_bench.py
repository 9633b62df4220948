#!/usr/bin/env python3
"""Estimator decode-fold kernel in isolation (ncu target): 32 tracked layers,
32 heads, width 8328 (the Llama-3-8B 8K decode step)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402

N, H, W = 32, 32, 8328
cfg = K.ModelConfig(n_layers=N, n_heads=H, head_dim=4, d_model=4 * H, vocab_size=8,
                    dtype=K.KRUL_F32, max_tokens=64)
ctx = K.Context(cfg, 0)
rows = np.random.default_rng(0).dirichlet(np.ones(W), (N, H)).astype(np.float32)
est = K.StreamingEstimator(ctx, list(range(N)))
for _ in range(3):
    est.fold_decode_rows(rows)
print("sums[0:4]", est.sums()[:4])
