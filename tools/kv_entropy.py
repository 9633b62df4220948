#!/usr/bin/env python3
"""Exponent statistics of the bf16 KV snapshot of the bench workload: how
compressible is the load stream losslessly (sign+mantissa raw, exponent coded)?"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2507_08045_b200 import native as K  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b-8k"
spec = CONFIGS[name]
L = spec["L"]
cfg = K.ModelConfig(n_layers=spec["n_layers"], n_heads=spec["n_heads"], n_kv_heads=spec["n_kv_heads"],
                    head_dim=spec["head_dim"], d_model=spec["d_model"], vocab_size=spec["vocab_size"],
                    ffn_mult=spec["ffn_mult"], ffn_kind=spec["ffn_kind"], rope_theta=spec["rope_theta"],
                    seed=1234, dtype=K.KRUL_BF16, max_tokens=L + 256)
ctx = K.Context(cfg, 0)
ctx.init_weights(1234)
rng = np.random.default_rng(1000)
hist = rng.integers(0, cfg.vocab_size, L, dtype=np.int32)
prev = ctx.conversation(L + 256)
ctx.prefill(prev, hist)
pairs = [(a, b, 0.0) for a, b in spec["pairs"]]
plan = K.build_plan(L, cfg.n_layers, 0.064, pairs)
snap = K.KVSnapshot.compress(ctx, prev, pairs, plan, L, K.MERGE_MEAN)


def H(c):
    p = c[c > 0] / c.sum()
    return float(-(p * np.log2(p)).sum())


tot = np.zeros(256, np.int64)
for b in range(snap.n_blobs()):
    o, sp, k, v = snap.blob(b)
    for name_, x in (("K", k), ("V", v)):
        bits = x.astype(np.float32).view(np.uint32) >> 16
        e = ((bits >> 7) & 0xFF).astype(np.int64)
        c = np.bincount(e.ravel(), minlength=256)
        tot += c
        if b in (0, snap.n_blobs() // 2, snap.n_blobs() - 1):
            top = np.argsort(-c)[:16]
            print(f"blob {b} owners {o} {name_}: H(exp) = {H(c):.3f} bits, top-15 cover "
                  f"{c[top[:15]].sum() / c.sum():.6f}, top-7 {c[top[:7]].sum() / c.sum():.4f}, "
                  f"range {e.min()}..{e.max()}", flush=True)
top = np.argsort(-tot)
print(f"ALL: H(exp) = {H(tot):.3f} bits -> bf16 {8 + H(tot):.2f} bits/elem "
      f"(ratio {(8 + H(tot)) / 16:.3f}); top-15 cover {tot[top[:15]].sum() / tot.sum():.7f}; "
      f"top-7 {tot[top[:7]].sum() / tot.sum():.5f}")
print("hist", {int(i): int(tot[i]) for i in top[:20]})
