#!/usr/bin/env python3
"""One restore + new-input prefill step inside a cuProfilerStart/Stop range,
for `ncu --profile-from-start off` (launch lists and per-kernel captures).

Same workload as bench.py (Llama-3-8B shape, 8K history) but with a fixed
recompute ratio so no calibration launches pollute the capture.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402
from paper_2507_08045_b200 import native as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama3-8b-8k")
    ap.add_argument("--rc", type=float, default=0.0)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    spec = CONFIGS[args.config]
    L, n_new = spec["L"], spec["n_new"]
    cfg = K.ModelConfig(n_layers=spec["n_layers"], n_heads=spec["n_heads"],
                        n_kv_heads=spec["n_kv_heads"], head_dim=spec["head_dim"],
                        d_model=spec["d_model"], vocab_size=spec["vocab_size"],
                        ffn_mult=spec["ffn_mult"], ffn_kind=spec["ffn_kind"],
                        rope_theta=spec["rope_theta"], seed=1234, dtype=K.KRUL_BF16,
                        max_tokens=L + n_new + 64)
    ctx = K.Context(cfg, 0)
    ctx.init_weights(1234)
    rng = np.random.default_rng(1000)
    hist = rng.integers(0, cfg.vocab_size, L, dtype=np.int32)
    new = rng.integers(0, cfg.vocab_size, n_new, dtype=np.int32)
    prev = ctx.conversation(L + n_new + 64)
    ctx.prefill(prev, hist)
    pairs = [(a, b, 0.0) for a, b in spec["pairs"]]
    plan = K.build_plan(L, cfg.n_layers, args.rc, pairs)
    snap = K.KVSnapshot.compress(ctx, prev, pairs, plan, L, K.MERGE_MEAN)
    conv = ctx.conversation(L + n_new + 64)
    ctx.set_capture(False)
    for _ in range(2):
        ctx.restore_and_prefill(conv, hist, snap, new)
    ctx.sync()
    cuda = ctypes.CDLL("libcuda.so.1")
    cuda.cuProfilerStart()
    for _ in range(args.steps):
        _, st, ttft = ctx.restore_and_prefill(conv, hist, snap, new)
    ctx.sync()
    cuda.cuProfilerStop()
    print(f"ttft_ms={ttft:.3f} stats={st}")


if __name__ == "__main__":
    main()
