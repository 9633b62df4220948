#!/usr/bin/env python3
"""TTFT of the restore DAG with/without CUDA-graph replay and kernel timing."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2507_08045_b200 import native as K  # noqa: E402


def main():
    spec = CONFIGS["llama3-8b-8k"]
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
    conv = ctx.conversation(L + n_new + 64)
    for rc in (0.068,):
        plan = K.build_plan(L, cfg.n_layers, rc, pairs)
        snap = K.KVSnapshot.compress(ctx, prev, pairs, plan, L, K.MERGE_MEAN)
        for kt in (False, True):
            ctx.ktime_enable(kt)
            t = []
            for i in range(8):
                _, st, ttft = ctx.restore_and_prefill(conv, hist, snap, new)
                t.append((round(ttft, 2), round(st["compute_ms"], 2), round(st["load_ms"], 2)))
            print(f"rc={rc} graphs={os.environ.get('KRUL_GRAPHS', '1')} ktime={kt}:", t, flush=True)
        ctx.ktime_enable(False)


if __name__ == "__main__":
    main()
