#!/usr/bin/env python3
"""Isolate the bimodal recompute time: recompute alone, restore alone, restore+prefill."""
import os
import sys
import time

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
    plan = K.build_plan(L, cfg.n_layers, 0.06, pairs)
    snap = K.KVSnapshot.compress(ctx, prev, pairs, plan, L, K.MERGE_MEAN)
    t = []
    for i in range(8):
        t0 = time.perf_counter()
        ctx.partial_prefix_recompute(conv, hist, plan)
        t.append(round((time.perf_counter() - t0) * 1e3, 2))
    print("partial_recompute wall ms:", t, flush=True)
    t = []
    for i in range(5):
        st = ctx.execute_restore(conv, hist, snap)
        t.append((round(st["compute_ms"], 2), round(st["load_ms"], 2)))
        tc, tl, _ = ctx.restore_timeline()
        print(f"run {i}: compute per layer", [round(float(x), 2) for x in tc[::4]], flush=True)
    print("restore (compute, load):", t, flush=True)
    t = []
    for i in range(8):
        _, st, ttft = ctx.restore_and_prefill(conv, hist, snap, new)
        t.append((round(ttft, 2), round(st["compute_ms"], 2), round(st["load_ms"], 2)))
        tc, tl, tn = ctx.restore_timeline()
        print(f"rp run {i}: compute", [round(float(x), 2) for x in tc[::4]], "new", [round(float(x), 2) for x in tn[::4]], flush=True)
    print("restore+prefill:", t, flush=True)
    t = []
    for i in range(8):
        t0 = time.perf_counter()
        ctx.partial_prefix_recompute(conv, hist, plan)
        t.append(round((time.perf_counter() - t0) * 1e3, 2))
    print("partial_recompute wall ms:", t, flush=True)


if __name__ == "__main__":
    main()
