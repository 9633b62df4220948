#!/usr/bin/env python3
"""TTFT vs r_c (measured restore + new-input prefill), coded and raw store."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2507_08045_b200 import native as K  # noqa: E402

spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b-8k"]
L, n_new = spec["L"], spec["n_new"]
cfg = K.ModelConfig(n_layers=spec["n_layers"], n_heads=spec["n_heads"], n_kv_heads=spec["n_kv_heads"],
                    head_dim=spec["head_dim"], d_model=spec["d_model"], vocab_size=spec["vocab_size"],
                    ffn_mult=spec["ffn_mult"], ffn_kind=spec["ffn_kind"], rope_theta=spec["rope_theta"],
                    seed=1234, dtype=K.KRUL_BF16, max_tokens=L + n_new + 64)
ctx = K.Context(cfg, 0)
ctx.init_weights(1234)
rng = np.random.default_rng(1000)
hist = rng.integers(0, cfg.vocab_size, L, dtype=np.int32)
new = rng.integers(0, cfg.vocab_size, n_new, dtype=np.int32)
prev = ctx.conversation(L + n_new + 64)
ctx.prefill(prev, hist)
conv = ctx.conversation(L + n_new + 64)
ctx.set_capture(False)
pairs = [(a, b, 0.0) for a, b in spec["pairs"]]
grid = [0.0, 0.004, 0.008, 0.012, 0.016, 0.02, 0.03, 0.04, 0.06, 0.08, 0.1]
for coding in (True, False):
    ctx.set_kv_coding(coding)
    r, tt = ctx.calibrate_rc_ttft(prev, conv, hist, new, pairs, grid, reps=5)
    print(f"coding={coding}: best r_c {r}: " + " ".join(f"{g}:{t:.3f}" for g, t in zip(grid, tt)), flush=True)
    for rc in (0.0, 0.02, 0.06):
        plan = K.build_plan(L, cfg.n_layers, rc, pairs)
        snap = K.KVSnapshot.compress(ctx, prev, pairs, plan, L, K.MERGE_MEAN)
        for _ in range(3):
            _, st, t = ctx.restore_and_prefill(conv, hist, snap, new)
        tl_c, tl_l, tl_n = ctx.restore_timeline()
        print(f"   rc={rc}: ttft {t:.3f} compute {st['compute_ms']:.2f} load {st['load_ms']:.2f} "
              f"h2d {st['h2d_ms']:.2f} ({st['h2d_bytes'] / 1e6:.0f} MB) last load {tl_l[-1]:.3f} "
              f"last new {tl_n[-1]:.3f}", flush=True)
