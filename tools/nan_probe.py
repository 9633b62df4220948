#!/usr/bin/env python3
"""Per-layer finiteness / magnitude of the prefill KV at the bench shape."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2507_08045_b200 import native as K  # noqa: E402

spec = CONFIGS["llama3-8b-8k"]
for L in [int(x) for x in (sys.argv[1:] or ["8192"])]:
    cfg = K.ModelConfig(n_layers=spec["n_layers"], n_heads=spec["n_heads"], n_kv_heads=spec["n_kv_heads"],
                        head_dim=spec["head_dim"], d_model=spec["d_model"], vocab_size=spec["vocab_size"],
                        ffn_mult=spec["ffn_mult"], ffn_kind=spec["ffn_kind"], rope_theta=spec["rope_theta"],
                        seed=1234, dtype=K.KRUL_F32 if os.environ.get("F32") else K.KRUL_BF16, max_tokens=L + 256)
    ctx = K.Context(cfg, 0)
    ctx.init_weights(1234)
    if os.environ.get("HIDDEN"):
        pass
    rng = np.random.default_rng(1000)
    hist = rng.integers(0, cfg.vocab_size, L, dtype=np.int32)
    conv = ctx.conversation(L + 256)
    logits = ctx.prefill(conv, hist)
    print(f"L={L} logits finite={np.isfinite(logits).all()} max={np.nanmax(np.abs(logits)):.3g}", flush=True)
    for l in range(cfg.n_layers):
        k, v = conv.kv(l, 0, L)
        bad_k = (~np.isfinite(k)).sum()
        bad_v = (~np.isfinite(v)).sum()
        rows_bad = np.where(~np.isfinite(k).all(axis=(0, 2)))[0]
        print(f"  layer {l:2d}: nonfinite K {bad_k} V {bad_v} first bad row "
              f"{rows_bad[0] if len(rows_bad) else -1}  max|K| {np.nanmax(np.abs(k)):.3g} "
              f"max|V| {np.nanmax(np.abs(v)):.3g}", flush=True)
        if bad_k and l > 0 and not os.environ.get("ALL"):
            break
    del ctx
