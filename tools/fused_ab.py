#!/usr/bin/env python3
"""A/B of the restore + prefill DAG modes (fused recompute vs separate
recompute stream) at a few r_c, coded store, graph-replayed steps."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2507_08045_b200 import native as K  # noqa: E402

spec = CONFIGS["llama3-8b-8k"]
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
rcs = [float(x) for x in (sys.argv[1:] or ["0.0", "0.02", "0.04"])]
snaps = {rc: K.KVSnapshot.compress(ctx, prev, pairs, K.build_plan(L, cfg.n_layers, rc, pairs), L, K.MERGE_MEAN)
         for rc in rcs}
for rep in range(2):
    for fused, tl in ((False, True), (True, True)):
        ctx.set_fused_recompute(fused)
        ctx.set_timeline(tl)
        for rc in rcs:
            tt = []
            for i in range(13):
                _, st, t = ctx.restore_and_prefill(conv, hist, snaps[rc], new)
                if i >= 3:
                    tt.append(t)
            tl_c, tl_l, tl_n = ctx.restore_timeline()
            print(f"rep {rep} fused={fused} timeline={tl} rc={rc}: ttft p50 {np.median(tt):.3f} min {min(tt):.3f} "
                  f"load {st['load_ms']:.2f} last load {tl_l[-1]:.3f} last new {tl_n[-1]:.3f} "
                  f"compute {st['compute_ms']:.2f}", flush=True)
