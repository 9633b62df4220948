#!/usr/bin/env python3
"""Attention tuning sweep: new-input-prefill shape (128 rows over 8K) and a
recompute shape (1024 causal rows) on the Llama-3-8B layout."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402


def main():
    cfg = K.ModelConfig(n_layers=2, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096,
                        vocab_size=1024, ffn_mult=3.5, ffn_kind=1, rope_theta=5e5, seed=1,
                        dtype=K.KRUL_BF16, max_tokens=8192 + 256)
    ctx = K.Context(cfg, 0)
    ctx.init_weights(1)
    conv = ctx.conversation(8192 + 256)
    toks = np.random.default_rng(0).integers(0, 1024, 8192 + 128, dtype=np.int32)
    ctx.prefill(conv, toks)
    lib = K.lib()
    for rows, pos0, name in ((128, 8192, "new-prefill 128x8320"), (1024, 0, "recompute 1024 causal")):
        vis = rows * pos0 + rows * (rows + 1) / 2
        fl = 4 * 128 * 32 * vis
        for dbg in [int(x) for x in os.environ.get("DBG", "0").split(",")]:
            for target in (0, 8, 16, 32):
                ms = C.c_float()
                rc = lib.krul_debug_attn_bench(ctx.h, conv.h, 0, C.c_int64(rows), C.c_int64(pos0),
                                               dbg, target, 20, C.byref(ms))
                assert rc == 0, rc
                print(f"{name} dbg={dbg} target={target}: {ms.value * 1e3:.1f} us "
                      f"{fl / (ms.value * 1e-3) / 1e12:.0f} TF/s", flush=True)


if __name__ == "__main__":
    main()
