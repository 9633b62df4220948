#!/usr/bin/env python3
"""Phase timeline of one tcgen05 attention launch (krul_debug_attn_timeline)
on the Llama-3-8B layout: per phase, the min / median / max over CTAs in us
from the first CTA's entry. usage: attn_timeline.py [rows pos0 target]..."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402

NAMES = ["entry", "prologue done", "Q in (MMA)", "MMA loop done", "softmax done", "epilogue done", "exit"]


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
    args = [int(x) for x in sys.argv[1:]] or [128, 8192, 0, 1024, 0, 0]
    for i in range(0, len(args), 3):
        rows, pos0, target = args[i:i + 3]
        n = 8 * 4096 + 5 * 64 * 4
        ts = (C.c_ulonglong * n)()
        rc = lib.krul_debug_attn_timeline(ctx.h, conv.h, 0, C.c_int64(rows), C.c_int64(pos0), target, ts,
                                          C.c_int64(n))
        assert rc == 0, rc
        a = np.frombuffer(ts, dtype=np.uint64).reshape(-1, 8).astype(np.float64)
        a = a[a[:, 0] > 0]
        t0 = a[:, 0].min()
        print(f"rows={rows} pos0={pos0} target={target}: {len(a)} CTAs")
        for k, nm in enumerate(NAMES):
            col = a[:, k]
            col = col[col > 0]
            if col.size:
                d = (col - t0) / 1e3
                print(f"   {nm:16s} min {d.min():7.2f}  p50 {np.median(d):7.2f}  max {d.max():7.2f} us")
        tr = np.frombuffer(ts, dtype=np.uint64)[8 * 4096:].reshape(5, 64, 4).astype(np.int64)
        c0 = tr[tr > 0].min() if (tr > 0).any() else 0
        roles = ["softmaxA [start, S in, S loaded, P stored]", "softmaxB", "MMA [K in, S issued, V in, PV issued]",
                 "Kprod [start, slot free, issued]", "Vprod [start, slot free, issued]"]
        for r in range(5):
            print("  ", roles[r])
            for i in range(64):
                if tr[r, i].any():
                    print("     ", i, " ".join(f"{(x - c0) if x else -1:7d}" for x in tr[r, i]))


if __name__ == "__main__":
    main()
