#!/usr/bin/env python3
"""Phase timeline of one weight-streaming GEMM launch (krul_debug_gemm_timeline):
CTA 0's phases and the spread of all CTAs' entry / exit, in us from the first
CTA's entry. usage: gemm_timeline.py [N K epi force splits]..."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402

NAMES = {0: "entry", 1: "prologue done", 2: "first stage full (MMA)", 3: "last MMA committed",
         4: "epilogue: accumulator ready", 5: "cluster: stash written", 6: "cluster: barrier 1 passed",
         7: "cluster: reduce+epilogue done", 8: "epilogue done", 9: "TMA stores complete"}
cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4, dtype=K.KRUL_BF16, max_tokens=64)
ctx = K.Context(cfg, 0)
lib = K.lib()
args = [int(x) for x in sys.argv[1:]] or [4096, 256, 2, 0, 0, 4096, 4096, 2, 0, 0, 6144, 4096, 0, 0, 0,
                                           28672, 4096, 4, 0, 0]
for i in range(0, len(args), 5):
    N, Kd, epi, force, sp = args[i:i + 5]
    ts = (C.c_ulonglong * 544)()
    rc = lib.krul_debug_gemm_timeline(ctx.h, C.c_int64(128), C.c_int64(N), C.c_int64(Kd), epi, force, sp, ts)
    assert rc == 0, rc
    ent = [ts[32 + b] for b in range(256) if ts[32 + b]]
    ext = [ts[288 + b] for b in range(256) if ts[288 + b]]
    t0 = min(ent)
    print(f"N={N} K={Kd} epi={epi} f{force}s{sp}: {len(ent)} CTAs, entry spread {(max(ent) - t0) / 1e3:.2f} us, "
          f"exit first {(min(ext) - t0) / 1e3:.2f} last {(max(ext) - t0) / 1e3:.2f} us")
    for k in range(10):
        if ts[k]:
            print(f"   {NAMES[k]:32s} {(ts[k] - t0) / 1e3:7.2f} us")
