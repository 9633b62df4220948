#!/usr/bin/env python3
"""Estimator decode-fold kernel in isolation (ncu target): 32 tracked layers,
32 heads, width 8328 (the Llama-3-8B 8K decode step)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08045_b200 import native as K  # noqa: E402

N, H, W = 32, 32, int(os.environ.get("FOLD_W", 8328))
cfg = K.ModelConfig(n_layers=N, n_heads=H, head_dim=4, d_model=4 * H, vocab_size=8,
                    dtype=K.KRUL_F32, max_tokens=64)
ctx = K.Context(cfg, 0)
if os.environ.get("FOLD_DATA") == "softmax":  # peaked rows with tiny (subnormal) tails, like decode attention
    z = np.random.default_rng(0).standard_normal((N, H, W)).astype(np.float32) * 12.0
    z = np.exp(z - z.max(axis=-1, keepdims=True))
    rows = (z / z.sum(axis=-1, keepdims=True)).astype(np.float32)
    print("subnormal fraction", float(np.mean((rows > 0) & (rows < np.finfo(np.float32).tiny))),
          "zero fraction", float(np.mean(rows == 0)))
else:
    rows = np.random.default_rng(0).dirichlet(np.ones(W), (N, H)).astype(np.float32)
est = K.StreamingEstimator(ctx, list(range(N)))
for _ in range(3):
    est.fold_decode_rows(rows)
print("sums[0:4]", est.sums()[:4])

if os.environ.get("FOLD_TIMELINE"):
    import ctypes as C
    lib = K.lib()
    n_ts = 256 * 8
    ts = np.zeros(n_ts, np.uint64)
    lib.krul_debug_fold_timeline(1, None, C.c_int64(n_ts))
    est.fold_decode_rows(rows)
    lib.krul_debug_fold_timeline(0, ts.ctypes.data_as(C.c_void_p), C.c_int64(n_ts))
    t = ts.reshape(256, 8).astype(np.int64)
    live = t[:, 0] > 0
    t0 = t[live, 0].min()
    r = t[live] - t0
    r[t[live] == 0] = -1
    print("ctas", int(live.sum()), "span us", (t[live].max() - t0) / 1e3)
    for k, name in enumerate(["entry", "setup", "loop"]):
        v = r[:, k][r[:, k] >= 0] / 1e3
        if len(v):
            print(f"{name:6s} min {v.min():7.2f} p50 {np.median(v):7.2f} max {v.max():7.2f}  (n={len(v)})")
    d = (r[:, 2] - r[:, 1])[r[:, 2] >= 0] / 1e3
    print("loop duration min/p50/max", d.min(), np.median(d), d.max())
    if os.environ.get("FOLD_TIMELINE") == "2":
        idx = np.nonzero(live)[0]
        for i in idx:
            if t[i, 2] > 0:
                print(f"cta {i:3d} sm {t[i, 7]:3d} start {(t[i, 1] - t0) / 1e3:6.2f} loop {(t[i, 2] - t[i, 1]) / 1e3:6.2f}"
                      " in " + " ".join(f"{(t[i, 3 + k] - t0) / 1e3:6.2f}" for k in range(4)) +
                      f" end {(t[i, 2] - t0) / 1e3:6.2f}")

if os.environ.get("FOLD_LOOP"):
    import ctypes as C
    ms = C.c_float()
    n_it = int(os.environ["FOLD_LOOP"])
    K.lib().krul_debug_fold_repeat(est.h, n_it, C.byref(ms))
    print(f"device ms/fold {ms.value:.5f}  ({N * H * W * 4 / ms.value / 1e6:.0f} GB/s)")
