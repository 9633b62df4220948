import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2507_08045_b200 import native as K
cfg = K.ModelConfig(n_layers=2, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096, vocab_size=1024, ffn_mult=3.5, ffn_kind=1, rope_theta=5e5, seed=1, dtype=K.KRUL_BF16, max_tokens=8192 + 256)
ctx = K.Context(cfg, 0); ctx.init_weights(1)
conv = ctx.conversation(8192 + 256)
ctx.prefill(conv, np.random.default_rng(0).integers(0, 1024, 8192 + 128, dtype=np.int32))
ms = C.c_float()
for dbg in (0, 2):
    print("dbg", dbg, flush=True)
    K.lib().krul_debug_attn_bench(ctx.h, conv.h, 0, C.c_int64(128), C.c_int64(8192), dbg, 64, 3, C.byref(ms))
    sys.stderr.flush()
