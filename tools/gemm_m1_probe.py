import ctypes as C, sys, os
sys.path.insert(0, '/root/repo')
from paper_2507_08045_b200 import native as K
M = int(sys.argv[1])
cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4, dtype=K.KRUL_BF16, max_tokens=64)
ctx = K.Context(cfg, 0)
ms = C.c_float()
print(K.lib().krul_debug_gemm_bench(ctx.h, C.c_int64(M), C.c_int64(28672), C.c_int64(4096), 4, 1, 1, 5, C.byref(ms)), ms.value)
