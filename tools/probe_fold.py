import sys, numpy as np
sys.path.insert(0, '.')
from paper_2507_08045_b200 import native as K
for n, H, W in [(64, 2, 515), (72, 2, 515), (80, 2, 515), (80, 2, 64), (40, 2, 515)]:
    cfg = K.ModelConfig(n_layers=n, n_heads=H, head_dim=4, d_model=4 * H, vocab_size=5, dtype=K.KRUL_F32, max_tokens=64)
    ctx = K.Context(cfg, 0)
    est = K.StreamingEstimator(ctx, list(range(n)))
    rows = np.random.default_rng(0).dirichlet(np.ones(W), (n, H)).astype(np.float32)
    try:
        est.fold_decode_rows(rows); print(n, H, W, "ok")
    except Exception as e:
        print(n, H, W, "ERR", e)
