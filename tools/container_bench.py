import sys, time, os
sys.path.insert(0, '.')
import numpy as np
from paper_2507_08045_b200 import native as K
from bench import CONFIGS, container_leg
spec = CONFIGS["llama3-8b-8k"]
L = spec["L"]
cfg = K.ModelConfig(n_layers=spec["n_layers"], n_heads=spec["n_heads"], n_kv_heads=spec["n_kv_heads"], head_dim=spec["head_dim"], d_model=spec["d_model"], vocab_size=spec["vocab_size"], ffn_mult=spec["ffn_mult"], ffn_kind=spec["ffn_kind"], rope_theta=spec["rope_theta"], seed=1234, dtype=K.KRUL_BF16, max_tokens=L + 256)
ctx = K.Context(cfg, 0); ctx.init_weights(1234)
rng = np.random.default_rng(1)
hist = rng.integers(0, cfg.vocab_size, L, dtype=np.int32)
prev = ctx.conversation(L + 256); ctx.prefill(prev, hist)
pairs = [(a, b, 0.0) for a, b in spec["pairs"]]
plan = K.build_plan(L, cfg.n_layers, 0.064, pairs)
snap = K.KVSnapshot.compress(ctx, prev, pairs, plan, L, K.MERGE_MEAN)
os.environ["KRUL_CONTAINER_PROFILE"] = "1"
print(container_leg(K, ctx, snap), flush=True)
t0=time.perf_counter(); snap.save_file("/tmp/x.krul"); t1=time.perf_counter()
b=K.KVSnapshot.load_file("/tmp/x.krul", ctx); t2=time.perf_counter()
print("file save %.1f ms load %.1f ms" % (1e3*(t1-t0), 1e3*(t2-t1)), flush=True)
