"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.

Tolerances (stated per SURVEY.md §8c):
  * f32 parity mode: K/V and logits max-abs <= 1e-4, probabilities <= 1e-5,
    estimator prefill sums rel <= 1e-12, with decode folds rel <= 1e-6 (the
    reference rounds decode differences to f32), D rel <= 1e-6; pairs, plans and blob layouts
    bit-exact.
  * bf16 perf mode: per-layer relative Frobenius error <= 2e-2 vs the f32
    oracle on identical weights; the selector bit-exact on identical D.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2507_08045_b200 import native
    native.lib()
    return native


def make_pair(K, O, dtype, max_tokens=1024, **kw):
    base = dict(n_layers=3, n_heads=2, head_dim=4, d_model=8, vocab_size=17, ffn_mult=2.0, seed=5)
    base.update(kw)
    ocfg = O.ModelConfig(**base)
    om = O.Model(ocfg)
    cfg = K.ModelConfig(**base, dtype=dtype, max_tokens=max_tokens)
    ctx = K.Context(cfg, 0)
    ctx.upload_weights(om.weights())
    return ocfg, om, cfg, ctx


def rel_fro(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


# ----------------------------------------------------------------- GEMM unit

@pytest.mark.parametrize("M,N,Kd", [(1, 16, 8), (7, 40, 24), (128, 128, 64), (200, 300, 136),
                                    (256, 2048, 512), (513, 4096, 1024), (64, 6144, 4096),
                                    # split-K (weight streaming, M <= 128) and multi-wave
                                    # persistent shapes of the Llama-3-8B recompute
                                    (128, 4096, 14336), (3, 6144, 4096), (983, 6144, 4096),
                                    (1500, 1024, 2048)])
def test_gemm_bf16_tcgen05(K, oracle, M, N, Kd):
    from paper_2507_08045_b200.native import _p, lib
    import ctypes as C
    cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4,
                        dtype=K.KRUL_BF16, max_tokens=64)
    ctx = K.Context(cfg, 0)
    rng = np.random.default_rng(M * 7 + N)
    A = rng.uniform(-1, 1, (M, Kd)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, Kd)).astype(np.float32)
    Ab = A.astype(np.float32)
    # reference on bf16-rounded inputs
    def bf(x):
        u = x.view(np.uint32).astype(np.uint64)
        u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
        return u.astype(np.uint32).view(np.float32)
    ref = bf(Ab).astype(np.float64) @ bf(B).astype(np.float64).T
    out = np.zeros((M, N), np.float32)
    rc = lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A), _p(B),
                               None, 0, _p(out))
    assert rc == 0
    err = np.abs(out - ref).max() / max(np.abs(ref).max(), 1)
    assert err < 1e-4, err


@pytest.mark.parametrize("M,N,Kd", [(128, 1024, 4096), (300, 512, 256)])
def test_gemm_epilogues_bf16_splitk(K, M, N, Kd):
    """Fused epilogues through both the single-pass and the split-K reduce
    paths (M=128, K=4096 plans split-K; M=300, K=256 does not)."""
    from paper_2507_08045_b200.native import _p, lib
    import ctypes as C
    cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4,
                        dtype=K.KRUL_BF16, max_tokens=64)
    ctx = K.Context(cfg, 0)
    rng = np.random.default_rng(M + N)
    A = (rng.uniform(-.5, .5, (M, Kd)) / np.sqrt(Kd / 64)).astype(np.float32)
    B = rng.uniform(-.5, .5, (N, Kd)).astype(np.float32)
    bias = rng.uniform(-.5, .5, N).astype(np.float32)
    acc = A.astype(np.float64) @ B.astype(np.float64).T
    tol = 5e-2
    out = np.zeros((M, N), np.float32)
    assert lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A),
                                 _p(B), _p(bias), 3, _p(out)) == 0
    assert np.abs(out - np.tanh(acc + bias)).max() < tol
    out = np.zeros((M, N // 2), np.float32)
    assert lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A),
                                 _p(B), None, 4, _p(out)) == 0
    g, u = acc[:, 0::2], acc[:, 1::2]
    assert np.abs(out - g / (1 + np.exp(-g)) * u).max() < tol * max(1.0, np.abs(g * u).max())
    resid = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    out = resid.copy()
    assert lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A),
                                 _p(B), _p(bias), 2, _p(out)) == 0
    assert np.abs(out - (resid + acc + bias)).max() < tol


def test_gemm_epilogues_f32(K):
    from paper_2507_08045_b200.native import _p, lib
    import ctypes as C
    for dtype in (K.KRUL_F32, K.KRUL_BF16):
        cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4,
                            dtype=dtype, max_tokens=64)
        ctx = K.Context(cfg, 0)
        rng = np.random.default_rng(1)
        M, N, Kd = 130, 256, 64
        A = rng.uniform(-.5, .5, (M, Kd)).astype(np.float32)
        B = rng.uniform(-.5, .5, (N, Kd)).astype(np.float32)
        bias = rng.uniform(-.5, .5, N).astype(np.float32)
        acc = A.astype(np.float64) @ B.astype(np.float64).T
        tol = 1e-5 if dtype == K.KRUL_F32 else 3e-2
        out = np.zeros((M, N), np.float32)
        assert lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A),
                                     _p(B), _p(bias), 3, _p(out)) == 0
        assert np.abs(out - np.tanh(acc + bias)).max() < tol
        out = np.zeros((M, N // 2), np.float32)
        assert lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A),
                                     _p(B), None, 4, _p(out)) == 0
        g, u = acc[:, 0::2], acc[:, 1::2]
        assert np.abs(out - g / (1 + np.exp(-g)) * u).max() < tol
        resid = rng.uniform(-1, 1, (M, N)).astype(np.float32)
        out = resid.copy()
        assert lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A),
                                     _p(B), _p(bias), 2, _p(out)) == 0
        assert np.abs(out - (resid + acc + bias)).max() < tol


# ----------------------------------------------------------------- engine

@pytest.mark.parametrize("kw", [dict(), dict(head_dim=5, d_model=10),
                                dict(n_layers=4, n_heads=4, head_dim=64, d_model=256,
                                     vocab_size=256, ffn_mult=4.0, seed=7),
                                dict(n_layers=3, n_heads=4, n_kv_heads=2, head_dim=16, d_model=64,
                                     vocab_size=50, ffn_kind=1, rope_theta=500000.0)])
def test_prefill_f32_matches_oracle(K, oracle, kw):
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_F32, **kw)
    toks = oracle.tokens(40, 3, ocfg.vocab_size)
    ctx.set_capture(True)
    conv = ctx.conversation(128)
    logits = ctx.prefill(conv, toks)
    opf = om.prefill(toks)
    assert np.abs(logits - opf.logits()).max() < 1e-4
    assert np.abs(ctx.captured_prefill() - opf.attn_all()).max() < 1e-5
    okv = opf.take_kv()
    for l in range(ocfg.n_layers):
        k, v = conv.kv(l, 0, 40)
        ok, ov = okv.layer(l)
        assert np.abs(k - ok).max() < 1e-4 and np.abs(v - ov).max() < 1e-4


def test_decode_f32_matches_oracle(K, oracle):
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_F32, n_layers=4, n_heads=4, head_dim=64,
                                   d_model=256, vocab_size=256, ffn_mult=4.0, seed=7)
    toks = oracle.tokens(33, 4, 256)
    conv = ctx.conversation(128)
    ctx.prefill(conv, toks[:-1])
    okv = om.prefill(toks[:-1]).take_kv()
    for step in range(3):
        t = int(toks[-1]) if step == 0 else step
        lg = ctx.decode_step(conv, t)
        olg, orows = om.decode(okv, t)
        assert np.abs(lg - olg).max() < 1e-4
        assert np.abs(ctx.captured_decode() - orows).max() < 1e-5
    assert len(conv) == 35


def test_partial_recompute_f32(K, oracle):
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_F32)
    toks = oracle.tokens(16, 7, 17)
    conv = ctx.conversation(64)
    ctx.partial_prefix_recompute(conv, toks, [12, 9, 4])
    opk = om.partial(toks, [12, 9, 4])
    for l, p in enumerate([12, 9, 4]):
        k, v = conv.kv(l, 0, p)
        ok, ov = opk.layer(l)
        assert np.abs(k - ok).max() < 1e-5 and np.abs(v - ov).max() < 1e-5
    with pytest.raises(K.PlanInvalidError):
        ctx.partial_prefix_recompute(conv, toks, [4, 6, 2])
    with pytest.raises(K.PlanInvalidError):
        ctx.partial_prefix_recompute(conv, toks, [4, 2])


def test_prefill_bf16_close_to_oracle(K, oracle):
    kw = dict(n_layers=4, n_heads=4, head_dim=64, d_model=256, vocab_size=256, ffn_mult=4.0, seed=7)
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_BF16, **kw)
    toks = oracle.tokens(300, 3, 256)
    conv = ctx.conversation(512)
    ctx.set_capture(True)
    logits = ctx.prefill(conv, toks)
    opf = om.prefill(toks)
    assert rel_fro(logits, opf.logits()) < 2e-2
    okv = opf.take_kv()
    for l in range(4):
        k, v = conv.kv(l, 0, 300)
        ok, ov = okv.layer(l)
        assert rel_fro(k, ok) < 2e-2 and rel_fro(v, ov) < 2e-2


@pytest.mark.parametrize("hd,L,n_new,H,Hkv", [(64, 300, 0, 4, 2), (128, 700, 0, 4, 2),
                                                 (128, 1000, 70, 4, 2), (64, 2500, 128, 4, 2),
                                                 (64, 900, 40, 3, 3), (128, 1500, 128, 8, 2),
                                                 (128, 3900, 128, 4, 1)])
def test_tcgen05_attention_matches_simt(K, oracle, hd, L, n_new, H, Hkv):
    """bf16: the tcgen05 flash-attention path (capture off) against the SIMT
    path (capture on) on the same weights; also the new-input prefill with
    split-KV and the in-kernel classifier mass. Covers GQA head pairs sharing
    a KV head, MHA pairs with two KV heads and an odd head count."""
    kw = dict(n_layers=3, n_heads=H, n_kv_heads=Hkv, head_dim=hd, d_model=H * hd, vocab_size=256,
              ffn_mult=2.0, seed=3)
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_BF16, **kw)
    cfg.max_tokens = 4096
    ctx = K.Context(cfg, 0)
    ctx.upload_weights(om.weights())
    toks = oracle.tokens(L + max(n_new, 1), 5, 256)
    res = {}
    for cap in (True, False):
        ctx.set_capture(cap)
        conv = ctx.conversation(4096)
        lg = ctx.prefill(conv, toks[:L])
        if n_new:
            lg = ctx.prefill_new(conv, toks[L:L + n_new])
        avg, ir, _ = ctx.classify_layers(gamma=0.1)
        kv = [conv.kv(l, 0, L + n_new) for l in range(3)]
        res[cap] = (lg, avg, kv)
    assert rel_fro(res[False][0], res[True][0]) < 1e-2
    assert np.abs(res[False][1] - res[True][1]).max() < 2e-3
    for l in range(3):
        assert rel_fro(res[False][2][l][0], res[True][2][l][0]) < 1e-2


# ----------------------------------------------------------------- estimator

def test_estimator_folds_match_oracle(K, oracle):
    cfg = K.ModelConfig(n_layers=8, n_heads=3, head_dim=4, d_model=12, vocab_size=5,
                        dtype=K.KRUL_F32, max_tokens=64)
    ctx = K.Context(cfg, 0)
    rng = np.random.default_rng(0)
    N, H, s = 8, 3, 700
    tracked = [0, 2, 3, 5, 7]
    pre = rng.dirichlet(np.ones(s), (N, H, 20)).astype(np.float32)
    est = K.StreamingEstimator(ctx, tracked)
    acc = oracle.Accumulator(tracked, H)
    est.fold_prefill_rows(pre)
    acc.fold_prefill(pre)
    # prefill: the reference's expanded f64 form (analysis.hpp:37-50) up to
    # summation order
    got, want = est.sums(), acc.sums()
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert rel.max() < 1e-12, (rel.max(), int(rel.argmax()))
    for t in range(5):
        rows = rng.dirichlet(np.ones(s + t), (N, H)).astype(np.float32)
        est.fold_decode_rows(rows)
        acc.fold_decode(rows)
    # decode: the reference rounds each difference to f32 before squaring
    # (analysis.cpp:146-147); the Gram form is exact in f64 -> <= 2^-23 per term
    got, want = est.sums(), acc.sums()
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert rel.max() < 1e-6, (rel.max(), int(rel.argmax()), got[rel.argmax()], want[rel.argmax()])
    D, Do = est.finish(), acc.finalize()
    assert np.allclose(D, Do, rtol=1e-6, atol=1e-12)
    assert est.counts() == (20, 5)
    with pytest.raises(K.AccountingError):
        est.fold_prefill_rows(pre)
    e2 = K.StreamingEstimator(ctx, tracked)
    with pytest.raises(K.AccountingError):
        e2.finish()


@pytest.mark.parametrize("n,H,W", [(40, 5, 3001), (80, 2, 515), (12, 200, 64), (32, 32, 8328), (2, 1, 3)])
def test_estimator_decode_fold_shapes(K, oracle, n, H, W):
    """K1 decode fold layouts: > 32 tracked layers (several unit rounds per
    CTA), several heads per CTA, a CTA range crossing heads, row ends inside
    a 64-column block and inside a 16-byte unit, the Llama-3-8B 8K shape."""
    cfg = K.ModelConfig(n_layers=n, n_heads=H, head_dim=4, d_model=4 * H, vocab_size=5,
                        dtype=K.KRUL_F32, max_tokens=64)
    ctx = K.Context(cfg, 0)
    rng = np.random.default_rng(n + H)
    tracked = list(range(n))
    est = K.StreamingEstimator(ctx, tracked)
    acc = oracle.Accumulator(tracked, H)
    for t in range(2):
        rows = rng.dirichlet(np.ones(W + t), (n, H)).astype(np.float32)
        est.fold_decode_rows(rows)
        acc.fold_decode(rows)
    got, want = est.sums(), acc.sums()
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert rel.max() < 1e-6, (rel.max(), int(rel.argmax()), got[rel.argmax()], want[rel.argmax()])


@pytest.mark.parametrize("stride,W", [(3, 1000), (2, 8328), (5, 130)])
def test_estimator_sampled_token_subset(K, stride, W):
    """Opt-in sampled decode folds (not a parity mode): step t folds the
    64-column blocks b with b % stride == t % stride, each pair-head sum
    scaled by W / sampled columns. Checked against the same sampled sum in
    numpy (f32 difference, f64 square-sum), rel <= 1e-6."""
    n, H = 12, 4
    cfg = K.ModelConfig(n_layers=n, n_heads=H, head_dim=4, d_model=4 * H, vocab_size=5,
                        dtype=K.KRUL_F32, max_tokens=64)
    ctx = K.Context(cfg, 0)
    rng = np.random.default_rng(stride * 7 + W)
    est = K.StreamingEstimator(ctx, list(range(n)))
    est.set_sampling(stride)
    want = np.zeros((n * (n - 1) // 2, H))
    for t in range(stride + 1):
        w = W + t
        rows = rng.dirichlet(np.ones(w), (n, H)).astype(np.float32)
        est.fold_decode_rows(rows)
        blocks = [np.arange(b * 64, min(w, b * 64 + 64)) for b in range((w + 63) // 64) if b % stride == t % stride]
        if not blocks:  # this step's phase has no block in a row this short: nothing is folded
            continue
        cols = np.concatenate(blocks)
        scale = w / len(cols)
        p = 0
        for a in range(n):
            for b in range(a + 1, n):
                d = (rows[a][:, cols] - rows[b][:, cols]).astype(np.float64)  # f32 difference, widened
                want[p] += scale * (d * d).sum(axis=1)
                p += 1
    got = est.sums().reshape(-1, H)
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert rel.max() < 1e-6, rel.max()
    with pytest.raises(K.ConfigError):
        est.set_sampling(0)


def test_estimator_on_engine_capture(K, oracle):
    kw = dict(n_layers=4, n_heads=4, head_dim=64, d_model=256, vocab_size=256, ffn_mult=4.0, seed=7)
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_F32, **kw)
    toks = oracle.tokens(64, 9, 256)
    ctx.set_capture(True)
    conv = ctx.conversation(256)
    ctx.prefill(conv, toks)
    avg, ir, _ = ctx.classify_layers(gamma=0.1)
    opf = om.prefill(toks)
    oavg, oir = opf.classify(gamma=0.1)
    assert np.allclose(avg, oavg, atol=1e-6) and ir == oir
    est = K.StreamingEstimator(ctx, [0, 1, 2, 3])
    est.fold_prefill()
    acc = oracle.Accumulator([0, 1, 2, 3], 4)
    acc.fold_prefill_handle(opf)
    okv = opf.take_kv()
    for t in range(4):
        ctx.decode_step(conv, t + 1)
        est.fold_decode()
        _, rows = om.decode(okv, t + 1)
        acc.fold_decode(rows)
    assert np.allclose(est.finish(), acc.finalize(), rtol=1e-5, atol=1e-7)


# ----------------------------------------------------------------- selector

def test_selector_bit_exact(K, oracle):
    cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4,
                        dtype=K.KRUL_F32, max_tokens=16)
    ctx = K.Context(cfg, 0)
    D = np.array([[0, 3, 1, 4], [3, 0, 5, 2], [1, 5, 0, 6], [4, 2, 6, 0]], np.float64)
    s = K.select_strategy(ctx, D, [0, 1, 2, 3], [0, 1, 2, 3], 1.0, 4)
    assert s.pairs == [(0, 2, 1.0), (1, 3, 2.0)] and not s.exhausted_before_quota
    s = K.select_strategy(ctx, np.ones((6, 6)) - np.eye(6), range(6), range(6), 1.0, 6)
    assert s.pairs == [(0, 1, 1.0), (2, 3, 1.0), (4, 5, 1.0)]
    rng = np.random.default_rng(303)
    for trial in range(300):
        N = 2 + int(rng.integers(80))
        n_ir = int(rng.integers(0, min(N, 40) + 1))
        ir = sorted(rng.permutation(N)[:n_ir].tolist())
        D = np.zeros((n_ir, n_ir))
        iu = np.triu_indices(n_ir, 1)
        vals = rng.uniform(0, 2, len(iu[0]))
        if trial % 3 == 0:
            vals = np.round(vals, 1)  # ties
        D[iu] = vals
        D = D + D.T
        r_l = 0.25 * int(rng.integers(5))
        got = K.select_strategy(ctx, D, ir, list(rng.permutation(ir)) if ir else [], r_l, N)
        want = oracle.select_strategy(D, ir, ir, r_l, N)
        assert got.pairs == want.pairs and got.exhausted_before_quota == want.exhausted


# ----------------------------------------------------------------- kvstore + restore

def test_selector_golden_kats(K):
    """K3 on the device against the reference's hand-built selector KATs
    (tests/golden/kat.json <- test_strategy.cpp:89-134)."""
    import json
    import os
    kat = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kat.json")))["kat"]
    ctx = K.Context(K.ModelConfig(n_layers=6, n_heads=1, head_dim=4, d_model=4, vocab_size=4,
                                  dtype=K.KRUL_F32, max_tokens=16), 0)
    h = kat["select_hand"]
    s = K.select_strategy(ctx, np.array(h["D"], float), h["layers"], h["layers"], h["r_l"],
                          h["n_layers"])
    assert [list(p) for p in s.pairs] == h["pairs"] and s.exhausted_before_quota == h["exhausted"]
    t = kat["select_ties"]
    D = np.ones((t["n"], t["n"])) - np.eye(t["n"])
    s = K.select_strategy(ctx, D, list(range(t["n"])), list(range(t["n"])), t["r_l"], t["n"])
    assert [list(p) for p in s.pairs] == t["pairs"]


def test_snapshot_compress_matches_oracle(K, oracle):
    kw = dict(n_layers=4, n_heads=2, head_dim=4, d_model=8, vocab_size=13, seed=21)
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_F32, **kw)
    hist = oracle.tokens(70, 77, 13)
    conv = ctx.conversation(128)
    ctx.prefill(conv, hist)
    okv = om.prefill(hist).take_kv()
    pairs = [(1, 3, 0.25)]
    p = K.build_plan(70, 4, 0.4, pairs)
    for mode in (0, 1):
        snap = K.KVSnapshot.compress(ctx, conv, pairs, p, 70, mode)
        osnap = oracle.Snapshot(okv, ocfg, oracle.Strategy(pairs), p, 70, mode=mode)
        assert snap.n_blobs() == osnap.n_blobs()
        for b in range(snap.n_blobs()):
            o1, s1, k1, v1 = snap.blob(b)
            o2, s2, k2, v2 = osnap.blob(b)
            assert o1 == o2 and tuple(s1) == tuple(s2)
            assert np.abs(k1 - k2).max() < 1e-5 and np.abs(v1 - v2).max() < 1e-5
        assert snap.storage_report() == osnap.storage()
        for l in range(4):
            (a, e), k, v = snap.expand(l)
            (a2, e2), k2, v2 = osnap.expand(l)
            assert (a, e) == (a2, e2) and np.abs(k - k2).max() < 1e-5
        with pytest.raises(K.RestorationGapError):
            snap.expand(4)


@pytest.mark.parametrize("r_c", [0.0, 0.25, 0.5, 0.75, 1.0])
def test_lossless_restore(K, oracle, r_c):  # test_scheduler.cpp:353-400
    kw = dict(n_layers=4, n_heads=2, head_dim=4, d_model=8, vocab_size=13, seed=21)
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_F32, **kw)
    hist = oracle.tokens(24, 77, 13)
    conv = ctx.conversation(64)
    ctx.prefill(conv, hist)
    p = K.build_plan(24, 4, r_c)
    snap = K.KVSnapshot.compress(ctx, conv, [], p, 24, K.MERGE_KEEP_DEEPER)
    conv2 = ctx.conversation(64)
    st = ctx.execute_restore(conv2, hist, snap)
    for l in range(4):
        k1, v1 = conv.kv(l, 0, 24)
        k2, v2 = conv2.kv(l, 0, 24)
        assert np.abs(k1 - k2).max() < 1e-6 and np.abs(v1 - v2).max() < 1e-6
    a = ctx.decode_step(conv2, int(hist[-1]))
    b = ctx.decode_step(conv, int(hist[-1]))
    assert np.abs(a - b).max() < 1e-5
    assert st["restore_ms"] >= 0


def test_restore_and_prefill_matches_oracle(K, oracle):
    kw = dict(n_layers=4, n_heads=4, head_dim=64, d_model=256, vocab_size=256, ffn_mult=4.0, seed=7)
    for dtype, tol in ((K.KRUL_F32, 1e-4), (K.KRUL_BF16, None)):
        ocfg, om, cfg, ctx = make_pair(K, oracle, dtype, **kw)
        hist = oracle.tokens(512, 11, 256)
        new = oracle.tokens(64, 12, 256)
        conv = ctx.conversation(1024)
        ctx.prefill(conv, hist)
        pairs = [(1, 2, 0.5)]
        p = K.build_plan(512, 4, 0.3, pairs)
        snap = K.KVSnapshot.compress(ctx, conv, pairs, p, 512, K.MERGE_MEAN)
        conv2 = ctx.conversation(1024)
        logits, st, ttft = ctx.restore_and_prefill(conv2, hist, snap, new)
        okv = om.prefill(hist).take_kv()
        osnap = oracle.Snapshot(okv, ocfg, oracle.Strategy(pairs), p, 512, mode=0)
        rest = om.restore(hist, osnap)
        want = om.prefill(np.concatenate([hist, new]), preload=rest.suffix([0] * 4)).logits()
        if tol:
            assert np.abs(logits - want).max() < tol
        else:
            assert rel_fro(logits, want) < 3e-2
        assert ttft > 0 and len(conv2) == 576


def test_restore_graph_replay_is_exact(K, oracle, monkeypatch):
    """The restore DAG is run eagerly, then captured into a CUDA graph, then
    replayed: all three produce bit-identical logits and KV, also after an
    unrelated call grew the workspaces (the graph must be re-captured, not
    replayed with stale addresses) and after the plan changed."""
    kw = dict(n_layers=4, n_heads=4, n_kv_heads=2, head_dim=64, d_model=256, vocab_size=256,
              ffn_mult=3.5, ffn_kind=1, rope_theta=500000.0, seed=9)
    monkeypatch.setenv("KRUL_KV_POOL_CONVS", "3")
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_BF16, **kw)
    hist = oracle.tokens(700, 21, 256)
    new = oracle.tokens(48, 22, 256)
    prev = ctx.conversation(1024)
    ctx.prefill(prev, hist)
    pairs = [(1, 2, 0.0)]
    snap = K.KVSnapshot.compress(ctx, prev, pairs, K.build_plan(700, 4, 0.2, pairs), 700,
                                 K.MERGE_MEAN)
    conv = ctx.conversation(1024)
    runs = [ctx.restore_and_prefill(conv, hist, snap, new)[0] for _ in range(4)]
    kv0 = [conv.kv(l, 0, 748) for l in range(4)]
    for r in runs[1:]:
        assert np.array_equal(r, runs[0])
    big = ctx.conversation(1024)
    ctx.prefill(big, oracle.tokens(1000, 23, 256))  # grows the shared workspaces
    again = ctx.restore_and_prefill(conv, hist, snap, new)[0]
    again2 = ctx.restore_and_prefill(conv, hist, snap, new)[0]
    assert np.array_equal(again, runs[0]) and np.array_equal(again2, runs[0])
    for l in range(4):
        k, v = conv.kv(l, 0, 748)
        assert np.array_equal(k, kv0[l][0]) and np.array_equal(v, kv0[l][1])
    # a new plan on the same snapshot object invalidates the graph: a larger
    # r_c still covers its load spans (recompute more, load a suffix of each
    # stored blob), a smaller one does not
    snap.set_plan(K.build_plan(700, 4, 0.35, pairs))
    more = [ctx.restore_and_prefill(conv, hist, snap, new)[0] for _ in range(3)]
    assert np.array_equal(more[1], more[0]) and np.array_equal(more[2], more[0])
    assert not np.array_equal(more[0], runs[0])  # rows [p_l(0.2), p_l(0.35)) recomputed, not merged
    snap.set_plan(K.build_plan(700, 4, 0.1, pairs))
    with pytest.raises(K.RestorationGapError):
        ctx.restore_and_prefill(conv, hist, snap, new)


def test_restore_rejects_mismatch(K, oracle):  # test_scheduler.cpp:402-430
    kw = dict(n_layers=2, n_heads=1, head_dim=4, d_model=4, vocab_size=7)
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_F32, **kw)
    hist = np.array([1, 2, 3, 4, 5, 6], np.int32)
    conv = ctx.conversation(16)
    ctx.prefill(conv, hist)
    snap = K.KVSnapshot.compress(ctx, conv, [], K.build_plan(6, 2, 0.5), 6, 1)
    c2 = ctx.conversation(16)
    with pytest.raises(K.RestorationGapError):
        ctx.execute_restore(c2, np.append(hist, 1), snap)
    snap.set_plan([2, 1])
    with pytest.raises(K.RestorationGapError):
        ctx.execute_restore(c2, hist, snap)
    with pytest.raises(K.ConfigError):
        ctx.prefill(c2, np.array([0, 7], np.int32))


# ----------------------------------------------------------------- full-size properties

@pytest.mark.parametrize("pairs,mode", [([], 1), ([(1, 2, 0.0)], 0)])
def test_full_size_restore_properties(K, pairs, mode, monkeypatch):
    """Llama-3-8B layer shape (d=4096, 32/8 heads, hd=128, SwiGLU 14336,
    theta 5e5; 4 layers to bound the run) with an 8K history -- size-
    independent properties instead of an oracle run (the CPU restatement
    needs minutes per layer at this size):
      * loaded spans [p_l, L) are bit-identical to the previous turn's KV
        (keep-deeper, no pairs), or equal to the mean merge 0.5*(a+b) of the
        pair members (kvstore.cpp:302-307) rounded to bf16;
      * recomputed spans [0, p_l) match the previous turn's prefill (rel
        Frobenius <= 1e-2; different GEMM tilings / split-K order);
      * the restored conversation's next-token logits match a plain prefill
        of history + new input (rel <= 3e-2), repeated replays bit-stable."""
    L, n = 8192, 128
    monkeypatch.setenv("KRUL_KV_POOL_CONVS", "3")
    cfg = K.ModelConfig(n_layers=4, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096,
                        vocab_size=32000, ffn_mult=3.5, ffn_kind=1, rope_theta=500000.0, seed=3,
                        dtype=K.KRUL_BF16, max_tokens=L + n + 64)
    ctx = K.Context(cfg, 0)
    ctx.init_weights(3)
    rng = np.random.default_rng(5)
    hist = rng.integers(0, cfg.vocab_size, L, dtype=np.int32)
    new = rng.integers(0, cfg.vocab_size, n, dtype=np.int32)
    prev = ctx.conversation(L + n + 64)
    ctx.prefill(prev, hist)
    ref = [prev.kv(l, 0, L) for l in range(4)]
    plan = K.build_plan(L, 4, 0.1, pairs)
    snap = K.KVSnapshot.compress(ctx, prev, pairs, plan, L, mode)
    conv = ctx.conversation(L + n + 64)
    outs = [ctx.restore_and_prefill(conv, hist, snap, new)[0] for _ in range(3)]
    assert np.isfinite(outs[0]).all()
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    bf = lambda x: (x.astype(np.float32).view(np.uint32) + 0x7FFF +  # noqa: E731
                    ((x.astype(np.float32).view(np.uint32) >> 16) & 1)) >> 16 << 16
    for l in range(4):
        p = int(plan[l])
        k, v = conv.kv(l, 0, L)
        rk, rv = ref[l]
        owners = [pp for pp in pairs if l in pp[:2]]
        if owners:  # pair member: the stored blob is the mean over the shallow member's span
            a, b = owners[0][:2]
            ka, va = ref[a]
            kb, vb = ref[b]
            s = int(plan[a])
            want_k = bf(0.5 * (ka[:, s:] + kb[:, s:])).astype(np.uint32).view(np.float32)
            want_v = bf(0.5 * (va[:, s:] + vb[:, s:])).astype(np.uint32).view(np.float32)
            assert np.array_equal(k[:, max(p, s):], want_k[:, max(p, s) - s:])
            assert np.array_equal(v[:, max(p, s):], want_v[:, max(p, s) - s:])
        else:
            assert np.array_equal(k[:, p:], rk[:, p:]) and np.array_equal(v[:, p:], rv[:, p:])
        if p:
            assert rel_fro(k[:, :p], rk[:, :p]) < 1e-2 and rel_fro(v[:, :p], rv[:, :p]) < 1e-2
    full = ctx.conversation(L + n + 64)
    want = ctx.prefill(full, np.concatenate([hist, new]))
    if not pairs:
        assert rel_fro(outs[0], want) < 3e-2


def test_llama_depth_stays_finite(K, monkeypatch):
    """All 32 layers of the bench model (Llama-3-8B shape, random init): the
    residual stream must stay bounded with depth (the SwiGLU block runs on
    RMSNorm(h_mid), as Llama) -- every layer's K/V and the logits finite."""
    monkeypatch.setenv("KRUL_KV_POOL_CONVS", "1")
    L = 512
    cfg = K.ModelConfig(n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096,
                        vocab_size=128256, ffn_mult=3.5, ffn_kind=1, rope_theta=500000.0, seed=1234,
                        dtype=K.KRUL_BF16, max_tokens=L + 64)
    ctx = K.Context(cfg, 0)
    ctx.init_weights(1234)
    hist = np.random.default_rng(1000).integers(0, cfg.vocab_size, L, dtype=np.int32)
    conv = ctx.conversation(L + 64)
    logits = ctx.prefill(conv, hist)
    assert np.isfinite(logits).all()
    for l in range(32):
        k, v = conv.kv(l, 0, L)
        assert np.isfinite(k).all() and np.isfinite(v).all(), l
        assert 0 < np.abs(k).max() < 64 and 0 < np.abs(v).max() < 64, l


# ------------------------------------------------ KRUL v1 container (f3)
def test_container_matches_oracle_f32(K, oracle, tmp_path):
    """krul_snapshot_save / _load against oracle/container.py (kvstore.cpp:360-511):
    bit-exact bytes for the same f32 store, exact metadata for a device
    compress, and a loaded container restores like the oracle's restore."""
    from oracle import container as OC
    kw = dict(n_layers=4, n_heads=2, head_dim=4, d_model=8, vocab_size=13, seed=21)
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_F32, **kw)
    hist = oracle.tokens(70, 77, 13)
    conv = ctx.conversation(128)
    ctx.prefill(conv, hist)
    okv = om.prefill(hist).take_kv()
    pairs = [(1, 3, 0.25)]
    p = K.build_plan(70, 4, 0.4, pairs)
    cls = ([0, 1, 2, 3], [], [0.75, 0.5, 1.0 / 3.0, 1e-5])
    for mode in (0, 1):
        st = oracle.Strategy(pairs)
        osnap = oracle.Snapshot(okv, ocfg, st, p, 70, mode=mode)
        want = OC.from_oracle(osnap, ocfg, st, p, 70, mode, b"conv-7", cls)
        # the oracle's blobs in the device store -> identical container bytes
        blobs = [osnap.blob(b)[2:] for b in range(osnap.n_blobs())]
        s1 = K.KVSnapshot.from_blobs(ctx, pairs, p, 70, mode, blobs)
        s1.set_meta("conv-7", False, *cls)
        raw = s1.save()
        assert raw == OC.save(want)
        # device compress -> same metadata, payload within the f32 tolerance
        s2 = K.KVSnapshot.compress(ctx, conv, pairs, p, 70, mode)
        s2.set_meta("conv-7", False, *cls)
        got = OC.load(s2.save(), ocfg.hash())
        assert OC.meta_text(got) == OC.meta_text(want)
        for (o1, sp1, k1, v1), (o2, sp2, k2, v2) in zip(got.blobs, want.blobs):
            assert o1 == o2 and sp1 == sp2
            assert np.abs(k1 - k2).max() < 1e-5 and np.abs(v1 - v2).max() < 1e-5
        # load into the context (pinned f32 store) and restore
        s3 = K.KVSnapshot.load(raw, ctx, ocfg.hash())
        assert s3.save() == raw and s3.meta()["conversation_id"] == "conv-7"
        conv2 = ctx.conversation(128)
        ctx.execute_restore(conv2, hist, s3)
        rest = om.restore(hist, osnap)
        for l in range(4):
            k, v = conv2.kv(l, 0, 70)
            (a, e), ko, vo = rest.span(l), *rest.layer(l)
            assert (a, e) == (0, 70)
            assert np.abs(k - ko).max() < 1e-4 and np.abs(v - vo).max() < 1e-4
        # file path, config guard
        path = str(tmp_path / f"m{mode}.krul")
        s3.save_file(path)
        assert open(path, "rb").read() == raw
        with pytest.raises(K.SnapshotLoadError) as e:
            K.KVSnapshot.load_file(path, ctx, ocfg.hash() + 1)
        assert e.value.field == "config"
    # a host-only snapshot cannot feed the restore DAG
    host = K.KVSnapshot.load(raw)
    with pytest.raises(K.SnapshotError):
        ctx.execute_restore(ctx.conversation(128), hist, host)


def test_container_bf16_round_trip_restores_bit_exact(K, oracle, tmp_path, monkeypatch):
    """bf16 store -> f32 container (exact widening) -> bf16 store: the same bits,
    so the restore + new-input prefill from the reloaded snapshot gives the
    same logits bit for bit; a container from another config is rejected."""
    monkeypatch.setenv("KRUL_KV_POOL_CONVS", "6")
    kw = dict(n_layers=4, n_heads=4, head_dim=64, d_model=256, vocab_size=256, ffn_mult=4.0, seed=7)
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_BF16, **kw)
    hist = oracle.tokens(512, 11, 256)
    new = oracle.tokens(64, 12, 256)
    conv = ctx.conversation(1024)
    ctx.prefill(conv, hist)
    pairs = [(1, 2, 0.5)]
    p = K.build_plan(512, 4, 0.3, pairs)
    snap = K.KVSnapshot.compress(ctx, conv, pairs, p, 512, K.MERGE_MEAN)
    snap.set_meta("turn-3", True, [1, 2], [0, 3], [0.9, 0.8, 0.7, 0.2])
    path = str(tmp_path / "bf16.krul")
    snap.save_file(path)
    raw = open(path, "rb").read()
    assert raw == snap.save()
    back = K.KVSnapshot.load_file(path, ctx, ocfg.hash())
    assert back.save() == raw
    for b in range(snap.n_blobs()):
        assert snap.blob(b)[2].tobytes() == back.blob(b)[2].tobytes()
    ctx.set_capture(False)
    c1, c2 = ctx.conversation(1024), ctx.conversation(1024)
    l1, _, _ = ctx.restore_and_prefill(c1, hist, snap, new)
    l2, _, _ = ctx.restore_and_prefill(c2, hist, back, new)
    assert np.array_equal(l1, l2)
    # header says another model: restore refuses (scheduler.cpp:324)
    other = bytearray(raw)
    other[8:16] = (ocfg.hash() ^ 1).to_bytes(8, "little")
    from oracle import oracle as O
    other = bytes(other[:-4]) + O.crc32(bytes(other[:-4])).to_bytes(4, "little")
    alien = K.KVSnapshot.load(other, ctx)
    with pytest.raises(K.SnapshotError):
        ctx.restore_and_prefill(ctx.conversation(1024), hist, alien, new)


# ---------------------------------------------- exponent-coded KV store
@pytest.mark.parametrize("n", [1, 33, 64, 2048, 2049, 5 * 2048 + 1000, 1 << 22])
def test_kvcode_device_matches_host(K, n):
    """Device histogram + encode produce the host codec's image byte for byte;
    the device decoder restores every element."""
    import ctypes as C
    cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4,
                        dtype=K.KRUL_BF16, max_tokens=64)
    ctx = K.Context(cfg, 0)
    rng = np.random.default_rng(n)
    u = (rng.standard_normal(n) * 0.5).astype(np.float32).view(np.uint32)
    x = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    if n > 100:
        x[::97] = np.uint16(0x0001)  # denormal exponent 0 -> long codes
    lib = K.lib()
    nb = C.c_uint64()
    assert lib.krul_ec_host_roundtrip(K._p(x), C.c_uint64(n), None, C.c_uint64(0), C.byref(nb), None) == 0
    himg = np.zeros(nb.value, np.uint8)
    lib.krul_ec_host_roundtrip(K._p(x), C.c_uint64(n), K._p(himg), C.c_uint64(himg.size), C.byref(nb), None)
    dimg = np.zeros(nb.value + 64, np.uint8)
    dec = np.zeros(n, np.uint16)
    rc = lib.krul_debug_ec_device(ctx.h, K._p(x), C.c_uint64(n), K._p(dimg), C.c_uint64(dimg.size),
                                  C.byref(nb), K._p(dec))
    assert rc == 0 and nb.value == himg.size
    assert np.array_equal(dimg[:nb.value], himg)
    assert np.array_equal(dec, x)


@pytest.mark.parametrize("hd", [64, 128])
def test_coded_store_restores_bit_exact(K, oracle, monkeypatch, hd):
    """The coded store (H2D of the coded image + device decode) restores the
    same bits as the raw store: identical logits, KV, blob values and
    container bytes; the load stream moves fewer bytes. At hd = 128 the two
    arms share no kernel: the raw store goes through the TMA-staged k_expand
    (bulk copies in, bulk stores out; ragged head / tail pages on the
    vector path), the coded one through the fused k_ec_decode_expand."""
    monkeypatch.setenv("KRUL_KV_POOL_CONVS", "6")
    kw = dict(n_layers=4, n_heads=4, head_dim=hd, d_model=4 * hd, vocab_size=256, ffn_mult=4.0, seed=7)
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_BF16, **kw)
    hist = oracle.tokens(700, 11, 256)
    new = oracle.tokens(64, 12, 256)
    conv = ctx.conversation(1024)
    ctx.prefill(conv, hist)
    pairs = [(1, 2, 0.5)]
    p = K.build_plan(700, 4, 0.3, pairs)
    ctx.set_kv_coding(False)
    raw = K.KVSnapshot.compress(ctx, conv, pairs, p, 700, K.MERGE_MEAN)
    ctx.set_kv_coding(True)
    cod = K.KVSnapshot.compress(ctx, conv, pairs, p, 700, K.MERGE_MEAN)
    assert not raw.coding()["coded"] and cod.coding()["coded"]
    assert cod.coding()["ratio"] < 0.8
    for b in range(raw.n_blobs()):
        assert raw.blob(b)[2].tobytes() == cod.blob(b)[2].tobytes()
        assert raw.blob(b)[3].tobytes() == cod.blob(b)[3].tobytes()
    assert raw.save() == cod.save()
    ctx.set_capture(False)
    c1, c2 = ctx.conversation(1024), ctx.conversation(1024)
    for _ in range(3):  # eager, capture, graph replay
        l1, s1, _ = ctx.restore_and_prefill(c1, hist, raw, new)
        l2, s2, _ = ctx.restore_and_prefill(c2, hist, cod, new)
        assert np.array_equal(l1, l2)
        assert s2["h2d_bytes"] < s1["h2d_bytes"]
    for l in range(4):
        k1, v1 = c1.kv(l, 0, 764)
        k2, v2 = c2.kv(l, 0, 764)
        assert np.array_equal(k1, k2) and np.array_equal(v1, v2)
    # a raw store re-encoded later is the same code / image
    raw.encode()
    assert raw.coding() == cod.coding()


def test_expand_cta_capped_loop_bit_exact():
    """KRUL_EXPAND_CTAS caps the k_expand grid, so each CTA walks several
    page tiles through the TMA-staged path (the mbarrier phase flips per
    tile, shared memory reused behind the bulk stores). The cap is read once
    per process: the hd-128 raw-vs-coded test runs again in a child."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, KRUL_EXPAND_CTAS="8")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        f"{__file__}::test_coded_store_restores_bit_exact[128]"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "1 passed" in r.stdout


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_fused_recompute_matches_separate_stream(K, oracle, dtype, monkeypatch):
    """The fused DAG (recompute rows inside the new-input prefill's layer
    steps) restores the same KV and logits as the separate recompute stream:
    loaded spans bit-identical, recomputed spans and logits within the
    f32 / bf16 tolerances; both against the oracle's restore + prefill."""
    monkeypatch.setenv("KRUL_KV_POOL_CONVS", "6")
    kw = dict(n_layers=4, n_heads=4, head_dim=64, d_model=256, vocab_size=256, ffn_mult=4.0, seed=7)
    dt = K.KRUL_F32 if dtype == "f32" else K.KRUL_BF16
    ocfg, om, cfg, ctx = make_pair(K, oracle, dt, **kw)
    L = 517  # not page aligned: the segments share pages
    hist = oracle.tokens(L, 11, 256)
    new = oracle.tokens(48, 12, 256)
    conv = ctx.conversation(1024)
    ctx.prefill(conv, hist)
    pairs = [(1, 2, 0.5)]
    p = K.build_plan(L, 4, 0.35, pairs)
    assert p[0] > 0
    snap = K.KVSnapshot.compress(ctx, conv, pairs, p, L, K.MERGE_MEAN)
    ctx.set_capture(False)
    outs = {}
    for fused in (True, False):
        ctx.set_fused_recompute(fused)
        cv = ctx.conversation(1024)
        for _ in range(3):  # eager, capture, replay
            lg, st, _ = ctx.restore_and_prefill(cv, hist, snap, new)
        outs[fused] = (lg, [cv.kv(l, 0, L + 48) for l in range(4)])
    ctx.set_fused_recompute(True)
    (lf, kvf), (ls, kvs) = outs[True], outs[False]
    for l in range(4):
        a = int(p[l])
        assert np.array_equal(kvf[l][0][:, a:L], kvs[l][0][:, a:L])  # loaded suffix
        tol = 1e-4 if dtype == "f32" else None
        for x, y in ((kvf[l][0], kvs[l][0]), (kvf[l][1], kvs[l][1])):
            if tol:
                assert np.abs(x - y).max() < tol
            else:
                assert rel_fro(x, y) < 2e-2
    okv = om.prefill(hist).take_kv()
    osnap = oracle.Snapshot(okv, ocfg, oracle.Strategy(pairs), p, L, mode=0)
    want = om.prefill(np.concatenate([hist, new]), preload=om.restore(hist, osnap).suffix([0] * 4)).logits()
    if dtype == "f32":
        assert np.abs(lf - want).max() < 1e-4 and np.abs(ls - want).max() < 1e-4
    else:
        assert rel_fro(lf, want) < 3e-2 and rel_fro(lf, ls) < 2e-2


@pytest.mark.parametrize("force,sp", [(0, 0), (5, 0), (6, 0), (11, 2), (11, 4), (12, 2), (12, 3), (12, 4)])
@pytest.mark.parametrize("M,N,Kd", [(128, 4096, 4096), (77, 1536, 14336), (1, 6144, 4096), (128, 28672 // 8, 4096)])
def test_gemm_stream_k_epilogues(K, force, sp, M, N, Kd):
    """Weight-streaming shapes (M <= 128) through the stream-K schedule
    (every CTA streams T / G weight blocks, tiles split into pieces reduced in
    fixed order; force 5 / 6) and the cluster split-K (cs CTAs per tile, fp32
    partials reduced over DSMEM inside the GEMM; force 11, cs = sp) vs the
    auto plan, for the F32 / tanh / SwiGLU / residual epilogues;
    deterministic across calls."""
    from paper_2507_08045_b200.native import _p, lib
    import ctypes as C
    cfg = K.ModelConfig(n_layers=2, n_heads=1, head_dim=8, d_model=8, vocab_size=4,
                        dtype=K.KRUL_BF16, max_tokens=64)
    ctx = K.Context(cfg, 0)
    rng = np.random.default_rng(M + N + Kd)
    A = (rng.uniform(-.5, .5, (M, Kd)) / np.sqrt(Kd / 64)).astype(np.float32)
    B = rng.uniform(-.5, .5, (N, Kd)).astype(np.float32)
    bias = rng.uniform(-.5, .5, N).astype(np.float32)
    acc = A.astype(np.float64) @ B.astype(np.float64).T
    tol = 5e-2
    assert lib().krul_debug_set_gemm_plan(force, sp) == 0
    try:
        outs = []
        for _ in range(2):
            out = np.zeros((M, N), np.float32)
            assert lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A),
                                         _p(B), None, 0, _p(out)) == 0
            outs.append(out)
        assert np.array_equal(outs[0], outs[1])
        assert np.abs(outs[0] - acc).max() < tol * 0.2
        out = np.zeros((M, N), np.float32)
        assert lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A),
                                     _p(B), _p(bias), 3, _p(out)) == 0
        assert np.abs(out - np.tanh(acc + bias)).max() < tol
        out = np.zeros((M, N // 2), np.float32)
        assert lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A),
                                     _p(B), None, 4, _p(out)) == 0
        g, u = acc[:, 0::2], acc[:, 1::2]
        assert np.abs(out - g / (1 + np.exp(-g)) * u).max() < tol * max(1.0, np.abs(g * u).max())
        resid = rng.uniform(-1, 1, (M, N)).astype(np.float32)
        out = resid.copy()
        assert lib().krul_debug_gemm(ctx.h, C.c_int64(M), C.c_int64(N), C.c_int64(Kd), _p(A),
                                     _p(B), _p(bias), 2, _p(out)) == 0
        assert np.abs(out - (resid + acc + bias)).max() < tol
    finally:
        lib().krul_debug_set_gemm_plan(0, 0)


def _decode_run(K, oracle, L, steps):
    import os
    cfg = K.ModelConfig(n_layers=2, n_heads=8, n_kv_heads=2, head_dim=128, d_model=1024,
                        vocab_size=512, ffn_mult=3.5, ffn_kind=1, rope_theta=500000.0, seed=3,
                        dtype=K.KRUL_BF16, max_tokens=L + 64)
    ctx = K.Context(cfg, 0)
    ctx.init_weights(3)
    conv = ctx.conversation(L + 64)
    ctx.prefill(conv, oracle.tokens(L, 9, 512))
    out = []
    for t in range(steps):
        lg = ctx.decode_step(conv, 7 + t)
        out.append((lg, ctx.captured_decode().copy()))
    return out


def test_decode_attention_split_keys_matches_simt(K, oracle):
    """bf16 decode attention split over key chunks (k_attn_decode1/2) vs the
    per-(row, head) SIMT kernel: logits, captured probability rows (row sums
    1) over ragged widths (chunk tails, page tails) and 4 heads per KV head."""
    import os
    import subprocess
    import sys
    import json
    for L in (1, 63, 700, 2049):
        fast = _decode_run(K, oracle, L, 3)
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        code = ("import json,sys;sys.path[:0]=[%r,%r];from test_gpu_parity import _decode_run;"
                "from paper_2507_08045_b200 import native as K;from oracle import oracle as O;O.lib();"
                "r=_decode_run(K,O,%d,3);json.dump([[a.tolist(),b.tolist()] for a,b in r],sys.stdout)"
                % (root, os.path.join(root, "tests"), L))
        env = dict(os.environ, KRUL_DECODE_ATTN="simt")
        ref = json.loads(subprocess.check_output([sys.executable, "-c", code], env=env))
        for (lg, rows), (lr, rr) in zip(fast, ref):
            lr, rr = np.asarray(lr, np.float32), np.asarray(rr, np.float32)
            assert rel_fro(lg, lr) < 2e-2
            assert rows.shape == rr.shape
            assert np.abs(rows[0] - rr[0]).max() < 1e-5  # layer 0: identical inputs
            assert rel_fro(rows, rr) < 2e-2              # deeper: bf16 hidden-state drift
            np.testing.assert_allclose(rows.reshape(-1, rows.shape[-1]).sum(axis=-1), 1.0, atol=1e-4)


@pytest.mark.parametrize("L", [63, 700, 2049])
def test_decode_attention_split_keys_matches_oracle(K, oracle, L):
    """The bf16 split-key decode (k_attn_decode1/2, GQA 4 heads per KV head,
    hd 128, SwiGLU) against the oracle's decode_step (engine.cpp:406-446)
    directly: logits and every layer's captured probability row after the
    same prefill, three steps (bf16 tolerance rel-Fro <= 3e-2; rows sum to 1)."""
    kw = dict(n_layers=2, n_heads=8, n_kv_heads=2, head_dim=128, d_model=1024, vocab_size=512,
              ffn_mult=3.5, ffn_kind=1, rope_theta=500000.0, seed=3)
    ocfg, om, cfg, ctx = make_pair(K, oracle, K.KRUL_BF16, max_tokens=L + 16, **kw)
    toks = oracle.tokens(L, 9, 512)
    conv = ctx.conversation(L + 16)
    ctx.prefill(conv, toks)
    okv = om.prefill(toks).take_kv()
    for t in range(3):
        lg = ctx.decode_step(conv, 7 + t)
        rows = ctx.captured_decode()
        olg, orows = om.decode(okv, 7 + t)
        assert rel_fro(lg, olg) < 3e-2, (L, t)
        assert rows.shape == orows.shape, (rows.shape, orows.shape)
        assert rel_fro(rows, orows) < 3e-2, (L, t)
        np.testing.assert_allclose(rows.reshape(-1, rows.shape[-1]).sum(axis=-1), 1.0, atol=1e-4)


def test_calibrate_rc_measured_contract(K, oracle):
    """calibrate_rc_measured (scheduler.cpp:402-443) on the device and its
    TTFT variant: the result is a grid member and the argmin of the measured
    objective the call returns (|T_C - T_L| with the reference's strict `<`,
    ties -> the smaller ratio; median TTFT); the measured stream rates feed a
    cost model whose analytic calibration is also a grid member."""
    shape = dict(n_layers=4, n_heads=4, n_kv_heads=2, head_dim=128, d_model=512, vocab_size=512,
                 ffn_mult=3.5, ffn_kind=1, seed=3)
    cfg = K.ModelConfig(**shape, dtype=K.KRUL_BF16, max_tokens=1280)
    ctx = K.Context(cfg, 0)
    ctx.init_weights(3)
    L = 1024
    hist = np.random.default_rng(1).integers(0, cfg.vocab_size, L, dtype=np.int32)
    new = np.random.default_rng(2).integers(0, cfg.vocab_size, 32, dtype=np.int32)
    prev, scratch = ctx.conversation(1280), ctx.conversation(1280)
    ctx.prefill(prev, hist)
    grid = [0.0, 0.1, 0.25, 0.5, 1.0]
    pairs = [(1, 2, 0.0)]
    r, tc, tl = ctx.calibrate_rc_measured(prev, scratch, hist, pairs, grid)
    assert r in grid
    d = np.abs(tc - tl)
    best = 0
    for i in range(1, len(grid)):
        if d[i] < d[best]:
            best = i
    assert r == sorted(grid)[best]
    assert tc[0] == 0 or tc[0] < tc[-1]  # more recompute costs more compute time
    assert tl[-1] <= tl[0]               # and less load
    r2, tt = ctx.calibrate_rc_ttft(prev, scratch, hist, new, pairs, grid, reps=3)
    assert r2 in grid and r2 == sorted(grid)[int(np.argmin(tt))]
    assert np.all(tt > 0)
    b, f = ctx.measure_rates(scratch)
    assert b > 1e9 and f > 1e12
    cm = K.CostModel.for_model(cfg, f, b)
    assert K.calibrate_rc(cm, cfg.n_layers, L, cfg.d_model, pairs) in list(K.default_rc_grid())


@pytest.mark.parametrize("r_c,gemm_force", [(0.0, 0), (0.25, 0), (0.0, 11), (0.0, 12)])
def test_llama_width_restore_matches_oracle(K, oracle, r_c, gemm_force):
    """Production shape against the CPU oracle (not the repo's own SIMT
    path): 2 layers at full Llama-3-8B width (d=4096, GQA 32/8, hd=128,
    SwiGLU F=14336, rope theta 5e5), bf16 tcgen05 kernels throughout --
    history prefill, exponent-coded snapshot, the two-stream restore (the
    r_c=0.25 plan recomputes a 1024 / 0 prefix on the CTA-pair GEMM + FA
    attention while the rest loads), the 128-row new-input prefill
    (weight-streaming GEMMs + FA attention), then a decode step (split-key
    decode attention). Restored K/V, new-input logits, decode logits and the
    decode attention rows vs the oracle's f32 prefill / decode on the same
    weights: relative Frobenius <= 2e-2 (bf16 tolerance).
    gemm_force 11: every weight-streaming GEMM with a non-SwiGLU epilogue
    (the fused RoPE / page-scatter QKV, O and FFN2 residual epilogues) runs
    as cluster split-K with the DSMEM reduce."""
    from paper_2507_08045_b200.native import lib
    assert lib().krul_debug_set_gemm_plan(gemm_force, 0) == 0
    try:
        _llama_width_restore(K, oracle, r_c)
    finally:
        lib().krul_debug_set_gemm_plan(0, 0)


def _llama_width_restore(K, oracle, r_c):
    shape = dict(n_layers=2, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096, vocab_size=512,
                 ffn_mult=3.5, ffn_kind=1, rope_theta=500000.0, seed=21)
    om = oracle.Model(oracle.ModelConfig(**shape))
    cfg = K.ModelConfig(**shape, dtype=K.KRUL_BF16, max_tokens=2304)
    ctx = K.Context(cfg, 0)
    ctx.upload_weights(om.weights())
    L, n = 2048, 128
    hist = oracle.tokens(L, 31, cfg.vocab_size)
    new = oracle.tokens(n, 32, cfg.vocab_size)
    prev = ctx.conversation(2304)
    ctx.prefill(prev, hist)
    plan = K.build_plan(L, 2, r_c)
    snap = K.KVSnapshot.compress(ctx, prev, [], plan, L, K.MERGE_KEEP_DEEPER)
    assert snap.coding()["coded"]
    conv = ctx.conversation(2304)
    for _ in range(2):  # eager, then the captured graph
        logits, _, _ = ctx.restore_and_prefill(conv, hist, snap, new)
    ref = om.prefill(np.concatenate([hist, new]), capture=False)
    assert rel_fro(logits, ref.logits()) <= 2e-2, rel_fro(logits, ref.logits())
    okv = ref.take_kv()
    for l in range(2):
        gk, gv = conv.kv(l, 0, L + n)
        ok_, ov = okv.layer(l)
        ek, ev = rel_fro(gk, ok_), rel_fro(gv, ov)
        assert ek <= 2e-2 and ev <= 2e-2, (l, ek, ev)
    tok = 7
    dl = ctx.decode_step(conv, tok)
    rows = ctx.captured_decode()
    ol, orows = om.decode(okv, tok)
    assert rel_fro(dl, ol) <= 2e-2, rel_fro(dl, ol)
    assert rel_fro(rows, orows) <= 2e-2, rel_fro(rows, orows)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_prefill_fold_recompute_matches_record(K, oracle, dtype):
    """K2 without the attention record: fold_prefill over capture mode 2
    (Q + softmax statistics, probabilities recomputed per key chunk) equals
    the fold over the materialised record (mode 1) -- f32: the recomputed
    probabilities are bit-identical, sums rel <= 1e-6 (the two folds sum in
    different orders); bf16: mode 2 keeps the tcgen05 FA kernel, mode 1 runs
    the SIMT kernel that writes the record, so the sums agree to the bf16
    attention tolerance (2e-2). The f32 sums also match the oracle's
    SimilarityAccumulator::fold_prefill (analysis.cpp:97-122) on the same
    weights and tokens."""
    kw = dict(n_layers=4, n_heads=4, head_dim=64, d_model=256, vocab_size=256, ffn_mult=4.0, seed=7)
    if dtype == "bf16":
        kw.update(n_kv_heads=2, head_dim=128, d_model=512, ffn_kind=1, ffn_mult=3.5)
    om = oracle.Model(oracle.ModelConfig(**kw))
    cfg = K.ModelConfig(**kw, dtype=K.KRUL_F32 if dtype == "f32" else K.KRUL_BF16, max_tokens=640)
    ctx = K.Context(cfg, 0)
    ctx.upload_weights(om.weights())
    hist, new = oracle.tokens(320, 41, cfg.vocab_size), oracle.tokens(48, 42, cfg.vocab_size)
    sums = {}
    for mode in (1, 2):
        conv = ctx.conversation(640)
        ctx.set_capture(0)
        ctx.prefill(conv, hist)
        ctx.set_capture(mode)
        ctx.prefill_new(conv, new)
        ctx.set_capture(0)
        est = K.StreamingEstimator(ctx, list(range(cfg.n_layers)))
        est.fold_prefill()
        sums[mode] = est.sums()
        assert est.counts()[0] == 48
        del conv
    rel = np.abs(sums[2] - sums[1]) / np.maximum(np.abs(sums[1]), 1e-30)
    assert rel.max() <= (1e-6 if dtype == "f32" else 2e-2), rel.max()
    if dtype == "f32":
        pf = om.prefill(np.concatenate([hist, new]), preload=om.prefill(hist).take_kv().suffix([0] * 4))
        acc = oracle.Accumulator(list(range(4)), 4)
        acc.fold_prefill_handle(pf)
        want = acc.sums()
        rel = np.abs(sums[2] - want) / np.maximum(np.abs(want), 1e-30)
        assert rel.max() <= 1e-5, rel.max()
