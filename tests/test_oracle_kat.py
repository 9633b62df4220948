"""Pins the CPU oracle against the reference's own known-answer tests.

Each test re-expresses a reference test case (cited file:line under
/root/reference/proj/tests) against the oracle restatement. These are the
golden vectors SURVEY.md §8c lists; the oracle is trusted as the parity
checker for the CUDA path only because it passes them.
"""
import numpy as np
import pytest

# ---------------------------------------------------------------- common


def test_fnv1a64_known_vectors(oracle):  # test_common.cpp:23-29
    assert oracle.fnv1a64(b"") == 0xCBF29CE484222325
    assert oracle.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert oracle.fnv1a64(b"foobar") == 0x85944171F73967E8
    assert oracle.fnv1a64(b"bar", oracle.fnv1a64(b"foo")) == oracle.fnv1a64(b"foobar")


def test_crc32_known_vectors(oracle):  # test_common.cpp:31-35
    assert oracle.crc32(b"") == 0
    assert oracle.crc32(b"123456789") == 0xCBF43926
    assert oracle.crc32(b"456789", oracle.crc32(b"123")) == 0xCBF43926


def test_uniform_stream(oracle):  # test_common.cpp:37-61
    a = oracle.uniform(42, -2.0, 3.0, 1000)
    b = oracle.uniform(42, -2.0, 3.0, 1000)
    c = oracle.uniform(43, -2.0, 3.0, 1000)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)
    assert a.min() >= -2.0 and a.max() < 3.0
    d = oracle.uniform_index(7, 13, 200)
    assert d.max() < 13 and len(set(d.tolist())) > 6
    # mt19937_64 first output for the default seed 5489 is the standard
    # 14514284786278117030; the 24-bit mapping follows common.hpp:73-77.
    top = 14514284786278117030 >> 40
    assert oracle.uniform(5489, 0.0, 1.0, 1)[0] == np.float32(top) * np.float32(1.0 / 16777216.0)


# ---------------------------------------------------------------- engine

def tiny(seed=5):  # test_engine.cpp:13-23
    from oracle.oracle import ModelConfig
    return ModelConfig(n_layers=3, n_heads=2, head_dim=4, d_model=8, vocab_size=17, ffn_mult=2.0,
                       seed=seed)


def test_model_config_validation(oracle):  # test_engine.cpp:53-71
    cfg = tiny()
    cfg.validate()
    assert cfg.ffn_hidden() == 16
    for bad in (dict(d_model=9), dict(n_layers=1), dict(vocab_size=1), dict(ffn_mult=0.0)):
        c = tiny()
        for k, v in bad.items():
            setattr(c, k, v)
        with pytest.raises(oracle.OracleError) as e:
            c.validate()
        assert e.value.kind == "ConfigError"


def test_config_hash_covers_fields(oracle):  # test_engine.cpp:73-85
    base = tiny()
    for k, v in (("n_layers", 4), ("seed", 99), ("ffn_mult", 3.0)):
        c = tiny()
        setattr(c, k, v)
        assert c.hash() != base.hash()
    assert tiny().hash() == base.hash()


def test_model_build_deterministic(oracle):  # test_engine.cpp:87-99
    a = oracle.Model(tiny(5)).weights()
    b = oracle.Model(tiny(5)).weights()
    c = oracle.Model(tiny(6)).weights()
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert np.abs(a).max() <= 1.0 / np.sqrt(np.float32(8.0))


def test_prefill_causal_row_stochastic(oracle):  # test_engine.cpp:101-120
    m = oracle.Model(tiny())
    toks = oracle.tokens(12, 3, 17)
    pr = m.prefill(toks)
    probs = pr.attn_all()
    assert probs.shape == (3, 2, 12, 12)
    assert np.allclose(probs.sum(-1), 1.0, atol=1e-5)
    assert np.all(np.triu(probs, 1) == 0.0)
    again = m.prefill(toks)
    assert np.array_equal(pr.logits(), again.logits())


def test_prefill_input_validation(oracle):  # test_engine.cpp:122-127
    m = oracle.Model(tiny())
    for toks in ([], [0, 17], [-1]):
        with pytest.raises(oracle.OracleError) as e:
            m.prefill(np.array(toks, np.int32))
        assert e.value.kind == "ConfigError"


def test_decode_extends_prefill(oracle):  # test_engine.cpp:129-148
    m = oracle.Model(tiny())
    toks = oracle.tokens(10, 11, 17)
    part = m.prefill(toks[:-1])
    kv = part.take_kv()
    logits, rows = m.decode(kv, int(toks[-1]))
    full = m.prefill(toks)
    assert np.abs(logits - full.logits()).max() < 1e-5
    fkv = full.take_kv()
    for l in range(3):
        assert kv.span(l) == (0, 10)
        k1, v1 = fkv.layer(l)
        k2, v2 = kv.layer(l)
        assert np.abs(k1 - k2).max() < 1e-5 and np.abs(v1 - v2).max() < 1e-5
    assert rows.shape == (3, 2, 10)
    assert np.allclose(rows.sum(-1), 1.0, atol=1e-5)


def test_partial_recompute_matches_full(oracle):  # test_engine.cpp:165-193
    m = oracle.Model(tiny())
    toks = oracle.tokens(16, 7, 17)
    fkv = m.prefill(toks).take_kv()
    pk = m.partial(toks, [12, 9, 4])
    for l, p in enumerate([12, 9, 4]):
        assert pk.span(l) == (0, p)
        k1, v1 = fkv.layer(l)
        k2, v2 = pk.layer(l)
        assert np.abs(k1[:, :p] - k2).max() < 1e-5 and np.abs(v1[:, :p] - v2).max() < 1e-5


def test_partial_recompute_rejects_bad_plans(oracle):  # test_engine.cpp:195-223
    m = oracle.Model(tiny())
    toks = oracle.tokens(8, 1, 17)
    for p in ([4, 6, 2], [9, 4, 2], [4, 2]):
        with pytest.raises(oracle.OracleError) as e:
            m.partial(toks, p)
        assert e.value.kind in ("PlanInvalidError",)
    none = m.partial(toks, [0, 0, 0])
    assert all(none.span(l) == (0, 0) for l in range(3))


def test_prefill_over_preloaded_suffixes(oracle):  # test_engine.cpp:225-260
    m = oracle.Model(tiny())
    hist = 14
    toks = oracle.tokens(hist + 5, 9, 17)
    full = m.prefill(toks)
    base = m.prefill(toks[:hist]).take_kv()
    pre = base.suffix([10, 6, 0])
    sp = m.prefill(toks, preload=pre)
    assert np.abs(sp.logits() - full.logits()).max() < 1e-4
    probs = sp.attn_all()
    assert probs.shape == (3, 2, 5, hist + 5)
    skv, fkv = sp.take_kv(), full.take_kv()
    for l in range(3):
        assert skv.span(l) == (0, hist + 5)
        assert np.abs(skv.layer(l)[0] - fkv.layer(l)[0]).max() < 1e-4


def test_preload_gap_errors(oracle):  # test_engine.cpp:262-308
    m = oracle.Model(tiny())
    toks = oracle.tokens(12, 4, 17)
    base = m.prefill(toks[:8]).take_kv()
    with pytest.raises(oracle.OracleError) as e:
        m.prefill(toks, preload=base.suffix([4, 6, 0]))
    assert e.value.kind == "RestorationGapError"
    with pytest.raises(oracle.OracleError) as e:
        m.prefill(toks[:8], preload=base.suffix([4, 2, 0]))
    assert e.value.kind == "RestorationGapError"


def test_rotary_keys_depend_on_position(oracle):  # test_engine.cpp:310-319
    m = oracle.Model(tiny())
    k, v = m.prefill(np.array([5, 5], np.int32)).take_kv().layer(0)
    assert np.abs(v[0, 0] - v[0, 1]).max() < 1e-6
    assert np.abs(k[0, 0] - k[0, 1]).max() > 1e-4


def test_odd_head_dim(oracle):  # test_engine.cpp:321-329
    from oracle.oracle import ModelConfig
    cfg = ModelConfig(n_layers=3, n_heads=2, head_dim=5, d_model=10, vocab_size=17, ffn_mult=2.0,
                      seed=5)
    p = oracle.Model(cfg).prefill(oracle.tokens(6, 8, 17)).attn_all()
    assert np.allclose(p.sum(-1), 1.0, atol=1e-5)


# ---------------------------------------------------------------- analysis

def causal_uniform(s):
    m = np.zeros((s, s), np.float32)
    for r in range(s):
        m[r, : r + 1] = np.float32(1.0) / np.float32(r + 1)
    return m


def first_column(s):
    m = np.zeros((s, s), np.float32)
    m[:, 0] = 1.0
    return m


def random_causal(rows, width, first_q, seed):
    # acceptance.cpp:71-85 style (deterministic numpy stand-in for the stream)
    rng = np.random.default_rng(seed)
    m = np.zeros((rows, width), np.float32)
    for r in range(rows):
        vis = first_q + r + 1
        w = rng.uniform(0.01, 1.0, vis).astype(np.float32)
        m[r, :vis] = w / w.sum(dtype=np.float32)
    return m


def test_stable_distance_hand(oracle):  # test_analysis.cpp:72-82
    assert oracle.stable_sq([1, 0], [0, 1]) == pytest.approx(2.0, rel=1e-12)
    assert oracle.stable_sq([1, 0], [1, 0]) == pytest.approx(0.0)


def test_stable_distance_vs_direct(oracle):  # test_analysis.cpp:84-97, acceptance.cpp:189-206
    rng = np.random.default_rng(404)
    for _ in range(50):
        a = rng.uniform(-2, 2, 64).astype(np.float32)
        b = rng.uniform(-2, 2, 64).astype(np.float32)
        direct = float(((a.astype(np.float64) - b) ** 2).sum())
        s = oracle.stable_sq(a, b)
        assert abs(s - direct) <= 1e-5 * max(1.0, direct) and s >= 0.0


def test_classifier_separates_layers(oracle):  # test_analysis.cpp:99-113
    probs = np.stack([first_column(100)[None], causal_uniform(100)[None]])
    avg, ir = oracle.classify(probs)
    assert avg[0] == pytest.approx(1.0)
    assert 0.0 < avg[1] < 0.5
    assert ir == [0]


def test_classifier_noncausal_uniform(oracle):  # test_analysis.cpp:115-126
    u = np.full((100, 100), np.float32(1.0) / np.float32(100), np.float32)
    avg, ir = oracle.classify(np.stack([np.stack([u, u])]))
    assert avg[0] == pytest.approx(0.2, rel=1e-5)
    assert ir == []


def test_classifier_rejects_degenerate(oracle):  # test_analysis.cpp:128-145
    with pytest.raises(oracle.OracleError) as e:
        oracle.classify(causal_uniform(5)[None, None])
    assert e.value.kind == "ClassificationError"
    with pytest.raises(oracle.OracleError) as e:
        oracle.classify(causal_uniform(100)[None, None], gamma=0.0)
    assert e.value.kind == "ConfigError"
    with pytest.raises(oracle.OracleError) as e:
        oracle.classify(causal_uniform(100)[None, None], initial_frac=0.6, recent_frac=0.5)
    assert e.value.kind == "ConfigError"


def test_classifier_24_of_32_fixture(oracle):  # acceptance.cpp:576-613
    s, N = 100, 32
    diffuse = set(range(3, N, 4))
    layers = []
    for l in range(N):
        if l in diffuse:
            m = causal_uniform(s)
        else:
            m = np.zeros((s, s), np.float32)
            m[:, 0] += 0.7
            m[np.arange(s), np.arange(s)] += 0.3
        layers.append(m[None])
    avg, ir = oracle.classify(np.stack(layers))
    assert ir == [l for l in range(N) if l not in diffuse] and len(ir) == 24


def test_pairwise_distance_hand(oracle):  # test_analysis.cpp:164-178
    acc = oracle.Accumulator([0, 1], 1)
    acc.fold_prefill(np.stack([first_column(2)[None], causal_uniform(2)[None]]))
    D = acc.finalize()
    assert D[0, 1] == pytest.approx(np.sqrt(0.5), rel=1e-6)
    assert D[1, 0] == D[0, 1] and D[0, 0] == 0.0


def test_streaming_matches_batch(oracle):  # test_analysis.cpp:180-250, acceptance.cpp:98-185
    rng = np.random.default_rng(77)
    H, s, N, steps = 2, 24, 4, 6
    tracked = [0, 2, 3]
    for trial in range(10):
        pre = np.stack([np.stack([random_causal(s, s, 0, rng.integers(1 << 30)) for _ in range(H)])
                        for _ in range(N)])
        dec = [np.stack([np.stack([random_causal(1, s + t + 1, s + t, rng.integers(1 << 30))[0]
                                   for _ in range(H)]) for _ in range(N)]) for t in range(steps)]
        acc = oracle.Accumulator(tracked, H)
        acc.fold_prefill(pre)
        for d in dec:
            acc.fold_decode(d)
        D = acc.finalize()
        W = s + steps

        def row(l, r, h):
            out = np.zeros(W)
            if r < s:
                out[:s] = pre[l, h, r]
            else:
                x = dec[r - s][l, h]
                out[: len(x)] = x
            return out

        for a in range(3):
            for b in range(a + 1, 3):
                i, j = tracked[a], tracked[b]
                want = np.mean([np.sqrt(sum(((row(i, r, h) - row(j, r, h)) ** 2).sum()
                                            for r in range(s + steps))) for h in range(H)])
                assert abs(D[a, b] - want) <= 1e-6 * max(1.0, want)


def test_accumulator_protocol(oracle):  # test_analysis.cpp:252-275
    rec = np.stack([causal_uniform(10)[None], causal_uniform(10)[None]])
    acc = oracle.Accumulator([0, 1], 1)
    with pytest.raises(oracle.OracleError) as e:
        acc.finalize()
    assert e.value.kind == "AccountingError"
    acc.fold_prefill(rec)
    with pytest.raises(oracle.OracleError) as e:
        acc.fold_prefill(rec)
    assert e.value.kind == "AccountingError"
    acc.fold_decode(np.zeros((2, 1, 11), np.float32))
    with pytest.raises(oracle.OracleError) as e:
        acc.fold_decode(np.zeros((1, 1, 12), np.float32))
    assert e.value.kind == "StateCorruptionError"
    with pytest.raises(oracle.OracleError) as e:
        acc.fold_decode(np.zeros((2, 2, 12), np.float32))
    assert e.value.kind == "StateCorruptionError"
    other = oracle.Accumulator([0, 1], 1)
    with pytest.raises(oracle.OracleError) as e:
        other.fold_prefill(causal_uniform(4)[None, None])
    assert e.value.kind == "ConfigError"
    with pytest.raises(oracle.OracleError):
        oracle.Accumulator([0], 0)
    with pytest.raises(oracle.OracleError):
        oracle.Accumulator([-1, 0], 1)


# ---------------------------------------------------------------- strategy

def test_quota_table(oracle):  # test_strategy.cpp:75-87
    for n, r, q in ((32, .5, 16), (5, .5, 3), (5, 0, 0), (4, 1, 4), (10, .25, 3), (10, .2, 2),
                    (0, .5, 0)):
        assert oracle.quota(n, r) == q
    for n, r in ((-1, .5), (4, -.1), (4, 1.5)):
        with pytest.raises(oracle.OracleError) as e:
            oracle.quota(n, r)
        assert e.value.kind == "ConfigError"


def test_select_hand_matrix(oracle):  # test_strategy.cpp:89-110
    D = np.array([[0, 3, 1, 4], [3, 0, 5, 2], [1, 5, 0, 6], [4, 2, 6, 0]], np.float64)
    s = oracle.select_strategy(D, [0, 1, 2, 3], [0, 1, 2, 3], 1.0, 4)
    assert s.pairs == [(0, 2, 1.0), (1, 3, 2.0)] and not s.exhausted


def test_select_ties_lexicographic(oracle):  # test_strategy.cpp:123-134
    D = np.ones((6, 6)) - np.eye(6)
    s = oracle.select_strategy(D, list(range(6)), list(range(6)), 1.0, 6)
    assert s.pairs == [(0, 1, 1.0), (2, 3, 1.0), (4, 5, 1.0)]


def test_select_quota_zero_and_exhaustion(oracle):  # test_strategy.cpp:112-158
    D = np.ones((4, 4)) - np.eye(4)
    s = oracle.select_strategy(D, [0, 1, 2, 3], [0, 1, 2, 3], 0.0, 4)
    assert s.pairs == [] and not s.exhausted
    s1 = oracle.select_strategy(np.zeros((1, 1)), [3], [3], 0.5, 8)
    assert s1.pairs == [] and s1.exhausted
    s3 = oracle.select_strategy(np.ones((3, 3)) - np.eye(3), [0, 1, 2], [0, 1, 2], 0.5, 8)
    assert len(s3.pairs) == 1 and s3.exhausted
    s0 = oracle.select_strategy(np.zeros((0, 0)), [], [], 0.5, 8)
    assert s0.pairs == [] and s0.exhausted


def iterative_min(D, layers, quota_n):  # test_strategy.cpp:37-71
    layers = sorted(layers)
    pos = {l: i for i, l in enumerate(layers)}
    taken, pairs = set(), []
    while len(taken) < quota_n:
        best = None
        for a in range(len(layers)):
            for b in range(a + 1, len(layers)):
                i, j = layers[a], layers[b]
                if i in taken or j in taken:
                    continue
                key = (D[pos[i], pos[j]], i, j)
                if best is None or key < best:
                    best = key
        if best is None:
            return pairs, True
        pairs.append((best[1], best[2], best[0]))
        taken |= {best[1], best[2]}
    return pairs, False


def test_select_vs_iterative_min_oracle(oracle):  # test_strategy.cpp:160-195
    rng = np.random.default_rng(2024)
    for _ in range(200):
        n_layers = 8 + int(rng.integers(9))
        n_ir = 2 + int(rng.integers(5))
        ir = sorted(rng.permutation(n_layers)[:n_ir].tolist())
        D = np.zeros((n_ir, n_ir))
        for a in range(n_ir):
            for b in range(a + 1, n_ir):
                D[a, b] = D[b, a] = float(np.float32(rng.uniform(0, 4)))
        q = oracle.quota(n_layers, 0.5)
        got = oracle.select_strategy(D, ir, list(rng.permutation(ir)), 0.5, n_layers)
        want, exh = iterative_min(D, ir, q)
        assert got.pairs == want and got.exhausted == exh


# ---------------------------------------------------------------- kvstore

def coded_kv(oracle, N, H, hd, L):  # test_kvstore.cpp:17-39
    from oracle.oracle import ModelConfig
    cfg = ModelConfig(n_layers=N, n_heads=H, head_dim=hd, d_model=H * hd, vocab_size=11)
    layers = []
    for l in range(N):
        k = np.zeros((H, L, hd), np.float32)
        for h in range(H):
            for r in range(L):
                for c in range(hd):
                    k[h, r, c] = np.float32(1000 * l + 100 * h + r) + np.float32(c) * np.float32(0.01)
        layers.append((0, L, k, -k))
    return cfg, oracle.KV.from_host(cfg, layers), layers


def test_blob_layout_golden(oracle):  # test_kvstore.cpp:87-105
    st = oracle.Strategy([(0, 5, .1), (2, 3, .2)])
    specs = oracle.blob_specs(12, [12, 10, 8, 6, 4, 2], st)
    assert specs == [([0, 5], (2, 12)), ([1], (10, 12)), ([2, 3], (6, 12)), ([4], (4, 12))]
    assert oracle.blob_specs(12, [12, 3]) == [([0], (12, 12)), ([1], (3, 12))]
    for bad in ([(1, 7, .1)], [(0, 1, .1), (1, 2, .2)]):
        with pytest.raises(oracle.OracleError) as e:
            oracle.blob_specs(6, [4, 3, 2, 1], oracle.Strategy(bad))
        assert e.value.kind == "SnapshotError"


def test_keep_deeper_and_mean_merge(oracle):  # test_kvstore.cpp:115-167
    cfg, kv, raw = coded_kv(oracle, 4, 2, 3, 10)
    st = oracle.Strategy([(1, 3, .25)])
    keep = oracle.Snapshot(kv, cfg, st, [8, 6, 4, 2], 10, mode=1)
    assert keep.n_blobs() == 3
    owners, span, k, v = keep.blob(1)
    assert owners == [1, 3] and span == (2, 10)
    assert np.array_equal(k, raw[3][2][:, 2:]) and np.array_equal(v, raw[3][3][:, 2:])
    sp, k3, _ = keep.expand(3)
    assert sp == (2, 10) and np.array_equal(k3, raw[3][2][:, 2:])
    sp, k1, _ = keep.expand(1)
    assert sp == (6, 10) and np.array_equal(k1, raw[3][2][:, 6:])
    sp, k0, _ = keep.expand(0)
    assert sp == (8, 10) and np.array_equal(k0, raw[0][2][:, 8:])
    mean = oracle.Snapshot(kv, cfg, st, [8, 6, 4, 2], 10, mode=0)
    _, _, k, _ = mean.blob(1)
    assert np.array_equal(k[:, :4], raw[3][2][:, 2:6])
    want = np.float32(0.5) * (raw[1][2][:, 6:] + raw[3][2][:, 6:])
    assert np.abs(k[:, 4:] - want).max() < 1e-6


def test_expand_rejects_gaps(oracle):  # test_kvstore.cpp:189-197
    cfg, kv, _ = coded_kv(oracle, 4, 2, 3, 10)
    snap = oracle.Snapshot(kv, cfg, oracle.Strategy([(1, 3, .25)]), [8, 6, 4, 2], 10)
    for layer in (4, -1):
        with pytest.raises(oracle.OracleError) as e:
            snap.expand(layer)
        assert e.value.kind == "RestorationGapError"
    snap.set_plan([7, 6, 4, 2])
    with pytest.raises(oracle.OracleError) as e:
        snap.expand(0)
    assert e.value.kind == "RestorationGapError"


def test_storage_exact(oracle):  # test_kvstore.cpp:199-242, acceptance.cpp:363-399
    cfg, kv, _ = coded_kv(oracle, 4, 2, 3, 10)
    snap = oracle.Snapshot(kv, cfg, oracle.Strategy([(1, 3, .25)]), [8, 6, 4, 2], 10)
    full, stored = snap.storage()
    assert full == 4 * 10 * 48 and stored == (2 + 8 + 6) * 48
    from oracle.oracle import ModelConfig
    N, L = 32, 40
    cfg = ModelConfig(n_layers=N, n_heads=1, head_dim=2, d_model=2, vocab_size=5)
    ones = [(0, L, np.ones((1, L, 2), np.float32), np.ones((1, L, 2), np.float32))] * N
    kv = oracle.KV.from_host(cfg, ones)
    st = oracle.Strategy([(2 * k, 2 * k + 1, 0.1) for k in range(8)])
    snap = oracle.Snapshot(kv, cfg, st, oracle.uniform_plan(L, N, 0.4), L, mode=1)
    full, stored = snap.storage()
    assert stored / full == 0.45


# ---------------------------------------------------------------- scheduler

def test_cost_hand_values(oracle):  # test_scheduler.cpp:52-71
    assert oracle.layer_flops(2, 4) == pytest.approx(816.0)
    assert oracle.layer_flops(0, 4) == 0.0
    whole = oracle.prefill_flops(48, 0, 64, 4)
    split = oracle.prefill_flops(16, 0, 64, 4) + oracle.prefill_flops(32, 16, 64, 4)
    assert whole == pytest.approx(split, rel=1e-12)
    assert oracle.prefill_flops(10, 0, 32, 1) == pytest.approx(oracle.layer_flops(10, 32))


def test_pyramid_plan_hand_values(oracle):  # test_scheduler.cpp:73-92
    assert oracle.build_plan(8, 4, 0.5).tolist() == [8, 5, 3, 0]
    assert oracle.build_plan(10, 3, 0.0).tolist() == [0, 0, 0]
    assert oracle.build_plan(10, 3, 1.0).tolist() == [10, 10, 10]
    assert oracle.build_plan(10, 1, 0.3).tolist() == [3]
    for args, kind in (((8, 0, 0.5), "ConfigError"), ((-1, 4, 0.5), "ConfigError"),
                       ((8, 4, 1.5), "ConfigError")):
        with pytest.raises(oracle.OracleError) as e:
            oracle.build_plan(*args)
        assert e.value.kind == kind
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_plan(8, 4, 0.5, oracle.Strategy([(1, 9, .1)]))
    assert e.value.kind == "PlanInvalidError"


def test_plan_invariants_random(oracle):  # test_scheduler.cpp:94-117, acceptance.cpp:535-572
    rng = np.random.default_rng(99)
    for _ in range(300):
        N = 1 + int(rng.integers(48))
        L = int(rng.integers(2000))
        r = int(rng.integers(1001)) / 1000.0
        p = oracle.build_plan(L, N, r)
        assert (p >= 0).all() and (p <= L).all() and (np.diff(p) <= 0).all()
        assert abs(p.sum() - r * L * N) <= N
        assert oracle.validate_plan(L, p) == 0
        for l in range(1, N):
            if p[l - 1] < L:
                q = p.copy()
                q[l] = p[l - 1] + 1
                assert oracle.validate_plan(L, q) & 2


def test_uniform_plan_and_grid(oracle):  # test_scheduler.cpp:119-136
    assert oracle.uniform_plan(10, 3, 0.42).tolist() == [4, 4, 4]
    assert oracle.uniform_plan(10, 2, 1.0).tolist() == [10, 10]
    g = oracle.default_rc_grid()
    assert len(g) == 21 and g[0] == 0.0 and g[-1] == 1.0 and g[10] == pytest.approx(0.5)
    assert len(oracle.default_rc_grid(0.5)) == 3


def test_calibration_limits_and_argmin(oracle):  # test_scheduler.cpp:138-183
    assert oracle.calibrate_rc(8, 500, 128, b_peak=1e30) == 0.0
    assert oracle.calibrate_rc(8, 500, 128, f_peak=1e30) == 1.0
    rng = np.random.default_rng(7)
    grid = oracle.default_rc_grid()
    for trial in range(40):
        f = 1e12 * (1 + int(rng.integers(500)))
        b = 1e9 * (1 + int(rng.integers(500)))
        N = 2 + int(rng.integers(31))
        L = 100 + int(rng.integers(900))
        d = 64 << int(rng.integers(5))
        st = oracle.Strategy([(0, N - 1, .1), (1, N - 2, .2)]) if trial % 2 == 0 and N >= 4 \
            else oracle.Strategy()
        got = oracle.calibrate_rc(N, L, d, st, grid, f_peak=f, b_peak=b)
        best, gap = None, None
        for r in grid:
            p = oracle.build_plan(L, N, r, st)
            tc = sum(oracle.layer_flops(int(x), d) for x in p) / f
            tl = sum(2.0 * (e - s) * d * 4.0 for _, (s, e) in oracle.blob_specs(L, p, st)) / b
            if best is None or abs(tc - tl) < gap:
                best, gap = r, abs(tc - tl)
        assert got == best


def test_calibration_regime_acceptance6(oracle):  # acceptance.cpp:403-441
    N, L, d, n_new = 32, 1000, 1024, 100
    t_rec = oracle.prefill_flops(L, 0, d, N) / 312e12
    full_bytes = N * 2.0 * L * d * 4.0
    b = full_bytes / (t_rec * 1.35 / 2.0)
    r = oracle.calibrate_rc(N, L, d, b_peak=b)

    def ttft(p):
        return oracle.simulate(L, p, None, d, b_peak=b)["makespan"] + \
            oracle.prefill_flops(n_new, L, d, N) / 312e12
    tk = ttft(oracle.build_plan(L, N, r))
    assert abs(r - 0.40) <= 0.05
    assert 1.6 <= ttft(oracle.uniform_plan(L, N, 1.0)) / tk <= 2.4
    assert 1.08 <= ttft(oracle.uniform_plan(L, N, 0.0)) / tk <= 1.62


def test_simulator_intervals(oracle):  # test_scheduler.cpp:255-331
    st = oracle.Strategy([(1, 3, .5)])
    p = oracle.build_plan(600, 4, 0.5, st)
    t = oracle.simulate(600, p, st, 128)
    assert t["n_compute"] == 3 and t["n_load"] == 2
    assert t["makespan"] == pytest.approx(max(t["compute_finish"], t["load_finish"]))
    a = oracle.simulate(100, oracle.uniform_plan(100, 4, 1.0), None, 64)
    assert a["n_load"] == 0 and a["bubble_load"] == 0.0
    z = oracle.simulate(0, oracle.uniform_plan(0, 4, 0.5), None, 64)
    assert z["makespan"] == 0.0
    un = oracle.simulate(400, oracle.uniform_plan(400, 4, 0.25), None, 128)
    pa = oracle.simulate(400, oracle.uniform_plan(400, 4, 0.25), oracle.Strategy([(0, 2, .1)]), 128)
    assert un["n_load"] == 4 and pa["n_load"] == 3 and pa["load_finish"] < un["load_finish"]


def test_lossless_restore(oracle):  # test_scheduler.cpp:353-400, acceptance.cpp:278-359
    from oracle.oracle import ModelConfig
    cfg = ModelConfig(n_layers=4, n_heads=2, head_dim=4, d_model=8, vocab_size=13, seed=21)
    m = oracle.Model(cfg)
    hist = oracle.tokens(24, 77, 13)
    full = m.prefill(hist).take_kv()
    for r in (0.0, 0.25, 0.5, 0.75, 1.0):
        p = oracle.build_plan(24, 4, r)
        snap = oracle.Snapshot(full, cfg, oracle.Strategy(), p, 24, mode=1)
        rest = m.restore(hist, snap)
        for l in range(4):
            assert rest.span(l) == (0, 24)
            assert np.abs(rest.layer(l)[0] - full.layer(l)[0]).max() < 1e-6
            assert np.abs(rest.layer(l)[1] - full.layer(l)[1]).max() < 1e-6
        la, _ = m.decode(rest, int(hist[-1]))
        lb, _ = m.decode(full.clone(), int(hist[-1]))
        assert np.abs(la - lb).max() < 1e-5


def test_restore_rejects_mismatch(oracle):  # test_scheduler.cpp:402-430
    from oracle.oracle import ModelConfig
    cfg = ModelConfig(n_layers=2, n_heads=1, head_dim=4, d_model=4, vocab_size=7)
    m = oracle.Model(cfg)
    hist = np.array([1, 2, 3, 4, 5, 6], np.int32)
    full = m.prefill(hist).take_kv()
    snap = oracle.Snapshot(full, cfg, oracle.Strategy(), oracle.build_plan(6, 2, 0.5), 6, mode=1)
    with pytest.raises(oracle.OracleError) as e:
        m.restore(np.append(hist, 1), snap)
    assert e.value.kind == "RestorationGapError"
    snap.set_plan([2, 1])
    with pytest.raises(oracle.OracleError) as e:
        m.restore(hist, snap)
    assert e.value.kind == "RestorationGapError"
