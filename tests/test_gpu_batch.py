"""Pipelined batch restore (krul_restore_batch, configs[3]): conversation i+1's
blob copies start under conversation i's new-input prefill tail. The batch
must produce exactly what one restore_and_prefill per conversation produces:
the same logits and the same restored K/V, bit for bit (same kernels, same
plans; only the inter-conversation ordering differs)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPE = dict(n_layers=4, n_heads=4, n_kv_heads=2, head_dim=128, d_model=512, vocab_size=512,
             ffn_mult=3.5, ffn_kind=1, rope_theta=10000.0, seed=7)


@pytest.mark.parametrize("coded", [True, False])
def test_restore_batch_matches_single_restores(coded, monkeypatch):
    from paper_2507_08045_b200 import native as K

    monkeypatch.setenv("KRUL_KV_POOL_CONVS", "6")
    cfg = K.ModelConfig(**SHAPE, dtype=K.KRUL_BF16, max_tokens=640)
    ctx = K.Context(cfg, 0)
    ctx.init_weights(3)
    ctx.set_kv_coding(coded)
    rng = np.random.default_rng(5)
    Ls = [448, 384, 512, 320]
    pairs = [(1, 3, 0.0)]
    items = []
    for i, L in enumerate(Ls):
        hist = rng.integers(0, cfg.vocab_size, L, dtype=np.int32)
        new = rng.integers(0, cfg.vocab_size, 64, dtype=np.int32)
        src = ctx.conversation(640)
        ctx.prefill(src, hist)
        plan = K.build_plan(L, cfg.n_layers, 0.1 * i, pairs)
        snap = K.KVSnapshot.compress(ctx, src, pairs, plan, L, K.MERGE_MEAN)
        src.close()
        items.append((hist, new, snap, plan))
    # reference: one restore_and_prefill per conversation into a fresh conversation
    want = []
    for hist, new, snap, plan in items:
        c = ctx.conversation(640)
        logits, _, _ = ctx.restore_and_prefill(c, hist, snap, new)
        kv = [c.kv(layer, 0, len(hist) + len(new)) for layer in range(cfg.n_layers)]
        want.append((logits, kv))
        c.close()
    convs = [ctx.conversation(640), ctx.conversation(640)]
    seq = [convs[i % 2] for i in range(len(items))]
    for rep in range(2):  # the second pass reuses the conversations' pages
        tt, total, logits = ctx.restore_batch(seq, [it[0] for it in items], [it[2] for it in items],
                                              [it[1] for it in items], logits=True)
        assert total > 0 and np.all(tt > 0) and tt.max() <= total + 1e-3
        for i, (hist, new, snap, plan) in enumerate(items):
            assert np.array_equal(logits[i], want[i][0]), (rep, i)
        # the last two conversations' pages are still intact
        for i in (len(items) - 2, len(items) - 1):
            hist, new = items[i][0], items[i][1]
            for layer in range(cfg.n_layers):
                k, v = seq[i].kv(layer, 0, len(hist) + len(new))
                assert np.array_equal(k, want[i][1][layer][0]) and np.array_equal(v, want[i][1][layer][1]), (i, layer)
    # a restore_and_prefill after a batch still works (graph key reset)
    hist, new, snap, _ = items[0]
    c = ctx.conversation(640)
    for _ in range(3):
        logits, _, _ = ctx.restore_and_prefill(c, hist, snap, new)
        assert np.array_equal(logits, want[0][0])


def test_restore_batch_rejects_same_conversation_twice(monkeypatch):
    from paper_2507_08045_b200 import native as K

    monkeypatch.setenv("KRUL_KV_POOL_CONVS", "4")
    cfg = K.ModelConfig(**SHAPE, dtype=K.KRUL_BF16, max_tokens=640)
    ctx = K.Context(cfg, 0)
    ctx.init_weights(3)
    rng = np.random.default_rng(1)
    hist = rng.integers(0, cfg.vocab_size, 256, dtype=np.int32)
    new = rng.integers(0, cfg.vocab_size, 16, dtype=np.int32)
    src = ctx.conversation(640)
    ctx.prefill(src, hist)
    snap = K.KVSnapshot.compress(ctx, src, [], K.build_plan(256, 4, 0.0), 256, K.MERGE_MEAN)
    c = ctx.conversation(640)
    with pytest.raises(K.ConfigError):
        ctx.restore_batch([c, c], [hist, hist], [snap, snap], [new, new])


def test_gemm_spans_do_not_change_results():
    """krul_span_enable (device-side GEMM spans): stamps every weight-streaming
    GEMM launch of a restore, sane totals, identical logits with spans on/off."""
    from paper_2507_08045_b200 import native as K

    cfg = K.ModelConfig(**SHAPE, dtype=K.KRUL_BF16, max_tokens=640)
    ctx = K.Context(cfg, 0)
    ctx.init_weights(3)
    rng = np.random.default_rng(9)
    hist = rng.integers(0, cfg.vocab_size, 448, dtype=np.int32)
    new = rng.integers(0, cfg.vocab_size, 64, dtype=np.int32)
    src = ctx.conversation(640)
    ctx.prefill(src, hist)
    snap = K.KVSnapshot.compress(ctx, src, [(1, 3, 0.0)], K.build_plan(448, 4, 0.1, [(1, 3, 0.0)]), 448,
                                 K.MERGE_MEAN)
    conv = ctx.conversation(640)
    want = None
    for _ in range(3):
        want, _, _ = ctx.restore_and_prefill(conv, hist, snap, new)
    ctx.span_enable(True)
    for _ in range(3):  # eager, capture, replay
        got, _, _ = ctx.restore_and_prefill(conv, hist, snap, new)
        assert np.array_equal(got, want)
        n, ms, by = ctx.span_read()
        # 4 GEMMs per layer of the new-input prefill (+ the pyramid's small-M layers)
        assert n >= 4 * cfg.n_layers and ms > 0 and by > 0, (n, ms, by)
    ctx.span_enable(False)
