"""End-to-end turn-loop parity: the reference's Krul turn
loop (harness.cpp:92-259) on the device -- restore -> new-input prefill ->
classify -> estimator (prefill + decode folds) -> select -> calibrate_rc ->
build_plan -> compress -- against the oracle's restatement of the same loop
(oracle/turns.py) on the same weights and teacher-forced tokens.

Bar (f32 parity mode): ir_layers, selected pairs, exhausted_before_quota,
r_c and recompute_len bit-equal to the oracle every turn; avg_weight_sum
abs <= 1e-6; D rel <= 1e-5; logits abs <= 1e-4. The minimum relative gap
between consecutive sorted candidate distances is printed (SURVEY §7 hard
part 2): a pair flip is only possible when it is below D's error.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG1 = dict(n_layers=4, n_heads=4, head_dim=64, d_model=256, vocab_size=256, ffn_mult=4.0, seed=7)


def candidate_gap(D, layers, ir):
    pos = {l: i for i, l in enumerate(layers)}
    ir = sorted(set(ir))
    d = sorted(D[pos[a], pos[b]] for k, a in enumerate(ir) for b in ir[k + 1:])
    if len(d) < 2:
        return float("inf")
    return min((d[k + 1] - d[k]) / max(d[k], 1e-300) for k in range(len(d) - 1))


@pytest.mark.parametrize("merge", [0, 1])
def test_turn_loop_cfg1_bit_exact(merge, oracle):
    from oracle import turns as OT
    from paper_2507_08045_b200 import native as K
    from paper_2507_08045_b200 import turns as T

    O = oracle
    om = O.Model(O.ModelConfig(**CFG1))
    user0 = O.tokens(64, 11, 256)
    user1 = O.tokens(64, 12, 256)
    traces = OT.reference_pass(om, [OT.OTurn(user0, 448), OT.OTurn(user1, 16)])
    assert traces[0][1].size == 448 and traces[1][1].size == 16
    knobs = dict(gamma=0.1, initial_frac=0.1, recent_frac=0.1, r_l=0.5, merge=merge)
    orecs, osnap = OT.run_krul(om, traces, **knobs)

    ctx = K.Context(K.ModelConfig(**CFG1, dtype=K.KRUL_F32, max_tokens=1024), 0)
    ctx.upload_weights(om.weights())
    recs, st = T.run_turns(ctx, [T.Turn(u, f) for u, f in traces], T.TurnConfig(**knobs), 1024)

    for t, (g, o) in enumerate(zip(recs, orecs)):
        assert g.history_len == o.history_len and g.total_len == o.total_len
        assert np.abs(g.logits - o.logits).max() <= 1e-4, t
        assert np.abs(g.avg_weight_sum - o.avg_weight_sum).max() <= 1e-6, t
        assert g.ir_layers == o.ir_layers, (t, g.ir_layers, o.ir_layers)
        rel = np.abs(g.D - o.D).max() / max(np.abs(o.D).max(), 1e-300)
        assert rel <= 1e-5, (t, rel)
        gap = candidate_gap(o.D, sorted(set(o.ir_layers)), o.ir_layers)
        print(f"turn {t}: ir={g.ir_layers} pairs={[p[:2] for p in g.pairs]} exhausted={g.exhausted} "
              f"r_c={g.r_c} plan={g.plan.tolist()} D rel err={rel:.2e} min candidate gap={gap:.3e}")
        assert [p[:2] for p in g.pairs] == [p[:2] for p in o.pairs], (t, g.pairs, o.pairs)
        for gp, op in zip(g.pairs, o.pairs):
            assert abs(gp[2] - op[2]) <= 1e-5 * max(abs(op[2]), 1e-300)
        assert g.exhausted == o.exhausted
        assert g.r_c == o.r_c
        assert np.array_equal(g.plan, o.plan), (t, g.plan, o.plan)
        if t >= 1:
            assert g.ttft_ms is not None and g.ttft_ms > 0
    # at least one turn actually shares a pair (quota 2 of 4 layers)
    assert any(r.pairs for r in recs)
    # the final snapshots: same layout, blobs within the f32 tolerance
    snap = st.snapshot
    assert snap.n_blobs() == osnap.n_blobs()
    for b in range(snap.n_blobs()):
        go, gspan, gk, gv = snap.blob(b)
        oo, ospan, ok, ov = osnap.blob(b)
        assert go == oo and gspan == ospan
        if gk.size:
            assert np.abs(gk - ok).max() <= 1e-5 and np.abs(gv - ov).max() <= 1e-5
    assert snap.storage_report() == osnap.storage()
