"""The reference's Krul turn loop (harness.cpp:92-259, the kKrul branch) on
the device, through the C ABI only.

Per turn t (harness.cpp:111-249):
  1. t == 0: fresh prefill of the user tokens (harness.cpp:124-126);
     t >= 1: restore the previous turn's snapshot and prefill the new input
     over it (execute_restore + prefill(tokens, restored), :127-131) -- one
     krul_restore_and_prefill call, device-timed (TTFT).
  2. classify_layers over the prefill just run (:175); the region masses
     come out of the attention kernel itself.
  3. StreamingEstimator(ir_layers) folds the prefill attention (:176-177),
     then every teacher-forced decode step's rows (:180-188).
  4. End of turn (:221-236): finish -> select_strategy -> calibrate_rc over
     default_rc_grid(step) with the configured CostModel -> build_plan ->
     compress_and_snapshot (K8 on the device), classifier report attached.

The forced decode tokens are inputs (the reference fixes them with a greedy
full-recompute pass, harness.cpp:39-66); the tests take them from the oracle.
This module is host orchestration only: every step is a library call.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import native as K


@dataclass
class Turn:
    """harness.hpp Turn + the replayed trace: user tokens and the forced
    decode tokens of the turn."""
    user: np.ndarray
    forced_decode: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))


@dataclass
class TurnConfig:
    """The BenchConfig fields the Krul branch reads (harness.hpp:45-66)."""
    gamma: float = 0.5            # ClassifierConfig::gamma
    initial_frac: float = 0.1
    recent_frac: float = 0.1
    r_l: float = 0.5              # StrategyConfig::r_l
    merge: int = K.MERGE_MEAN     # BenchConfig::merge
    cost: K.CostModel = field(default_factory=K.CostModel)  # reference defaults F=312e12, B=139e9
    rc_grid_step: float = 0.05
    # prefill attention for the estimator: 2 = recompute (K2, no record; the
    # attention stays on the tcgen05 path), 1 = the materialised record
    capture: int = 2
    # B200 extension: the split from measured stream rates (calibrate_rc_measured,
    # scheduler.cpp:402-443). Called as calibrate(state, pairs, total_len) -> r_c at
    # the end of the turn, with the turn's full KV in state.conv; None keeps the
    # reference's analytic calibrate_rc over `cost`.
    calibrate: object = None


@dataclass
class TurnRecord:
    history_len: int
    new_len: int
    logits: np.ndarray
    ttft_ms: float | None
    restore_stats: dict | None
    avg_weight_sum: np.ndarray
    ir_layers: list
    non_ir_layers: list
    D: np.ndarray
    pairs: list
    exhausted: bool
    r_c: float
    plan: np.ndarray
    total_len: int


class KrulTurns:
    """run_method(kKrul) state across turns: history, the conversation's paged
    cache and the last snapshot."""

    def __init__(self, ctx: K.Context, cfg: TurnConfig, capacity: int | None = None):
        self.ctx = ctx
        self.cfg = cfg
        self.conv = ctx.conversation(capacity)
        self.history = np.zeros(0, np.int32)
        self.snapshot: K.KVSnapshot | None = None
        ctx.set_classifier_regions(cfg.initial_frac, cfg.recent_frac)

    def start_from(self, history):
        """Seeds the loop with a conversation whose previous turns are not
        replayed: a fresh prefill of `history` and a full-load snapshot
        (uniform_plan(L, N, 0), keep-deeper, no pairs -- the kFullLoad
        snapshot of harness.cpp:202-207). The next turn() then restores it."""
        ctx, N = self.ctx, self.ctx.cfg.n_layers
        h = np.ascontiguousarray(history, np.int32)
        ctx.prefill(self.conv, h)
        self.snapshot = K.KVSnapshot.compress(ctx, self.conv, [], K.uniform_plan(h.size, N, 0.0), h.size,
                                              K.MERGE_KEEP_DEEPER)
        self.history = h

    def turn(self, t: int, trace: Turn) -> TurnRecord:
        ctx, cfg, mc = self.ctx, self.cfg, self.ctx.cfg
        hist_len = int(self.history.size)
        user = np.ascontiguousarray(trace.user, np.int32)
        tokens = np.concatenate([self.history, user]).astype(np.int32)
        ttft, stats = None, None
        # the estimator's prefill fold reads this prefill's attention record
        ctx.set_capture(cfg.capture)
        try:
            if t == 0 or self.snapshot is None:                      # harness.cpp:124-126
                logits = ctx.prefill(self.conv, tokens)
            else:                                                   # harness.cpp:127-131
                logits, stats, ttft = ctx.restore_and_prefill(self.conv, self.history, self.snapshot, user)
            # the adaptive path analyses the turn it just prefilled (harness.cpp:171-178)
            avg, ir, non_ir = ctx.classify_layers(cfg.gamma, cfg.initial_frac, cfg.recent_frac)
            est = K.StreamingEstimator(ctx, ir)
            est.fold_prefill()
        finally:
            ctx.set_capture(False)
        for tok in np.asarray(trace.forced_decode, np.int32):  # harness.cpp:180-188
            ctx.decode_step(self.conv, int(tok))
            est.fold_decode()
        end_tokens = np.concatenate([tokens, np.asarray(trace.forced_decode, np.int32)]).astype(np.int32)
        total = int(end_tokens.size)
        # end-of-turn snapshot, kKrul (harness.cpp:221-236)
        D = est.finish()
        strat = K.select_strategy(ctx, D, est.layers, ir, cfg.r_l, mc.n_layers)
        self.history = end_tokens
        if cfg.calibrate is None:
            r_c = K.calibrate_rc(cfg.cost, mc.n_layers, total, mc.d_model, strat.pairs,
                                 K.default_rc_grid(cfg.rc_grid_step))
        else:
            r_c = float(cfg.calibrate(self, strat.pairs, total))
        plan = K.build_plan(total, mc.n_layers, r_c, strat.pairs)
        snap = K.KVSnapshot.compress(ctx, self.conv, strat.pairs, plan, total, cfg.merge)
        snap.set_meta("bench", strat.exhausted_before_quota, ir, non_ir, list(avg))
        self.snapshot = snap
        return TurnRecord(hist_len, int(user.size), logits, ttft, stats, avg, ir, non_ir, D,
                          list(strat.pairs), bool(strat.exhausted_before_quota), float(r_c), plan, total)


def run_turns(ctx: K.Context, turns, cfg: TurnConfig, capacity: int | None = None):
    """All turns of one conversation -> (records, final KrulTurns state)."""
    st = KrulTurns(ctx, cfg, capacity)
    return [st.turn(t, tr) for t, tr in enumerate(turns)], st
