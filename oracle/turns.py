"""CPU restatement of the reference's turn replay (TEST INFRASTRUCTURE ONLY:
imported by tests/ and bench.py's CPU legs, never by the product package).

  reference_pass   harness.cpp:39-66   greedy full-recompute pass that fixes
                                       every turn's forced decode tokens
  run_krul         harness.cpp:92-259  run_method, kKrul branch: restore ->
                                       prefill(tokens, restored) -> classify
                                       -> estimator (prefill + decode folds)
                                       -> select -> calibrate_rc ->
                                       build_plan -> compress_and_snapshot
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import oracle as O


@dataclass
class OTurn:
    user: np.ndarray
    decode_len: int = 0


def reference_pass(model: O.Model, turns):
    """harness.cpp:39-66 -> list of (user, forced_decode) per turn."""
    out = []
    history = np.zeros(0, np.int32)
    for tr in turns:
        tokens = np.concatenate([history, np.asarray(tr.user, np.int32)]).astype(np.int32)
        pf = model.prefill(tokens, capture=False)
        logits = pf.logits()
        kv = pf.take_kv()
        forced = []
        for _ in range(tr.decode_len):
            tok = int(np.argmax(logits))  # greedy_pick: first maximum (engine.cpp:491-495)
            forced.append(tok)
            logits, _ = model.decode(kv, tok)
        forced = np.asarray(forced, np.int32)
        out.append((np.asarray(tr.user, np.int32), forced))
        history = np.concatenate([tokens, forced]).astype(np.int32)
    return out


@dataclass
class ORecord:
    history_len: int
    logits: np.ndarray
    avg_weight_sum: np.ndarray
    ir_layers: list
    D: np.ndarray
    pairs: list
    exhausted: bool
    r_c: float
    plan: np.ndarray
    total_len: int
    restore_prefill_s: float


def run_krul(model: O.Model, traces, gamma=0.5, initial_frac=0.1, recent_frac=0.1, r_l=0.5, merge=0,
             rc_grid_step=0.05, f_peak=312e12, b_peak=139e9, cost_ffn_mult=4.0, rc_override=None):
    """harness.cpp:92-259 (kKrul). traces: [(user, forced_decode)]."""
    cfg = model.cfg
    N, H, d = cfg.n_layers, cfg.n_heads, cfg.d_model
    history = np.zeros(0, np.int32)
    snap = None
    recs = []
    for t, (user, forced) in enumerate(traces):
        tokens = np.concatenate([history, user]).astype(np.int32)
        t0 = time.perf_counter()
        if t == 0 or snap is None:
            pf = model.prefill(tokens, capture=True)                       # :124-126
        else:
            restored = model.restore(history, snap)                         # :127-131
            pf = model.prefill(tokens, preload=restored.suffix([0] * N), capture=True)
        dt = time.perf_counter() - t0
        logits = pf.logits()
        avg, ir = pf.classify(gamma, initial_frac, recent_frac)             # :175
        acc = O.Accumulator(ir, H)                                          # :176-177
        acc.fold_prefill_handle(pf)
        kv = pf.take_kv()
        for tok in forced:                                                  # :180-188
            _, rows = model.decode(kv, int(tok))
            acc.fold_decode(rows)
        end_tokens = np.concatenate([tokens, forced]).astype(np.int32)
        total = int(end_tokens.size)
        D = acc.finalize()                                                  # :222
        strat = O.select_strategy(D, acc.layers, ir, r_l, N)                # :223-224
        r_c = (O.calibrate_rc(N, total, d, strat, O.default_rc_grid(rc_grid_step), f_peak, b_peak,
                              cost_ffn_mult) if rc_override is None else rc_override)  # :225-227
        plan = O.build_plan(total, N, r_c, strat)                           # :228-229
        snap = O.Snapshot(kv, cfg, strat, plan, total, mode=merge)         # :230-231
        recs.append(ORecord(int(history.size), logits, avg, ir, D, list(strat.pairs), bool(strat.exhausted),
                            float(r_c), plan, total, dt))
        history = end_tokens
    return recs, snap
