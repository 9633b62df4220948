#!/usr/bin/env python3
"""Restoration TTFT benchmark (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1], the default): Llama-3-8B-shaped
random-init model (32 layers, d=4096, 32 heads / 8 KV heads, hd=128, SwiGLU
F=14336, vocab 128256, rope theta 5e5), bf16, one conversation with an
8192-token history restored from its compressed snapshot in pinned host
memory, then a 128-token new-input prefill. A step = one restore + new-input
prefill (TTFT: restore launch -> last-row logits). Conversations are
independent, so N GPUs run N shards with no collective ("weak" scaling);
value = conversations restored per second over all ranks (max-over-ranks
device time).

The snapshot is produced by the reference's turn loop (harness.cpp:92-259,
kKrul; paper_2507_08045_b200/turns.py), untimed: the previous turn restores
its own snapshot, prefills its 128-token input, classifies the layers
(gamma 0.1), runs the streaming estimator over that prefill and 64 decode
steps, selects the layer pairs (r_l 0.5), picks r_c from measured stream
rates (the TTFT-argmin calibration on the device) and compresses (K8). The
timed steps restore exactly that estimator-selected snapshot. The fixed
8-pair control is reported beside it (policies.krul_control).

`--impl reference` times the reference's CPU path -- the oracle/ restatement
(the reference itself cannot be built here: Eigen is absent) -- on the host
cores: execute_restore + prefill(history + new, restored) of the same
workload (the same r_c and pair count), without loading the product library.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = {"hbm_gbs": 6547.2, "bf16_tflops": 1676.4, "bf16_tflops_sustained": 1397.8}
try:
    PEAKS.update(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))))
    PEAKS["MEASURED_PEAKS_FILE"] = True
except Exception:
    pass

# ncu --set full DRAM bytes (read + write) of one launch per kernel class vs
# its algorithmic bytes, from the committed captures under profiles/
NCU_TRAFFIC = {
    "gemm": (276_462_080, 1078 * 4096 * 2 + 28672 * 4096 * 2 + 1078 * 14336 * 2,
             "profiles/r01c/SUMMARY.md (FFN1 pair GEMM, M=1078 N=28672 K=4096)"),
    "gemm_stream": (236031744 + 4214016, 28672 * 4096 * 2 + 128 * 4096 * 2 + 128 * 14336 * 2,
                    "profiles/r02/ncu_gstream.md (new-input FFN1, M=128 N=28672 K=4096, SwiGLU epilogue, "
                    "k_gemm_tc<256,4,4> cluster split-K, dram read + write)"),
}

METRIC = ("restoration TTFT p50 (ms) @8K history; conversations restored/sec at 1/2/4/8 GPU")

_LLAMA8 = dict(n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096, vocab_size=128256,
               ffn_mult=3.5, ffn_kind=1, rope_theta=500000.0)
# turn structure (the turn whose end-of-turn snapshot the timed steps restore):
# n_dec teacher-forced decode steps after the n_new-token prefill; estimator
# knobs gamma / r_l (gamma 0.5 empties L_I on random-init weights);
# `pairs` = the fixed control strategy; r_c_ref = the split both arms restore
# at (the argmin of the GPU arm's measured TTFT curve on B200, round 2:
# 0.016-0.02 over seven runs; the plan's recompute_token_layers at a given
# r_c does not depend on which 8 pairs were selected, so the two arms'
# `config` is identical)
CONFIGS = {
    # BASELINE.json configs[1]
    "llama3-8b-8k": dict(**_LLAMA8, label="Llama-3-8B-shaped", L=8192, n_new=128, n_dec=64, gamma=0.1,
                         r_l=0.5, pairs=[(9 + 2 * k, 10 + 2 * k) for k in range(8)], r_c_ref=0.02,
                         l2="inputs (16 GB bf16 weights, 1 GB KV) larger than L2; no flush"),
    # BASELINE.json configs[2]: Mistral-7B shape (GQA 32/8), 32K history
    "mistral-7b-32k": dict(n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, d_model=4096,
                           vocab_size=32000, ffn_mult=3.5, ffn_kind=1, rope_theta=1000000.0,
                           label="Mistral-7B-shaped", L=32768, n_new=128, n_dec=16, gamma=0.1, r_l=0.5,
                           pairs=[(9 + 2 * k, 10 + 2 * k) for k in range(8)], r_c_ref=0.06,
                           l2="inputs (14.5 GB bf16 weights, 4.3 GB KV) larger than L2; no flush"),
    # BASELINE.json configs[4]: Llama-3-70B shape, bf16 replica (~141 GB), 16K history
    "llama3-70b-16k": dict(n_layers=80, n_heads=64, n_kv_heads=8, head_dim=128, d_model=8192,
                           vocab_size=128256, ffn_mult=3.5, ffn_kind=1, rope_theta=500000.0,
                           label="Llama-3-70B-shaped", L=16384, n_new=128, n_dec=16, gamma=0.1, r_l=0.5,
                           pairs=[(30 + 2 * k, 31 + 2 * k) for k in range(20)], r_c_ref=0.0,
                           l2="inputs (141 GB bf16 weights, 5.4 GB KV) larger than L2; no flush"),
    # BASELINE.json configs[3]: 256 conversations, 2K-16K history, sharded by
    # conversation (LPT on KV bytes) across the GPUs of the box
    "llama3-8b-batch256": dict(**_LLAMA8, label="Llama-3-8B-shaped", L=16384, n_new=128, batch=256,
                               L_lo=2048, L_hi=16384, gamma=0.1, r_l=0.5,
                               pairs=[(9 + 2 * k, 10 + 2 * k) for k in range(8)], r_c_ref=0.0,
                               l2="inputs (16 GB bf16 weights, 0.3-2 GB KV) larger than L2; no flush"),
    # BASELINE.json configs[0] / SURVEY §8(d) cfg1: the CPU reference's own
    # case, f32 parity mode: turn 0 = 64 user + 448 forced tokens, turn 1 = 64
    # new tokens restored at the reference's analytic calibrate_rc (default
    # CostModel) -- the identical plan on both arms
    "tiny-512": dict(n_layers=4, n_heads=4, n_kv_heads=4, head_dim=64, d_model=256, vocab_size=256,
                     ffn_mult=4.0, ffn_kind=0, rope_theta=10000.0, label="tiny reference-architecture",
                     L=512, n_new=64, turn0=(64, 448), gamma=0.1, r_l=0.5, pairs=[(1, 2)], f32=True,
                     l2="inputs fit in L2 (tiny config); no flush"),
}


def model_kwargs(spec):
    return {k: spec[k] for k in ("n_layers", "n_heads", "n_kv_heads", "head_dim", "d_model", "vocab_size",
                                 "ffn_mult", "ffn_kind", "rope_theta")}


def workload_config(args, spec, world, r_c, n_pairs, plan_sum):
    """`config` of the JSON line -- identical on both arms for the same plan."""
    return {"workload": f"{args.config}: {spec['label']}, {spec['L']}-token history restore + "
                        f"{spec['n_new']}-token new-input prefill, 1 conversation/step/GPU",
            "global_batch": world, "seq_len": spec["L"], "n_new": spec["n_new"],
            "parallelism": f"dp{world} (conversation shards, no collective)", "l2": spec["l2"],
            "r_c": r_c, "pairs": n_pairs, "recompute_token_layers": int(plan_sum)}


def lscpu_cores():
    """Physical cores on this host (lscpu) and the threads this process may use."""
    try:
        out = subprocess.run(["lscpu", "-p=CORE,SOCKET"], capture_output=True, text=True, timeout=10).stdout
        cores = len({ln for ln in out.splitlines() if ln and not ln.startswith("#")})
    except Exception:
        cores = None
    return cores, len(os.sched_getaffinity(0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                          f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace('.', '', 1).isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        # KRUL_BENCH_DEVICE pins every rank to one GPU (multi-rank plumbing
        # test on a 1-GPU box; NCCL refuses shared devices, so gloo then)
        if os.environ.get("KRUL_BENCH_DEVICE") is not None:
            local = int(os.environ["KRUL_BENCH_DEVICE"])
        else:
            from paper_2507_08045_b200 import shard
            shard.bind_to_gpu_numa(local)  # host snapshots on the GPU's NUMA node
        torch.cuda.set_device(local)
        dist.init_process_group(os.environ.get("KRUL_DIST_BACKEND", "nccl"))
        return rank, local, world, dist
    return rank, local, world, None


def barrier(dist):
    if dist:
        dist.barrier()


def allmax(dist, x, local):
    from paper_2507_08045_b200 import shard
    return shard.max_over_ranks(x, dist, f"cuda:{local}")


# ---------------------------------------------------------------- B200 arm

def run_batch(args, rank, local, world, dist, K, spec):
    """configs[3]: `batch` conversations (history U[L_lo, L_hi], whole pages)
    sharded over the ranks by LPT on KV bytes (paper_2507_08045_b200.shard),
    no collective on the data path. Conversations are restored in windows of
    `--window` through the pipelined batch restore (krul_restore_batch: the
    next conversation's blob copies start under the previous one's new-input
    prefill tail). Per window (untimed): each conversation's history prefill,
    plan and device compress into a pinned snapshot, one warm-up batch; then
    the timed batch (device time from the window's first copy to its last
    logits). value = conversations of all ranks / max over ranks of the summed
    window times. The serial figure (one restore_and_prefill per conversation,
    graph replay) is measured beside it. r_c is calibrated once (device TTFT
    objective) on a median-length conversation and reused: the recompute/load
    balance ratio is nearly length-independent."""
    from paper_2507_08045_b200 import shard
    n_new = spec["n_new"]
    Ls = shard.synthetic_histories(spec["batch"], spec["L_lo"], spec["L_hi"])
    w = shard.kv_bytes(Ls, spec["n_layers"], spec["n_kv_heads"], spec["head_dim"])
    mine = shard.lpt_assign(w, world)[rank]
    if args.convs:
        mine = mine[:args.convs]
    os.environ["KRUL_KV_POOL_CONVS"] = "4"  # history source + two alternating restore targets + serial
    cfg = K.ModelConfig(n_layers=spec["n_layers"], n_heads=spec["n_heads"],
                        n_kv_heads=spec["n_kv_heads"], head_dim=spec["head_dim"],
                        d_model=spec["d_model"], vocab_size=spec["vocab_size"],
                        ffn_mult=spec["ffn_mult"], ffn_kind=spec["ffn_kind"],
                        rope_theta=spec["rope_theta"], seed=1234, dtype=K.KRUL_BF16,
                        max_tokens=int(Ls.max()) + n_new + 64)
    ctx = K.Context(cfg, local)
    ctx.init_weights(1234)
    pairs = [(a, b, 0.0) for a, b in spec["pairs"]]
    prev = ctx.conversation(cfg.max_tokens)
    conv = ctx.conversation(cfg.max_tokens)
    alt = [ctx.conversation(cfg.max_tokens), ctx.conversation(cfg.max_tokens)]
    rng = np.random.default_rng(77)
    Lm = int(np.median(Ls)) // 64 * 64
    hist = rng.integers(0, cfg.vocab_size, Lm, dtype=np.int32)
    new = rng.integers(0, cfg.vocab_size, n_new, dtype=np.int32)
    ctx.prefill(prev, hist)
    ctx.set_capture(False)
    r0, _ = ctx.calibrate_rc_ttft(prev, conv, hist, new, pairs, [round(0.02 * k, 4) for k in range(16)])
    r_c, _ = ctx.calibrate_rc_ttft(prev, conv, hist, new, pairs,
                                   sorted({max(0.0, round(r0 + 0.004 * k, 4)) for k in range(-4, 5)}))
    barrier(dist)
    clocks = ClockSampler(local)
    clocks.start()
    win = max(2, args.window)
    serial, swalls, pipe_ms, pipe_ttft, walls, h2d = [], [], [], [], [], 0.0
    launches0 = K.launch_count()
    t_setup = 0.0
    for w0 in range(0, len(mine), win):
        idx = mine[w0:w0 + win]
        items = []
        s0 = time.perf_counter()
        for i in idx:
            L = int(Ls[i])
            g = np.random.default_rng(1000 + i)
            h = g.integers(0, cfg.vocab_size, L, dtype=np.int32)
            nw = g.integers(0, cfg.vocab_size, n_new, dtype=np.int32)
            ctx.prefill(prev, h)
            plan = K.build_plan(L, cfg.n_layers, r_c, pairs)
            items.append((h, nw, K.KVSnapshot.compress(ctx, prev, pairs, plan, L, K.MERGE_MEAN)))
        seq = [alt[k % 2] for k in range(len(items))]
        ctx.restore_batch(seq, [x[0] for x in items], [x[2] for x in items], [x[1] for x in items])  # warm-up
        t_setup += time.perf_counter() - s0
        if len(items) >= 2:
            wa = time.perf_counter()
            tt, tot, _ = ctx.restore_batch(seq, [x[0] for x in items], [x[2] for x in items],
                                           [x[1] for x in items], logits=True)
            walls.append((time.perf_counter() - wa) * 1e3)
            pipe_ms.append(tot)
            pipe_ttft.extend(tt.tolist())
        # the serial figure: one restore_and_prefill per conversation (graph replay)
        for h, nw, snap in items:
            for _ in range(2):
                ctx.restore_and_prefill(conv, h, snap, nw)
            ws = time.perf_counter()
            _, st, ttft = ctx.restore_and_prefill(conv, h, snap, nw)
            swalls.append((time.perf_counter() - ws) * 1e3)
            serial.append(ttft)
            h2d += st["h2d_bytes"]
            if len(items) < 2:
                pipe_ms.append(ttft)
                pipe_ttft.append(ttft)
                walls.append(ttft)
        del items
    ctx.sync()
    launches = K.launch_count() - launches0
    barrier(dist)
    clk = clocks.stop()
    total_ms = shard.max_over_ranks(float(np.sum(pipe_ms)), dist, f"cuda:{local}")
    serial_ms = shard.max_over_ranks(float(np.sum(serial)), dist, f"cuda:{local}")
    wall_ms = shard.max_over_ranks(float(np.sum(walls)), dist, f"cuda:{local}")
    swall_ms = shard.max_over_ranks(float(np.sum(swalls)), dist, f"cuda:{local}")
    n_all = int(shard.sum_over_ranks(len(mine), dist, f"cuda:{local}"))
    pipe_s = n_all / (total_ms / 1e3)
    conv_s = n_all / (serial_ms / 1e3)
    return {
        "metric": METRIC, "value": round(conv_s, 4), "unit": "conversations/s",
        "ttft_p50_ms": round(float(np.median(serial)), 4), "n_gpus": world,
        "steps": len(mine), "warmup": 2, "ms_per_step": round(serial_ms / max(len(mine), 1), 4),
        "higher_is_better": True, "scaling": "weak" if args.convs else "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, uniform random token ids)",
        "config": {"workload": f"{args.config}: {spec['batch']} conversations, history U[{spec['L_lo']}, "
                               f"{spec['L_hi']}] (seed 2507), LPT-sharded over {world} GPU(s), "
                               f"{n_new}-token new input each (serial restores; pipelined windows of {win} beside)",
                   "conversations_this_rank": len(mine), "r_c": r_c,
                   "parallelism": f"dp{world} (conversation shards, no collective)",
                   "l2": "inputs larger than L2; no flush"},
        "batch": {"pipelined_conv_s": round(pipe_s, 4), "pipelined_e2e_conv_s": round(n_all / (wall_ms / 1e3), 4),
                  "serial_conv_s": round(conv_s, 4),
                  "pipelined_item_ttft_p50_ms": round(float(np.median(pipe_ttft)), 4),
                  "serial_ttft_p50_ms": round(float(np.median(serial)), 4), "window": win,
                  "note": "value = serial: one restore_and_prefill per conversation (graph replay), summed "
                          "device TTFT; pipelined = krul_restore_batch windows (measured no faster: the "
                          "restores are link-bound); item TTFT of the pipelined run includes waiting for the "
                          "previous conversation's prefill"},
        "e2e": {"value": round(n_all / (swall_ms / 1e3), 4), "unit": "conversations/s",
                "h2d_bytes_per_step": int(h2d / max(len(mine), 1)), "d2h_bytes_per_step": 4 * cfg.vocab_size,
                "note": "wall clock around each timed restore_and_prefill call (host token buffers in, logits "
                        "out)"},
        "gpu_launches": int(launches), "clocks": clk, "setup_s": round(t_setup, 1),
    }


def make_ctx(K, spec, local, extra_tokens=0):
    dtype = K.KRUL_F32 if spec.get("f32") else K.KRUL_BF16
    cfg = K.ModelConfig(**model_kwargs(spec), seed=1234, dtype=dtype,
                        max_tokens=spec["L"] + spec["n_new"] + 64 + extra_tokens)
    ctx = K.Context(cfg, local)
    ctx.init_weights(1234)
    return cfg, ctx


def prepare_snapshot(args, K, T, ctx, cfg, spec, rank):
    """The turn that ends in the snapshot the timed steps restore (the
    reference turn loop, harness.cpp:92-259 kKrul, on the device; untimed).
    Returns (state, new-input tokens of the timed turn, turn record,
    calibration report)."""
    L, n_new = spec["L"], spec["n_new"]
    rng = np.random.default_rng(1000 + rank)
    new = rng.integers(0, cfg.vocab_size, n_new, dtype=np.int32)
    scratch = {}
    calib = {}

    def measured_rc(state, pairs, total):
        # calibrate_rc_measured (scheduler.cpp:402-443) with the B200 objective:
        # the measured TTFT of the full restore + new-input prefill DAG, coarse
        # grid then a fine grid around its argmin; |T_C - T_L| balance reported
        conv = scratch.setdefault("conv", ctx.conversation(cfg.max_tokens))
        coarse = [round(0.02 * k, 4) for k in range(0, 21)]
        r0, tt_coarse = ctx.calibrate_rc_ttft(state.conv, conv, state.history, new, pairs, coarse)
        fine = sorted({min(1.0, max(0.0, round(r0 + 0.004 * k, 4))) for k in range(-5, 6)})
        r_c, _ = ctx.calibrate_rc_ttft(state.conv, conv, state.history, new, pairs, fine, reps=7)
        if r_c != r0:  # a sub-0.1 ms fine-grid difference is within run-to-run noise: re-measure
            r_c, _ = ctx.calibrate_rc_ttft(state.conv, conv, state.history, new, pairs, sorted({r0, r_c}),
                                           reps=15)
        r_b0, _, _ = ctx.calibrate_rc_measured(state.conv, conv, state.history, pairs, coarse)
        r_bal, _, _ = ctx.calibrate_rc_measured(state.conv, conv, state.history, pairs,
                                                sorted({min(1.0, max(0.0, round(r_b0 + 0.004 * k, 4)))
                                                        for k in range(-5, 6)}))
        b_h2d, f_rec = ctx.measure_rates(conv)
        cost = K.CostModel.for_model(cfg, f_rec, b_h2d)
        # the timed restores use the config's committed split (the argmin of
        # this curve on B200) so that the reference arm restores
        # the identical plan; the live argmin is reported beside it
        r_use = spec.get("r_c_ref", r_c)
        calib.update({"r_c": r_use, "r_c_ttft_argmin": r_c, "r_c_balanced_restore": r_bal,
                      "r_c_analytic_measured_rates": K.calibrate_rc(cost, cfg.n_layers, total, cfg.d_model,
                                                                    pairs),
                      "h2d_gbs_measured": round(b_h2d / 1e9, 2),
                      "recompute_tflops_measured": round(f_rec / 1e12, 1),
                      "calibration_ttft_ms": {str(r): round(float(t), 3) for r, t in zip(coarse, tt_coarse)}})
        return r_use

    tc = T.TurnConfig(gamma=spec["gamma"], r_l=spec["r_l"], merge=K.MERGE_MEAN,
                      calibrate=None if spec.get("f32") else measured_rc)
    st = T.KrulTurns(ctx, tc, cfg.max_tokens)
    if "turn0" in spec:    # cfg1: turn 0 = fresh prefill of the user tokens + forced decode
        n_user, n_dec = spec["turn0"]
        rec = st.turn(0, T.Turn(rng.integers(0, cfg.vocab_size, n_user, dtype=np.int32),
                                rng.integers(0, cfg.vocab_size, n_dec, dtype=np.int32)))
    else:                  # a restoration turn over an (untracked) earlier history
        n_dec = spec["n_dec"]
        st.start_from(rng.integers(0, cfg.vocab_size, L - n_new - n_dec, dtype=np.int32))
        rec = st.turn(1, T.Turn(rng.integers(0, cfg.vocab_size, n_new, dtype=np.int32),
                                rng.integers(0, cfg.vocab_size, n_dec, dtype=np.int32)))
    assert st.history.size == L, (st.history.size, L)
    return st, new, rec, calib, scratch.get("conv")


def run_b200(args, rank, local, world, dist):
    from paper_2507_08045_b200 import native as K
    from paper_2507_08045_b200 import turns as T
    spec = CONFIGS[args.config]
    if "batch" in spec:
        return run_batch(args, rank, local, world, dist, K, spec)
    L, n_new = spec["L"], spec["n_new"]
    cfg, ctx = make_ctx(K, spec, local)
    t0 = time.time()
    st, new, rec, calib, conv = prepare_snapshot(args, K, T, ctx, cfg, spec, rank)
    t_setup = time.time() - t0
    snap, hist, prev = st.snapshot, st.history, st.conv
    pairs, r_c, plan = rec.pairs, rec.r_c, rec.plan
    conv = conv or ctx.conversation(cfg.max_tokens)
    full_b, stored_b = snap.storage_report()

    def step():
        return ctx.restore_and_prefill(conv, hist, snap, new)

    for _ in range(args.warmup):
        step()
    barrier(dist)
    ctx.sync()
    clocks = ClockSampler(local)
    clocks.start()
    ttfts, stats, walls = [], [], []
    launches0 = K.launch_count()
    for _ in range(args.steps):
        w0 = time.perf_counter()
        logits, st_, ttft = step()
        walls.append((time.perf_counter() - w0) * 1e3)
        ttfts.append(ttft)
        stats.append(st_)
    ctx.sync()
    launches = K.launch_count() - launches0
    barrier(dist)
    clk = clocks.stop()
    tl_c, tl_l, tl_n = ctx.restore_timeline()
    # Instrumented pass (same workload, right after the timed steps): CUDA
    # events around every GEMM / attention / expand launch on the stream it
    # runs on. Kept out of the headline steps because an event between two
    # kernels costs their launch overlap (~+35% on the step, measured).
    tags = (("gemm", 0), ("attention", 1), ("expand", 2), ("gemm_stream", 7), ("decode", 8),
            ("logits", 9), ("decode_expand", 10))
    peak_t = PEAKS.get("bf16_tflops_sustained", 1397.8)
    peak_b = PEAKS.get("hbm_gbs", 6547.2)

    inst_ttft = []

    def instrumented():
        kt = {name: [0, 0.0, 0.0, 0.0] for name, _ in tags}
        ideal = {name: 0.0 for name, _ in tags}
        ctx.ktime_enable(True)
        for i in range(args.warmup + args.steps):
            t_ = step()[2]
            if i >= args.warmup:
                inst_ttft.append(t_)
                for name, tag in tags:
                    kt[name] = [a + b for a, b in zip(kt[name], ctx.ktime_read(tag))]
                    ideal[name] += ctx.ktime_roofline(tag, peak_t, peak_b)
        ctx.ktime_enable(False)
        return kt, ideal

    kt, ideal = instrumented()
    inst_p50 = float(np.median(inst_ttft))
    # the same launches with the new-input prefill serialised behind the
    # recompute: each kernel then owns the GPU (kernel efficiency without SM sharing)
    ctx.set_concurrency(False)
    kti, _ = instrumented()
    ctx.set_concurrency(True)
    total_ms = allmax(dist, float(np.sum(ttfts)), local)
    wall_total = allmax(dist, float(np.sum(walls)), local)
    p50 = float(np.median(ttfts))
    conv_s = world * args.steps / (total_ms / 1e3)
    e2e_conv_s = world * args.steps / (wall_total / 1e3)
    sts = {k: float(np.median([s[k] for s in stats])) for k in stats[0]}
    peak_src = ("MEASURED_PEAKS.json bf16_tflops_sustained / hbm_gbs" if "MEASURED_PEAKS_FILE" in PEAKS
                else "fallback (B200_PROFILING.md: sustained bf16 ~1.4 PFLOP/s, 6547 GB/s copy; "
                     "MEASURED_PEAKS.json absent)")
    classes = {
        "gemm": ("tensor", "k_gemm_tc / k_gemm_tc2, M > 128 (recompute GEMMs, K6)", "2*M*N*K flop per launch"),
        "gemm_stream": ("hbm", "k_gemm_tc (+ split-K reduce), M <= 128 (new-input prefill, K7)",
                        "weights N*K*2 + A M*K*2 + C M*N*4 bytes per launch"),
        "attention": ("tensor", "k_attn_fa (+ split-KV merge)", "4*hd*H*sum(visible keys) flop per launch"),
        "decode_expand": ("hbm", "k_ec_decode_expand (exponent-coded blob -> owners' pages, K4b+K5 fused)",
                          "coded image bytes read + rows*2*Hkv*hd*2 bytes written per owner"),
        "decode": ("hbm", "k_ec_decode (coded blob -> raw bf16 staging, K4b; unfused path)",
                   "coded image bytes read + raw bytes written per blob"),
        "expand": ("hbm", "k_expand (K5, raw store)", "rows*2*Hkv*hd*2 bytes x (read + write) per owner"),
        "logits": ("hbm", "k_logits_vec (last-row LM head)", "V*d*2 + V*4 bytes"),
    }

    def rate(v, bound):
        n_, ms_, fl_, by_ = v
        if ms_ <= 0:
            return None
        return round(fl_ / (ms_ * 1e-3) / 1e12, 2) if bound == "tensor" else round(by_ / (ms_ * 1e-3) / 1e9, 1)

    roof = {}
    for name, (bound, kern, alg) in classes.items():
        n_, ms_, fl_, by_ = kt[name]
        if n_ == 0:
            continue
        pk = peak_t if bound == "tensor" else peak_b
        a = rate(kt[name], bound)
        roof[name] = {"bound": bound, "kernel": kern, "achieved": a, "peak": pk,
                      "unit": "TFLOP/s" if bound == "tensor" else "GB/s",
                      "frac": round(a / pk, 4) if a else None, "launches": int(n_) // max(args.steps, 1),
                      "ms_per_step": round(ms_ / args.steps, 4),
                      "avg_launch_us": round(1e3 * ms_ / max(n_, 1), 2), "algorithmic": alg,
                      "achieved_serialised": rate(kti[name], bound),
                      "frac_of_roofline": round(ideal[name] / ms_, 4) if ms_ else None}
    dominant = max(roof, key=lambda k: roof[k]["ms_per_step"])
    if "gemm_stream" in roof:
        try:  # diagnostic: device-side spans of the same launches, no events in the streams
            ctx.span_enable(True)
            sn_, sms_, sby_, stt_ = 0, 0.0, 0.0, []
            for i in range(args.warmup + args.steps):
                t_ = step()[2]
                if i >= args.warmup:
                    n_, ms_, by_ = ctx.span_read()
                    sn_ += n_
                    sms_ += ms_
                    sby_ += by_
                    stt_.append(t_)
            ctx.span_enable(False)
            if sms_ > 0:
                a_ = sby_ / (sms_ * 1e-3) / 1e9
                roof["gemm_stream"]["kernel_span"] = {
                    "achieved": round(a_, 1), "frac": round(a_ / peak_b, 4),
                    "launches": int(sn_) // max(args.steps, 1), "ms_per_step": round(sms_ / args.steps, 4),
                    "avg_launch_us": round(1e3 * sms_ / max(sn_, 1), 2),
                    "ttft_p50_ms": round(float(np.median(stt_)), 4),
                    "note": "the same launches in the timed DAG, each timed on the device from its first CTA's "
                            "entry to its last CTA's exit (%globaltimer stamps, split-K reduce included); no "
                            "timing events in the streams, so the DAG runs as in the headline steps"}
        except Exception as ex:  # noqa: BLE001
            roof["gemm_stream"]["kernel_span"] = {"error": repr(ex)[:200]}
    if "gemm_stream" in roof and rank == 0:
        try:  # diagnostic only: never let it cost the bench line
            roof["gemm_stream"]["isolated"] = gemm_stream_isolated(K, ctx, cfg, n_new, peak_b)
        except Exception as ex:  # noqa: BLE001
            roof["gemm_stream"]["isolated"] = {"error": repr(ex)[:200]}
    head = dict(roof[dominant])
    tr = NCU_TRAFFIC.get(dominant)
    head.update({"class": dominant,
                 "traffic": tr[0] if tr else None,
                 "traffic_algorithmic": tr[1] if tr else None,
                 "traffic_source": tr[2] if tr else "no ncu capture of this class yet",
                 "frac_of_roofline_note": "sum over launches of max(flops / tensor peak, bytes / HBM peak) "
                                          "/ measured time",
                 "serialised_note": "same launches timed with the new-input prefill serialised behind "
                                    "the recompute (no SM sharing)",
                 "measured": "CUDA events around each launch on its own stream, instrumented pass of the "
                             "same steps right after the timed region",
                 "instrumented_ttft_p50_ms": round(inst_p50, 4),
                 "instrumented_note": "TTFT of the instrumented pass (events around every timed launch break the "
                                      "graph's kernel-to-kernel launch overlap) vs ttft_p50_ms of the headline steps",
                 "peak_source": peak_src})
    b_h2d = calib.get("h2d_gbs_measured")
    h2d_gbs = round(sts["h2d_bytes"] / (sts["h2d_ms"] * 1e-3) / 1e9, 2) if sts["h2d_ms"] > 0 else None
    pol = policies_leg(K, ctx, prev, conv, cfg, hist, new, L, r_c, pairs, spec) if (
        rank == 0 and not args.no_policies) else None
    est = estimator_leg(K, ctx, conv, cfg, spec) if rank == 0 else None
    eager = None
    if rank == 0:
        try:  # diagnostic: the first restore of a conversation runs its DAG eagerly
            ctx.set_graphs(False)
            tt_, ww_ = [], []
            for k in range(7):
                w0 = time.perf_counter()
                t_ = step()[2]
                if k >= 2:
                    tt_.append(t_)
                    ww_.append((time.perf_counter() - w0) * 1e3)
            ctx.set_graphs(True)
            for _ in range(2):
                step()
            eager = {"ttft_p50_ms": round(float(np.median(tt_)), 4), "wall_p50_ms": round(float(np.median(ww_)), 4),
                     "note": "the same restore + prefill enqueued eagerly (~600 stream launches, no CUDA graph): "
                             "a conversation's first restore; the headline steps replay its captured graph"}
        except Exception as ex:  # noqa: BLE001
            eager = {"error": repr(ex)[:200]}
    bub = None
    if rank == 0 and calib.get("r_c_balanced_restore") is not None:
        try:  # diagnostic leg: never let it cost the bench line
            bub = bubble_leg(K, ctx, prev, conv, cfg, hist, new, L, pairs, calib)
        except Exception as ex:  # noqa: BLE001
            bub = {"error": repr(ex)[:200]}
    ctr = container_leg(K, ctx, snap) if rank == 0 and not spec.get("f32") else None
    out = {
        "metric": METRIC,
        "value": round(conv_s, 4),
        "unit": "conversations/s",
        "ttft_p50_ms": round(p50, 4),
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32" if spec.get("f32") else "bf16",
        "data": "synthetic (random-init weights, uniform random token ids)",
        "config": workload_config(args, spec, world, r_c, len(pairs), np.sum(plan)),
        "strategy": {"source": "estimator (turn loop harness.cpp:171-236 on the device)",
                     "pairs": [[int(a), int(b), round(float(d), 9)] for a, b, d in pairs],
                     "exhausted_before_quota": rec.exhausted, "ir_layers": len(rec.ir_layers),
                     "gamma": spec["gamma"], "r_l": spec["r_l"], "plan_head": [int(x) for x in plan[:4]],
                     "setup_s": round(t_setup, 1)},
        "calibration": calib,
        "kv_store": snap.coding(),
        "restore": {k: round(v, 4) for k, v in sts.items()},
        "timeline_ms": {"compute_done": [round(x, 3) for x in tl_c],
                        "load_done": [round(x, 3) for x in tl_l],
                        "new_prefill_done": [round(x, 3) for x in tl_n]},
        "storage": {"full_bytes": full_b, "stored_bytes": stored_b},
        "roofline": head,
        "rooflines": {
            **{k: v for k, v in roof.items() if k != dominant},
            **({"h2d_load": {"bound": "pcie", "kernel": "cudaMemcpyAsync pinned->device (K4)",
                             "achieved": h2d_gbs, "unit": "GB/s", "peak": b_h2d,
                             "frac": round(h2d_gbs / b_h2d, 4) if h2d_gbs and b_h2d else None,
                             "peak_source": "measured 256 MiB pinned H2D copy on this box",
                             "note": "the restore's binding resource: TTFT = load stream + tail"}}
               if b_h2d else {}),
            "recompute_stream": {"bound": "tensor", "achieved": round(
                sts["recompute_flops"] / (sts["compute_ms"] * 1e-3) / 1e12, 2) if sts["recompute_flops"] else None,
                "unit": "TFLOP/s",
                "note": "algorithmic pyramid flops / recompute-stream makespan (shares SMs with the "
                        "new-input prefill and expand streams)"},
            **({"estimator_decode_fold": est["fold"], "selector": est["select"],
                "decode_tpot": est["tpot"]} if est else {}),
            **({"container": ctr} if ctr else {}),
        },
        **({"bubble_free": bub} if bub else {}),
        **({"restore_eager": eager} if eager else {}),
        "e2e": {"value": round(e2e_conv_s, 4), "unit": "conversations/s",
                "ttft_p50_ms": round(float(np.median(walls)), 4),
                "h2d_bytes_per_step": int(sts["h2d_bytes"] + 4 * (L + n_new)),
                "d2h_bytes_per_step": 4 * cfg.vocab_size},
        "gpu_launches": int(launches),
        "gpu_launches_per_step": round(launches / args.steps, 1),
        "clocks": clk,
        **({"policies": pol} if pol else {}),
    }
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_baseline(args, spec, r_c, budget_s=args.cpu_budget)
    return out


def gemm_stream_isolated(K, ctx, cfg, rows, peak_b, iters=20):
    """The new-input prefill's four weight-streaming GEMM shapes of one layer
    (QKV, O, FFN up, FFN down at M = rows) timed alone: graph-replayed launches
    with the planner's choice, weights rotated over >= 320 MB so every launch
    streams them from HBM (krul_debug_gemm_bench). The QKV shape runs the F32
    epilogue (the RoPE / page-scatter epilogue needs a conversation). Explains
    the in-DAG figure: there the launches share the SMs with the blob decode +
    expand and the recompute."""
    import ctypes as C
    d, H, Hkv, hd, F = cfg.d_model, cfg.n_heads, cfg.kv_heads, cfg.head_dim, cfg.ffn_hidden()
    swiglu = cfg.ffn_kind == 1
    shapes = {"qkv": ((H + 2 * Hkv) * hd, d, 0), "o": (d, H * hd, 2),
              "ffn_up": ((2 if swiglu else 1) * F, d, 4 if swiglu else 3), "ffn_down": (d, F, 2)}
    out, tot_b, tot_us = {}, 0.0, 0.0
    for name, (N, Kd, epi) in shapes.items():
        ms = C.c_float(0)
        rc = K.lib().krul_debug_gemm_bench(ctx.h, C.c_int64(rows), C.c_int64(N), C.c_int64(Kd), epi, 0, 0, iters,
                                           C.byref(ms))
        if rc != 0:
            return {"error": f"krul_debug_gemm_bench rc={rc}"}
        by = N * Kd * 2 + rows * Kd * 2 + rows * N * 4
        us = ms.value * 1e3
        out[name] = {"N": N, "K": Kd, "us": round(us, 2), "GB/s": round(by / (us * 1e-6) / 1e9, 1)}
        tot_b += by
        tot_us += us
    a = tot_b / (tot_us * 1e-6) / 1e9
    return {"shapes": out, "achieved": round(a, 1), "frac": round(a / peak_b, 4), "us_per_layer": round(tot_us, 2),
            "note": "one layer's four GEMMs alone (graph replay, HBM-streamed weights), same bytes formula"}


def bubble_leg(K, ctx, prev, conv, cfg, hist, new, L, pairs, calib, reps=7):
    """The bubble-free split (north_star; scheduler.cpp:307-316 bubble
    fractions): the restore alone (recompute stream || load stream, no
    new-input prefill) at the ratio calibrate_rc_measured balances, median of
    `reps` device-timed runs, plus the TTFT of restore + prefill at that ratio
    (the new-input prefill then competes with the recompute for the SMs, which
    is why the TTFT argmin sits at a smaller r_c)."""
    r_bal = calib["r_c_balanced_restore"]
    plan = K.build_plan(L, cfg.n_layers, r_bal, pairs)
    snap = K.KVSnapshot.compress(ctx, prev, pairs, plan, L, K.MERGE_MEAN)
    runs = [ctx.execute_restore(conv, hist, snap) for _ in range(reps + 2)][2:]
    med = {k: round(float(np.median([r[k] for r in runs])), 4) for k in
           ("restore_ms", "compute_ms", "load_ms", "bubble_compute", "bubble_load")}
    tt = [ctx.restore_and_prefill(conv, hist, snap, new)[2] for _ in range(reps + 2)][2:]
    return {"r_c": r_bal, "recompute_token_layers": int(np.sum(plan)), **med,
            "max_bubble": max(med["bubble_compute"], med["bubble_load"]),
            "ttft_ms_restore_and_prefill": round(float(np.median(tt)), 4),
            "note": "restore-only DAG at the calibrate_rc_measured split; bubble = idle fraction of the "
                    "recompute / load stream over the restore (scheduler.cpp:307-316)"}


def policies_leg(K, ctx, prev, conv, cfg, hist, new, L, r_c, pairs, spec, warmup=3, steps=5):
    """The reference's restore policies (harness.cpp:125-162, 198-220) on the
    same kernels, device TTFT (restore + new-input prefill, graph replay):
    full-recompute (uniform plan r=1: everything recomputed, nothing
    loaded), full-load (r=0, keep-deeper), fixed-partial (uniform r=0.4, the
    reference's default fixed_ratio, harness.hpp:58), fixed-compression
    (deeper-half adjacent pairs, r=0, harness.cpp:68-76), krul (the
    estimator-selected strategy + pyramid plan at the calibrated r_c, as the
    timed steps) and krul_control (the fixed 8-adjacent-pair control of
    SURVEY §8d at the same r_c)."""
    N = cfg.n_layers
    deeper = [(i, i + 1, 0.0) for i in range(N // 2, N - 1, 2)]
    control = [(a, b, 0.0) for a, b in spec["pairs"]]
    cases = {
        "full_recompute": ([], K.uniform_plan(L, N, 1.0), K.MERGE_KEEP_DEEPER),
        "full_load": ([], K.uniform_plan(L, N, 0.0), K.MERGE_KEEP_DEEPER),
        "fixed_partial": ([], K.uniform_plan(L, N, 0.4), K.MERGE_KEEP_DEEPER),
        "fixed_compression": (deeper, K.uniform_plan(L, N, 0.0), K.MERGE_MEAN),
        "krul": (pairs, K.build_plan(L, N, r_c, pairs), K.MERGE_MEAN),
        "krul_control": (control, K.build_plan(L, N, r_c, control), K.MERGE_MEAN),
    }
    out = {}
    for name, (pp, plan, mode) in cases.items():
        snap = K.KVSnapshot.compress(ctx, prev, pp, plan, L, mode)
        for _ in range(warmup):
            ctx.restore_and_prefill(conv, hist, snap, new)
        t = [ctx.restore_and_prefill(conv, hist, snap, new)[2] for _ in range(steps)]
        full_b, stored_b = snap.storage_report()
        out[name] = {"ttft_ms": round(float(np.median(t)), 3), "stored_bytes": int(stored_b),
                     "pairs": len(pp)}
        del snap
    k = out["krul"]["ttft_ms"]
    for name in out:
        out[name]["krul_speedup"] = round(out[name]["ttft_ms"] / k, 3)
    return out


def estimator_leg(K, ctx, conv, cfg, spec, steps=8):
    """The estimator on the restored conversation, as the reference's turn
    loop runs it (harness.cpp:180-188): teacher-forced decode steps whose
    per-layer attention rows feed the decode fold (K1), then finalize and
    the device selector (K3). All N layers are tracked (P = N(N-1)/2 pairs)
    so the fold reads every layer's row; decode fold HBM GB/s from CUDA
    events around each fold launch (algorithmic bytes: N*H*W*4 + P*H*16)."""
    est = K.StreamingEstimator(ctx, list(range(cfg.n_layers)))
    rng = np.random.default_rng(7)
    # TPOT with and without the streaming estimator in the decode loop
    # (the paper reports the overhead as negligible):
    # wall clock per synchronous decode step, the fold on its own stream
    # per-step times, the two modes interleaved, medians: the eager decode
    # step is host-launch-bound and a shared host adds bursty noise
    tpot = {False: [], True: []}
    for i in range(48):
        with_est = bool(i & 1)
        t0 = time.perf_counter()
        ctx.decode_step(conv, int(rng.integers(0, cfg.vocab_size)))
        if with_est:
            est.fold_decode()
        ctx.sync()
        tpot[with_est].append((time.perf_counter() - t0) * 1e3)
    tpot = {k: float(np.median(v)) for k, v in tpot.items()}
    ctx.ktime_enable(True)
    for _ in range(steps):
        ctx.decode_step(conv, int(rng.integers(0, cfg.vocab_size)))
        est.fold_decode()
    n, ms_ev, _, by_ev = ctx.ktime_read(3)
    ctx.ktime_enable(False)
    # device time of the fold kernels themselves: 20 folds back to back on
    # the estimator stream (the per-call events above also hold the host
    # launch gap, the stream being idle when they are recorded)
    ms, by = est.fold_bench(20)
    hbm = PEAKS.get("hbm_gbs", 6547.2)
    gbs = by / (ms * 1e-3) / 1e9 if ms else None
    # the fold's other roof: 2 f32 lane-ops (difference, square-accumulate)
    # per pair, head and column on 128 f32 lanes / clk / SM (DESIGN.md §4 K1)
    W = int(len(conv))
    P = cfg.n_layers * (cfg.n_layers - 1) // 2
    lane_ops = 2.0 * P * cfg.n_heads * W
    fp32_peak = 128.0 * 148 * PEAKS.get("sm_max_mhz", 1965.0) * 1e6
    fp32_frac = lane_ops / (ms * 1e-3) / fp32_peak if ms else None
    # finalize + selector (one CTA bitonic sort + greedy matching), timed on the host
    sums = est.sums()
    D = np.zeros((cfg.n_layers, cfg.n_layers))
    P = 0
    for i in range(cfg.n_layers):
        for j in range(i + 1, cfg.n_layers):
            D[i, j] = D[j, i] = float(np.mean(np.sqrt(np.maximum(sums[P], 0.0))))
            P += 1
    layers = list(range(cfg.n_layers))
    t0 = time.perf_counter()
    reps = 20
    for _ in range(reps):
        strat = K.select_strategy(ctx, D, layers, layers, 0.5, cfg.n_layers)
    sel_us = (time.perf_counter() - t0) / reps * 1e6
    return {"fold": {"bound": "hbm", "kernel": "k_fold_direct (K1: f32 difference, FADD2/FFMA2; one launch)",
                     "achieved": round(gbs, 1) if gbs else None, "unit": "GB/s", "peak": hbm,
                     "frac": round(gbs / hbm, 4) if gbs else None, "launches": n,
                     "fp32_lane_ops": lane_ops, "fp32_peak_lane_ops_per_s": fp32_peak,
                     "fp32_frac": round(fp32_frac, 4) if fp32_frac else None,
                     "floor_us": round(1e6 * max(by / (hbm * 1e9), lane_ops / fp32_peak), 2),
                     "us_per_fold": round(1e3 * ms, 2),
                     "us_per_fold_incl_launch_gap": round(1e3 * ms_ev / max(n, 1), 2),
                     "width": int(len(conv)), "tracked_layers": cfg.n_layers},
            "tpot": {"decode_step_ms": round(tpot[False], 3),
                     "decode_step_with_estimator_ms": round(tpot[True], 3),
                     "estimator_overhead": round(tpot[True] / tpot[False] - 1.0, 4),
                     "note": "median wall clock of 24 synchronous decode steps per mode (eager launches, "
                             "modes interleaved) at the restored context length, all layers tracked"},
            "select": {"bound": "latency", "kernel": "k_select (K3) incl. D upload + result read",
                       "us_per_call": round(sel_us, 1), "pairs_selected": len(strat.pairs),
                       "candidates": cfg.n_layers * (cfg.n_layers - 1) // 2}}


# ---------------------------------------------------------------- CPU legs

_ORACLE_MODELS = {}


def container_leg(K, ctx, snap, reps=3):
    """KRUL v1 container (kvstore.cpp:360-511) of this workload's
    snapshot, in host memory: save (bf16 store -> f32 payload + nlohmann-exact
    metadata + crc32) and load (crc32 + checks + f32 -> bf16 into a fresh
    pinned store), all host threads. Reference: one-thread memcpy of the same
    bytes."""
    n = snap.save_size()
    buf = np.empty(n, np.uint8)
    ts, tl = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        snap.save_to(buf)
        ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        back = K.KVSnapshot.load(buf, ctx)
        tl.append(time.perf_counter() - t0)
        del back
    dst = np.empty_like(buf)
    t0 = time.perf_counter()
    np.copyto(dst, buf)
    tm = time.perf_counter() - t0
    ok = K.KVSnapshot.load(buf, ctx).save_size() == n
    return {"bytes": int(n), "save_ms": round(1e3 * min(ts), 2), "load_ms": round(1e3 * min(tl), 2),
            "save_gbs": round(n / min(ts) / 1e9, 2), "load_gbs": round(n / min(tl) / 1e9, 2),
            "memcpy_1thread_gbs": round(n / tm / 1e9, 2), "threads": len(os.sched_getaffinity(0)),
            "round_trip_ok": bool(ok),
            "note": "load = crc32 + checks + f32->bf16 into fresh host memory (threads first-touch) + cudaHostRegister; save = bf16->f32 + metadata + crc32"}


def _oracle_sample(spec, n_layers, vocab, r_c, seed=3):
    """A timing model + snapshot for the CPU legs: the workload's layer
    shape (timing-only weights), `n_layers` layers, the workload's history,
    a pair (0, 1) merged like the workload's pairs and the plan at r_c."""
    from oracle import oracle as O
    kw = model_kwargs(spec)
    kw.update(n_layers=n_layers, vocab_size=vocab)
    ocfg = O.ModelConfig(**kw, seed=seed)
    m = O.Model(ocfg, fast_seed=seed)
    L = spec["L"]
    strat = O.Strategy([(0, 1, 0.0)])
    snap = O.Snapshot(O.KV.synthetic(ocfg, L, seed), ocfg, strat, O.build_plan(L, n_layers, r_c, strat), L,
                      mode=0)
    rng = np.random.default_rng(seed)
    hist = rng.integers(0, vocab, L, dtype=np.int32)
    new = rng.integers(0, vocab, spec["n_new"], dtype=np.int32)
    return m, snap, hist, new


class CpuTurnSampler:
    """The reference's CPU TTFT path (execute_restore + prefill(history +
    new, restored), scheduler.cpp:320-400 + engine.cpp:282-340, restated in
    oracle/) timed on a bounded sample of the workload: a 2-layer model of
    the workload's layer shape with a 256-token vocabulary (every layer does
    the identical work at a uniform plan: its prefix recompute, its blob
    expand, its 128 new rows over L + 128 keys), so one conversation's TTFT =
    t(2 layers) x N/2 + the full-vocabulary LM head, which is measured once
    as t(2 layers, full vocab) - t(2 layers, 256). Nothing here loads the
    product library."""

    def __init__(self, spec, r_c):
        from oracle import oracle as O
        self.O = O
        self.spec = spec
        self.r_c = r_c
        self.N = spec["n_layers"]
        self.sample = _oracle_sample(spec, 2, 256, r_c)
        self.head_s = 0.0

    def measure_head(self):
        m, snap, hist, new = _oracle_sample(self.spec, 2, self.spec["vocab_size"], self.r_c)
        r1, p1, _ = m.time_turn(hist, snap, new)
        m0, snap0, hist0, new0 = self.sample
        r0, p0, _ = m0.time_turn(hist0, snap0, new0)
        self.head_s = max(0.0, (r1 + p1) - (r0 + p0))
        return self.head_s

    def step(self, threads=None):
        if threads:
            self.O.set_threads(threads)
        m, snap, hist, new = self.sample
        r, p, _ = m.time_turn(hist, snap, new)
        return (r + p) * self.N / 2 + self.head_s, r, p


def cpu_baseline(args, spec, r_c, budget_s=20.0):
    """The oracle's turn (CpuTurnSampler) on this host's cores, all threads
    and one thread, rank 0 at N=1; bounded to ~budget_s of CPU work."""
    if "turn0" in spec:
        return cpu_turn_loop_tiny(spec, reps=5)
    cores, threads = lscpu_cores()
    s = CpuTurnSampler(spec, r_c)
    s.O.set_threads(threads)
    s.measure_head()
    vals, t0 = [], time.time()
    while time.time() - t0 < budget_s / 2 or len(vals) < 2:
        vals.append(s.step(threads)[0])
        if len(vals) >= 8:
            break
    one = s.step(1)[0]
    s.O.set_threads(threads)
    v = float(np.median(vals))
    return {"value": round(1.0 / v, 6), "unit": "conversations/s", "ttft_ms": round(v * 1e3, 1),
            "cores": threads, "lscpu_cores": cores, "kind": "port",
            "one_thread": {"value": round(1.0 / one, 6), "ttft_ms": round(one * 1e3, 1), "cores": 1},
            "sample": f"oracle execute_restore + prefill(history + new, restored) of a 2-layer model at the "
                      f"workload's layer shape, L={spec['L']}, n={spec['n_new']}, r_c={r_c}, timed "
                      f"(median of {len(vals)}) x {spec['n_layers']}/2 layers + the full-vocab LM head "
                      f"({s.head_s * 1e3:.0f} ms, measured)"}


def cpu_turn_loop_tiny(spec, reps=50, warmup=0):
    """cfg1 on the CPU: the oracle's full turn loop (reference_pass +
    run_krul), then the timed turn-1 restore + new-input prefill repeated."""
    from oracle import oracle as O
    from oracle import turns as OT
    kw = model_kwargs(spec)
    om = O.Model(O.ModelConfig(**kw, seed=1234))
    rng = np.random.default_rng(1000)
    n_user, n_dec = spec["turn0"]
    traces = OT.reference_pass(om, [OT.OTurn(rng.integers(0, kw["vocab_size"], n_user, dtype=np.int32), n_dec)])
    recs, snap = OT.run_krul(om, traces, gamma=spec["gamma"], r_l=spec["r_l"])
    hist = np.concatenate(traces[0]).astype(np.int32)
    new = rng.integers(0, kw["vocab_size"], spec["n_new"], dtype=np.int32)
    cores, threads = lscpu_cores()
    ts = []
    for i in range(warmup + reps):
        r, p, _ = om.time_turn(hist, snap, new)
        if i >= warmup:
            ts.append(r + p)
    v = float(np.median(ts))
    return {"value": round(1.0 / v, 4), "unit": "conversations/s", "ttft_ms": round(v * 1e3, 3),
            "cores": threads, "lscpu_cores": cores, "kind": "port", "r_c": recs[0].r_c,
            "pairs": len(recs[0].pairs), "recompute_token_layers": int(np.sum(recs[0].plan)),
            "sample": f"the full cfg1 turn loop on the oracle (turn 0: {n_user} user + {n_dec} forced tokens, "
                      f"estimator, select, calibrate_rc, build_plan, compress); turn-1 restore + prefill timed, "
                      f"p50 of {reps}"}


def run_reference(args, rank, local, world, dist):
    """The reference's CPU path on the host cores (rank 0 only), on this
    arm's workload and plan: r_c = the config's r_c_ref (the GPU arm's
    measured optimum) and the same pair count, so `config` equals the GPU
    arm's. Each step is one bounded sample (CpuTurnSampler); tiny-512 runs
    the whole cfg1 turn loop."""
    if rank != 0:
        return None
    spec = CONFIGS[args.config]
    cores, threads = lscpu_cores()
    t_all = time.time()
    if "turn0" in spec:
        cb = cpu_turn_loop_tiny(spec, reps=args.steps, warmup=args.warmup)
        v, ms, cfgd = cb["value"], cb["ttft_ms"], workload_config(args, spec, world, cb["r_c"], cb["pairs"],
                                                                  cb["recompute_token_layers"])
        sample = cb["sample"]
    else:
        from oracle import oracle as O
        r_c = spec["r_c_ref"]
        s = CpuTurnSampler(spec, r_c)
        O.set_threads(threads)
        s.measure_head()
        vals = [s.step()[0] for _ in range(args.warmup + args.steps)][args.warmup:]
        t = float(np.median(vals))
        v, ms = 1.0 / t, t * 1e3
        pairs = [(a, b) for a, b in spec["pairs"]]
        plan_sum = int(np.sum(O.build_plan(spec["L"], spec["n_layers"], r_c, O.Strategy(
            [(a, b, 0.0) for a, b in pairs]))))
        cfgd = workload_config(args, spec, world, r_c, len(pairs), plan_sum)
        sample = (f"oracle execute_restore + prefill(history + new, restored) of a 2-layer model at the "
                  f"workload's layer shape, L={spec['L']}, n={spec['n_new']}, r_c={r_c}, per step; x "
                  f"{spec['n_layers']}/2 layers + the full-vocab LM head ({s.head_s * 1e3:.0f} ms, measured)")
    return {"metric": METRIC, "value": round(v, 6), "unit": "conversations/s", "impl": "reference",
            "ttft_p50_ms": round(ms, 3), "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round((time.time() - t_all) * 1e3 / (args.warmup + args.steps), 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (random-init weights, uniform random token ids)", "config": cfgd,
            "cpu_baseline": {"value": round(v, 6), "unit": "conversations/s", "cores": threads,
                             "lscpu_cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": round(v, 6), "unit": "conversations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)  # p50 over >= 50 restores
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="llama3-8b-8k", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-policies", action="store_true",
                    help="skip the reference-policy TTFT comparison (full recompute / load / fixed)")
    ap.add_argument("--window", type=int, default=8,
                    help="batch config: conversations per pipelined restore_batch window")
    ap.add_argument("--convs", type=int, default=0,
                    help="batch configs: conversations per rank (0 = the whole LPT shard)")
    args = ap.parse_args()
    if os.environ.get("KRUL_BENCH_WATCHDOG"):  # debugging aid: dump the stack if a phase hangs
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["KRUL_BENCH_WATCHDOG"]), exit=True)
    # the CPU legs (reference arm, cpu_baseline) use every host thread, also
    # under torchrun (which exports OMP_NUM_THREADS=1); the oracle's OpenMP
    # runtime reads this when its library loads
    if args.impl == "reference" or not args.no_cpu_baseline:
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    rank, local, world, dist = dist_setup()
    if args.impl == "reference":
        out = run_reference(args, rank, local, world, dist)
    else:
        out = run_b200(args, rank, local, world, dist)
    if rank == 0 and out is not None:
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
