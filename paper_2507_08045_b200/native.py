"""ctypes binding of include/krul_b200.h — the Python mirror of the
reference's hot-path interface (/root/reference/proj/include/krul/*.hpp).

Names follow the reference (classify_layers, StreamingEstimator,
select_strategy, build_plan, calibrate_rc, compress_and_snapshot, expand,
execute_restore, ...). Every call goes through libkrul_b200.so; there is no
CPU fallback: importing this module on a machine without the built library
raises, and any device entry fails loudly with CudaError when no GPU exists.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# KRUL_LIB: an alternate build of the same library (A/B timing experiments)
LIB_PATH = os.environ.get("KRUL_LIB") or os.path.join(HERE, "_lib", "libkrul_b200.so")

KRUL_F32, KRUL_BF16 = 0, 1
FFN_TANH, FFN_SWIGLU = 0, 1
MERGE_MEAN, MERGE_KEEP_DEEPER = 0, 1


# ---- reference exception types (common.hpp:25-63) ---------------------------
class KrulError(RuntimeError):
    code = -1


class ConfigError(KrulError):
    code = 1


class RestorationGapError(KrulError):
    code = 2


class StateCorruptionError(KrulError):
    code = 3


class AccountingError(KrulError):
    code = 4


class PlanInvalidError(KrulError):
    code = 5


class ClassificationError(KrulError):
    code = 6


class SnapshotError(KrulError):
    code = 7


class SnapshotLoadError(KrulError):
    """kvstore::load failure; `field` names the container field that failed
    (kvstore.hpp SnapshotLoadError::field)."""
    code = 8
    field = ""


class CudaError(KrulError):
    code = 9


class ArgError(KrulError):
    code = 10


_ERRORS = {c.code: c for c in (ConfigError, RestorationGapError, StateCorruptionError,
                               AccountingError, PlanInvalidError, ClassificationError,
                               SnapshotError, SnapshotLoadError, CudaError, ArgError)}


class ModelDesc(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int), ("n_heads", C.c_int), ("n_kv_heads", C.c_int),
        ("head_dim", C.c_int), ("d_model", C.c_int), ("vocab_size", C.c_int),
        ("ffn_mult", C.c_float), ("ffn_kind", C.c_int), ("seed", C.c_uint64),
        ("rope_theta", C.c_double), ("dtype", C.c_int), ("max_tokens", C.c_int64),
    ]


class Pair(C.Structure):
    _fields_ = [("shallow", C.c_int), ("deep", C.c_int), ("distance", C.c_double)]


class CostModelC(C.Structure):
    _fields_ = [("f_peak", C.c_double), ("b_peak", C.c_double), ("ffn_mult", C.c_double),
                ("kv_dim", C.c_int64), ("q_dim", C.c_int64), ("ffn_hidden", C.c_int64),
                ("bytes_per_elem", C.c_double), ("ffn_kind", C.c_int)]


class BlobSpecC(C.Structure):
    _fields_ = [("owners", C.c_int * 2), ("start", C.c_int64), ("end", C.c_int64)]


class SnapshotMetaC(C.Structure):
    _fields_ = [("conversation_id", C.c_char_p), ("exhausted_before_quota", C.c_int),
                ("ir_layers", C.c_void_p), ("n_ir_layers", C.c_int),
                ("non_ir_layers", C.c_void_p), ("n_non_ir_layers", C.c_int),
                ("avg_weight_sum", C.c_void_p), ("n_avg_weight_sum", C.c_int)]


class RestoreStats(C.Structure):
    _fields_ = [("restore_ms", C.c_double), ("compute_ms", C.c_double), ("load_ms", C.c_double),
                ("bubble_compute", C.c_double), ("bubble_load", C.c_double),
                ("h2d_bytes", C.c_double), ("expand_bytes", C.c_double),
                ("recompute_flops", C.c_double), ("h2d_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Loads the B200 library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                              "(the CUDA extension is required; there is no CPU path)")
        _lib = C.CDLL(LIB_PATH)
        _lib.krul_snapshot_n_blobs.argtypes = [C.c_void_p]
        _lib.krul_crc32.restype = C.c_uint32
        _lib.krul_crc32.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32]
    return _lib


def crc32(data: bytes, crc: int = 0) -> int:
    """common.cpp:34-42 (host threads for large buffers)."""
    return lib().krul_crc32(data, len(data), crc)


def _check(rc):
    if rc != 0:
        buf = C.create_string_buffer(1024)
        lib().krul_last_error(buf, 1024)
        raise _ERRORS.get(rc, KrulError)(buf.value.decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _pairs(pairs):
    pairs = list(pairs or [])
    arr = (Pair * max(1, len(pairs)))()
    for i, p in enumerate(pairs):
        arr[i] = Pair(int(p[0]), int(p[1]), float(p[2]) if len(p) > 2 else 0.0)
    return arr, len(pairs)


@dataclass
class ModelConfig:
    """engine.hpp:17-29 ModelConfig + extensions (n_kv_heads, ffn_kind, rope_theta)."""
    n_layers: int = 4
    n_heads: int = 2
    head_dim: int = 8
    d_model: int = 16
    vocab_size: int = 64
    ffn_mult: float = 4.0
    seed: int = 0
    n_kv_heads: int = 0
    ffn_kind: int = FFN_TANH
    rope_theta: float = 10000.0
    dtype: int = KRUL_F32
    max_tokens: int = 1024

    def desc(self):
        return ModelDesc(self.n_layers, self.n_heads, self.n_kv_heads, self.head_dim, self.d_model,
                         self.vocab_size, self.ffn_mult, self.ffn_kind, self.seed, self.rope_theta,
                         self.dtype, self.max_tokens)

    @property
    def kv_heads(self):
        return self.n_kv_heads or self.n_heads

    def ffn_hidden(self):
        return int(np.round(np.float32(self.ffn_mult) * np.float32(self.d_model)))

    def hash(self):
        out = C.c_uint64()
        d = self.desc()
        _check(lib().krul_config_hash(C.byref(d), C.byref(out)))
        return out.value


# ---- context / conversations -------------------------------------------------

class Context:
    """One CUDA device + weights + streams (krul_ctx)."""

    def __init__(self, cfg: ModelConfig, device: int = 0):
        self.cfg = cfg
        h = C.c_void_p()
        d = cfg.desc()
        _check(lib().krul_ctx_create(device, C.byref(d), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().krul_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload_weights(self, w: np.ndarray):
        w = np.ascontiguousarray(w, np.float32)
        _check(lib().krul_weights_upload_f32(self.h, _p(w), C.c_int64(w.size)))

    def init_weights(self, seed: int):
        _check(lib().krul_weights_init_device(self.h, C.c_uint64(seed)))

    def conversation(self, capacity=None) -> "Conversation":
        return Conversation(self, capacity or self.cfg.max_tokens)

    def set_kv_coding(self, on: bool):
        """Exponent-code bf16 snapshots at compress (lossless; default on)."""
        _check(lib().krul_set_kv_coding(self.h, int(bool(on))))

    def set_capture(self, mode):
        """Attention capture of later prefills: False/0 off, True/1 the
        reference's materialised probability record, 2 the estimator's
        recompute mode (Q rows + softmax statistics; fold_prefill recomputes
        the probabilities chunk by chunk)."""
        _check(lib().krul_set_capture(self.h, int(mode)))

    def set_classifier_regions(self, initial_frac=0.1, recent_frac=0.1):
        _check(lib().krul_set_classifier_regions(self.h, C.c_double(initial_frac),
                                                  C.c_double(recent_frac)))

    def sync(self):
        _check(lib().krul_ctx_sync(self.h))

    # -- engine (engine.hpp:106-139)
    def prefill(self, conv, tokens):
        t = np.ascontiguousarray(tokens, np.int32)
        out = np.empty(self.cfg.vocab_size, np.float32)
        _check(lib().krul_prefill(self.h, conv.h, _p(t), C.c_int64(t.size), _p(out)))
        return out

    def prefill_new(self, conv, tokens):
        t = np.ascontiguousarray(tokens, np.int32)
        out = np.empty(self.cfg.vocab_size, np.float32)
        _check(lib().krul_prefill_new(self.h, conv.h, _p(t), C.c_int64(t.size), _p(out)))
        return out

    def decode_step(self, conv, token: int):
        out = np.empty(self.cfg.vocab_size, np.float32)
        _check(lib().krul_decode_step(self.h, conv.h, C.c_int32(int(token)), _p(out)))
        return out

    def partial_prefix_recompute(self, conv, tokens, recompute_len):
        t = np.ascontiguousarray(tokens, np.int32)
        p = np.ascontiguousarray(recompute_len, np.int64)
        _check(lib().krul_partial_recompute(self.h, conv.h, _p(t), C.c_int64(t.size), _p(p),
                                            len(p)))

    def captured_prefill(self):
        """[N, H, rows, width] f32 of the last prefill (capture must be on)."""
        cfg = self.cfg
        r, w = C.c_int64(), C.c_int64()
        _check(lib().krul_capture_prefill(self.h, 0, 0, None, C.byref(r), C.byref(w)))
        out = np.empty((cfg.n_layers, cfg.n_heads, r.value, w.value), np.float32)
        for l in range(cfg.n_layers):
            for hh in range(cfg.n_heads):
                buf = np.empty((r.value, w.value), np.float32)
                _check(lib().krul_capture_prefill(self.h, l, hh, _p(buf), None, None))
                out[l, hh] = buf
        return out

    def captured_decode(self):
        w = C.c_int64()
        _check(lib().krul_capture_decode(self.h, None, C.byref(w)))
        cfg = self.cfg
        out = np.empty((cfg.n_layers, cfg.n_heads, w.value), np.float32)
        _check(lib().krul_capture_decode(self.h, _p(out), None))
        return out

    def classify_layers(self, gamma=0.5, initial_frac=0.1, recent_frac=0.1):
        """analysis.cpp:20-63 over the last prefill -> (avg_weight_sum, ir, non_ir)."""
        N = self.cfg.n_layers
        avg = np.empty(N, np.float64)
        ir = np.empty(N, np.int32)
        _check(lib().krul_classify(self.h, C.c_double(gamma), C.c_double(initial_frac),
                                   C.c_double(recent_frac), _p(avg), _p(ir)))
        return avg, [l for l in range(N) if ir[l]], [l for l in range(N) if not ir[l]]

    def restore_timeline(self):
        """Per-layer ms from restore launch: (compute[l], load[l], new_prefill[l])."""
        N = self.cfg.n_layers
        a, b, c = (np.zeros(N, np.float64) for _ in range(3))
        _check(lib().krul_restore_timeline(self.h, _p(a), _p(b), _p(c)))
        return a, b, c

    def calibrate_rc_measured(self, prev, scratch, history, pairs, grid, mode=1):
        """scheduler.cpp:402-443 on the device -> (r_c, tc[ms], tl[ms]) over the sorted grid."""
        t = np.ascontiguousarray(history, np.int32)
        arr, n = _pairs(pairs)
        g = np.ascontiguousarray(sorted(grid), np.float64)
        tc, tl = np.zeros(len(g)), np.zeros(len(g))
        r = C.c_double()
        _check(lib().krul_calibrate_rc_measured(self.h, prev.h, scratch.h, _p(t), C.c_int64(t.size),
                                                arr, n, _p(g), len(g), mode, C.byref(r), _p(tc),
                                                _p(tl)))
        return r.value, tc, tl

    def calibrate_rc_ttft(self, prev, scratch, history, new_tokens, pairs, grid, mode=1, reps=3):
        """calibrate_rc_measured with the measured TTFT of restore + new-input
        prefill as the objective -> (r_c, ttft[ms]) over the sorted grid."""
        t = np.ascontiguousarray(history, np.int32)
        nt = np.ascontiguousarray(new_tokens, np.int32)
        arr, n = _pairs(pairs)
        g = np.ascontiguousarray(sorted(grid), np.float64)
        tt = np.zeros(len(g))
        r = C.c_double()
        _check(lib().krul_calibrate_rc_ttft(self.h, prev.h, scratch.h, _p(t), C.c_int64(t.size),
                                            _p(nt), C.c_int64(nt.size), arr, n, _p(g), len(g),
                                            mode, reps, C.byref(r), _p(tt)))
        return r.value, tt

    def set_timeline(self, on: bool):
        """Record per-layer timeline events in the restore DAG (diagnostic)."""
        _check(lib().krul_set_timeline(self.h, int(bool(on))))

    def span_enable(self, on: bool):
        """Stamp device-side spans of the weight-streaming GEMMs of each restore."""
        _check(lib().krul_span_enable(self.h, int(bool(on))))

    def span_read(self):
        """(launches, span ms, algorithmic bytes) of the last restore's stamped GEMMs."""
        n, ms, by = C.c_int64(), C.c_double(), C.c_double()
        _check(lib().krul_span_read(self.h, C.byref(n), C.byref(ms), C.byref(by)))
        return n.value, ms.value, by.value

    def set_graphs(self, on: bool):
        """Graph-capture repeated restore DAGs (default) or enqueue every restore eagerly."""
        _check(lib().krul_set_graphs(self.h, int(bool(on))))

    def set_fused_recompute(self, on: bool):
        """Fold the recompute rows into the new-input prefill's layer steps (default off)."""
        _check(lib().krul_set_fused_recompute(self.h, int(bool(on))))

    def set_concurrency(self, two_stream: bool):
        """Restore DAG mode: new-input prefill concurrent with the recompute (default)
        or serialised behind it."""
        _check(lib().krul_set_concurrency(self.h, int(bool(two_stream))))

    def ktime_enable(self, on: bool):
        _check(lib().krul_ktime_enable(self.h, int(bool(on))))

    def ktime_read(self, tag: int):
        """(launches, ms, flops, bytes) of the timed launches of a kernel class."""
        n, ms, fl, by = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
        _check(lib().krul_ktime_read(self.h, tag, C.byref(n), C.byref(ms), C.byref(fl), C.byref(by)))
        return n.value, ms.value, fl.value, by.value

    def ktime_roofline(self, tag: int, peak_tflops: float, peak_gbs: float) -> float:
        """ms the timed launches of a class would take at their binding roof."""
        v = C.c_double()
        _check(lib().krul_ktime_roofline(self.h, tag, C.c_double(peak_tflops), C.c_double(peak_gbs),
                                         C.byref(v)))
        return v.value

    def measure_rates(self, scratch):
        b, f = C.c_double(), C.c_double()
        _check(lib().krul_measure_rates(self.h, scratch.h, C.byref(b), C.byref(f)))
        return b.value, f.value

    # -- restore (scheduler.cpp:320-400)
    def execute_restore(self, conv, history, snapshot):
        t = np.ascontiguousarray(history, np.int32)
        st = RestoreStats()
        _check(lib().krul_restore(self.h, conv.h, snapshot.h, _p(t), C.c_int64(t.size),
                                  C.byref(st)))
        return st.as_dict()

    def restore_and_prefill(self, conv, history, snapshot, new_tokens):
        t = np.ascontiguousarray(history, np.int32)
        n = np.ascontiguousarray(new_tokens, np.int32)
        out = np.empty(self.cfg.vocab_size, np.float32)
        st = RestoreStats()
        ttft = C.c_double()
        _check(lib().krul_restore_and_prefill(self.h, conv.h, snapshot.h, _p(t),
                                              C.c_int64(t.size), _p(n), C.c_int64(n.size),
                                              _p(out), C.byref(st), C.byref(ttft)))
        return out, st.as_dict(), ttft.value


    def restore_batch(self, convs, histories, snapshots, new_tokens, logits=False):
        """Pipelined restore + new-input prefill of a batch (conversation i+1's
        copies under conversation i's prefill tail) -> (ttft_ms[n], total_ms,
        logits[n][V] or None). Consecutive items need different conversations."""
        n = len(convs)
        hs = [np.ascontiguousarray(h, np.int32) for h in histories]
        ns = [np.ascontiguousarray(t, np.int32) for t in new_tokens]
        cv = (C.c_void_p * n)(*[c.h.value if isinstance(c.h, C.c_void_p) else c.h for c in convs])
        sv = (C.c_void_p * n)(*[s.h.value if isinstance(s.h, C.c_void_p) else s.h for s in snapshots])
        hp = (C.c_void_p * n)(*[h.ctypes.data for h in hs])
        npp = (C.c_void_p * n)(*[t.ctypes.data for t in ns])
        Ls = np.array([h.size for h in hs], np.int64)
        nn = np.array([t.size for t in ns], np.int64)
        tt = np.zeros(n, np.float64)
        tot = C.c_double()
        out = np.empty((n, self.cfg.vocab_size), np.float32) if logits else None
        _check(lib().krul_restore_batch(self.h, n, cv, sv, hp, _p(Ls), npp, _p(nn),
                                        _p(out) if out is not None else None, _p(tt), C.byref(tot)))
        return tt, tot.value, out


class Conversation:
    """Paged KV cache of one conversation (krul_conv)."""

    def __init__(self, ctx: Context, capacity: int):
        self.ctx = ctx
        h = C.c_void_p()
        _check(lib().krul_conv_create(ctx.h, C.c_int64(capacity), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().krul_conv_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self):
        n = C.c_int64()
        _check(lib().krul_conv_length(self.h, C.byref(n)))
        return n.value

    def kv(self, layer, start, end):
        cfg = self.ctx.cfg
        k = np.zeros((cfg.kv_heads, max(0, end - start), cfg.head_dim), np.float32)
        v = np.zeros_like(k)
        _check(lib().krul_conv_kv_read(self.h, layer, C.c_int64(start), C.c_int64(end), _p(k),
                                       _p(v)))
        return k, v

    def write_kv(self, layer, start, end, k, v):
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        _check(lib().krul_conv_kv_write(self.h, layer, C.c_int64(start), C.c_int64(end), _p(k),
                                        _p(v)))


# ---- analysis: streaming estimator (analysis.hpp:96-126) ---------------------

class StreamingEstimator:
    def __init__(self, ctx: Context, ir_layers):
        self.ctx = ctx
        ir = np.ascontiguousarray(list(ir_layers) or [0], np.int32)
        h = C.c_void_p()
        _check(lib().krul_est_create(ctx.h, _p(ir), len(list(ir_layers)), C.byref(h)))
        self.h = h
        self.layers = sorted(set(int(x) for x in ir_layers))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib().krul_est_destroy(self.h)

    def fold_prefill(self):
        _check(lib().krul_est_fold_prefill(self.h))

    def fold_decode(self):
        _check(lib().krul_est_fold_decode(self.h))

    def fold_prefill_rows(self, probs):
        p = np.ascontiguousarray(probs, np.float32)
        N, H, R, W = p.shape
        _check(lib().krul_est_fold_prefill_host(self.h, _p(p), N, C.c_int64(R), C.c_int64(W)))

    def set_sampling(self, stride: int):
        """Opt-in sampled token subset for the decode folds (every stride-th
        64-column block, rotating per step, scaled to the full width); 1 =
        every column, the reference's fold."""
        _check(lib().krul_est_set_sampling(self.h, int(stride)))

    def fold_decode_rows(self, rows):
        r = np.ascontiguousarray(rows, np.float32)
        N, H, W = r.shape
        _check(lib().krul_est_fold_decode_host(self.h, _p(r), N, C.c_int64(W)))

    def sums(self):
        n = len(self.layers)
        out = np.zeros(max(1, n * (n - 1) // 2 * self.ctx.cfg.n_heads), np.float64)
        _check(lib().krul_est_sums(self.h, _p(out)))
        return out[: n * (n - 1) // 2 * self.ctx.cfg.n_heads]

    def finish(self):
        n = len(self.layers)
        D = np.zeros((max(n, 1), max(n, 1)), np.float64)
        _check(lib().krul_est_finalize(self.h, _p(D)))
        return D[:n, :n]

    def fold_bench(self, iters=20):
        """(ms, algorithmic bytes) of one decode fold on the last captured
        decode rows, device-timed back to back (state untouched)."""
        ms, by = C.c_float(), C.c_double()
        _check(lib().krul_est_fold_bench(self.h, iters, C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def counts(self):
        a, b = C.c_int64(), C.c_int64()
        _check(lib().krul_est_counts(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value


# ---- strategy (strategy.hpp:37-44) -------------------------------------------

@dataclass
class CompressionStrategy:
    pairs: list = field(default_factory=list)  # [(shallow, deep, distance)]
    exhausted_before_quota: bool = False

    @property
    def shared(self):
        return sorted({x for p in self.pairs for x in p[:2]})


def launch_count() -> int:
    """Kernels launched by this library in this process (bench evidence)."""
    v = C.c_uint64()
    _check(lib().krul_launch_count(C.byref(v)))
    return v.value


def shared_layer_quota(n_layers, r_l):
    out = C.c_int()
    _check(lib().krul_quota(n_layers, C.c_double(r_l), C.byref(out)))
    return out.value


def select_strategy(ctx: Context, D, dm_layers, ir_layers, r_l, n_layers) -> CompressionStrategy:
    """K3 on the device: sort (d, i, j) + greedy disjoint matching."""
    D = np.ascontiguousarray(D, np.float64)
    dl = np.ascontiguousarray(list(dm_layers) or [0], np.int32)
    ir = np.ascontiguousarray(list(ir_layers) or [0], np.int32)
    out = (Pair * max(1, len(list(ir_layers))))()
    n, ex = C.c_int(), C.c_int()
    _check(lib().krul_select(ctx.h, _p(D), _p(dl), len(list(dm_layers)), _p(ir),
                             len(list(ir_layers)), C.c_double(r_l), n_layers, out, C.byref(n),
                             C.byref(ex)))
    return CompressionStrategy([(out[i].shallow, out[i].deep, out[i].distance)
                                for i in range(n.value)], bool(ex.value))


VIOLATION_KINDS = {1: "pair orientation", 2: "layer range", 4: "non-I-R member", 8: "layer reuse",
                   16: "distance order", 32: "shared size", 64: "quota shortfall"}


def validate_strategy(strategy: CompressionStrategy, ir_layers, n_layers, r_l, shared=None):
    """strategy.cpp:76-131 -> (bitmask, ["kind: detail", ...]). `shared`
    defaults to the union of the pair members (CompressionStrategy::shared)."""
    arr, n = _pairs(strategy.pairs)
    sh = list(strategy.shared if shared is None else shared)
    sd = np.ascontiguousarray(sh or [0], np.int32)
    ir = np.ascontiguousarray(list(ir_layers) or [0], np.int32)
    m = C.c_int()
    buf = C.create_string_buffer(8192)
    _check(lib().krul_validate_strategy(arr, n, _p(sd), len(sh), int(bool(strategy.exhausted_before_quota)),
                                        _p(ir), len(list(ir_layers)), n_layers, C.c_double(r_l),
                                        C.byref(m), buf, C.c_size_t(len(buf))))
    return m.value, [x for x in buf.value.decode().split("\n") if x]


# ---- scheduler (scheduler.hpp:14-112) ----------------------------------------

@dataclass
class CostModel:
    f_peak: float = 312e12
    b_peak: float = 139e9
    ffn_mult: float = 4.0
    kv_dim: int = 0
    q_dim: int = 0
    ffn_hidden: int = 0
    bytes_per_elem: float = 0.0
    ffn_kind: int = 0

    def c(self):
        return CostModelC(self.f_peak, self.b_peak, self.ffn_mult, self.kv_dim, self.q_dim,
                          self.ffn_hidden, self.bytes_per_elem, self.ffn_kind)

    @staticmethod
    def for_model(cfg: ModelConfig, f_peak, b_peak):
        """Cost model with the model's real KV width, FFN and storage dtype."""
        return CostModel(f_peak, b_peak, cfg.ffn_mult, cfg.kv_heads * cfg.head_dim,
                         cfg.n_heads * cfg.head_dim, cfg.ffn_hidden(),
                         2.0 if cfg.dtype == KRUL_BF16 else 4.0, cfg.ffn_kind)


def build_plan(L, N, r_c, pairs=()):
    arr, n = _pairs(pairs)
    out = np.empty(N, np.int64)
    _check(lib().krul_build_plan(C.c_int64(L), N, C.c_double(r_c), arr, n, _p(out)))
    return out


def uniform_plan(L, N, r_c):
    out = np.empty(N, np.int64)
    _check(lib().krul_uniform_plan(C.c_int64(L), N, C.c_double(r_c), _p(out)))
    return out


def default_rc_grid(step=0.05):
    n = C.c_int()
    _check(lib().krul_default_rc_grid(C.c_double(step), None, C.byref(n)))
    out = np.empty(n.value, np.float64)
    _check(lib().krul_default_rc_grid(C.c_double(step), _p(out), C.byref(n)))
    return out


def calibrate_rc(cost: CostModel, N, L, d, pairs=(), grid=None):
    arr, n = _pairs(pairs)
    g = np.ascontiguousarray(default_rc_grid() if grid is None else grid, np.float64)
    out = C.c_double()
    cm = cost.c()
    _check(lib().krul_calibrate_rc(C.byref(cm), N, C.c_int64(L), C.c_int64(d), arr, n, _p(g),
                                   len(g), C.byref(out)))
    return out.value


def validate_plan(L, p, pairs=()):
    arr, n = _pairs(pairs)
    pp = np.ascontiguousarray(p, np.int64)
    m = C.c_int()
    _check(lib().krul_validate_plan(C.c_int64(L), _p(pp), len(pp), arr, n, C.byref(m)))
    return m.value


def plan_blob_specs(L, p, pairs=()):
    arr, n = _pairs(pairs)
    pp = np.ascontiguousarray(p, np.int64)
    out = (BlobSpecC * max(1, len(pp)))()
    cnt = C.c_int()
    _check(lib().krul_blob_specs(C.c_int64(L), _p(pp), len(pp), arr, n, out, C.byref(cnt)))
    res = []
    for i in range(cnt.value):
        o = [out[i].owners[0]] + ([out[i].owners[1]] if out[i].owners[1] >= 0 else [])
        res.append((o, (out[i].start, out[i].end)))
    return res


def simulate_pipeline(L, p, pairs, cost: CostModel, d):
    arr, n = _pairs(pairs)
    pp = np.ascontiguousarray(p, np.int64)
    out = np.empty(5, np.float64)
    cm = cost.c()
    _check(lib().krul_simulate(C.c_int64(L), _p(pp), len(pp), arr, n, C.byref(cm), C.c_int64(d),
                               _p(out)))
    return dict(makespan=out[0], compute_finish=out[1], load_finish=out[2],
                bubble_compute=out[3], bubble_load=out[4])


# ---- kvstore (kvstore.hpp:16-89) -----------------------------------------------

class KVSnapshot:
    """Compressed KV store: pinned host blobs + plan + strategy."""

    def __init__(self, h, ctx):
        self.h = h
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib().krul_snapshot_destroy(self.h)

    @classmethod
    def compress(cls, ctx: Context, conv: Conversation, pairs, recompute_len, L, mode=MERGE_MEAN):
        """compress_and_snapshot (kvstore.cpp:243-314), K8 on the device."""
        arr, n = _pairs(pairs)
        p = np.ascontiguousarray(recompute_len, np.int64)
        h = C.c_void_p()
        _check(lib().krul_snapshot_compress(ctx.h, conv.h, arr, n, _p(p), C.c_int64(L), mode,
                                            C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_blobs(cls, ctx: Context, pairs, recompute_len, L, mode, blobs):
        """blobs: list of (K[kvh,rows,hd], V[kvh,rows,hd]) in service order."""
        arr, n = _pairs(pairs)
        p = np.ascontiguousarray(recompute_len, np.int64)
        ks = [np.ascontiguousarray(b[0], np.float32) for b in blobs]
        vs = [np.ascontiguousarray(b[1], np.float32) for b in blobs]
        kp = (C.c_void_p * max(1, len(ks)))(*[k.ctypes.data for k in ks])
        vp = (C.c_void_p * max(1, len(vs)))(*[v.ctypes.data for v in vs])
        h = C.c_void_p()
        _check(lib().krul_snapshot_from_host(ctx.h, arr, n, _p(p), C.c_int64(L), mode, kp, vp,
                                             C.byref(h)))
        return cls(h, ctx)

    def n_blobs(self):
        return lib().krul_snapshot_n_blobs(self.h)

    def blob(self, b):
        spec = BlobSpecC()
        _check(lib().krul_snapshot_blob(self.h, b, C.byref(spec), None, None))
        hd = self.header()
        rows = spec.end - spec.start
        k = np.empty((hd["n_heads"], rows, hd["head_dim"]), np.float32)
        v = np.empty_like(k)
        _check(lib().krul_snapshot_blob(self.h, b, C.byref(spec), _p(k), _p(v)))
        o = [spec.owners[0]] + ([spec.owners[1]] if spec.owners[1] >= 0 else [])
        return o, (spec.start, spec.end), k, v

    def storage_report(self):
        f, s = C.c_uint64(), C.c_uint64()
        _check(lib().krul_snapshot_storage(self.h, C.byref(f), C.byref(s)))
        return f.value, s.value

    def plan(self):
        N = self.header()["n_layers"]
        p = np.empty(max(N, 1), np.int64)
        L = C.c_int64()
        _check(lib().krul_snapshot_plan(self.h, _p(p), C.byref(L)))
        return p[:N], L.value

    def set_plan(self, p):
        pp = np.ascontiguousarray(p, np.int64)
        _check(lib().krul_snapshot_set_plan(self.h, _p(pp)))

    def expand(self, layer):
        hd = self.header()
        p, L = self.plan()
        rows = max(0, L - int(p[layer])) if 0 <= layer < len(p) else L
        k = np.empty((hd["n_heads"], max(rows, 1), hd["head_dim"]), np.float32)
        v = np.empty_like(k)
        s, e = C.c_int64(), C.c_int64()
        _check(lib().krul_expand(self.h, layer, _p(k), _p(v), C.byref(s), C.byref(e)))
        r = e.value - s.value
        return (s.value, e.value), k[:, :r], v[:, :r]

    def encode(self):
        """Exponent-code a raw bf16 store (lossless)."""
        _check(lib().krul_snapshot_encode(self.h))

    def coding(self) -> dict:
        c, r, k = C.c_int(), C.c_uint64(), C.c_uint64()
        _check(lib().krul_snapshot_coding(self.h, C.byref(c), C.byref(r), C.byref(k)))
        return {"coded": bool(c.value), "raw_bytes": r.value, "coded_bytes": k.value,
                "ratio": (k.value / r.value) if r.value else 1.0}

    # ---- KRUL v1 container (kvstore.cpp:360-511) ----
    def header(self) -> dict:
        h, n, kvh, hd, L, mode, npairs = (C.c_uint64(), C.c_int(), C.c_int(), C.c_int(),
                                          C.c_int64(), C.c_int(), C.c_int())
        _check(lib().krul_snapshot_header(self.h, C.byref(h), C.byref(n), C.byref(kvh), C.byref(hd),
                                          C.byref(L), C.byref(mode), C.byref(npairs)))
        return {"config_hash": h.value, "n_layers": n.value, "n_heads": kvh.value,
                "head_dim": hd.value, "history_len": L.value, "mode": mode.value,
                "n_pairs": npairs.value}

    def pairs(self):
        n = self.header()["n_pairs"]
        arr = (Pair * max(1, n))()
        _check(lib().krul_snapshot_pairs(self.h, arr))
        return [(arr[i].shallow, arr[i].deep, arr[i].distance) for i in range(n)]

    def set_meta(self, conversation_id: str = "", exhausted_before_quota: bool = False,
                 ir_layers=(), non_ir_layers=(), avg_weight_sum=()):
        ir = np.ascontiguousarray(list(ir_layers) or [0], np.int32)
        nir = np.ascontiguousarray(list(non_ir_layers) or [0], np.int32)
        avg = np.ascontiguousarray(list(avg_weight_sum) or [0.0], np.float64)
        m = SnapshotMetaC(conversation_id.encode("utf-8", "surrogateescape"), int(bool(exhausted_before_quota)),
                          ir.ctypes.data, len(ir_layers), nir.ctypes.data, len(non_ir_layers),
                          avg.ctypes.data, len(avg_weight_sum))
        _check(lib().krul_snapshot_set_meta(self.h, C.byref(m)))

    def meta(self) -> dict:
        m = SnapshotMetaC()
        _check(lib().krul_snapshot_get_meta(self.h, C.byref(m)))

        def arr(ptr, n, t):
            return [] if n == 0 else list(C.cast(ptr, C.POINTER(t))[:n])

        return {"conversation_id": (m.conversation_id or b"").decode("utf-8", "surrogateescape"),
                "exhausted_before_quota": bool(m.exhausted_before_quota),
                "ir_layers": arr(m.ir_layers, m.n_ir_layers, C.c_int32),
                "non_ir_layers": arr(m.non_ir_layers, m.n_non_ir_layers, C.c_int32),
                "avg_weight_sum": arr(m.avg_weight_sum, m.n_avg_weight_sum, C.c_double)}

    def save(self) -> bytes:
        """kvstore::save into memory: the container bytes."""
        n = C.c_uint64()
        _check(lib().krul_snapshot_save(self.h, None, C.c_uint64(0), C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        _check(lib().krul_snapshot_save(self.h, buf, C.c_uint64(n.value), C.byref(n)))
        return buf.raw[:n.value]

    def save_size(self) -> int:
        n = C.c_uint64()
        _check(lib().krul_snapshot_save(self.h, None, C.c_uint64(0), C.byref(n)))
        return n.value

    def save_to(self, buf: np.ndarray) -> int:
        """Save into a caller-owned contiguous uint8 array; returns the bytes written."""
        n = C.c_uint64()
        _check(lib().krul_snapshot_save(self.h, _p(buf), C.c_uint64(buf.nbytes), C.byref(n)))
        return n.value

    def save_file(self, path: str):
        _check(lib().krul_snapshot_save_file(self.h, os.fsencode(path)))

    @classmethod
    def _load(cls, fn, ctx, expected_config_hash):
        h = C.c_void_p()
        field = C.create_string_buffer(32)
        eh = C.byref(C.c_uint64(expected_config_hash)) if expected_config_hash is not None else None
        rc = fn(ctx.h if ctx is not None else None, eh, C.byref(h), field)
        if rc != 0:
            try:
                _check(rc)
            except SnapshotLoadError as e:
                e.field = field.value.decode()
                raise
        return cls(h, ctx)

    @classmethod
    def load(cls, data: bytes, ctx: "Context | None" = None, expected_config_hash: int | None = None):
        """kvstore::load. With ctx: pinned store in the ctx dtype, ready to
        restore. Without: host-only f32 snapshot (inspect / expand / save)."""
        if isinstance(data, np.ndarray):
            if not data.flags.c_contiguous:
                raise ValueError("container buffer must be contiguous")
            ptr, n = _p(data), data.nbytes
        else:
            data = bytes(data)
            ptr, n = data, len(data)
        return cls._load(lambda c, eh, out, f: lib().krul_snapshot_load(
            c, ptr, C.c_uint64(n), eh, out, f, 32), ctx, expected_config_hash)

    @classmethod
    def load_file(cls, path: str, ctx: "Context | None" = None, expected_config_hash: int | None = None):
        return cls._load(lambda c, eh, out, f: lib().krul_snapshot_load_file(
            c, os.fsencode(path), eh, out, f, 32), ctx, expected_config_hash)
