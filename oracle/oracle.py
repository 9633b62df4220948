"""ctypes view of the CPU oracle (oracle/_build/libkrul_oracle.so).

TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py — never by the product package. The library is a
restatement of /root/reference/proj (see krul_oracle.hpp); this module only
marshals numpy arrays across its C ABI (kro_capi.cpp).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libkrul_oracle.so")

# kro::Status <-> reference exception names (common.hpp:25-63)
STATUS_NAMES = {
    1: "ConfigError",
    2: "RestorationGapError",
    3: "StateCorruptionError",
    4: "AccountingError",
    5: "PlanInvalidError",
    6: "ClassificationError",
    7: "SnapshotError",
    8: "SnapshotLoadError",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS_NAMES.get(code, str(code))


def build():
    import subprocess

    subprocess.check_call(["make", "-s", "-C", HERE])


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.kro_model_weights.restype = C.c_int64
        _lib.kro_fnv1a64.restype = C.c_uint64
        _lib.kro_fnv1a64.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
        _lib.kro_crc32.restype = C.c_uint32
        _lib.kro_crc32.argtypes = [C.c_void_p, C.c_size_t, C.c_uint32]
        _lib.kro_stable_sq.restype = C.c_double
        _lib.kro_layer_flops.restype = C.c_double
        _lib.kro_layer_flops.argtypes = [C.c_double, C.c_int64, C.c_int64]
        _lib.kro_prefill_flops.restype = C.c_double
        _lib.kro_prefill_flops.argtypes = [C.c_double, C.c_int64, C.c_int64, C.c_int64, C.c_int]
        _lib.kro_time_partial.restype = C.c_double
        _lib.kro_kv_synthetic.restype = C.c_void_p
        _lib.kro_kv_synthetic.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_uint64]
        _lib.kro_set_threads.argtypes = [C.c_int]
        for name in ("kro_prefill_take_kv", "kro_kv_clone", "kro_kv_suffix", "kro_kv_from_host"):
            getattr(_lib, name).restype = C.c_void_p
        _lib.kro_kv_suffix.argtypes = [C.c_void_p, C.c_void_p]
        _lib.kro_kv_clone.argtypes = [C.c_void_p]
        _lib.kro_prefill_take_kv.argtypes = [C.c_void_p]
        for name in ("kro_kv_free", "kro_prefill_free", "kro_model_free", "kro_acc_free",
                     "kro_snapshot_free"):
            getattr(_lib, name).argtypes = [C.c_void_p]
    return _lib


def _check(rc: int):
    if rc != 0:
        buf = C.create_string_buffer(512)
        lib().kro_last_error(buf, 512)
        raise OracleError(rc, buf.value.decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class KroCfg(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int), ("n_heads", C.c_int), ("n_kv_heads", C.c_int),
        ("head_dim", C.c_int), ("d_model", C.c_int), ("vocab", C.c_int),
        ("ffn_mult", C.c_float), ("ffn_kind", C.c_int), ("seed", C.c_uint64),
        ("rope_theta", C.c_double),
    ]


@dataclass
class ModelConfig:
    """engine.hpp:17-29 ModelConfig (+ n_kv_heads / ffn_kind / rope_theta extensions)."""
    n_layers: int = 4
    n_heads: int = 2
    head_dim: int = 8
    d_model: int = 16
    vocab_size: int = 64
    ffn_mult: float = 4.0
    seed: int = 0
    n_kv_heads: int = 0
    ffn_kind: int = 0
    rope_theta: float = 10000.0

    def c(self) -> KroCfg:
        return KroCfg(self.n_layers, self.n_heads, self.n_kv_heads, self.head_dim, self.d_model,
                      self.vocab_size, self.ffn_mult, self.ffn_kind, self.seed, self.rope_theta)

    @property
    def kv_heads(self):
        return self.n_kv_heads or self.n_heads

    def ffn_hidden(self) -> int:
        out = C.c_int()
        cfg = self.c()
        _check(lib().kro_config_ffn_hidden(C.byref(cfg), C.byref(out)))
        return out.value

    def hash(self) -> int:
        out = C.c_uint64()
        cfg = self.c()
        _check(lib().kro_config_hash(C.byref(cfg), C.byref(out)))
        return out.value

    def validate(self):
        cfg = self.c()
        _check(lib().kro_config_validate(C.byref(cfg)))


def fnv1a64(data: bytes, basis: int = 0xCBF29CE484222325) -> int:
    return lib().kro_fnv1a64(data, len(data), basis)


def crc32(data: bytes, crc: int = 0) -> int:
    return lib().kro_crc32(data, len(data), crc)


def uniform(seed: int, lo: float, hi: float, n: int) -> np.ndarray:
    out = np.empty(n, np.float32)
    lib().kro_uniform_fill(C.c_uint64(seed), C.c_float(lo), C.c_float(hi), _p(out), C.c_int64(n))
    return out


def uniform_index(seed: int, mod: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().kro_uniform_index(C.c_uint64(seed), C.c_uint64(mod), _p(out), C.c_int64(n))
    return out


def tokens(n: int, seed: int, vocab: int) -> np.ndarray:
    """UniformStream(seed).next_index(vocab) draws (test_engine.cpp:18-26)."""
    return uniform_index(seed, vocab, n).astype(np.int32)


class KV:
    """A vector<KVCacheLayer> held by the oracle."""

    def __init__(self, h, cfg: ModelConfig):
        self.h = C.c_void_p(h)
        self.cfg = cfg

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib().kro_kv_free(self.h)
            self.h = C.c_void_p(None)

    def span(self, layer):
        s, e = C.c_int64(), C.c_int64()
        _check(lib().kro_kv_span(self.h, layer, C.byref(s), C.byref(e)))
        return s.value, e.value

    def layer(self, layer):
        """(K, V) as [kv_heads, rows, hd] f32."""
        s, e = self.span(layer)
        rows = max(0, e - s)
        k = np.zeros((self.cfg.kv_heads, rows, self.cfg.head_dim), np.float32)
        v = np.zeros_like(k)
        _check(lib().kro_kv_get(self.h, layer, self.cfg.head_dim, _p(k), _p(v)))
        return k, v

    def clone(self):
        return KV(lib().kro_kv_clone(self.h), self.cfg)

    def suffix(self, starts):
        st = np.ascontiguousarray(starts, np.int64)
        return KV(lib().kro_kv_suffix(self.h, _p(st)), self.cfg)

    @staticmethod
    def synthetic(cfg: ModelConfig, L: int, seed: int = 1):
        """Timing-only KV: every layer [0, L) filled with U(-1, 1)."""
        return KV(lib().kro_kv_synthetic(cfg.n_layers, cfg.kv_heads, cfg.head_dim, L, seed), cfg)

    @staticmethod
    def from_host(cfg: ModelConfig, layers):
        """layers: list of (start, end, K[kvh,rows,hd], V[kvh,rows,hd])."""
        N = len(layers)
        starts = np.array([l[0] for l in layers], np.int64)
        ends = np.array([l[1] for l in layers], np.int64)
        ks = [np.ascontiguousarray(l[2], np.float32) for l in layers]
        vs = [np.ascontiguousarray(l[3], np.float32) for l in layers]
        kp = (C.c_void_p * N)(*[k.ctypes.data for k in ks])
        vp = (C.c_void_p * N)(*[v.ctypes.data for v in vs])
        h = lib().kro_kv_from_host(N, cfg.kv_heads, cfg.head_dim, _p(starts), _p(ends), kp, vp)
        return KV(h, cfg)


class Prefill:
    def __init__(self, h, model):
        self.h = C.c_void_p(h)
        self.model = model

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib().kro_prefill_free(self.h)

    def logits(self):
        out = np.empty(self.model.cfg.vocab_size, np.float32)
        lib().kro_prefill_logits(self.h, _p(out))
        return out

    def attn(self, layer, head):
        r, w = C.c_int64(), C.c_int64()
        _check(lib().kro_prefill_attn(self.h, layer, head, None, C.byref(r), C.byref(w)))
        out = np.empty((r.value, w.value), np.float32)
        _check(lib().kro_prefill_attn(self.h, layer, head, _p(out), None, None))
        return out

    def attn_all(self):
        """[N, H, rows, width] f32 prefill probabilities."""
        cfg = self.model.cfg
        return np.stack([np.stack([self.attn(l, h) for h in range(cfg.n_heads)])
                         for l in range(cfg.n_layers)])

    def take_kv(self) -> KV:
        return KV(lib().kro_prefill_take_kv(self.h), self.model.cfg)

    def classify(self, gamma=0.5, initial_frac=0.1, recent_frac=0.1):
        N = self.model.cfg.n_layers
        avg = np.empty(N, np.float64)
        ir = np.empty(N, np.int32)
        _check(lib().kro_classify_prefill(self.h, C.c_double(gamma), C.c_double(initial_frac),
                                          C.c_double(recent_frac), _p(avg), _p(ir)))
        return avg, [l for l in range(N) if ir[l]]


def set_threads(n: int):
    """OpenMP threads of the oracle's GEMM / attention loops."""
    lib().kro_set_threads(int(n))


def max_threads() -> int:
    return lib().kro_max_threads()


class Model:
    def __init__(self, cfg: ModelConfig, fast_seed: int | None = None):
        """build_model (engine.cpp:361-395); fast_seed: timing-only weights
        from a parallel counter-based fill instead of the reference draw."""
        self.cfg = cfg
        h = C.c_void_p()
        c = cfg.c()
        if fast_seed is None:
            _check(lib().kro_model_build(C.byref(c), C.byref(h)))
        else:
            _check(lib().kro_model_build_fast(C.byref(c), C.c_uint64(fast_seed), C.byref(h)))
        self.h = h

    def time_turn(self, history, snap: "Snapshot", new_tokens):
        """execute_restore + prefill(history + new, restored), timed in C++
        -> (restore_s, prefill_s, logits)."""
        t = np.ascontiguousarray(history, np.int32)
        nt = np.ascontiguousarray(new_tokens, np.int32)
        out = np.zeros(2, np.float64)
        lg = np.empty(self.cfg.vocab_size, np.float32)
        _check(lib().kro_time_turn(self.h, _p(t), C.c_int64(t.size), snap.h, _p(nt), C.c_int64(nt.size),
                                   _p(out), _p(lg)))
        return float(out[0]), float(out[1]), lg

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib().kro_model_free(self.h)

    def weights(self) -> np.ndarray:
        n = lib().kro_model_weights(self.h, None)
        out = np.empty(n, np.float32)
        lib().kro_model_weights(self.h, _p(out))
        return out

    def prefill(self, toks, preload: KV | None = None, capture=True) -> Prefill:
        t = np.ascontiguousarray(toks, np.int32)
        h = C.c_void_p()
        _check(lib().kro_prefill(self.h, _p(t), C.c_int64(len(t)),
                                 preload.h if preload is not None else None, int(capture),
                                 C.byref(h)))
        return Prefill(h.value, self)

    def decode(self, kv: KV, tok: int):
        """Returns (logits[V], rows[N, H, s+1]); grows kv in place."""
        s, e = kv.span(0)
        cfg = self.cfg
        logits = np.empty(cfg.vocab_size, np.float32)
        rows = np.empty((cfg.n_layers, cfg.n_heads, e + 1), np.float32)
        _check(lib().kro_decode(self.h, kv.h, C.c_int32(tok), _p(logits), _p(rows)))
        return logits, rows

    def partial(self, toks, recompute_len) -> KV:
        t = np.ascontiguousarray(toks, np.int32)
        p = np.ascontiguousarray(recompute_len, np.int64)
        h = C.c_void_p()
        _check(lib().kro_partial(self.h, _p(t), C.c_int64(len(t)), _p(p), len(p), C.byref(h)))
        return KV(h.value, self.cfg)

    def restore(self, history, snap: "Snapshot") -> KV:
        t = np.ascontiguousarray(history, np.int32)
        h = C.c_void_p()
        _check(lib().kro_restore(self.h, _p(t), C.c_int64(len(t)), snap.h, C.byref(h)))
        return KV(h.value, self.cfg)


# ---- analysis --------------------------------------------------------------

def classify(probs: np.ndarray, first_q=0, gamma=0.5, initial_frac=0.1, recent_frac=0.1):
    """probs [N, H, rows, W] -> (avg_weight_sum[N], ir_layers)."""
    p = np.ascontiguousarray(probs, np.float32)
    N, H, R, W = p.shape
    avg = np.empty(N, np.float64)
    ir = np.empty(N, np.int32)
    _check(lib().kro_classify(_p(p), N, H, C.c_int64(R), C.c_int64(W), C.c_int64(first_q),
                              C.c_double(gamma), C.c_double(initial_frac), C.c_double(recent_frac),
                              _p(avg), _p(ir)))
    return avg, [l for l in range(N) if ir[l]]


class Accumulator:
    """SimilarityAccumulator (analysis.hpp:66-94)."""

    def __init__(self, ir_layers, n_heads):
        ir = np.ascontiguousarray(ir_layers, np.int32)
        h = C.c_void_p()
        _check(lib().kro_acc_create(_p(ir), len(ir), n_heads, C.byref(h)))
        self.h = h
        self.layers = sorted(set(int(x) for x in ir_layers))
        self.H = n_heads

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib().kro_acc_free(self.h)

    def fold_prefill(self, probs: np.ndarray):
        p = np.ascontiguousarray(probs, np.float32)
        N, H, R, W = p.shape
        _check(lib().kro_acc_fold_prefill(self.h, _p(p), N, H, C.c_int64(R), C.c_int64(W)))

    def fold_prefill_handle(self, pf: Prefill):
        _check(lib().kro_acc_fold_prefill_handle(self.h, pf.h))

    def fold_decode(self, rows: np.ndarray):
        r = np.ascontiguousarray(rows, np.float32)
        N, H, W = r.shape
        _check(lib().kro_acc_fold_decode(self.h, _p(r), N, H, C.c_int64(W)))

    def sums(self):
        n = len(self.layers)
        out = np.empty(n * (n - 1) // 2 * self.H, np.float64)
        _check(lib().kro_acc_sums(self.h, _p(out)))
        return out

    def finalize(self):
        n = len(self.layers)
        out = np.empty((n, n), np.float64)
        _check(lib().kro_acc_finalize(self.h, _p(out)))
        return out


def stable_sq(a, b) -> float:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    lib().kro_stable_sq.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    return lib().kro_stable_sq(_p(a), _p(b), a.size)


# ---- strategy ---------------------------------------------------------------

@dataclass
class Strategy:
    pairs: list = field(default_factory=list)  # [(shallow, deep, distance)]
    exhausted: bool = False

    @property
    def shared(self):
        return sorted({x for p in self.pairs for x in p[:2]})

    def arrays(self):
        sh = np.array([p[0] for p in self.pairs] or [0], np.int32)
        dp = np.array([p[1] for p in self.pairs] or [0], np.int32)
        ds = np.array([p[2] if len(p) > 2 else 0.0 for p in self.pairs] or [0.0], np.float64)
        return sh, dp, ds, len(self.pairs)


def quota(n_layers, r_l) -> int:
    out = C.c_int()
    _check(lib().kro_quota(n_layers, C.c_double(r_l), C.byref(out)))
    return out.value


def select_strategy(D, dm_layers, ir_layers, r_l, n_layers) -> Strategy:
    D = np.ascontiguousarray(D, np.float64)
    dl = np.ascontiguousarray(dm_layers, np.int32)
    ir = np.ascontiguousarray(ir_layers if len(ir_layers) else [0], np.int32)
    cap = max(1, len(ir_layers))
    sh = np.zeros(cap, np.int32)
    dp = np.zeros(cap, np.int32)
    ds = np.zeros(cap, np.float64)
    npairs, exh = C.c_int(), C.c_int()
    _check(lib().kro_select(_p(D), _p(dl), len(dm_layers), _p(ir), len(ir_layers), C.c_double(r_l),
                            n_layers, _p(sh), _p(dp), _p(ds), C.byref(npairs), C.byref(exh)))
    return Strategy([(int(sh[i]), int(dp[i]), float(ds[i])) for i in range(npairs.value)],
                    bool(exh.value))


def validate_strategy(pairs, shared, exhausted, ir_layers, n_layers, r_l) -> int:
    """strategy.cpp:76-131 -> violation bitmask (krul_oracle.hpp)."""
    sh = np.ascontiguousarray([p[0] for p in pairs] or [0], np.int32)
    dp = np.ascontiguousarray([p[1] for p in pairs] or [0], np.int32)
    ds = np.ascontiguousarray([p[2] for p in pairs] or [0.0], np.float64)
    sd = np.ascontiguousarray(list(shared) or [0], np.int32)
    ir = np.ascontiguousarray(list(ir_layers) or [0], np.int32)
    m = C.c_int()
    _check(lib().kro_validate_strategy(_p(sh), _p(dp), _p(ds), len(pairs), _p(sd), len(list(shared)),
                                       int(bool(exhausted)), _p(ir), len(list(ir_layers)), n_layers,
                                       C.c_double(r_l), C.byref(m)))
    return m.value


# ---- scheduler --------------------------------------------------------------

def build_plan(L, N, r_c, strategy: Strategy | None = None):
    s = strategy or Strategy()
    sh, dp, _, n = s.arrays()
    out = np.empty(N, np.int64)
    _check(lib().kro_build_plan(C.c_int64(L), N, C.c_double(r_c), _p(sh), _p(dp), n, _p(out)))
    return out


def uniform_plan(L, N, r_c):
    out = np.empty(N, np.int64)
    _check(lib().kro_uniform_plan(C.c_int64(L), N, C.c_double(r_c), _p(out)))
    return out


def default_rc_grid(step=0.05):
    n = C.c_int()
    _check(lib().kro_default_grid(C.c_double(step), None, C.byref(n)))
    out = np.empty(n.value, np.float64)
    _check(lib().kro_default_grid(C.c_double(step), _p(out), C.byref(n)))
    return out


def calibrate_rc(N, L, d, strategy: Strategy | None = None, grid=None, f_peak=312e12,
                 b_peak=139e9, ffn_mult=4.0):
    s = strategy or Strategy()
    sh, dp, _, n = s.arrays()
    g = np.ascontiguousarray(default_rc_grid() if grid is None else grid, np.float64)
    out = C.c_double()
    _check(lib().kro_calibrate(C.c_double(f_peak), C.c_double(b_peak), C.c_double(ffn_mult), N,
                               C.c_int64(L), C.c_int64(d), _p(sh), _p(dp), n, _p(g), len(g),
                               C.byref(out)))
    return out.value


def validate_plan(L, p, strategy: Strategy | None = None) -> int:
    s = strategy or Strategy()
    sh, dp, _, n = s.arrays()
    pp = np.ascontiguousarray(p, np.int64)
    m = C.c_int()
    _check(lib().kro_validate_plan(C.c_int64(L), _p(pp), len(pp), _p(sh), _p(dp), n, C.byref(m)))
    return m.value


def blob_specs(L, p, strategy: Strategy | None = None):
    s = strategy or Strategy()
    sh, dp, _, n = s.arrays()
    pp = np.ascontiguousarray(p, np.int64)
    N = len(pp)
    owners = np.empty(2 * N, np.int32)
    spans = np.empty(2 * N, np.int64)
    cnt = C.c_int()
    _check(lib().kro_blob_specs(C.c_int64(L), _p(pp), N, _p(sh), _p(dp), n, _p(owners), _p(spans),
                                C.byref(cnt)))
    out = []
    for i in range(cnt.value):
        o = [int(owners[2 * i])] + ([int(owners[2 * i + 1])] if owners[2 * i + 1] >= 0 else [])
        out.append((o, (int(spans[2 * i]), int(spans[2 * i + 1]))))
    return out


def simulate(L, p, strategy: Strategy | None, d, f_peak=312e12, b_peak=139e9, ffn_mult=4.0):
    s = strategy or Strategy()
    sh, dp, _, n = s.arrays()
    pp = np.ascontiguousarray(p, np.int64)
    out = np.empty(6, np.float64)
    _check(lib().kro_simulate(C.c_int64(L), _p(pp), len(pp), _p(sh), _p(dp), n, C.c_double(f_peak),
                              C.c_double(b_peak), C.c_double(ffn_mult), C.c_int64(d), _p(out)))
    return dict(makespan=out[0], compute_finish=out[1], load_finish=out[2], bubble_compute=out[3],
                bubble_load=out[4], n_compute=int(out[5]) // 1000, n_load=int(out[5]) % 1000)


def layer_flops(p, d, ffn_mult=4.0):
    return lib().kro_layer_flops(ffn_mult, p, d)


def prefill_flops(n, hist, d, N, ffn_mult=4.0):
    return lib().kro_prefill_flops(ffn_mult, n, hist, d, N)


# ---- kvstore ------------------------------------------------------------------

class Snapshot:
    def __init__(self, kv: KV, cfg: ModelConfig, strategy: Strategy, p, L, mode=0):
        sh, dp, ds, n = strategy.arrays()
        pp = np.ascontiguousarray(p, np.int64)
        c = cfg.c()
        h = C.c_void_p()
        _check(lib().kro_snapshot(kv.h, C.byref(c), _p(sh), _p(dp), _p(ds), n, _p(pp),
                                  C.c_int64(L), mode, C.byref(h)))
        self.h = h
        self.cfg = cfg

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib().kro_snapshot_free(self.h)

    def n_blobs(self):
        return lib().kro_snapshot_n_blobs(self.h)

    def blob(self, b):
        owners = np.empty(2, np.int32)
        span = np.empty(2, np.int64)
        _check(lib().kro_snapshot_blob(self.h, b, _p(owners), _p(span), None, None))
        rows = int(span[1] - span[0])
        k = np.empty((self.cfg.kv_heads, rows, self.cfg.head_dim), np.float32)
        v = np.empty_like(k)
        _check(lib().kro_snapshot_blob(self.h, b, _p(owners), _p(span), _p(k), _p(v)))
        o = [int(owners[0])] + ([int(owners[1])] if owners[1] >= 0 else [])
        return o, (int(span[0]), int(span[1])), k, v

    def storage(self):
        full, stored = C.c_uint64(), C.c_uint64()
        _check(lib().kro_snapshot_storage(self.h, C.byref(full), C.byref(stored)))
        return full.value, stored.value

    def set_plan(self, p):
        pp = np.ascontiguousarray(p, np.int64)
        _check(lib().kro_snapshot_set_plan(self.h, _p(pp)))

    def expand(self, layer):
        span = np.empty(2, np.int64)
        # size from the plan is unknown here: probe with a generous buffer
        cap = self.cfg.kv_heads * self._max_rows() * self.cfg.head_dim
        k = np.empty(max(cap, 1), np.float32)
        v = np.empty_like(k)
        _check(lib().kro_expand(self.h, layer, _p(k), _p(v), _p(span)))
        rows = int(span[1] - span[0])
        n = self.cfg.kv_heads * rows * self.cfg.head_dim
        shape = (self.cfg.kv_heads, rows, self.cfg.head_dim)
        return (int(span[0]), int(span[1])), k[:n].reshape(shape), v[:n].reshape(shape)

    def _max_rows(self):
        return max(self.blob(b)[1][1] - self.blob(b)[1][0] for b in range(self.n_blobs()))
