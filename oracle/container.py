"""CPU restatement of the KRUL v1 snapshot container.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): imported by tests/ and
tests/golden/make_container_golden.py as the checker of the library's
krul_snapshot_save / krul_snapshot_load — never by the product package.

Follows /root/reference/proj/src/kvstore.cpp:
  * framing of save()                      kvstore.cpp:360-392
  * metadata object (key-sorted JSON)      kvstore.cpp:100-143, 362-371
  * load() checks, order and field names   kvstore.cpp:394-511
  * crc32                                  common.cpp:34-42 (oracle.crc32,
                                           pinned to the reference's own
                                           common.cpp by tests/test_golden.py)
The metadata text is nlohmann::json::dump() (json.hpp is not vendored in the
reference — CMakeLists.txt's vendor/ is absent — so nlohmann/json 3.11.3, the
copy in this image, is the pinned version): std::map key order, compact
separators, strings escaped per nlohmann's serializer, doubles by Grisu2
(Loitsch 2010) with nlohmann's boundaries and its fixed/exponent switch
(fixed for 1e-5 < |v| < 1e15). Python's repr is NOT a substitute: Grisu2 is
not always shortest (~0.2% of random doubles print one digit longer), so the
digit generation is restated here and pinned against nlohmann's own dump in
tests/golden/container.json.
"""
from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import oracle as O

MAGIC = b"KRUL"
FORMAT_VERSION = 1
MODE_NAMES = {0: "mean", 1: "keep-deeper"}  # merge_mode_name (kvstore.cpp:146-154)


class SnapshotLoadError(Exception):
    """kvstore::SnapshotLoadError: `field` names the failing container field."""

    def __init__(self, fld: str, msg: str):
        super().__init__(f"{fld}: {msg}")
        self.field = fld


# ---------------------------------------------------------------- Grisu2
_M64 = (1 << 64) - 1


def _pow10_table():
    out = []
    for k in range(-300, 325, 8):
        c = Fraction(10) ** k
        e = c.numerator.bit_length() - c.denominator.bit_length() - 64
        while c / Fraction(2) ** e >= 2 ** 64:
            e += 1
        while c / Fraction(2) ** e < 2 ** 63:
            e -= 1
        q = c / Fraction(2) ** e
        out.append((int(q) + (1 if q - int(q) >= Fraction(1, 2) else 0), e, k))
    return out


_POW10 = _pow10_table()


def _mul(xf, xe, yf, ye):
    return ((xf * yf + (1 << 63)) >> 64) & _M64, xe + ye + 64


def _norm(f, e):
    while not f >> 63:
        f <<= 1
        e -= 1
    return f, e


def _grisu2(v: float):
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    vf, ve = (F, -1074) if E == 0 else (F + (1 << 52), E - 1075)
    mpf, mpe = _norm(2 * vf + 1, ve - 1)
    mmf, mme = (4 * vf - 1, ve - 2) if (F == 0 and E > 1) else (2 * vf - 1, ve - 1)
    mmf, mme = mmf << (mme - mpe), mpe
    wf, we = _norm(vf, ve)
    f = -60 - mpe - 1
    k = (f * 78913) >> 18 if f >= 0 else -((-f * 78913) >> 18)  # C division truncates
    k += 1 if f > 0 else 0
    cf, ce, ck = _POW10[(300 + k + 7) // 8]
    w = _mul(wf, we, cf, ce)
    wm = _mul(mmf, mme, cf, ce)
    wp = _mul(mpf, mpe, cf, ce)
    Mm, Mp = wm[0] + 1, wp[0] - 1
    sh = -wp[1]
    dec = -ck
    delta, dist = (Mp - Mm) & _M64, (Mp - w[0]) & _M64
    one = 1 << sh
    p1, p2 = Mp >> sh, Mp & (one - 1)
    n = len(str(p1))
    pow10 = 10 ** (n - 1)
    buf = []

    def rnd(dist, delta, rest, ten_k):
        while rest < dist and delta - rest >= ten_k and (rest + ten_k < dist or dist - rest > rest + ten_k - dist):
            buf[-1] -= 1
            rest += ten_k

    while n > 0:
        d, p1 = divmod(p1, pow10)
        buf.append(d)
        n -= 1
        rest = (p1 << sh) + p2
        if rest <= delta:
            rnd(dist, delta, rest, pow10 << sh)
            return buf, dec + n
        pow10 //= 10
    m = 0
    while True:
        p2 *= 10
        buf.append(p2 >> sh)
        p2 &= one - 1
        m += 1
        delta *= 10
        dist *= 10
        if p2 <= delta:
            break
    rnd(dist, delta, p2, one)
    return buf, dec - m


def dump_double(v: float) -> str:
    """nlohmann::json(v).dump() for a double."""
    if not math.isfinite(v):
        return "null"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0:
        return sign + "0.0"
    digits, dec = _grisu2(abs(v))
    d = "".join(chr(48 + x) for x in digits)
    k = len(d)
    n = k + dec
    if k <= n <= 15:
        out = d + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        out = d[:n] + "." + d[n:]
    elif -4 < n <= 0:
        out = "0." + "0" * (-n) + d
    else:
        ex = n - 1
        out = (d if k == 1 else d[0] + "." + d[1:]) + "e" + ("-" if ex < 0 else "+") + "%02d" % abs(ex)
    return sign + out


def dump_string(s: bytes) -> str:
    """nlohmann string serialisation (ensure_ascii=false, strict UTF-8)."""
    text = s.decode("utf-8")  # UnicodeDecodeError = nlohmann's type_error 316
    out = ['"']
    esc = {'"': '\\"', "\\": "\\\\", "\b": "\\b", "\f": "\\f", "\n": "\\n", "\r": "\\r", "\t": "\\t"}
    for ch in text:
        if ch in esc:
            out.append(esc[ch])
        elif ord(ch) < 0x20:
            out.append("\\u%04x" % ord(ch))
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


# ------------------------------------------------------------- snapshot
@dataclass
class Container:
    """KVSnapshot (kvstore.hpp:46-59) with blobs as f32 arrays [heads, rows, hd]."""
    conversation_id: bytes = b""
    config_hash: int = 0
    n_layers: int = 0
    n_heads: int = 0
    head_dim: int = 0
    history_len: int = 0
    mode: str = "mean"
    pairs: list = field(default_factory=list)       # [(shallow, deep, distance)]
    shared: list | None = None                      # None = derived from pairs
    exhausted_before_quota: bool = False
    recompute_len: list = field(default_factory=list)
    plan_history_len: int | None = None             # None = history_len
    ir_layers: list = field(default_factory=list)
    non_ir_layers: list = field(default_factory=list)
    avg_weight_sum: list = field(default_factory=list)
    blobs: list = field(default_factory=list)       # [(owners, (start, end), K, V)]
    version: int = FORMAT_VERSION

    def shared_layers(self):
        if self.shared is not None:
            return sorted(set(self.shared))
        return sorted({x for p in self.pairs for x in p[:2]})


def from_oracle(snap: "O.Snapshot", cfg: "O.ModelConfig", strategy: "O.Strategy", p, L, mode=0,
                conversation_id: bytes = b"", classifier=None) -> Container:
    """compress_and_snapshot's KVSnapshot fields (kvstore.cpp:263-273) around
    the oracle's blobs; `classifier` = (ir, non_ir, avg_weight_sum)."""
    ir, non_ir, avg = classifier or ([], [], [])
    blobs = [snap.blob(b) for b in range(snap.n_blobs())]
    return Container(conversation_id=conversation_id, config_hash=cfg.hash(), n_layers=cfg.n_layers,
                     n_heads=cfg.kv_heads, head_dim=cfg.head_dim, history_len=int(L),
                     mode=MODE_NAMES[mode], pairs=[tuple(x) for x in strategy.pairs],
                     exhausted_before_quota=bool(strategy.exhausted),
                     recompute_len=[int(x) for x in p], ir_layers=list(ir), non_ir_layers=list(non_ir),
                     avg_weight_sum=[float(x) for x in avg], blobs=blobs)


def meta_text(c: Container) -> bytes:
    """kvstore.cpp:362-372 — json meta{...}.dump()."""
    ints = lambda v: "[" + ",".join(str(int(x)) for x in v) + "]"  # noqa: E731
    dbls = lambda v: "[" + ",".join(dump_double(float(x)) for x in v) + "]"  # noqa: E731
    pairs = "[" + ",".join(f"[{int(s)},{int(d)},{dump_double(float(x))}]" for s, d, x in c.pairs) + "]"
    ph = c.history_len if c.plan_history_len is None else c.plan_history_len
    t = ('{"classifier":{"avg_weight_sum":' + dbls(c.avg_weight_sum)
         + ',"ir_layers":' + ints(c.ir_layers) + ',"non_ir_layers":' + ints(c.non_ir_layers)
         + '},"conversation_id":' + dump_string(c.conversation_id)
         + ',"head_dim":' + str(c.head_dim) + ',"history_len":' + str(c.history_len)
         + ',"mode":' + dump_string(c.mode.encode()) + ',"n_heads":' + str(c.n_heads)
         + ',"n_layers":' + str(c.n_layers)
         + ',"plan":{"history_len":' + str(ph) + ',"recompute_len":' + ints(c.recompute_len)
         + '},"strategy":{"exhausted_before_quota":' + ("true" if c.exhausted_before_quota else "false")
         + ',"pairs":' + pairs + ',"shared":' + ints(c.shared_layers()) + "}}")
    return t.encode("utf-8")


def save(c: Container) -> bytes:
    """kvstore::save (kvstore.cpp:360-392)."""
    meta = meta_text(c)
    out = bytearray()
    out += MAGIC
    out += struct.pack("<IQQ", c.version, c.config_hash, len(meta))
    out += meta
    out += struct.pack("<I", len(c.blobs))
    for owners, (start, end), k, v in c.blobs:
        out += struct.pack("<I", len(owners))
        for o in owners:
            out += struct.pack("<i", int(o))
        k = np.ascontiguousarray(k, "<f4")
        v = np.ascontiguousarray(v, "<f4")
        out += struct.pack("<qqQ", int(start), int(end), k.nbytes + v.nbytes)
        out += k.tobytes() + v.tobytes()
    out += struct.pack("<I", O.crc32(bytes(out)))
    return bytes(out)


class _Reader:
    def __init__(self, buf: bytes):
        self.buf, self.pos = buf, 0

    def remaining(self):
        return len(self.buf) - self.pos

    def take(self, n, fld):
        if self.remaining() < n:
            raise SnapshotLoadError(fld, "container ends mid-field")
        b = self.buf[self.pos:self.pos + n]
        self.pos += n
        return b

    def u32(self, f):
        return struct.unpack("<I", self.take(4, f))[0]

    def u64(self, f):
        return struct.unpack("<Q", self.take(8, f))[0]

    def i32(self, f):
        return struct.unpack("<i", self.take(4, f))[0]

    def i64(self, f):
        return struct.unpack("<q", self.take(8, f))[0]


class _JErr(Exception):
    pass


def _at(v, key):
    if isinstance(key, int):
        if not isinstance(v, list) or key >= len(v):
            raise _JErr("at()")
        return v[key]
    if not isinstance(v, dict) or key not in v:
        raise _JErr(f"key '{key}' not found")
    return v[key]


def _num(v, conv, bits=64):
    """get<T>() of a number (or boolean); a double converts like static_cast on
    x86-64: out-of-range -> the integer-indefinite INT_MIN."""
    if isinstance(v, bool):
        return conv(int(v))
    if isinstance(v, float) and conv is int:
        lim = 2 ** (bits - 1)
        return int(v) if -lim - 1 < v < lim else -lim
    if isinstance(v, (int, float)):
        return conv(v)
    raise _JErr("type must be number")


def _parse_float(s):
    v = float(s)
    if not math.isfinite(v):
        raise _JErr("number overflow")
    return v


def _parse_int(s):
    v = int(s)
    return v if -(2 ** 63) <= v < 2 ** 64 else _parse_float(s)  # beyond (u)int64: a double


def _check_strings(o):
    """nlohmann's lexer rejects lone surrogate escapes anywhere in the text."""
    if isinstance(o, str):
        try:
            o.encode("utf-8")
        except UnicodeEncodeError:
            raise _JErr("invalid string: surrogate")
    elif isinstance(o, list):
        for x in o:
            _check_strings(x)
    elif isinstance(o, dict):
        for k, x in o.items():
            _check_strings(k)
            _check_strings(x)


def _arr(v):
    if not isinstance(v, list):
        raise _JErr("type must be array")
    return v


def _str(v):
    if not isinstance(v, str):
        raise _JErr("type must be string")
    return v


def _i32(x):  # static_cast<int> of a 64-bit integer (a double: see _num)
    x &= 0xFFFFFFFF
    return x - (1 << 32) if x >> 31 else x


def _int32(v):
    """get<int>(): a double converts directly (32-bit indefinite), an integer wraps."""
    return _num(v, int, 32) if isinstance(v, float) else _i32(_num(v, int))


def _no_const(name):
    raise _JErr(f"invalid literal {name}")


def load(buf: bytes, expected_config_hash: int | None = None) -> Container:
    """kvstore::load (kvstore.cpp:394-511): same checks, order and fields."""
    buf = bytes(buf)
    if len(buf) >= 4 and buf[:4] != MAGIC:
        raise SnapshotLoadError("magic", "not a snapshot container")
    if len(buf) < 8:
        raise SnapshotLoadError("checksum", "container shorter than its framing")
    if struct.unpack("<I", buf[-4:])[0] != O.crc32(buf[:-4]):
        raise SnapshotLoadError("checksum", "container checksum mismatch")
    r = _Reader(buf)
    r.take(4, "magic")
    c = Container()
    c.version = r.u32("version")
    if c.version != FORMAT_VERSION:
        raise SnapshotLoadError("version", f"unsupported format version {c.version}")
    c.config_hash = r.u64("config")
    if expected_config_hash is not None and c.config_hash != expected_config_hash:
        raise SnapshotLoadError("config", "snapshot was taken under a different model configuration")
    meta_len = r.u64("metadata")
    raw = r.take(meta_len, "metadata")
    try:
        try:
            m = json.loads(raw.decode("utf-8"), parse_constant=_no_const, parse_float=_parse_float,
                           parse_int=_parse_int)
        except (ValueError, UnicodeDecodeError) as e:
            raise _JErr(str(e))
        _check_strings(m)
        c.conversation_id = _str(_at(m, "conversation_id")).encode("utf-8")
        c.n_layers = _int32(_at(m, "n_layers"))
        c.n_heads = _int32(_at(m, "n_heads"))
        c.head_dim = _int32(_at(m, "head_dim"))
        c.history_len = _num(_at(m, "history_len"), int)
        mode = _str(_at(m, "mode"))
        if mode not in ("mean", "keep-deeper"):
            raise SnapshotLoadError("metadata", "unknown merge mode")
        c.mode = mode
        st = _at(m, "strategy")
        c.pairs = [(_int32(_at(p, 0)), _int32(_at(p, 1)), float(_num(_at(p, 2), float)))
                   for p in _arr(_at(st, "pairs"))]
        c.shared = sorted({_int32(x) for x in _arr(_at(st, "shared"))})
        ex = _at(st, "exhausted_before_quota")
        if not isinstance(ex, bool):
            raise _JErr("type must be boolean")
        c.exhausted_before_quota = ex
        pl = _at(m, "plan")
        c.plan_history_len = _num(_at(pl, "history_len"), int)
        c.recompute_len = [_num(x, int) for x in _arr(_at(pl, "recompute_len"))]
        cl = _at(m, "classifier")
        c.ir_layers = [_int32(x) for x in _arr(_at(cl, "ir_layers"))]
        c.non_ir_layers = [_int32(x) for x in _arr(_at(cl, "non_ir_layers"))]
        c.avg_weight_sum = [float(_num(x, float)) for x in _arr(_at(cl, "avg_weight_sum"))]
    except _JErr as e:
        raise SnapshotLoadError("metadata", str(e))
    if len(c.recompute_len) != c.n_layers or c.plan_history_len != c.history_len:
        raise SnapshotLoadError("plan", "plan does not match the snapshot header")
    n_blobs = r.u32("blob")
    covered = [False] * max(c.n_layers, 0)
    for _ in range(n_blobs):
        no = r.u32("blob")
        if no < 1 or no > 2:
            raise SnapshotLoadError("blob", "blob must have one or two owners")
        owners = []
        for _ in range(no):
            o = r.i32("blob")
            if o < 0 or o >= c.n_layers:
                raise SnapshotLoadError("blob", "blob owner outside the layer range")
            if covered[o]:
                raise SnapshotLoadError("coverage", "layer covered by more than one blob")
            covered[o] = True
            owners.append(o)
        start, end = r.i64("blob"), r.i64("blob")
        if start < 0 or start > end or end != c.history_len:
            raise SnapshotLoadError("blob", "blob span must end at the history")
        plen = r.u64("blob")
        rows = end - start
        if plen != 2 * c.n_heads * rows * c.head_dim * 4:
            raise SnapshotLoadError("blob", "payload length mismatch")
        half = plen // 2
        k = np.frombuffer(r.take(half, "blob"), "<f4").reshape(c.n_heads, rows, c.head_dim).copy()
        v = np.frombuffer(r.take(half, "blob"), "<f4").reshape(c.n_heads, rows, c.head_dim).copy()
        c.blobs.append((owners, (start, end), k, v))
    if r.remaining() != 4:
        raise SnapshotLoadError("blob", "trailing bytes after the blob table")
    for layer, cov in enumerate(covered):
        if not cov:
            raise SnapshotLoadError("coverage", f"layer {layer} is not covered by any blob")
    return c


def equal(a: Container, b: Container) -> bool:
    """operator== on KVSnapshot (kvstore.cpp:210-241): bytewise blobs."""
    head = lambda c: (c.version, c.conversation_id, c.config_hash, c.n_layers, c.n_heads,  # noqa: E731
                      c.head_dim, c.history_len, c.mode, [tuple(p) for p in c.pairs], c.shared_layers(),
                      c.exhausted_before_quota, list(c.recompute_len),
                      c.history_len if c.plan_history_len is None else c.plan_history_len,
                      list(c.ir_layers), list(c.non_ir_layers), list(c.avg_weight_sum), len(c.blobs))
    if head(a) != head(b):
        return False
    for (oa, sa, ka, va), (ob, sb, kb, vb) in zip(a.blobs, b.blobs):
        if list(oa) != list(ob) or tuple(sa) != tuple(sb):
            return False
        if np.asarray(ka, "<f4").tobytes() != np.asarray(kb, "<f4").tobytes():
            return False
        if np.asarray(va, "<f4").tobytes() != np.asarray(vb, "<f4").tobytes():
            return False
    return True
