#!/usr/bin/env python3
"""Generates tests/golden/container.json (committed; the GPU box has neither
/root/reference nor the reference-side shims).

Everything here comes from REAL reference-side code compiled by oracle/ref.mk:
  * `doubles` / `strings`: nlohmann::json(x).dump() from nlohmann/json 3.11.3
    (oracle/_ref/libkrul_ref_json.so) — the library kvstore.cpp:11 includes
    for the container metadata;
  * `meta`: the metadata object built with the reference's C++ types and key
    set (kvstore.cpp:100-143, 362-371) and dumped by nlohmann;
  * `containers`: full KRUL v1 containers of the reference's own test
    snapshot (test_kvstore.cpp:17-73: coded_kv(4, 2, 3, 10), pair {1, 3,
    0.25}, plan {8, 6, 4, 2}, "conv-7") in both merge modes — metadata from
    nlohmann, crc32 from the reference's common.cpp
    (oracle/_ref/libkrul_ref_common.so), blobs from the oracle's
    compress_and_snapshot restatement (itself pinned by tests/test_oracle_kat.py),
    framing per kvstore.cpp:374-390.

usage: make -C oracle -f ref.mk && python tests/golden/make_container_golden.py
"""
import ctypes as C
import json
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "container.json")

from oracle import container as OC  # noqa: E402
from oracle import oracle as O  # noqa: E402


def ref_json():
    lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libkrul_ref_json.so"))
    lib.ref_json_double.argtypes = [C.c_double, C.c_char_p, C.c_uint64]
    lib.ref_json_double.restype = C.c_long
    lib.ref_json_string.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64]
    lib.ref_json_string.restype = C.c_long
    lib.ref_json_meta.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64]
    lib.ref_json_meta.restype = C.c_long
    return lib


def ref_crc():
    lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libkrul_ref_common.so"))
    lib.ref_crc32.restype = C.c_uint32
    lib.ref_crc32.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32]
    return lib


def call(fn, *args, cap=1 << 20):
    buf = C.create_string_buffer(cap)
    n = fn(*args, buf, cap)
    return None if n < 0 else buf.raw[:n]


def coded_kv(n_layers, n_heads, head_dim, history):
    """test_kvstore.cpp:17-40: entry = 1000 l + 100 h + r + 0.01 c (f32)."""
    layers = []
    for l in range(n_layers):
        k = np.empty((n_heads, history, head_dim), np.float32)
        for h in range(n_heads):
            for r in range(history):
                for c in range(head_dim):
                    k[h, r, c] = np.float32(1000 * l + 100 * h + r) + np.float32(c) * np.float32(0.01)
        layers.append((0, history, k, -k))
    return layers


def meta_spec(c: OC.Container) -> str:
    """The typed field values for ref_json_meta (doubles as repr: exact)."""
    return json.dumps({
        "conversation_id": c.conversation_id.decode("utf-8"), "head_dim": c.head_dim,
        "history_len": c.history_len, "mode": c.mode, "n_heads": c.n_heads, "n_layers": c.n_layers,
        "plan_history_len": c.history_len, "recompute_len": list(c.recompute_len),
        "exhausted_before_quota": c.exhausted_before_quota, "ir_layers": list(c.ir_layers),
        "non_ir_layers": list(c.non_ir_layers), "avg_weight_sum": [float(x) for x in c.avg_weight_sum],
        "pairs": [[int(s), int(d), float(x)] for s, d, x in c.pairs]})


def main():
    J = ref_json()
    crc = ref_crc()
    rng = np.random.default_rng(2507)
    special = [0.0, -0.0, 0.1, 0.25, 1.0 / 3.0, 2.0 / 3.0, 1e-5, 1e-4, 1.5e-5, 9.99e-6, 1e15, 1e16,
               123456789012345.0, 1234567890123456.0, 1e21, 1e22, 1e100, 1e-100, 5e-324,
               2.2250738585072014e-308, 2.225073858507201e-308, 1.7976931348623157e308, 2.0 ** 60,
               2.0 ** -1074 * 3, 0.30000000000000004, 100.0, 1e-7, 0.001, 12.5, -7.25, float("inf"),
               float("nan"), 0.48787876305978217, 0.049359571966566707]
    vals = special + list(rng.random(1500)) + list(rng.standard_normal(750) * 10.0 ** rng.integers(-30, 30, 750))
    bits = rng.integers(0, 2 ** 63, 750, dtype=np.int64)
    vals += [struct.unpack("<d", struct.pack("<q", int(b)))[0] for b in bits]
    doubles = []
    for v in vals:
        v = float(v)
        doubles.append([struct.pack("<d", v).hex(), call(J.ref_json_double, v).decode()])

    strings = []
    for s in [b"", b"conv-7", b'quote" back\\slash /slash', b"\x00\x01\x08\x09\x0a\x0c\x0d\x1f\x20\x7f",
              "café 中文 \U0001F600".encode(), b"tab\tnew\nline", b"\xff\xfe bad utf8",
              b"\xc0\x80 overlong", b"\xed\xa0\x80 surrogate"]:
        r = call(J.ref_json_string, s, len(s))
        strings.append([s.hex(), None if r is None else r.decode("utf-8")])

    cases = []

    def add_container(name, cfg, strategy, plan, L, mode, conv_id, classifier, kv_layers):
        kv = O.KV.from_host(cfg, kv_layers)
        snap = O.Snapshot(kv, cfg, strategy, plan, L, mode)
        c = OC.from_oracle(snap, cfg, strategy, plan, L, mode, conv_id, classifier)
        meta = call(J.ref_json_meta, meta_spec(c).encode())
        assert meta is not None
        out = bytearray(b"KRUL")
        out += struct.pack("<IQQ", 1, c.config_hash, len(meta)) + meta
        out += struct.pack("<I", len(c.blobs))
        for owners, (start, end), k, v in c.blobs:
            out += struct.pack("<I", len(owners)) + b"".join(struct.pack("<i", o) for o in owners)
            out += struct.pack("<qqQ", start, end, k.nbytes + v.nbytes)
            out += np.ascontiguousarray(k, "<f4").tobytes() + np.ascontiguousarray(v, "<f4").tobytes()
        out += struct.pack("<I", crc.ref_crc32(bytes(out), len(out), 0))
        cases.append({"name": name, "meta": meta.decode("utf-8"), "container": bytes(out).hex(),
                      "config": {"n_layers": cfg.n_layers, "n_heads": cfg.n_heads, "head_dim": cfg.head_dim,
                                 "d_model": cfg.d_model, "vocab_size": cfg.vocab_size, "seed": cfg.seed},
                      "pairs": [list(p) for p in strategy.pairs], "exhausted": strategy.exhausted,
                      "plan": [int(x) for x in plan], "L": L, "mode": mode,
                      "conversation_id": conv_id.hex(),
                      "classifier": [list(classifier[0]), list(classifier[1]), list(classifier[2])]})

    # test_kvstore.cpp:66-73 sample_snapshot (both merge modes)
    cfg = O.ModelConfig(n_layers=4, n_heads=2, head_dim=3, d_model=6, vocab_size=11)
    for mode in (0, 1):
        add_container(f"sample_{OC.MODE_NAMES[mode]}", cfg, O.Strategy([(1, 3, 0.25)]), [8, 6, 4, 2], 10,
                      mode, b"conv-7", ([], [], []), coded_kv(4, 2, 3, 10))
    # awkward metadata: Grisu2-non-shortest distances, classifier report,
    # escapes in the id, exhausted flag, a layer with an empty load span
    cfg6 = O.ModelConfig(n_layers=6, n_heads=1, head_dim=2, d_model=2, vocab_size=11, seed=9)
    add_container("classifier_escapes", cfg6,
                  O.Strategy([(2, 4, 0.48787876305978217), (1, 5, 1e-5), (0, 3, 0.049359571966566707)], True),
                  [12, 12, 9, 7, 4, 2], 12, 0, 'id "q"\té\n'.encode(),
                  ([0, 1, 2, 3, 4, 5][1:], [0], [0.1, 0.9, 1.0 / 3.0, 0.5, 2e-7, 1e16]),
                  coded_kv(6, 1, 2, 12))

    metas = []
    for spec in [
        {"conversation_id": "", "head_dim": 128, "history_len": 8192, "mode": "mean", "n_heads": 8,
         "n_layers": 2, "plan_history_len": 8192, "recompute_len": [1049, 1015], "exhausted_before_quota": False,
         "ir_layers": [], "non_ir_layers": [], "avg_weight_sum": [], "pairs": []},
        {"conversation_id": "x", "head_dim": 8, "history_len": 0, "mode": "keep-deeper", "n_heads": 2,
         "n_layers": 3, "plan_history_len": 0, "recompute_len": [0, 0, 0], "exhausted_before_quota": True,
         "ir_layers": [0, 2], "non_ir_layers": [1], "avg_weight_sum": [1.0, 0.0, 0.5000000000000001],
         "pairs": [[0, 2, 0.0]]},
    ]:
        metas.append([spec, call(J.ref_json_meta, json.dumps(spec).encode()).decode("utf-8")])

    with open(OUT, "w") as f:
        json.dump({"source": "nlohmann/json 3.11.3 (cudnn_frontend/thirdparty) + reference common.cpp crc32",
                   "doubles": doubles, "strings": strings, "meta": metas, "containers": cases}, f, indent=0)
    print(f"wrote {OUT}: {len(doubles)} doubles, {len(strings)} strings, {len(metas)} metas, "
          f"{len(cases)} containers")


if __name__ == "__main__":
    main()
