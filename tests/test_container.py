"""KRUL v1 snapshot container (kvstore.cpp:360-511).

CPU only, no device calls:
  * the oracle restatement (oracle/container.py) against golden vectors made
    by the reference-side code — nlohmann/json 3.11.3's dump of doubles,
    strings and the metadata object, and whole containers of the reference's
    own test snapshot (test_kvstore.cpp:66-73) framed with the reference's
    crc32 (tests/golden/make_container_golden.py);
  * the reference's container tests (test_kvstore.cpp:244-313) on the oracle;
  * the product library's host-only container path (krul_snapshot_load with
    no context, krul_snapshot_save, krul_crc32) bit-exact with both, and its
    load errors naming the same field as the oracle over truncations and
    CRC-fixed corruptions of every byte.
"""
import json
import os
import struct

import numpy as np
import pytest

from oracle import container as OC

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "container.json")))


@pytest.fixture(scope="module")
def K():
    from paper_2507_08045_b200 import native
    native.lib()
    return native


def with_crc(b: bytes) -> bytes:
    from oracle import oracle as O
    return b[:-4] + struct.pack("<I", O.crc32(b[:-4]))


# ---------------------------------------------------------------- oracle
def test_oracle_doubles_match_nlohmann():
    bad = [(h, d) for h, d in G["doubles"]
           if OC.dump_double(struct.unpack("<d", bytes.fromhex(h))[0]) != d]
    assert not bad, bad[:5]
    assert len(G["doubles"]) > 3000


def test_oracle_strings_match_nlohmann():
    for h, d in G["strings"]:
        s = bytes.fromhex(h)
        if d is None:
            with pytest.raises(UnicodeDecodeError):
                OC.dump_string(s)
        else:
            assert OC.dump_string(s) == d


def test_oracle_meta_matches_nlohmann():
    for spec, want in G["meta"]:
        c = OC.Container(conversation_id=spec["conversation_id"].encode(), n_layers=spec["n_layers"],
                         n_heads=spec["n_heads"], head_dim=spec["head_dim"],
                         history_len=spec["history_len"], mode=spec["mode"],
                         pairs=[tuple(p) for p in spec["pairs"]],
                         exhausted_before_quota=spec["exhausted_before_quota"],
                         recompute_len=spec["recompute_len"], ir_layers=spec["ir_layers"],
                         non_ir_layers=spec["non_ir_layers"], avg_weight_sum=spec["avg_weight_sum"])
        assert OC.meta_text(c).decode() == want


def test_oracle_rebuilds_golden_containers(oracle):
    for case in G["containers"]:
        cfg = oracle.ModelConfig(**case["config"])
        L = case["L"]
        layers = []
        for l in range(cfg.n_layers):  # coded_kv (test_kvstore.cpp:17-40)
            k = np.empty((cfg.kv_heads, L, cfg.head_dim), np.float32)
            for h in range(cfg.kv_heads):
                for r in range(L):
                    for c in range(cfg.head_dim):
                        k[h, r, c] = np.float32(1000 * l + 100 * h + r) + np.float32(c) * np.float32(0.01)
            layers.append((0, L, k, -k))
        st = oracle.Strategy([tuple(p) for p in case["pairs"]], case["exhausted"])
        snap = oracle.Snapshot(oracle.KV.from_host(cfg, layers), cfg, st, case["plan"], L, case["mode"])
        c = OC.from_oracle(snap, cfg, st, case["plan"], L, case["mode"],
                           bytes.fromhex(case["conversation_id"]), case["classifier"])
        assert OC.meta_text(c).decode() == case["meta"]
        assert OC.save(c) == bytes.fromhex(case["container"]), case["name"]


def test_oracle_round_trip_and_config_guard():  # test_kvstore.cpp:244-263
    raw = bytes.fromhex(G["containers"][0]["container"])
    back = OC.load(raw)
    assert back.mode == "mean" and back.recompute_len == [8, 6, 4, 2]
    assert back.pairs == [(1, 3, 0.25)] and back.conversation_id == b"conv-7"
    assert OC.equal(back, OC.load(OC.save(back)))
    OC.load(raw, back.config_hash)
    with pytest.raises(OC.SnapshotLoadError) as e:
        OC.load(raw, back.config_hash + 1)
    assert e.value.field == "config"


def field_of(loader, data, h=None):
    try:
        loader(data, h)
    except OC.SnapshotLoadError as e:
        return e.field
    return ""


def test_oracle_loader_names_the_field():  # test_kvstore.cpp:265-313
    b = bytes.fromhex(G["containers"][0]["container"])
    h = OC.load(b).config_hash
    assert field_of(OC.load, b[:-1]) == "checksum"
    assert field_of(OC.load, b[:10]) == "checksum"
    assert field_of(OC.load, b"") == "checksum"
    assert field_of(OC.load, b"KR") == "checksum"
    c = bytearray(b)
    c[len(b) // 2] ^= 0x40
    assert field_of(OC.load, bytes(c)) == "checksum"
    assert field_of(OC.load, with_crc(b"X" + b[1:])) == "magic"
    assert field_of(OC.load, with_crc(b[:4] + b"\x09" + b[5:])) == "version"
    assert field_of(OC.load, b, h + 1) == "config"
    assert field_of(OC.load, b, h) == ""


# --------------------------------------------------------------- library
def lib_load(K):
    def f(data, h=None):
        try:
            return K.KVSnapshot.load(data, None, h)
        except K.SnapshotLoadError as e:
            raise OC.SnapshotLoadError(e.field, str(e))
    return f


def test_library_crc32_matches_reference(K, oracle):
    kat = json.load(open(os.path.join(ROOT, "tests", "golden", "kat.json")))
    assert K.crc32(b"123456789") == 0xCBF43926 and K.crc32(b"") == 0
    rng = np.random.default_rng(3)
    for n in (1, 7, 8, 9, 63, 4097, (8 << 20) + 13, (21 << 20) + 5):  # serial + threaded combine
        d = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert K.crc32(d) == oracle.crc32(d), n
        assert K.crc32(d[3:], 77) == oracle.crc32(d[3:], 77)
    assert kat  # the oracle crc32 itself is pinned to common.cpp in test_golden.py


def test_library_saves_golden_containers_bit_exact(K):
    for case in G["containers"]:
        raw = bytes.fromhex(case["container"])
        s = K.KVSnapshot.load(raw)  # host-only (no device)
        assert s.save() == raw, case["name"]
        hd = s.header()
        ref = OC.load(raw)
        assert (hd["n_layers"], hd["n_heads"], hd["head_dim"], hd["history_len"]) == \
            (ref.n_layers, ref.n_heads, ref.head_dim, ref.history_len)
        assert hd["config_hash"] == ref.config_hash
        assert s.pairs() == ref.pairs
        m = s.meta()
        assert m["conversation_id"].encode() == ref.conversation_id
        assert (m["ir_layers"], m["non_ir_layers"], m["avg_weight_sum"]) == \
            (ref.ir_layers, ref.non_ir_layers, ref.avg_weight_sum)
        p, L = s.plan()
        assert list(p) == ref.recompute_len and L == ref.history_len
        for b, (owners, span, k, v) in enumerate(ref.blobs):
            o, sp, kk, vv = s.blob(b)
            assert o == owners and sp == span
            assert kk.tobytes() == k.tobytes() and vv.tobytes() == v.tobytes()


def test_library_set_meta_round_trip(K):
    raw = bytes.fromhex(G["containers"][2]["container"])
    s = K.KVSnapshot.load(raw)
    ref = OC.load(raw)
    s.set_meta("conv-9 é", True, [3, 1], [0], [0.1, 1e-5, 2.0 / 3.0])
    ref.conversation_id, ref.exhausted_before_quota = "conv-9 é".encode(), True
    ref.ir_layers, ref.non_ir_layers, ref.avg_weight_sum = [3, 1], [0], [0.1, 1e-5, 2.0 / 3.0]
    assert s.save() == OC.save(ref)
    with pytest.raises(K.SnapshotError):  # nlohmann rejects invalid UTF-8
        s.set_meta("bad \udcff", False)
        s.save()


def test_library_file_round_trip(K, tmp_path):
    raw = bytes.fromhex(G["containers"][1]["container"])
    s = K.KVSnapshot.load(raw)
    path = str(tmp_path / "snap.krul")
    s.save_file(path)
    assert open(path, "rb").read() == raw
    t = K.KVSnapshot.load_file(path, None, s.header()["config_hash"])
    assert t.save() == raw
    with pytest.raises(K.SnapshotLoadError) as e:
        K.KVSnapshot.load_file(path, None, 1)
    assert e.value.field == "config"
    with pytest.raises(K.SnapshotError):
        K.KVSnapshot.load_file(str(tmp_path / "missing.krul"))


def test_library_errors_match_oracle_truncations(K):
    raw = bytes.fromhex(G["containers"][0]["container"])
    L = lib_load(K)
    for n in range(len(raw)):
        cut = raw[:n]
        assert field_of(L, cut) == field_of(OC.load, cut), n
        if n >= 8:  # crc repaired: exercises the structural checks
            fixed = with_crc(cut)
            assert field_of(L, fixed) == field_of(OC.load, fixed), n


def test_library_errors_match_oracle_corruptions(K):
    raw = bytes.fromhex(G["containers"][2]["container"])
    L = lib_load(K)
    rng = np.random.default_rng(11)
    seen = set()
    for i in range(len(raw) - 4):
        for flip in (0x01, 0x80, int(rng.integers(1, 256))):
            c = bytearray(raw)
            c[i] ^= flip
            c = with_crc(bytes(c))
            want = field_of(OC.load, c)
            assert field_of(L, c) == want, (i, flip)
            seen.add(want)
            if want == "":  # accepted: both must read back the same snapshot
                assert K.KVSnapshot.load(c).save() == OC.save(OC.load(c))
    assert {"magic", "version", "metadata", "plan", "blob", "coverage", ""} <= seen, seen


def test_library_metadata_edge_cases_match_oracle(K):
    base = OC.load(bytes.fromhex(G["containers"][0]["container"]))
    meta0 = OC.meta_text(base).decode()
    L = lib_load(K)

    def frame(meta: bytes) -> bytes:
        raw = bytes.fromhex(G["containers"][0]["container"])
        old = struct.unpack("<Q", raw[16:24])[0]
        body = raw[:16] + struct.pack("<Q", len(meta)) + meta + raw[24 + old:]
        return with_crc(body)

    variants = [
        meta0.replace('"mode":"mean"', '"mode":"slerp"'),
        meta0.replace('"n_layers":4', '"n_layers":3'),
        meta0.replace('"history_len":10,"mode"', '"history_len":11,"mode"'),
        meta0.replace('"n_layers":4', '"n_layers":4.0'),
        meta0.replace('"n_layers":4', '"n_layers":"4"'),
        meta0.replace('"exhausted_before_quota":false', '"exhausted_before_quota":0'),
        meta0.replace('"shared":[1,3]', '"shared":[3,1,1]'),
        meta0.replace('"conversation_id":"conv-7"', '"conversation_id":"c\\u00e9\\ud83d\\ude00\\/"'),
        meta0.replace('"conversation_id":"conv-7"', '"conversation_id":"\\ud83d"'),
        meta0.replace('"pairs":[[1,3,0.25]]', '"pairs":[[1,3,25e-2]]'),
        meta0.replace('"pairs":[[1,3,0.25]]', '"pairs":[[1,3]]'),
        meta0.replace('{"classifier"', ' \n{"classifier"') + " ",
        meta0[:-1],
        meta0 + "x",
        meta0.replace('"n_heads":2', '"n_heads":2,"n_heads":2'),
        meta0.replace('"avg_weight_sum":[]', '"avg_weight_sum":[NaN]'),
        meta0.replace('"avg_weight_sum":[]', '"avg_weight_sum":[1e400]'),
        meta0.replace('"ir_layers":[]', '"ir_layers":[-0]'),
        meta0.replace('"ir_layers":[]', '"ir_layers":[true,1e20,-1e20,99999999999,18446744073709551616]'),
        meta0.replace('"avg_weight_sum":[]', '"avg_weight_sum":[-0,true,7]'),
        meta0.replace('"shared":[1,3]', '"shared":[1,3,"x"]'),
        meta0.replace('"recompute_len":[8,6,4,2]', '"recompute_len":[8,6,4,2.9]'),
        meta0.replace('"conversation_id":"conv-7"', '"conversation_id":"conv-7","extra\\ud800":1'),
    ]
    for v in variants:
        c = frame(v.encode())
        want = field_of(OC.load, c)
        assert field_of(L, c) == want, v
        if want == "":
            assert K.KVSnapshot.load(c).save() == OC.save(OC.load(c)), v
