#!/usr/bin/env python3
"""Generates tests/golden/kat.json (committed; the GPU box has no /root/reference).

Two kinds of entries:
  * `kat`: the reference's own known-answer tests, transcribed with their
    file:line (proj/tests/*.cpp) -- the values the reference asserts.
  * `ref_generated`: outputs of the REAL reference code compiled here from
    /root/reference/proj/src/common.cpp + include/krul/common.hpp by
    oracle/ref.mk (oracle/_ref/libkrul_ref_common.so): fnv1a64 / crc32 of
    seeded byte strings and UniformStream draws (next(lo, hi), next_index),
    which also define the model weights (engine.cpp:368-393 draw order) and
    the token ids of the parity tests (test_engine.cpp:18-26).
The rest of the reference needs Eigen3 (absent) and is not built.

usage: make -C oracle -f ref.mk && python tests/golden/make_golden.py
"""
import ctypes as C
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "tests", "golden", "kat.json")


def ref_lib():
    lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libkrul_ref_common.so"))
    lib.ref_fnv1a64.restype = C.c_uint64
    lib.ref_fnv1a64.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
    lib.ref_crc32.restype = C.c_uint32
    lib.ref_crc32.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32]
    lib.ref_uniform_next.argtypes = [C.c_uint64, C.c_int64, C.c_float, C.c_float, C.c_void_p]
    lib.ref_uniform_index.argtypes = [C.c_uint64, C.c_int64, C.c_uint64, C.c_void_p]
    return lib


KAT = {
    "fnv1a64": {  # test_common.cpp:23-28
        "": "cbf29ce484222325", "a": "af63dc4c8601ec8c", "foobar": "85944171f73967e8"},
    "crc32": {"": 0, "123456789": 0xCBF43926},  # test_common.cpp:31-35
    "quota": [  # test_strategy.cpp:75-87: (n_layers, r_l, quota)
        [32, 0.5, 16], [5, 0.5, 3], [5, 0.0, 0], [4, 1.0, 4], [10, 0.25, 3], [10, 0.2, 2],
        [0, 0.5, 0]],
    "select_hand": {  # test_strategy.cpp:89-110 (values(2,1) = values(1,2))
        "D": [[0, 3, 1, 4], [3, 0, 5, 2], [1, 5, 0, 6], [4, 2, 6, 0]], "layers": [0, 1, 2, 3],
        "r_l": 1.0, "n_layers": 4, "pairs": [[0, 2, 1.0], [1, 3, 2.0]], "exhausted": False},
    "select_ties": {  # test_strategy.cpp:123-134: ones - identity, 6 layers
        "n": 6, "r_l": 1.0, "pairs": [[0, 1, 1.0], [2, 3, 1.0], [4, 5, 1.0]]},
    "blob_layout": {  # test_kvstore.cpp:87-105
        "pairs": [[0, 5, 0.1], [2, 3, 0.2]], "plan": [12, 10, 8, 6, 4, 2], "L": 12,
        "specs": [[[0, 5], [2, 12]], [[1, -1], [10, 12]], [[2, 3], [6, 12]], [[4, -1], [4, 12]]],
        "full_plan": [12, 3], "full_specs": [[[0, -1], [12, 12]], [[1, -1], [3, 12]]]},
    "cost": {"layer_flops_2_4": 816.0, "blob_bytes_3_4": 96.0},  # test_scheduler.cpp:52-58
    "plans": [  # test_scheduler.cpp:73-92, 119-125: (L, N, r_c, recompute_len)
        [8, 4, 0.5, [8, 5, 3, 0]], [10, 3, 0.0, [0, 0, 0]], [10, 3, 1.0, [10, 10, 10]],
        [10, 1, 0.3, [3]]],
    "uniform_plans": [[10, 3, 0.42, [4, 4, 4]], [10, 2, 1.0, [10, 10]]],
    "grid": {"n": 21, "first": 0.0, "last": 1.0, "mid": 0.5, "coarse_0.5": [0.0, 0.5, 1.0]},
    "storage_fraction": 0.45,  # acceptance.cpp:363-399 / test_kvstore.cpp:223-242
}


def main():
    lib = ref_lib()
    rng = np.random.default_rng(2507)
    gen = {"fnv1a64": [], "crc32": [], "uniform": [], "uniform_index": []}
    for n in (0, 1, 7, 64, 1000):
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        buf = C.create_string_buffer(data, max(n, 1))
        gen["fnv1a64"].append({"hex": data.hex(), "value": "%016x" % lib.ref_fnv1a64(buf, n, 0xCBF29CE484222325)})
        gen["crc32"].append({"hex": data.hex(), "value": int(lib.ref_crc32(buf, n, 0))})
    for seed, lo, hi, n in ((42, -2.0, 3.0, 256), (43, -2.0, 3.0, 64), (7, -0.0625, 0.0625, 4096),
                            (11, 0.0, 1.0, 256)):
        out = np.empty(n, np.float32)
        lib.ref_uniform_next(seed, n, lo, hi, out.ctypes.data)
        gen["uniform"].append({"seed": seed, "lo": lo, "hi": hi,
                               "bits": [int(x) for x in out.view(np.uint32)]})
    for seed, mod, n in ((7, 13, 200), (11, 256, 512), (3, 17, 64)):
        out = np.empty(n, np.uint64)
        lib.ref_uniform_index(seed, n, mod, out.ctypes.data)
        gen["uniform_index"].append({"seed": seed, "mod": mod, "values": [int(x) for x in out]})
    json.dump({"kat": KAT, "ref_generated": gen,
               "source": "proj/tests/*.cpp (kat) and proj/src/common.cpp compiled by oracle/ref.mk"},
              open(OUT, "w"), indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
