"""Exponent-coded bf16 KV store (kvcode.hpp): the host codec is lossless on
every distribution the store can see — Gaussian-like KV, all 256 exponents
(forces the 12-bit length limit), a single exponent, ragged chunk tails,
empty input — and its image layout is what the device decoder reads.
CPU only (krul_ec_host_roundtrip); the device codec is checked against it
bit for bit in tests/test_gpu_parity.py."""
import ctypes as C
import struct

import numpy as np
import pytest


@pytest.fixture(scope="module")
def K():
    from paper_2507_08045_b200 import native
    native.lib()
    return native


def roundtrip(K, x):
    x = np.ascontiguousarray(x, np.uint16)
    n = C.c_uint64()
    lib = K.lib()
    assert lib.krul_ec_host_roundtrip(K._p(x), C.c_uint64(x.size), None, C.c_uint64(0), C.byref(n), None) == 0
    img = np.zeros(max(n.value, 1), np.uint8)
    dec = np.zeros(max(x.size, 1), np.uint16)
    assert lib.krul_ec_host_roundtrip(K._p(x), C.c_uint64(x.size), K._p(img), C.c_uint64(img.size),
                                      C.byref(n), K._p(dec)) == 0
    return img[:n.value], dec[:x.size]


def bf16_bits(a):
    u = np.asarray(a, np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


@pytest.mark.parametrize("n", [0, 1, 31, 63, 64, 65, 2047, 2048, 2049, 3 * 2048 + 77, 5 * 8192 + 5])
def test_gaussian_roundtrip_and_layout(K, n):
    x = bf16_bits(np.random.default_rng(n).standard_normal(n) * 0.7)
    img, dec = roundtrip(K, x)
    assert np.array_equal(dec, x)
    magic, ne, nch, base_off, cnt_off, sm_off, exp_off, words = struct.unpack("<8I", img[:32].tobytes())
    assert magic == 0x37314345 and ne == n and nch == (n + 4095) // 4096
    assert base_off == 32 and cnt_off >= base_off + 4 * (nch + 1)
    assert sm_off % 16 == 0 and exp_off % 16 == 0 and exp_off >= sm_off + n
    assert img.size == ((exp_off + 4 * (words + 1) + 15) // 16) * 16
    base = np.frombuffer(img[base_off:base_off + 4 * (nch + 1)].tobytes(), np.uint32)
    cnt = img[cnt_off:cnt_off + 32 * nch].astype(np.int64)
    assert base[0] == 0 and base[-1] == words and cnt.sum() == words and cnt.max(initial=0) <= 48
    assert np.array_equal(np.diff(base), cnt.reshape(nch, 32).sum(axis=1))
    # sign+mantissa plane is the raw low bits
    sm = img[sm_off:sm_off + n]
    assert np.array_equal(sm, (((x >> 8) & 0x80) | (x & 0x7F)).astype(np.uint8))
    if n >= 8192:  # ~10.7 of 16 bits per element on Gaussian data
        assert img.size < 0.72 * 2 * n


def test_all_exponents_force_length_limit(K):
    rng = np.random.default_rng(7)
    # geometric exponent distribution over all 256 values: optimal Huffman
    # lengths exceed 12 bits and must be limited
    e = np.minimum(rng.geometric(0.5, 200000) - 1, 255)
    e[:256] = np.arange(256)
    x = ((rng.integers(0, 2, e.size) << 15) | (e << 7) | rng.integers(0, 128, e.size)).astype(np.uint16)
    img, dec = roundtrip(K, x)
    assert np.array_equal(dec, x)


def test_single_exponent_and_specials(K):
    x = np.full(20000, 0x3F80, np.uint16)  # 1.0 everywhere: one symbol, 1-bit codes
    img, dec = roundtrip(K, x)
    assert np.array_equal(dec, x)
    sp = np.array([0x0000, 0x8000, 0x7F80, 0xFF80, 0x7FC0, 0x0001, 0x807F, 0x3F80] * 5000, np.uint16)
    img, dec = roundtrip(K, sp)  # zeros, infs, NaN, denormals keep their bits
    assert np.array_equal(dec, sp)
