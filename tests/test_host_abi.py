"""CPU-only checks of the product library: it loads, exports every symbol the
C ABI header declares, and its host-side scheduler arithmetic (plans,
calibration, blob layout, quota) is bit-exact with the oracle restatement of
proj/src/scheduler.cpp / kvstore.cpp / strategy.cpp. No device calls."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def K():
    from paper_2507_08045_b200 import native
    native.lib()
    return native


def test_exports_every_declared_symbol(K):
    hdr = open(os.path.join(ROOT, "include", "krul_b200.h")).read()
    names = set(re.findall(r"^(?:int|uint32_t|uint64_t)\s+(krul_\w+)\s*\(", hdr, re.M))
    assert len(names) > 40
    lib = ctypes.CDLL(K.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.krul_abi_version() == 1


def test_quota_matches_oracle(K, oracle):
    for n in range(0, 40):
        for r in (0, .1, .2, .25, .3, .5, .75, 1.0):
            assert K.shared_layer_quota(n, r) == oracle.quota(n, r)
    with pytest.raises(K.ConfigError):
        K.shared_layer_quota(4, 1.5)


def test_plan_hand_values(K):  # test_scheduler.cpp:73-92
    assert K.build_plan(8, 4, 0.5).tolist() == [8, 5, 3, 0]
    assert K.build_plan(10, 3, 0.0).tolist() == [0, 0, 0]
    assert K.build_plan(10, 3, 1.0).tolist() == [10, 10, 10]
    assert K.build_plan(10, 1, 0.3).tolist() == [3]
    assert K.uniform_plan(10, 3, 0.42).tolist() == [4, 4, 4]
    with pytest.raises(K.ConfigError):
        K.build_plan(8, 0, 0.5)
    with pytest.raises(K.PlanInvalidError):
        K.build_plan(8, 4, 0.5, [(1, 9, .1)])


def test_plans_bit_exact_random(K, oracle):
    rng = np.random.default_rng(5)
    for _ in range(2000):
        N = 1 + int(rng.integers(80))
        L = int(rng.integers(40000))
        r = int(rng.integers(10001)) / 10000.0
        assert np.array_equal(K.build_plan(L, N, r), oracle.build_plan(L, N, r)), (L, N, r)
        assert np.array_equal(K.uniform_plan(L, N, r), oracle.uniform_plan(L, N, r))


def test_grid_matches(K, oracle):
    for step in (0.05, 0.5, 0.01, 0.3, 1.0):
        assert np.array_equal(K.default_rc_grid(step), oracle.default_rc_grid(step))


def random_pairs(rng, N):
    perm = rng.permutation(N)
    k = int(rng.integers(0, N // 2 + 1))
    pairs = []
    for i in range(k):
        a, b = sorted((int(perm[2 * i]), int(perm[2 * i + 1])))
        pairs.append((a, b, 0.1 * (i + 1)))
    return pairs


def test_calibration_bit_exact(K, oracle):
    rng = np.random.default_rng(11)
    grid = K.default_rc_grid()
    for _ in range(300):
        N = 2 + int(rng.integers(40))
        L = 1 + int(rng.integers(20000))
        d = 64 << int(rng.integers(6))
        f = 1e12 * (1 + int(rng.integers(2000)))
        b = 1e9 * (1 + int(rng.integers(500)))
        pairs = random_pairs(rng, N)
        got = K.calibrate_rc(K.CostModel(f, b), N, L, d, pairs, grid)
        want = oracle.calibrate_rc(N, L, d, oracle.Strategy(pairs), grid, f_peak=f, b_peak=b)
        assert got == want


def test_blob_specs_match(K, oracle):  # test_kvstore.cpp:87-113
    assert K.plan_blob_specs(12, [12, 10, 8, 6, 4, 2], [(0, 5, .1), (2, 3, .2)]) == \
        [([0, 5], (2, 12)), ([1], (10, 12)), ([2, 3], (6, 12)), ([4], (4, 12))]
    rng = np.random.default_rng(3)
    for _ in range(300):
        N = 2 + int(rng.integers(40))
        L = int(rng.integers(5000))
        p = K.build_plan(L, N, float(rng.uniform()))
        pairs = random_pairs(rng, N)
        assert [(o, tuple(s)) for o, s in K.plan_blob_specs(L, p, pairs)] == \
            [(o, tuple(s)) for o, s in oracle.blob_specs(L, p, oracle.Strategy(pairs))]
    for bad in ([(1, 7, .1)], [(0, 1, .1), (1, 2, .2)]):
        with pytest.raises(K.SnapshotError):
            K.plan_blob_specs(6, [4, 3, 2, 1], bad)


def test_validate_plan_matches(K, oracle):
    rng = np.random.default_rng(8)
    for _ in range(500):
        N = 1 + int(rng.integers(20))
        L = int(rng.integers(100))
        p = rng.integers(-2, L + 3, N)
        pairs = random_pairs(rng, N)
        assert K.validate_plan(L, p, pairs) == oracle.validate_plan(L, p, oracle.Strategy(pairs))


def test_simulator_matches(K, oracle):
    rng = np.random.default_rng(9)
    for _ in range(200):
        N = 2 + int(rng.integers(30))
        L = int(rng.integers(3000))
        d = 64 << int(rng.integers(5))
        pairs = random_pairs(rng, N)
        p = K.build_plan(L, N, float(rng.uniform()), pairs)
        got = K.simulate_pipeline(L, p, pairs, K.CostModel(), d)
        want = oracle.simulate(L, p, oracle.Strategy(pairs), d)
        for k in ("makespan", "compute_finish", "load_finish", "bubble_compute", "bubble_load"):
            assert got[k] == pytest.approx(want[k], rel=1e-12, abs=1e-18)


def test_extended_cost_model_reduces_to_reference(K):
    # kv_dim = q_dim = d and tanh FFN: the extended formula is the reference one.
    d, F = 256, 1024
    ref = K.CostModel()
    ext = K.CostModel(kv_dim=d, q_dim=d, ffn_hidden=F, bytes_per_elem=4.0, ffn_kind=0)
    for L in (10, 500, 4000):
        p = K.build_plan(L, 8, 0.3)
        a = K.simulate_pipeline(L, p, [], ref, d)
        b = K.simulate_pipeline(L, p, [], ext, d)
        assert a["makespan"] == pytest.approx(b["makespan"], rel=1e-12)


def test_config_hash_matches_oracle(K, oracle):
    for kw in (dict(n_layers=4, n_heads=4, head_dim=64, d_model=256, vocab_size=256, seed=7),
               dict(n_layers=3, n_heads=2, head_dim=4, d_model=8, vocab_size=17, ffn_mult=2.0,
                    seed=5),
               dict(n_layers=32, n_heads=32, head_dim=128, d_model=4096, vocab_size=128256,
                    n_kv_heads=8, ffn_kind=1, rope_theta=500000.0, ffn_mult=3.5)):
        assert K.ModelConfig(**kw).hash() == oracle.ModelConfig(**kw).hash()


def test_validate_strategy_reference_kats(K):  # test_strategy.cpp:200-254
    ir, n, r_l = [0, 1, 2, 3], 8, 0.5
    S = K.CompressionStrategy

    def kinds(s, shared=None):
        return {line.split(":")[0] for line in K.validate_strategy(s, ir, n, r_l, shared)[1]}

    good = S([(0, 1, 0.5), (2, 3, 0.7)])
    assert K.validate_strategy(good, ir, n, r_l) == (0, [])
    assert "pair orientation" in kinds(S([(1, 0, 0.5), (2, 3, 0.7)]))
    assert "layer range" in kinds(S([(0, 1, 0.5), (2, 9, 0.7)]))
    assert "non-I-R member" in kinds(S([(0, 1, 0.5), (2, 4, 0.7)]))
    assert "layer reuse" in kinds(S([(0, 1, 0.5), (1, 2, 0.7)]), shared=[0, 1, 2])
    assert "distance order" in kinds(S([(2, 3, 0.7), (0, 1, 0.5)]))
    assert "shared size" in kinds(good, shared=[0, 1, 2])
    short = S([(0, 1, 0.5)])
    assert "quota shortfall" in kinds(short)
    short.exhausted_before_quota = True
    assert "quota shortfall" not in kinds(short)


def test_validate_strategy_matches_oracle_random(K, oracle):
    rng = np.random.default_rng(11)
    for _ in range(500):
        n = 2 + int(rng.integers(20))
        ir = sorted(set(int(x) for x in rng.integers(-1, n + 2, int(rng.integers(0, n + 1)))))
        pairs = []
        for _ in range(int(rng.integers(0, 5))):
            a, b = (int(x) for x in rng.integers(-1, n + 1, 2))
            pairs.append((a, b, float(rng.integers(0, 4)) / 4))
        shared = sorted({x for p in pairs for x in p[:2]})
        if rng.random() < 0.3 and shared:
            shared = shared[:-1]
        ex = bool(rng.random() < 0.3)
        r_l = float(rng.integers(0, 5)) / 4
        m, lines = K.validate_strategy(K.CompressionStrategy(pairs, ex), ir, n, r_l, shared)
        assert m == oracle.validate_strategy(pairs, shared, ex, ir, n, r_l), (pairs, shared, ex, ir, n, r_l)
        assert bool(lines) == bool(m)
