"""Multi-GPU host logic on CPU (gloo, world_size 2): conversation sharding,
the max-over-ranks timing reduction, and the per-rank restore plan
(the path shards by conversation with no data collective).

The device restores themselves are covered by the -m gpu parity tests; here
every rank runs the same host-side planning the bench runs before its timed
region, and the ranks check they agree without exchanging anything but the
final gather used for verification."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_08045_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_lpt_partition_properties():
    L = shard.synthetic_histories(256)
    assert L.min() >= 2048 and L.max() <= 16384 and np.all(L % 64 == 0)
    w = shard.kv_bytes(L, 32, 8, 128)
    for n in (1, 2, 4, 8):
        sh = shard.lpt_assign(w, n)
        flat = sorted(i for s in sh for i in s)
        assert flat == list(range(256))  # a partition
        loads = shard.shard_loads(w, sh)
        # LPT bound: max load - min load <= the largest single item
        assert max(loads) - min(loads) <= int(w.max())
        # and within 4/3 of the ideal makespan
        assert max(loads) <= 4 / 3 * (w.sum() / n) + w.max()
    assert shard.lpt_assign([5, 5, 5], 2) == [[0, 2], [1]]  # deterministic ties
    with pytest.raises(ValueError):
        shard.lpt_assign([1], 0)


def test_numa_binding_is_safe_without_a_gpu():
    # NVML absent / no device: returns None and leaves the affinity alone
    before = os.sched_getaffinity(0)
    r = shard.bind_to_gpu_numa(0)
    assert r is None or (r and set(r) <= set(range(os.cpu_count())))
    if r is None:
        assert os.sched_getaffinity(0) == before


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_08045_b200 import native as K

        L = shard.synthetic_histories(64, seed=11)
        w = shard.kv_bytes(L, 32, 8, 128)
        mine = shard.lpt_assign(w, world)[rank]
        # the per-conversation plan each rank builds before its timed region
        cost = K.CostModel(f_peak=1.2e15, b_peak=55e9, kv_dim=1024, q_dim=4096, ffn_hidden=14336,
                           bytes_per_elem=2.0, ffn_kind=1)
        pairs = [(9 + 2 * k, 10 + 2 * k, 0.0) for k in range(8)]
        plans = {}
        for i in mine:
            r = K.calibrate_rc(cost, 32, int(L[i]), 4096, pairs)
            plans[i] = (r, [int(x) for x in K.build_plan(int(L[i]), 32, r, pairs)])
        # device time of the slowest rank is the job time
        t = shard.max_over_ranks(10.0 + rank, dist)
        assert shard.sum_over_ranks(1.0, dist) == float(world)
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, mine, plans, t))
        q.put(gathered if rank == 0 else None)
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gathered = next(r for r in res if r is not None)
    L = shard.synthetic_histories(64, seed=11)
    w = shard.kv_bytes(L, 32, 8, 128)
    ref = shard.lpt_assign(w, world)
    seen = []
    from paper_2507_08045_b200 import native as K
    for rank, mine, plans, t in gathered:
        assert mine == ref[rank]  # every rank computes the same partition alone
        assert t == 11.0           # max over ranks
        seen += mine
        for i, (r, p) in plans.items():
            # identical to a single-process plan: split points bit-exact
            assert p == [int(x) for x in K.build_plan(int(L[i]), 32, r, [(9 + 2 * k, 10 + 2 * k, 0.0)
                                                                          for k in range(8)])]
    assert sorted(seen) == list(range(64))
