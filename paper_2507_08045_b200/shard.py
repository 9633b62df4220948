"""Conversation sharding across the GPUs of one box.

Every hot-path object (estimator, snapshot, plan, restore) is per
conversation and only the immutable weights are shared, so N GPUs restore N
disjoint sets of conversations with no data-path collective (BASELINE.json
configs[3]: 256 conversations of 2K-16K history over 8 GPUs). The load stream
is H2D-bound, so shards are balanced on the bytes each conversation moves
over its GPU's link (longest-processing-time-first on stored bytes); the
per-GPU link is the fabric that matters, NVLink is idle on this path.

torch.distributed is plumbing only: the barrier around the timed region and
the max-over-ranks of device time.
"""
from __future__ import annotations

import numpy as np


def synthetic_histories(n: int, lo: int = 2048, hi: int = 16384, seed: int = 2507) -> np.ndarray:
    """History lengths of the batch workload (configs[3]): U[lo, hi] tokens,
    rounded to whole KV pages (64 tokens), deterministic in `seed`."""
    rng = np.random.default_rng(seed)
    L = rng.integers(lo, hi + 1, size=n)
    return (L // 64 * 64).astype(np.int64)


def kv_bytes(L, n_layers: int, n_kv_heads: int, head_dim: int, elem_bytes: int = 2) -> np.ndarray:
    """Full (uncompressed) KV bytes of each conversation: the balancing
    weight. The compressed snapshot is a fixed fraction of it for a given
    strategy and r_c, so the ordering (all LPT needs) is the same."""
    return np.asarray(L, np.int64) * n_layers * 2 * n_kv_heads * head_dim * elem_bytes


def lpt_assign(weights, n_ranks: int) -> list[list[int]]:
    """Longest-processing-time-first: conversations in decreasing weight
    (ties by index), each to the currently least-loaded rank (ties to the
    lowest rank). Deterministic, so every rank computes the same partition
    without communicating. Returns the conversation indices per rank in
    assignment order."""
    if n_ranks < 1:
        raise ValueError("n_ranks must be >= 1")
    w = np.asarray(weights, np.int64)
    order = sorted(range(len(w)), key=lambda i: (-int(w[i]), i))
    load = [0] * n_ranks
    out: list[list[int]] = [[] for _ in range(n_ranks)]
    for i in order:
        r = min(range(n_ranks), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += int(w[i])
    return out


def shard_loads(weights, shards) -> list[int]:
    w = np.asarray(weights, np.int64)
    return [int(w[s].sum()) if len(s) else 0 for s in shards]


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar over the process group (device time of the
    slowest rank is the job's time). CUDA tensor under NCCL, CPU under gloo."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    dev = device if (device is not None and dist.get_backend() == "nccl") else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    """Sum of a per-rank scalar (e.g. conversations restored) over the group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    dev = device if (device is not None and dist.get_backend() == "nccl") else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def bind_to_gpu_numa(device: int) -> list[int] | None:
    """Pin this process to the CPUs NVML reports as local to `device`, so the
    pinned host snapshots it allocates (first touch) sit on the GPU's NUMA
    node: with 8 GPUs each load stream pulls ~55 GB/s from host DRAM and
    cross-socket traffic would cap the aggregate. Returns the CPU list or
    None when NVML is unavailable."""
    try:
        import os

        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = [64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1]
        cpus = [c for c in cpus if c < (os.cpu_count() or 0)]
        if cpus:
            os.sched_setaffinity(0, cpus)
        return cpus or None
    except Exception:
        return None
