"""Multi-GPU sharding of a batched call (host logic only).

The batch of independent problems shards with NO exchange step (SURVEY
section 8.5): GPU g of G owns the contiguous range
[floor(g*B/G), floor((g+1)*B/G)) of the global problem index space, builds
its own inputs for those indices (counter-based generator, so no data moves)
and calls the library on its own stream.  Results are bitwise identical to a
one-GPU run because every C element is one fixed-order FMA chain that does
not depend on the batch split (tests/test_gpu_parity.py).

No collective is on the data path; torch.distributed is used by bench.py
only for the barrier around the timed region and the max-over-ranks time.
"""
from __future__ import annotations


def shard_range(total: int, rank: int, world: int):
    """Contiguous [lo, hi) share of `total` problems for `rank` of `world`
    (strong scaling: the global batch is fixed)."""
    if world <= 0 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard arguments")
    return (total * rank) // world, (total * (rank + 1)) // world


def weak_range(per_rank: int, rank: int):
    """Global problem ids of `rank` when every rank processes `per_rank`
    problems (weak scaling: per-GPU work fixed)."""
    return rank * per_rank, (rank + 1) * per_rank


def aggregate_gflops(flops_per_rank, times_s):
    """Whole-job GFLOP/s: total flops over the SLOWEST rank's time."""
    t = max(times_s)
    return sum(flops_per_rank) / t / 1e9 if t > 0 else 0.0


def gemm_on_devices(calls):
    """Single-process multi-GPU driver (SURVEY 8.5's process model): `calls`
    is a list of (device_index, kwargs of iaat.gemm_strided_batched) whose
    tensors live on that device.  Each call is enqueued on its device's
    current stream (asynchronous; the library keeps per-device kernel
    attributes and plans), and the list returns once everything is enqueued.
    Use one shard per device from shard_range(); no data crosses devices."""
    import torch

    from . import iaat
    for dev, kw in calls:
        with torch.cuda.device(dev):
            iaat.gemm_strided_batched(**kw)
