"""Multi-GPU plumbing for the batched decrypt: one process per GPU, torch.distributed.

The path partitions trivially — ciphertexts are independent — so rank r owns the contiguous slice
[r*B, (r+1)*B) of the seeded workload (weak scaling) and the timed region holds no collective. After
timing, one MAX all-reduce of the elapsed time (the job's time is the slowest rank's) and one SUM
all-reduce of the mismatch count. Backend "nccl" on GPUs; the same code runs on "gloo" in the CPU
tests (tests/test_dist_cpu.py).
"""
from __future__ import annotations

import os


def env() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(rank: int, per_rank: int) -> tuple[int, int]:
    """Global index range [i0, i0 + n) of this rank's ciphertexts (weak scaling: n = per_rank)."""
    return rank * per_rank, per_rank


def split_even(total: int, world: int, rank: int) -> tuple[int, int]:
    """Strong-scaling split of `total` ciphertexts: contiguous, sizes differ by at most one."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi - lo


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(count, device=None) -> int:
    """count: python int or a 1-element int64 tensor (summed in place when it is a tensor)."""
    import torch
    import torch.distributed as dist

    t = count if isinstance(count, torch.Tensor) else torch.tensor([int(count)], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())
