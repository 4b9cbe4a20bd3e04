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
    if dist.get_backend() == "gloo":  # gloo reduces host tensors
        device = "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(count, device=None) -> int:
    """count: python int or a 1-element int64 tensor (summed in place when it is a tensor)."""
    import torch
    import torch.distributed as dist

    t = count if isinstance(count, torch.Tensor) else torch.tensor([int(count)], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        if dist.get_backend() == "gloo":  # gloo reduces host tensors
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


def gather_objects(obj) -> list:
    """Every rank's `obj` (picklable), in rank order; [obj] for a single process."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def merge_clocks(per_rank: list) -> dict:
    """Clock records of all ranks (each {"sm_mhz", "sm_mhz_min", "sm_max_mhz", "reasons", "samples"}) ->
    one record: the median SM clock of the slowest rank, the minimum over ranks, the union of the
    throttle reasons, and the per-rank medians (a throttled rank is visible, not averaged away)."""
    med = [c.get("sm_mhz") for c in per_rank if c.get("sm_mhz") is not None]
    mins = [c.get("sm_mhz_min", c.get("sm_mhz")) for c in per_rank if c.get("sm_mhz") is not None]
    reasons = sorted({r for c in per_rank for r in c.get("reasons", [])})
    maxes = [c.get("sm_max_mhz") for c in per_rank if c.get("sm_max_mhz") is not None]
    return {"sm_mhz": min(med) if med else None, "sm_mhz_min": min(mins) if mins else None,
            "sm_max_mhz": max(maxes) if maxes else None, "reasons": reasons,
            "samples": sum(int(c.get("samples", 0)) for c in per_rank),
            "per_rank_sm_mhz": [c.get("sm_mhz") for c in per_rank]}


def scaling_run(levels, total: int, world: int, rank: int, run_shard, ops_per_unit: dict, peak_per_gpu: float,
                device=None) -> dict:
    """Strong-scaling measurement of BASELINE configs[4]: for each level, `total` units split
    evenly and contiguously over the ranks (split_even); run_shard(level, i0, n) runs this rank's shard
    and returns (ms_per_step, mismatches, clocks); the job's time is the MAX over ranks, the mismatches the
    SUM, the clocks are gathered from every rank. The same function runs under gloo in the CPU tests."""
    res = {}
    for level in levels:
        i0, n = split_even(total, world, rank)
        ms, bad, clk = run_shard(level, i0, n)
        ms_max = max_over_ranks(ms, device)
        bad_sum = sum_over_ranks(int(bad), device)
        clocks = merge_clocks(gather_objects(clk))
        shards = gather_objects((i0, n))
        val = total / (ms_max / 1e3)
        res[str(level)] = {"value": val, "unit": "decryptions/s", "total_batch": total, "n_gpus": world,
                           "ms_per_step": ms_max, "per_gpu_value": val / world,
                           "alu_roofline_frac": val / world * ops_per_unit[level] / peak_per_gpu,
                           "mismatches_vs_message": bad_sum, "shards": [list(s) for s in shards],
                           "clocks": clocks}
    return res
