"""The N > 1 host logic on CPU with the gloo backend, world size 2: shards are
disjoint and cover the job, every rank regenerates its shard of the seeded workload bit-identically
to a single-process generation of the whole range, and the MAX-time / SUM-mismatch reductions."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2512_12904_b200 import dist as hdist
from paper_2512_12904_b200 import gen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, r, lr = hdist.env()
    i0, n = hdist.shard(r, per_rank)
    sup = gen.support(77, gen.TAG_R2, i0, n, 35851, 114, 116)
    dense = gen.dense(77, gen.TAG_H, i0, n, 35851, 562)
    t = hdist.max_over_ranks(1.5 + r)
    c = hdist.sum_over_ranks(10 * (r + 1))
    ct = torch.tensor([3 + r], dtype=torch.int64)
    c2 = hdist.sum_over_ranks(ct)
    q.put((r, w, i0, n, sup, dense, t, c, c2))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_sharding_and_reductions(world):
    per_rank = 96
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    whole_sup = gen.support(77, gen.TAG_R2, 0, world * per_rank, 35851, 114, 116)
    whole_dense = gen.dense(77, gen.TAG_H, 0, world * per_rank, 35851, 562)
    covered = []
    for r, w, i0, n, sup, dense, t, c, c2 in res:
        assert w == world
        covered += list(range(i0, i0 + n))
        assert (sup == whole_sup[i0:i0 + n]).all() and (dense == whole_dense[i0:i0 + n]).all()
        assert t == 1.5 + world - 1
        assert c == sum(10 * (k + 1) for k in range(world))
        assert c2 == sum(3 + k for k in range(world))
    assert covered == list(range(world * per_rank))


def test_split_even():
    for total in (0, 1, 7, 4194304, 4194305):
        for world in (1, 2, 4, 8):
            parts = [hdist.split_even(total, world, r) for r in range(world)]
            assert sum(n for _, n in parts) == total
            assert all(parts[r][0] + parts[r][1] == (parts[r + 1][0] if r + 1 < world else total) for r in range(world))
            assert max(n for _, n in parts) - min(n for _, n in parts) <= 1


def _scaling_worker(rank, world, port, total, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seen = []

    def run_shard(level, i0, n):  # stands in for bench.config5_block's device part
        seen.append((level, i0, n))
        # rank r is slower by r ms; rank 1 sees one mismatch and a throttle reason at level 3
        clk = {"sm_mhz": 1965.0 - 10 * rank, "sm_mhz_min": 1900.0 - rank, "sm_max_mhz": 1965.0,
               "reasons": ["sw_power_cap"] if (rank == 1 and level == 3) else [], "samples": 5}
        return 10.0 * level + rank, int(rank == 1), clk

    ops = {1: 100, 3: 200, 5: 400}
    res = hdist.scaling_run((1, 3, 5), total, world, rank, run_shard, ops, peak_per_gpu=1e9)
    q.put((rank, seen, res))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_scaling_run():
    """bench.config5_block's host logic (hdist.scaling_run) at world size 2: even contiguous shards of the
    total, job time = MAX over ranks, rate = total / that time, mismatches SUMmed, clocks from both ranks
    (slowest median, union of reasons)."""
    world, total = 2, 4_194_305
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_scaling_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = [hdist.split_even(total, world, r) for r in range(world)]
    for rank, seen, out in res:
        assert [s[1:] for s in seen] == [shards[rank]] * 3
        assert out == res[0][2]  # every rank holds the same reduced result
    out = res[0][2]
    for level in (1, 3, 5):
        r = out[str(level)]
        assert r["ms_per_step"] == 10.0 * level + 1  # the slower rank
        assert r["value"] == pytest.approx(total / ((10.0 * level + 1) / 1e3))
        assert r["per_gpu_value"] == pytest.approx(r["value"] / world)
        assert r["alu_roofline_frac"] == pytest.approx(r["value"] / world * {1: 100, 3: 200, 5: 400}[level] / 1e9)
        assert r["mismatches_vs_message"] == 1
        assert r["shards"] == [list(s) for s in shards]
        assert r["clocks"]["sm_mhz"] == 1955.0 and r["clocks"]["sm_mhz_min"] == 1899.0
        assert r["clocks"]["per_rank_sm_mhz"] == [1965.0, 1955.0]
        assert r["clocks"]["reasons"] == (["sw_power_cap"] if level == 3 else [])
