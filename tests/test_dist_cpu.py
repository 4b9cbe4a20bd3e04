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
