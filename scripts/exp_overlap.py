#!/usr/bin/env python
"""Experiment: the decrypt as a software pipeline over chunks — the product (hqc_sparse_dense_mul_batch with
v, r to HBM) of chunk i+1 on one stream while stages 2 and 3 (hqc_rm_decode_batch, hqc_rs_decode_batch) of
chunk i run on another, so the decoders' FMA/ALU work can co-run with the shared-memory-bound product.
Compares: the fused kernel, the stages back to back on one stream, and the two-stream pipeline.
Usage: exp_overlap.py LEVEL BATCH CHUNK[,CHUNK...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402

level, B = int(sys.argv[1]), int(sys.argv[2])
chunks = [int(x) for x in sys.argv[3].split(",")]
dev = torch.device("cuda:0")
p = hqc.params(level)
u, v, y, m_ref = bench.make_valid_workload(level, 0, B, p, dev)
U, V, Y = u.view(B, -1), v.view(B, -1), y.view(B, -1)
m = torch.empty((B, p.k), dtype=torch.uint8, device=dev)


def timed(fn, steps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


res = {"env": {k: v for k, v in os.environ.items() if k.startswith("HQC_")}, "level": level, "B": B, "fused_ms": timed(lambda: hqc.hqc_decrypt_batch(level, u, v, y, m.view(-1)))}
for C in chunks:
    n = (B + C - 1) // C
    r = [torch.empty((C, p.v_words * 8), dtype=torch.uint8, device=dev) for _ in range(2)]
    sym = [torch.empty((C, p.n1), dtype=torch.uint8, device=dev) for _ in range(2)]
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()

    def parts(i):
        a, b = i * C, min(B, (i + 1) * C)
        return a, b, b - a

    def seq():
        for i in range(n):
            a, b, k = parts(i)
            hqc.hqc_sparse_dense_mul_batch(level, U[a:b], Y[a:b], V[a:b], r[i % 2][:k])
            hqc.hqc_rm_decode_batch(level, r[i % 2][:k], sym[i % 2][:k])
            hqc.hqc_rs_decode_batch(level, sym[i % 2][:k], m[a:b])

    def ovl(rm_on_a=False):
        cur = torch.cuda.current_stream()
        sA.wait_stream(cur)
        sB.wait_stream(cur)
        done = [None] * n
        for i in range(n):
            a, b, k = parts(i)
            if i >= 2:
                sA.wait_event(done[i - 2])  # r[i % 2] is free once chunk i-2 is decoded
            hqc.hqc_sparse_dense_mul_batch(level, U[a:b], Y[a:b], V[a:b], r[i % 2][:k], stream=sA)
            if rm_on_a:  # stage 2 with the product, only stage 3 on the second stream
                hqc.hqc_rm_decode_batch(level, r[i % 2][:k], sym[i % 2][:k], stream=sA)
            ev = torch.cuda.Event()
            ev.record(sA)
            sB.wait_event(ev)
            if not rm_on_a:
                hqc.hqc_rm_decode_batch(level, r[i % 2][:k], sym[i % 2][:k], stream=sB)
            hqc.hqc_rs_decode_batch(level, sym[i % 2][:k], m[a:b], stream=sB)
            done[i] = torch.cuda.Event()
            done[i].record(sB)
        cur.wait_stream(sA)
        cur.wait_stream(sB)

    m.zero_()
    res[f"seq_{C}_ms"] = timed(seq)
    ok1 = bool(torch.equal(m.view(-1), m_ref))
    m.zero_()
    res[f"ovl_{C}_ms"] = timed(ovl)
    ok2 = bool(torch.equal(m.view(-1), m_ref))
    m.zero_()
    res[f"ovl2_{C}_ms"] = timed(lambda: ovl(True))
    res[f"ok_{C}"] = ok1 and ok2 and bool(torch.equal(m.view(-1), m_ref))
print(json.dumps({k: (round(x, 4) if isinstance(x, float) else x) for k, x in res.items()}), flush=True)
