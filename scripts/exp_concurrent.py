#!/usr/bin/env python
"""Can RM/RS decoding hide under the shared-memory-bound product? Time the standalone stage kernels of
one level alone and concurrently on two streams over independent batches:
  A = hqc_sparse_dense_mul_batch (stage 1) on batch X;  B = hqc_rm_decode_batch + hqc_rs_decode_batch on batch Y.
If A || B takes ~max(A, B) the SM overlaps them; ~A + B means they compete for the same resource."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import make_inputs  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402


def main(level=3, B=65536, iters=10):
    p = hqc.params(level)
    u, v, y = make_inputs(level, 0, B, p)
    du, dv, dy = (torch.from_numpy(a.view(np.uint8)).cuda() for a in (u, v, y))
    r1 = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device="cuda")
    r2 = torch.empty_like(r1)
    hqc.hqc_sparse_dense_mul_batch(level, du, dy, dv, r2)
    sym = torch.empty(B * p.n1, dtype=torch.uint8, device="cuda")
    m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()

    def A():
        with torch.cuda.stream(sA):
            hqc.hqc_sparse_dense_mul_batch(level, du, dy, dv, r1)

    def Bf():
        with torch.cuda.stream(sB):
            hqc.hqc_rm_decode_batch(level, r2, sym)
            hqc.hqc_rs_decode_batch(level, sym, m)

    def t(fns):
        for _ in range(2):
            for f in fns:
                f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ev = e0
        for s in (sA, sB):
            s.wait_event(ev)
        for _ in range(iters):
            for f in fns:
                f()
        for s in (sA, sB):
            x = torch.cuda.Event()
            x.record(s)
            torch.cuda.current_stream().wait_event(x)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    res = {"level": level, "A_stage1": t([A]), "B_stage2+3": t([Bf]), "A||B": t([A, Bf])}
    print(json.dumps(res))


if __name__ == "__main__":
    for L in (1, 3, 5):
        main(L)
