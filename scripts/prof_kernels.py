#!/usr/bin/env python
"""Per-kernel timing (CUDA events) of the fused decrypt and the three per-stage kernels on the bench's
synthetic inputs; also the target command for ncu captures (scripts/gpu_*.sh)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import algorithmic_ops, make_inputs  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=3)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default="all", choices=["all", "fused", "s1", "s1n", "s2", "s3"])
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    p = hqc.params(a.level)
    B = a.batch
    u, v, y = make_inputs(a.level, 0, B, p)
    du, dv, dy = (torch.from_numpy(x.view(np.uint8).reshape(-1)).to(dev) for x in (u, v, y))
    dm = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
    dr = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device=dev)
    ds = torch.empty(B * p.n1, dtype=torch.uint8, device=dev)
    ops = {
        "fused": lambda: hqc.hqc_decrypt_batch(a.level, du, dv, dy, dm),
        "s1": lambda: hqc.hqc_sparse_dense_mul_batch(a.level, du, dy, dv, dr),
        "s1n": lambda: hqc.hqc_sparse_dense_mul_batch(a.level, du, dy, None, dr),  # standalone product, v = NULL
        "s2": lambda: hqc.hqc_rm_decode_batch(a.level, dr, ds),
        "s3": lambda: hqc.hqc_rs_decode_batch(a.level, ds, dm),
    }
    names = [n for n in ops if n != "s1n"] if a.only == "all" else [a.only]
    if a.only in ("s2", "s3"):
        ops["s1"]()
        if a.only == "s3":
            ops["s2"]()
    res = {}
    for name in names:
        for _ in range(3):
            ops[name]()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            ops[name]()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        res[name] = {"ms": ms, "decryptions_per_s": B / (ms / 1e3)}
    res["ops"] = algorithmic_ops(p)
    res["level"], res["batch"] = a.level, B
    print(json.dumps(res))


if __name__ == "__main__":
    main()
