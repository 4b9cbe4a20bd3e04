#!/usr/bin/env python
"""Step a6 alone, the three GF-product methods of hqc_rs_syndromes_batch (the paper's
nibble-sliced tables vs log/antilog vs the fused kernel's GF(2)-linear map), CUDA-event timed per level
on random received words; also the ncu target (scripts/gpu_syn.sh)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_12904_b200 import hqc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", default="1,3,5")
    ap.add_argument("--methods", default="linear,nibble,logexp")
    ap.add_argument("--batch", type=int, default=262144)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    res = {}
    for level in map(int, a.levels.split(",")):
        p = hqc.params(level)
        B = a.batch
        sym = torch.from_numpy(np.random.default_rng(level).integers(0, 256, B * p.n1, dtype=np.uint8)).to(dev)
        outs = {}
        for m in a.methods.split(","):
            out = torch.empty(B * 2 * p.delta, dtype=torch.uint8, device=dev)
            for _ in range(3):
                hqc.hqc_rs_syndromes_batch(level, sym, out, m)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                hqc.hqc_rs_syndromes_batch(level, sym, out, m)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            outs[m] = out
            res[f"L{level}.{m}"] = {"ms": ms, "words_per_s": B / (ms / 1e3),
                                    "gf_macs_per_s": B * 2 * p.delta * p.n1 / (ms / 1e3)}
        ms = list(outs.values())
        res[f"L{level}.agree"] = all(torch.equal(ms[0], x) for x in ms[1:])
    print(json.dumps(res))


if __name__ == "__main__":
    main()
