#!/usr/bin/env python
"""KEM row timing (CUDA events): GPU Encaps and Decaps next to the fused decrypt
on the same batch; keys by the library's keygen, one keypair per 256 ciphertexts (BASELINE recipe).
Also the target command for ncu launch lists of the KEM pipeline."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import CONFIG_SEED, gen_shape  # noqa: E402
from paper_2512_12904_b200 import gen, hqc  # noqa: E402


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", default="1,3,5")
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    out = {}
    for level in [int(x) for x in a.levels.split(",")]:
        p = hqc.params(level)
        B = a.batch
        sh = gen_shape(p)
        seed = CONFIG_SEED[level]
        key = gen.key_of(0, B)
        nk = int(key[-1]) + 1
        h, x, y = gen.key_draws(seed, sh, 0, nk)

        def d(t):
            return torch.from_numpy(np.ascontiguousarray(t).view(np.uint8).reshape(-1)).to(dev)

        dh, dy = d(h), d(y)
        ds = torch.empty(nk * p.u_stride * 8, dtype=torch.uint8, device=dev)
        hqc.hqc_keygen_batch(level, dh, d(x), dy, ds)
        hpk = torch.empty(nk * 32, dtype=torch.uint8, device=dev)
        hqc.hqc_kem_hpk_batch(level, dh, ds, hpk)
        sigma = d(gen.rand_bytes(seed, gen.TAG_TEST, 0, nk, p.k))
        m = d(gen.rand_bytes(seed, gen.TAG_TEST, 1 << 20, B, p.k))
        dkey = d(key.astype(np.uint32))
        u = torch.empty(B * p.u_stride * 8, dtype=torch.uint8, device=dev)
        v = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device=dev)
        K1, K2 = (torch.empty(B * 64, dtype=torch.uint8, device=dev) for _ in range(2))
        acc = torch.empty(B, dtype=torch.uint8, device=dev)
        ws = torch.empty(hqc.hqc_kem_workspace_bytes(level, B), dtype=torch.uint8, device=dev)
        yrow = d(y[key])
        mo = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
        enc = timed(lambda: hqc.hqc_kem_encaps_batch(level, dh, ds, hpk, dkey, m, u, v, K1, ws), a.iters)
        dec = timed(lambda: hqc.hqc_kem_decaps_batch(level, dh, ds, hpk, sigma, dkey, dy, u, v, K2, acc, ws),
                    a.iters)
        pke = timed(lambda: hqc.hqc_decrypt_batch(level, u, v, yrow, mo), a.iters)
        ok = int(acc.sum()) == B and torch.equal(K1, K2) and torch.equal(mo, m)
        out[f"hqc{level}"] = {"batch": B, "encaps_ms": enc, "decaps_ms": dec, "pke_decrypt_ms": pke,
                              "encaps_per_s": B / enc * 1e3, "decaps_per_s": B / dec * 1e3,
                              "all_accepted_and_K_equal": ok}
        print(json.dumps({f"hqc{level}": out[f"hqc{level}"]}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
