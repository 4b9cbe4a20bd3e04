#!/usr/bin/env python
"""Randomised parity soak of hqc_decrypt_batch (default launch policy) against the ORACLE, bit-exact.

Each trial draws a level, a batch size and a seed; builds D distinct ciphertexts with the oracle (valid rows,
rows with t RM blocks of v randomised around the RS decoding radius and far beyond it, uniformly random u / v:
the categories of BASELINE configs[3], R#17), decrypts them with the oracle, then decrypts on the GPU a batch
of B rows drawn from them with repetition in random order (row i = ciphertext idx[i]) and compares every
row. Batch sizes: tiny, a few chunks with a ragged tail, and sizes on both sides of every switch of the
launch policy, so that each default kernel and each split meets mixed rows.

    python scripts/soak_parity.py [trials_per_level] [seed]      (test infrastructure: it loads oracle/)
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_2512_12904_b200 import gen, hqc  # noqa: E402
from workloads import valid_batch  # noqa: E402

# batch sizes around the policy's switches (kernels.cuh dec_kernel_for / dec_split), per level
AROUND = {1: [40000, 65536, 73728, 131072], 3: [44000, 65536, 75776, 150000], 5: [16000, 24000, 65536, 262144 + 40000]}
D = 1024


def mixed_rows(level, seed, i0):
    W = valid_batch(level, i0, D, seed)
    p, sh = W["params"], W["shape"]
    rows = np.arange(D)
    cat = rows % 8  # 0-3 valid, 4-5 around the radius, 6 far beyond, 7 random u and v
    near = (cat == 4) | (cat == 5)
    gen.randomise_blocks(W["v"], i0, seed + 1, sh, max(p.delta - 2, 0), p.delta + 3, row_mask=near)
    gen.randomise_blocks(W["v"], i0, seed + 2, sh, p.delta + 1, 2 * p.delta, row_mask=cat == 6)
    r = np.nonzero(cat == 7)[0]
    W["u"][r] = gen.dense(seed, gen.TAG_U_RAND, i0, r.size, p.n, sh.u_stride)
    W["v"][r] = gen.dense(seed, gen.TAG_V_RAND, i0, r.size, p.n12, sh.v_words)
    ref = oracle.decrypt_batch(p, W["u"], W["v"], W["y"])
    assert (ref[cat < 4] == W["m"][cat < 4]).all()
    return W, ref, cat


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 20251021
    rng = np.random.default_rng(seed0)
    dev = torch.device("cuda:0")
    total = bad_total = 0
    for level in (1, 3, 5):
        p = hqc.params(level)
        for t in range(trials):
            seed = int(rng.integers(1, 2**31))
            t0 = time.time()
            W, ref, cat = mixed_rows(level, seed, int(rng.integers(0, 1 << 20)))
            du, dv, dy = (torch.from_numpy(np.ascontiguousarray(W[k]).view(np.uint8).reshape(D, -1)).to(dev)
                          for k in ("u", "v", "y"))
            sizes = [1, int(rng.integers(2, 200)), int(rng.integers(1000, 5000))]
            sizes += [int(b + rng.integers(-3000, 3000)) for b in AROUND[level]]
            for B in sizes:
                idx = rng.integers(0, D, B)
                ti = torch.from_numpy(idx).to(dev)
                u, v, y = (x.index_select(0, ti).reshape(-1).contiguous() for x in (du, dv, dy))
                m = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
                hqc.hqc_decrypt_batch(level, u, v, y, m)
                torch.cuda.synchronize()
                got = m.cpu().numpy().reshape(B, p.k)
                bad = int((got != ref[idx]).any(axis=1).sum())
                total += B
                bad_total += bad
                print(json.dumps({"level": level, "seed": seed, "B": B, "kernel": hqc.hqc_decrypt_launch_kernel(level, B),
                                  "launches": hqc.hqc_decrypt_launch_count(level, B), "mismatching_rows": bad,
                                  "garbage_rows": int((got != W["m"][idx]).any(axis=1).sum())}), flush=True)
                del u, v, y, m
            print(json.dumps({"level": level, "trial": t, "seconds": round(time.time() - t0, 1)}), flush=True)
    print(json.dumps({"rows_compared": total, "mismatching_rows": bad_total}), flush=True)
    sys.exit(1 if bad_total else 0)


if __name__ == "__main__":
    main()
