#!/usr/bin/env python
"""Parity of an experiment build (scripts/libx_*.so) against the oracle: valid and adversarial batches,
all levels, fused decrypt + stage-3 alone. Usage: par_lib.py LIB.so"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402

hqc.LIB_PATH = os.path.abspath(sys.argv[1])
from workloads import adversarial_batch, valid_batch  # noqa: E402

ok = True
for level in (1, 3, 5):
    p = hqc.params(level)
    for W in (valid_batch(level, 40000, 150), adversarial_batch(0, 256, 256) if level == 1 else None):
        if W is None:
            continue
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).cuda()  # noqa: E731
        B = W["u"].shape[0]
        m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
        hqc.hqc_decrypt_batch(level, d(W["u"]), d(W["v"]), d(W["y"]), m)
        torch.cuda.synchronize()
        ref = oracle.decrypt_batch(W["params"], W["u"], W["v"], W["y"])
        good = bool((m.cpu().numpy().reshape(B, p.k) == ref).all())
        ok &= good
        print("level", level, "B", B, "parity", good)
    rng = np.random.default_rng(level)
    sym = rng.integers(0, 256, (300, p.n1)).astype(np.uint8)
    for i in range(0, 300, 3):  # within capacity
        c = oracle.rs_encode(rng.integers(0, 256, p.k).astype(np.uint8), p.n1, p.k)
        pos = rng.choice(p.n1, p.delta, replace=False)
        c[pos] ^= rng.integers(1, 256, p.delta).astype(np.uint8)
        sym[i] = c
    mm = torch.empty(300 * p.k, dtype=torch.uint8, device="cuda")
    hqc.hqc_rs_decode_batch(level, torch.from_numpy(sym.reshape(-1)).cuda(), mm)
    torch.cuda.synchronize()
    ref, _ = oracle.rs_decode_batch(oracle.params(level), sym)
    good = bool((mm.cpu().numpy().reshape(300, p.k) == ref).all())
    ok &= good
    print("level", level, "rs parity", good)
print("ALL_OK" if ok else "MISMATCH")
