"""Parity of an experiment build's standalone product (hqc_sparse_dense_mul_batch with v; HQC_S1_KERNEL from
the environment) against a numpy roll-and-XOR of a few rows per level. Usage: par_s1_lib.py LIB.so"""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch
from paper_2512_12904_b200 import hqc
hqc.LIB_PATH = os.path.abspath(sys.argv[1])
from bench import make_inputs
ok = True
for level in (1, 3, 5):
    p = hqc.params(level)
    B = 600
    u, v, y = make_inputs(level, 0, B, p)
    du, dv, dy = (torch.from_numpy(a.view(np.uint8)).cuda() for a in (u, v, y))
    dr = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device="cuda")
    hqc.hqc_sparse_dense_mul_batch(level, du, dy, dv, dr)
    torch.cuda.synchronize()
    got = dr.cpu().numpy().view(np.uint64).reshape(B, p.v_words)
    # reference by plain numpy bit arithmetic on a few rows
    n = p.n
    for b in range(0, B, 97):
        ub = np.unpackbits(u[b].view(np.uint8), bitorder="little")[:n]
        acc = np.zeros(n, np.uint8)
        for yi in y[b][: p.w]:
            acc ^= np.roll(ub, int(yi))
        vb = np.unpackbits(v[b].view(np.uint8), bitorder="little")[: p.n12]
        ref = np.packbits(acc[: p.n12] ^ vb, bitorder="little").view(np.uint64)
        if not (ref == got[b]).all():
            ok = False
            print("MISMATCH level", level, "row", b)
            break
print("S1T_PARITY", ok)
