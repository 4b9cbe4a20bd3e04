#!/usr/bin/env python
"""Time the standalone product hqc_sparse_dense_mul_batch (v = NULL, as bench.py's standalone_product)
of an experiment build. Usage: time_s1_lib.py LIB.so LEVELS"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import make_inputs  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402

hqc.LIB_PATH = os.path.abspath(sys.argv[1])
res = {}
for level in [int(x) for x in sys.argv[2].split(",")]:
    p = hqc.params(level)
    B = 65536
    u, _, y = make_inputs(level, 0, B, p)
    du, dy = (torch.from_numpy(a.view(np.uint8)).cuda() for a in (u, y))
    dr = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        hqc.hqc_sparse_dense_mul_batch(level, du, dy, None, dr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        hqc.hqc_sparse_dense_mul_batch(level, du, dy, None, dr)
    e1.record()
    torch.cuda.synchronize()
    res[f"L{level}"] = round(e0.elapsed_time(e1) / 20, 4)
print(os.path.basename(sys.argv[1]), json.dumps(res), flush=True)
