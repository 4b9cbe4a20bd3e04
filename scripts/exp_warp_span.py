#!/usr/bin/env python
"""When do the warps of one k_decrypt_sb launch start and finish? (%globaltimer per warp, HQC_EXP_TIMING
build = scripts/libhqc_exp_timing.so). Prints quantiles of start and end times relative to the earliest
start, for HQC-3 at a few batch sizes."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402

hqc.LIB_PATH = os.path.join(ROOT, "scripts", "libhqc_exp_timing.so")
L = hqc.lib()
for level, B in ((3, 65536), (3, 262144), (1, 1024)):
    p = hqc.params(level)
    u, v, y = (torch.from_numpy(a.view(np.uint8).reshape(-1)).cuda() for a in bench.make_inputs(level, 0, B, p))
    m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        hqc.hqc_decrypt_batch(level, u, v, y, m)
    torch.cuda.synchronize()
    g, w = hqc.hqc_decrypt_launch_shape(level, B)
    n = g * w
    buf = (ctypes.c_ulonglong * (2 * n))()
    getattr(L, f"hqc_exp_warp_span_l{level}")(buf, n)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 2).astype(np.float64)
    t0 = a[:, 0].min()
    st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
    q = [0, 0.01, 0.1, 0.5, 0.9, 0.99, 1.0]
    cta_end = en.reshape(g, w).max(axis=1)
    cta_mean = en.reshape(g, w).mean(axis=1)
    print(json.dumps({"level": level, "B": B, "warps": n, "start_us": np.quantile(st, q).round(2).tolist(),
                      "end_us": np.quantile(en, q).round(2).tolist(), "quantiles": q,
                      "cta_end_us": np.quantile(cta_end, q).round(1).tolist(),
                      "cta_end_by_quarter_of_blockIdx": [float(c.mean().round(1)) for c in np.array_split(cta_end, 4)],
                      "cta_end_even_odd_blockIdx": [float(cta_end[0::2].mean().round(1)), float(cta_end[1::2].mean().round(1))],
                      "within_cta_spread_us_median": float(np.median(cta_end - en.reshape(g, w).min(axis=1)).round(1))}),
          flush=True)
