#!/usr/bin/env python
"""When do the two warps (u, v) of each k_encrypt2 CTA finish? (HQC_EXP_TIMING build,
scripts/libhqc_exp_timing.so; %globaltimer per warp.)"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_12904_b200 import gen, hqc  # noqa: E402

hqc.LIB_PATH = os.path.join(ROOT, "scripts", "libhqc_exp_timing.so")
L = hqc.lib()
dev = torch.device("cuda:0")
B = 65536
for level in (1, 3):
    p = hqc.params(level)
    sh = bench.gen_shape(p)
    nk = B // 256
    h, x, y = gen.key_draws(0x5EED, sh, 0, nk)
    m, r1, r2, e = gen.ct_draws(0x5EED, sh, 0, B)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1)).to(dev)  # noqa: E731
    dh = d(h)
    ds = torch.empty(nk * p.u_stride * 8, dtype=torch.uint8, device=dev)
    hqc.hqc_keygen_batch(level, dh, d(x), d(y), ds)
    key = d((np.arange(B) // 256).astype(np.uint32))
    u = torch.empty(B * p.u_stride * 8, dtype=torch.uint8, device=dev)
    v = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device=dev)
    dm, d1, d2, de = d(m), d(r1), d(r2), d(e)
    for _ in range(3):
        hqc.hqc_encrypt_batch(level, dh, ds, key, dm, d1, d2, de, u, v, check_keys=False)
    torch.cuda.synchronize()
    n = 2 * 1024
    buf = (ctypes.c_ulonglong * (2 * 8192))()
    getattr(L, f"hqc_exp_warp_span_l{level}")(buf, 8192)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 2).astype(np.float64)
    g = int((a[:, 1] > 0).sum() // 2)
    a = a[: 2 * g]
    t0 = a[:, 0].min()
    end = (a[:, 1] - t0) / 1e3
    st = (a[:, 0] - t0) / 1e3
    eu, ev = end[0::2], end[1::2]
    dur = (end - st)[1::2]
    q = [0, 0.1, 0.5, 0.9, 1.0]
    print(json.dumps({"level": level, "ctas": g, "u_end_us": np.quantile(eu, q).round(1).tolist(),
                      "v_end_us": np.quantile(ev, q).round(1).tolist(),
                      "v_minus_u_us_median": float(np.median(ev - eu).round(1)), "quantiles": q,
                      "start_us": np.quantile(st, q).round(1).tolist(),
                      "v_duration_us": np.quantile(dur, q).round(1).tolist(),
                      "v_duration_by_blockIdx_eighths": [float(c.mean().round(1)) for c in np.array_split(dur, 8)]}),
          flush=True)
