#!/usr/bin/env python
"""Time the fused decrypt against its stages run as separate launches (hqc_sparse_dense_mul_batch with v,
hqc_rm_decode_batch, hqc_rs_decode_batch) on the same valid ciphertexts: how much each stage costs
alone, and what a split pipeline would cost. Usage: time_stages.py [LEVEL:BATCH ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import make_valid_workload  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402

hqc.LIB_PATH = os.environ.get("HQC_LIB", hqc.LIB_PATH)  # A/B of experiment builds


def timed(fn, steps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


cases = sys.argv[1:] or ["1:65536", "3:65536", "5:262144"]
dev = torch.device("cuda:0")
for c in cases:
    level, B = (int(x) for x in c.split(":"))
    p = hqc.params(level)
    u, v, y, m_ref = make_valid_workload(level, 0, B, p, dev)
    m = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
    r = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device=dev)
    sym = torch.empty(B * p.n1, dtype=torch.uint8, device=dev)
    m2 = torch.empty_like(m)
    t = {
        "fused": timed(lambda: hqc.hqc_decrypt_batch(level, u, v, y, m)),
        "s1_with_v": timed(lambda: hqc.hqc_sparse_dense_mul_batch(level, u, y, v, r)),
        "rm": timed(lambda: hqc.hqc_rm_decode_batch(level, r, sym)),
        "rs": timed(lambda: hqc.hqc_rs_decode_batch(level, sym, m2)),
    }
    t["split_sum"] = t["s1_with_v"] + t["rm"] + t["rs"]
    ok = bool(torch.equal(m, m_ref)) and bool(torch.equal(m2, m_ref))
    print(json.dumps({"level": level, "B": B, "ms": {k: round(x, 4) for k, x in t.items()}, "outputs_ok": ok}),
          flush=True)
