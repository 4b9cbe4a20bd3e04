#!/usr/bin/env python
"""Time hqc_decrypt_batch on VALID ciphertexts (bench.make_valid_workload) under the current environment
(HQC_DEC_KERNEL, HQC_DEC_SPLIT, HQC_S12_STAGGER ... are read by the library). Usage: time_kind.py L:B[,L:B]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402

dev = torch.device("cuda:0")
tag = {k: v for k, v in os.environ.items() if k.startswith("HQC_")}
for c in sys.argv[1].split(","):
    level, B = (int(x) for x in c.split(":"))
    p = hqc.params(level)
    u, v, y, m_ref = bench.make_valid_workload(level, 0, B, p, dev)
    m = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
    run = lambda: hqc.hqc_decrypt_batch(level, u, v, y, m)  # noqa: E731
    run()
    torch.cuda.synchronize()
    ms = bench._timed_ms(run, 10 if B >= 65536 else 50)
    print(json.dumps({"env": tag, "level": level, "B": B, "ms": round(ms, 4), "rate": B / ms * 1e3,
                      "ok": bool(torch.equal(m, m_ref))}), flush=True)
