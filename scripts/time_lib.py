#!/usr/bin/env python
"""Time hqc_decrypt_batch of an experiment build (scripts/exp_build.py) on the bench's inputs.
Usage: time_lib.py LIB.so LEVELS [batch]   (HQC_DEC_KERNEL etc. from the environment)"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import make_inputs  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402


def main():
    hqc.LIB_PATH = os.path.abspath(sys.argv[1])
    levels = [int(x) for x in sys.argv[2].split(",")]
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
    res = {}
    for level in levels:
        p = hqc.params(level)
        u, v, y = make_inputs(level, 0, B, p)
        du, dv, dy = (torch.from_numpy(a.view(np.uint8)).cuda() for a in (u, v, y))
        dm = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
        e1.record()
        torch.cuda.synchronize()
        res[f"L{level}"] = round(e0.elapsed_time(e1) / 20, 4)
    print(os.path.basename(sys.argv[1]), os.environ.get("HQC_DEC_KERNEL", ""), json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
