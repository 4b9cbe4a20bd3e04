#!/usr/bin/env python
"""Occupancy sweep of the fused kernel: __launch_bounds__ min-CTAs variants (build here, run there)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VALUES = [int(x) for x in os.environ.get("OCC_VALUES", "6,7,8,9,10,11,12,14").split(",")]
MACRO = os.environ.get("OCC_MACRO", "HQC_DEC_MINCTAS")


def build():
    from concurrent.futures import ThreadPoolExecutor

    from paper_2512_12904_b200 import build as b

    def one(m):
        return b.build_variant(os.path.join(ROOT, "scripts", f"libhqc_occ_{m}.so"), [f"{MACRO}={m}"])

    with ThreadPoolExecutor(4) as ex:
        list(ex.map(one, VALUES))


def run():
    import numpy as np
    import torch

    from bench import make_inputs
    from paper_2512_12904_b200 import hqc

    inputs = {}
    res = {}
    for m in VALUES:
        hqc._lib = None
        hqc._cparams.clear()
        hqc.LIB_PATH = os.path.join(ROOT, "scripts", f"libhqc_occ_{m}.so")
        for level in (1, 3, 5):
            p = hqc.params(level)
            B = 65536
            if level not in inputs:
                u, v, y = make_inputs(level, 0, B, p)
                inputs[level] = [torch.from_numpy(a.view(np.uint8)).cuda() for a in (u, v, y)]
            du, dv, dy = inputs[level]
            dm = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
            for _ in range(3):
                hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(20):
                hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
            e1.record()
            torch.cuda.synchronize()
            res[f"m{m}_L{level}"] = round(e0.elapsed_time(e1) / 20, 4)
    print(json.dumps(res))


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
