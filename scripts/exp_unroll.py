#!/usr/bin/env python
"""Stage-1 loop unroll experiment (HQC_S1_UNROLL) on the fused kernel."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARS = {"u1": ["HQC_S1_UNROLL=1"], "u2": ["HQC_S1_UNROLL=2"], "u3": ["HQC_S1_UNROLL=3"]}


def build():
    from concurrent.futures import ThreadPoolExecutor

    from paper_2512_12904_b200 import build as b
    with ThreadPoolExecutor(3) as ex:
        list(ex.map(lambda kv: b.build_variant(os.path.join(ROOT, "scripts", f"libhqc_{kv[0]}.so"), kv[1]), VARS.items()))


def run():
    import numpy as np
    import torch

    from bench import make_inputs
    from paper_2512_12904_b200 import hqc
    res, inputs = {}, {}
    for name in VARS:
        hqc._lib = None
        hqc._cparams.clear()
        hqc.LIB_PATH = os.path.join(ROOT, "scripts", f"libhqc_{name}.so")
        for level in (1, 3, 5):
            p = hqc.params(level)
            B = 65536
            if level not in inputs:
                inputs[level] = [torch.from_numpy(a.view(np.uint8)).cuda() for a in make_inputs(level, 0, B, p)]
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
            res[f"{name}_L{level}"] = round(e0.elapsed_time(e1) / 20, 4)
    print(json.dumps(res))


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
