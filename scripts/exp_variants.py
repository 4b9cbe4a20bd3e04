#!/usr/bin/env python
"""Timing experiments: the fused kernel with stage 2 and/or stage 3 compiled out (results invalid,
time only) to attribute the fused kernel's time. Build here (nvcc), run on the GPU box."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = {"full": 0, "no_s2": 1, "no_s3": 2, "no_s2s3": 3}
PHASES = ["wait_uy", "stage_d+buildE+sync", "product", "sync_after_product", "combine+wait_v+store",
          "stage2", "sync_after_stage2", "stage3",
          "ws.P.wait_u", "ws.P.build", "ws.P.wait_empty", "ws.P.product", "ws.P.combine",
          "ws.D.wait_full", "ws.D.stage2", "ws.Q.wait_sfull"]


def build():
    from paper_2512_12904_b200 import build as b
    for name, skip in VAR.items():
        b.build_variant(os.path.join(ROOT, "scripts", f"libhqc_exp_{name}.so"), [f"HQC_EXP_SKIP={skip}"])
    b.build_variant(os.path.join(ROOT, "scripts", "libhqc_exp_timing.so"), ["HQC_EXP_TIMING=1"])


def timing():
    """Per-phase warp-cycle totals of the fused kernel (lane 0 of each warp, clock64)."""
    import ctypes

    import numpy as np
    import torch

    from bench import make_inputs
    from paper_2512_12904_b200 import hqc

    hqc.LIB_PATH = os.path.join(ROOT, "scripts", "libhqc_exp_timing.so")
    L = hqc.lib()
    out = {}
    for level in (1, 3, 5):
        p = hqc.params(level)
        B = 65536
        u, v, y = make_inputs(level, 0, B, p)
        du, dv, dy = (torch.from_numpy(a.view(np.uint8)).cuda() for a in (u, v, y))
        dm = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
        f = getattr(L, f"hqc_exp_phases_l{level}")
        buf = (ctypes.c_ulonglong * 16)()
        hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
        f(buf)
        hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
        f(buf)
        out[level] = {PHASES[i]: round(buf[i] / B, 0) for i in range(16) if buf[i]}
    print(json.dumps(out))


def run():
    import numpy as np
    import torch

    from bench import make_inputs
    from paper_2512_12904_b200 import hqc

    res = {}
    for name in VAR:
        hqc._lib = None
        hqc._cparams.clear()
        hqc.LIB_PATH = os.path.join(ROOT, "scripts", f"libhqc_exp_{name}.so")
        for level in (1, 3, 5):
            p = hqc.params(level)
            B = 65536
            u, v, y = make_inputs(level, 0, B, p)
            du, dv, dy = (torch.from_numpy(a.view(np.uint8)).cuda() for a in (u, v, y))
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
    {"build": build, "timing": timing, "run": run}[sys.argv[1]]()
