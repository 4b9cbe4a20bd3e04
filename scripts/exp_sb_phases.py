#!/usr/bin/env python
"""Where a small-batch launch spends its time: per-phase warp-cycle totals (clock64, lane 0 of each warp)
of k_decrypt_sb from the HQC_EXP_TIMING experiment build (results of that build are not used otherwise).
    python scripts/exp_sb_phases.py build      (here)
    python scripts/exp_sb_phases.py run        (GPU box)"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SO = os.path.join(ROOT, "scripts", "libhqc_exp_timing.so")
PH = ["prologue", "run.wait_uy", "run.stage_d+build_E", "run.product", "run.wait_v+store", "stage2", "-",
      "rs_decode_warp", "-", "rs.syndromes", "rs.bm", "rs.chien", "rs.omega", "rs.forney"]


def build():
    from paper_2512_12904_b200 import build as b
    b.build_variant(SO, ["HQC_EXP_TIMING=1"])


def run():
    import numpy as np
    import torch

    import bench
    from paper_2512_12904_b200 import hqc

    hqc.LIB_PATH = SO
    L = hqc.lib()
    buf = (ctypes.c_ulonglong * 16)()
    for level in (1, 3, 5):
        p = hqc.params(level)
        f = getattr(L, f"hqc_exp_phases_l{level}")
        for B in (1, 1024):
            u, v, y = (torch.from_numpy(a.view(np.uint8).reshape(-1)).cuda() for a in bench.make_inputs(level, 0, B, p))
            m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
            for rep in range(3):
                f(buf)
                hqc.hqc_decrypt_batch(level, u, v, y, m)
                torch.cuda.synchronize()
                f(buf)
                ms = bench._timed_ms(lambda: hqc.hqc_decrypt_batch(level, u, v, y, m), 1)
            print(json.dumps({"level": level, "B": B, "ms_one_launch": ms,
                              "cycles_per_warp": {PH[i]: round(buf[i] / B) for i in range(len(PH))}}), flush=True)


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
