#!/usr/bin/env python
"""A/B timing of two builds of the library (the product .so and an experiment .so from
build.build_variant) on the same inputs: graph-timed launches per (level, batch).
    python scripts/exp_lib_ab.py LIB_A LIB_B level:batch[,level:batch...]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, "ROOT")
import bench
from paper_2512_12904_b200 import hqc
sys.path.insert(0, "ROOT/scripts")
from sweep_launch import graph_ms
hqc.LIB_PATH = sys.argv[1]
for c in sys.argv[2].split(","):
    level, B = map(int, c.split(":"))
    p = hqc.params(level)
    u, v, y = (torch.from_numpy(a.view(np.uint8).reshape(-1)).cuda() for a in bench.make_inputs(level, 0, B, p))
    m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
    run = lambda: hqc.hqc_decrypt_batch(level, u, v, y, m)
    run(); torch.cuda.synchronize()
    ms = graph_ms(run, G=16, R=5) if B <= 16384 else bench._timed_ms(run, 10)
    print(json.dumps({"lib": sys.argv[1].split("/")[-1], "level": level, "B": B, "ms": ms, "rate": B / ms * 1e3}), flush=True)
'''.replace("ROOT", ROOT)

if __name__ == "__main__":
    # an argument "KERNEL=k@LIB" runs LIB with HQC_DEC_KERNEL=k
    for rep in range(2):
        for lib in sys.argv[1:3]:
            env = dict(os.environ)
            if "@" in lib:
                kv, lib = lib.split("@")
                env["HQC_DEC_KERNEL"] = kv.split("=")[1]
            r = subprocess.run([sys.executable, "-c", CODE, lib, sys.argv[3]], capture_output=True, text=True, cwd=ROOT,
                               env=env)
            if "HQC_DEC_KERNEL" in env:
                sys.stdout.write(f"# HQC_DEC_KERNEL={env['HQC_DEC_KERNEL']}\n")
            sys.stdout.write(r.stdout + (r.stderr[-2000:] if r.returncode else ""))
            sys.stdout.flush()
