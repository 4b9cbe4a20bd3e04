#!/usr/bin/env python
"""A/B of two library builds on the standalone product (v = NULL) and the fused decrypt, same inputs."""
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
hqc.LIB_PATH = sys.argv[1]
for c in sys.argv[2].split(","):
    what, level, B = c.split(":")
    level, B = int(level), int(B)
    p = hqc.params(level)
    u, v, y = (torch.from_numpy(a.view(np.uint8).reshape(-1)).cuda() for a in bench.make_inputs(level, 0, B, p))
    m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
    r = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device="cuda")
    run = (lambda: hqc.hqc_decrypt_batch(level, u, v, y, m)) if what == "dec" else \
          (lambda: hqc.hqc_sparse_dense_mul_batch(level, u, y, None, r))
    run(); torch.cuda.synchronize()
    ms = bench._timed_ms(run, 20)
    print(json.dumps({"lib": sys.argv[1].split("/")[-1], "what": what, "level": level, "B": B, "ms": round(ms, 5),
                      "rate": B / ms * 1e3}), flush=True)
'''.replace("ROOT", ROOT)

if __name__ == "__main__":
    # an argument "S1=k@LIB" runs LIB with HQC_S1_KERNEL=k
    for rep in range(2):
        for lib in sys.argv[1:3]:
            env = dict(os.environ)
            if "@" in lib:
                kv, lib = lib.split("@")
                env["HQC_S1_KERNEL"] = kv.split("=")[1]
                sys.stdout.write(f"# HQC_S1_KERNEL={env['HQC_S1_KERNEL']}\n")
            r = subprocess.run([sys.executable, "-c", CODE, lib, sys.argv[3]], capture_output=True, text=True, cwd=ROOT,
                               env=env)
            sys.stdout.write(r.stdout + (r.stderr[-2000:] if r.returncode else ""))
            sys.stdout.flush()
