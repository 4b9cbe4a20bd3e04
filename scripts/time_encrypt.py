#!/usr/bin/env python
"""PKE Encrypt alone: 65,536 ciphertexts per level, one key per 256, CUDA events;
rate and fraction of the ALU roofline (bench.kem_ops). Optional HQC_ENC_KERNEL in the environment."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_12904_b200 import gen, hqc  # noqa: E402

hqc.LIB_PATH = os.environ.get("HQC_LIB", hqc.LIB_PATH)  # A/B of experiment builds


def main(B=65536, levels=(1, 3, 5)):
    dev = torch.device("cuda:0")
    for level in levels:
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
        dm, d1, d2, de = d(m), d(r1), d(r2), d(e)
        u = torch.empty(B * p.u_stride * 8, dtype=torch.uint8, device=dev)
        v = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device=dev)
        run = lambda: hqc.hqc_encrypt_batch(level, dh, ds, key, dm, d1, d2, de, u, v, check_keys=False)  # noqa: E731
        run()
        ms = bench._timed_ms(run, 10)
        ops = bench.kem_ops(p)["encrypt"]
        rate = B / ms * 1e3
        print(json.dumps({"level": level, "B": B, "ms": ms, "rate": rate,
                          "alu_roofline_frac": rate * ops / bench._alu_peak(dev)}), flush=True)


if __name__ == "__main__":
    main(levels=tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (1, 3, 5))
