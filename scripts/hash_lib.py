#!/usr/bin/env python
"""Hash the fused decrypt output of a library build on bench.py's seeded inputs, to compare experiment
builds against the default at batches the oracle cannot check directly (also prints mismatches against
the generator's messages when the inputs are valid ciphertexts). Usage: hash_lib.py LIB.so LEVEL BATCH"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import make_inputs  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402

hqc.LIB_PATH = os.path.abspath(sys.argv[1])
level, B = int(sys.argv[2]), int(sys.argv[3])
p = hqc.params(level)
u, v, y = make_inputs(level, 0, B, p)
du, dv, dy = (torch.from_numpy(a.view(np.uint8)).cuda() for a in (u, v, y))
dm = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
torch.cuda.synchronize()
print(os.path.basename(sys.argv[1]), level, B, hashlib.sha256(dm.cpu().numpy().tobytes()).hexdigest()[:16], flush=True)
