"""GPU parity of the warp RS decoder (stage3_warp.cuh: riBM, Chien, Forney) around the decoding radius
at every level, through the kernels that use it: k_decrypt_sb (HQC_DEC_KERNEL=5) and k_decrypt_sp (7),
and the library's default for the same batch. Each row has t ~ U{delta-2 .. delta+3} RM blocks replaced
by random bits (R#17), so the received RS words carry errors just inside and just beyond delta; the
outputs (corrected messages or the uncorrected garbage) must equal the oracle's bit for bit."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, numpy as np, torch
sys.path.insert(0, "tests")
import oracle
from paper_2512_12904_b200 import gen, hqc
from workloads import valid_batch
for level in (1, 3, 5):
    B = 300
    W = valid_batch(level, 123_456, B)
    p = W["params"]
    t = gen.randomise_blocks(W["v"], 123_456, 777 + level, W["shape"], max(p.delta - 2, 0), p.delta + 3)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).cuda()
    m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
    hqc.hqc_decrypt_batch(level, d(W["u"]), d(W["v"]), d(W["y"]), m)
    torch.cuda.synchronize()
    got = m.cpu().numpy().reshape(B, p.k)
    ref = oracle.decrypt_batch(p, W["u"], W["v"], W["y"])
    bad = np.nonzero((got != ref).any(axis=1))[0]
    assert bad.size == 0, (level, bad[:8], t[bad[:8]])
    # both sides of the radius occur: some rows decode to m, some do not
    ok = (got == W["m"]).all(axis=1)
    assert ok.any() and (~ok).any(), (level, ok.mean())
print("ok")
'''


@pytest.mark.parametrize("kernel", ["", "5", "7"])
def test_warp_rs_decoder_around_the_radius(kernel):
    env = dict(os.environ)
    env.pop("HQC_DEC_KERNEL", None)
    if kernel:
        env["HQC_DEC_KERNEL"] = kernel
    r = subprocess.run([sys.executable, "-c", CODE], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr[-3000:]
