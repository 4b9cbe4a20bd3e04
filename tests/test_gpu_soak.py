"""One seed per level of the randomised parity soak (scripts/soak_parity.py): 1,024 distinct oracle-built
ciphertexts per level (valid / RM blocks randomised around the RS radius / far beyond it / random u and v),
decrypted by the oracle, then GPU batches of rows drawn from them in random order at sizes on both sides of
every switch of the launch policy — every row bit-exact. The full soak (84 seeds) is under
profiles/r02/soak_parity*.log."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU only with -m gpu
    pytest.skip("no CUDA device", allow_module_level=True)

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
import soak_parity  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402


@pytest.mark.parametrize("level", [1, 3, 5])
def test_mixed_rows_across_the_launch_policy(level):
    rng = np.random.default_rng(1000 + level)
    dev = torch.device("cuda:0")
    p = hqc.params(level)
    W, ref, cat = soak_parity.mixed_rows(level, int(rng.integers(1, 2**31)), int(rng.integers(0, 1 << 20)))
    assert (ref[cat == 7] != W["m"][cat == 7]).any(axis=1).mean() > 0.9  # random ciphertexts decode to garbage
    du, dv, dy = (torch.from_numpy(np.ascontiguousarray(W[k]).view(np.uint8).reshape(soak_parity.D, -1)).to(dev)
                  for k in ("u", "v", "y"))
    kernels = set()
    for B in [1, 31, 33, 1500] + [int(b + rng.integers(-3000, 3000)) for b in soak_parity.AROUND[level]]:
        idx = rng.integers(0, soak_parity.D, B)
        ti = torch.from_numpy(idx).to(dev)
        u, v, y = (x.index_select(0, ti).reshape(-1).contiguous() for x in (du, dv, dy))
        m = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
        hqc.hqc_decrypt_batch(level, u, v, y, m)
        torch.cuda.synchronize()
        got = m.cpu().numpy().reshape(B, p.k)
        bad = np.nonzero((got != ref[idx]).any(axis=1))[0]
        assert bad.size == 0, f"HQC-{level} B={B}: {bad.size} rows differ, first {bad[:8]}, categories {cat[idx[bad[:8]]]}"
        kernels.add(hqc.hqc_decrypt_launch_kernel(level, B))
        del u, v, y, m
    assert len(kernels) >= 3  # the sizes really crossed the policy's switches
