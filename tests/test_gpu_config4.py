"""BASELINE configs[3] on its own seeded inputs: 1,048,576 HQC-1 ciphertexts in four quarters (valid; delta RM
blocks of v randomised; delta+1..2delta blocks randomised; uniformly random u and v), built chunk by chunk by
tests/workloads.adversarial_batch (generator draws, ORACLE keygen + encrypt), decrypted by the GPU in ONE
hqc_decrypt_batch call over the whole batch (the launch configuration bench.py's config4 block times), and
compared row by row with the oracle's decryption of every row — garbage outputs included.
The oracle work (~1M encryptions and decryptions on the host cores) makes this the slowest GPU test."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2512_12904_b200 import hqc  # noqa: E402
from workloads import adversarial_batch  # noqa: E402

DEV = torch.device("cuda:0")
BATCH = 1 << 20
CHUNK = 1 << 16


def test_config4_full_seeded_batch_vs_oracle():
    g = hqc.params(1)
    du = torch.empty((BATCH, g.u_stride * 8), dtype=torch.uint8, device=DEV)
    dv = torch.empty((BATCH, g.v_words * 8), dtype=torch.uint8, device=DEV)
    dy = torch.empty((BATCH, g.y_stride * 4), dtype=torch.uint8, device=DEV)
    ref = np.empty((BATCH, g.k), np.uint8)
    msg = np.empty((BATCH, g.k), np.uint8)
    quarter = np.empty(BATCH, np.int64)
    tblocks = np.empty(BATCH, np.uint8)
    for c0 in range(0, BATCH, CHUNK):
        W = adversarial_batch(c0, CHUNK, BATCH)
        sl = slice(c0, c0 + CHUNK)
        du[sl] = torch.from_numpy(np.ascontiguousarray(W["u"]).view(np.uint8)).to(DEV)
        dv[sl] = torch.from_numpy(np.ascontiguousarray(W["v"]).view(np.uint8)).to(DEV)
        dy[sl] = torch.from_numpy(np.ascontiguousarray(W["y"]).view(np.uint8)).to(DEV)
        ref[sl] = oracle.decrypt_batch(W["params"], W["u"], W["v"], W["y"])
        msg[sl], quarter[sl], tblocks[sl] = W["m"], W["quarter"], W["t_blocks"]
    m = torch.empty(BATCH * g.k, dtype=torch.uint8, device=DEV)
    hqc.hqc_decrypt_batch(1, du.view(-1), dv.view(-1), dy.view(-1), m)
    torch.cuda.synchronize()
    got = m.cpu().numpy().reshape(BATCH, g.k)
    bad = np.nonzero((got != ref).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} rows differ from the oracle; first {bad[:8]}, quarters {quarter[bad[:8]]}"
    # the construction itself (R#17): quarter sizes, randomised-block counts, and what the outputs must be
    assert [(quarter == q).sum() for q in range(4)] == [BATCH // 4] * 4
    assert (tblocks[quarter == 1] == 15).all()
    assert ((tblocks[quarter == 2] >= 16) & (tblocks[quarter == 2] <= 30)).all()
    assert (got[quarter == 0] == msg[quarter == 0]).all()  # valid ciphertexts decrypt to m
    eq = (got == msg).all(axis=1)
    assert 0.95 < eq[quarter == 1].mean() < 1.0  # at capacity: ~1.1% hit a natural RM failure on top
    assert eq[quarter == 2].mean() < 0.05 and eq[quarter == 3].mean() < 1e-3
