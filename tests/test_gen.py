"""The seeded generator (paper_2512_12904_b200/gen): determinism, shard independence (a row depends
only on (seed, tag, index) — SURVEY §8(d) config 5), support validity, adversarial quarters."""
import numpy as np

import oracle
from paper_2512_12904_b200 import gen
from workloads import adversarial_batch, shape_for


def test_shard_independence():
    a = gen.support(1, gen.TAG_R1, 0, 1000, 17669, 75, 76)
    b = gen.support(1, gen.TAG_R1, 600, 400, 17669, 75, 76)
    assert (a[600:] == b).all()
    d1 = gen.dense(9, gen.TAG_H, 0, 50, 35851, 562)
    d2 = gen.dense(9, gen.TAG_H, 25, 25, 35851, 562)
    assert (d1[25:] == d2).all()


def test_support_rows_valid():
    s = gen.support(3, gen.TAG_E, 0, 2000, 57637, 149, 152)
    assert (np.diff(s[:, :149].astype(np.int64), axis=1) > 0).all(), "sorted, distinct"
    assert (s[:, :149] < 57637).all() and (s[:, 149:] == 0).all()


def test_dense_pad_zero_and_balance():
    d = gen.dense(4, gen.TAG_U_RAND, 0, 64, 17669, 278)
    assert (d[:, 277:] == 0).all()
    assert (d[:, 276] >> np.uint64(17669 % 64) == 0).all()
    ones = np.unpackbits(d.view(np.uint8)).sum() / (64 * 17669)
    assert abs(ones - 0.5) < 0.01


def test_tags_are_independent():
    assert not (gen.dense(5, 1, 0, 1, 640, 10) == gen.dense(5, 2, 0, 1, 640, 10)).all()


def test_adversarial_quarters():
    p = oracle.params(1)
    W = adversarial_batch(0, 64, 64)
    q = W["quarter"]
    assert (np.bincount(q, minlength=4) == 16).all()
    t = W["t_blocks"]
    assert (t[q == 1] == p.delta).all()
    assert ((t[q == 2] >= p.delta + 1) & (t[q == 2] <= 2 * p.delta)).all()
    assert (t[(q == 0) | (q == 3)] == 0).all()
    m = oracle.decrypt_batch(p, W["u"], W["v"], W["y"])
    assert (m[q == 0] == W["m"][q == 0]).all()
    sh = shape_for(1)
    assert W["u"].shape[1] == sh.u_stride
