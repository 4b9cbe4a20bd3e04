"""Pins for the oracle's PKE (oracle/pke.c): decrypt(encrypt(m)) = m, all-zero ciphertext
decrypts to 0^k, the algebraic identity v + u*y = mG + x*r2 + r1*y + e (truncated; h*r2*y
cancels), stage 1 against the schoolbook product, printed sizes."""
import numpy as np
import pytest

import oracle
from bitutil import schoolbook_mul, support_to_bits, words_to_bits
from golden_values import printed
from workloads import shape_for, valid_batch


@pytest.mark.parametrize("level", [1, 3, 5])
def test_round_trip(level):
    p = oracle.params(level)
    W = valid_batch(level, 0, 24)
    m = oracle.decrypt_batch(p, W["u"], W["v"], W["y"])
    assert (m == W["m"]).all()


@pytest.mark.parametrize("level", [1, 5])
def test_algebraic_identity_and_schoolbook(level):
    p = oracle.params(level)
    W = valid_batch(level, 300, 2)
    for i in range(2):
        kx = W["key"][i]
        r = oracle.decrypt_stage1(p, W["u"][i], W["v"][i], W["y"][i])
        x, r1, r2, e = W["x"][kx][: p.w], W["r1"][i][: p.wr], W["r2"][i][: p.wr], W["e"][i][: p.wr]
        mg = oracle.code_encode(p, W["m"][i])
        rhs = words_to_bits(mg, p.n12)
        for a, b in ((x, r2), (r1, W["y"][i][: p.w])):
            rhs ^= schoolbook_mul(support_to_bits(a, p.n), support_to_bits(b, p.n))[: p.n12]
        rhs ^= support_to_bits(e, p.n)[: p.n12]
        assert (words_to_bits(r, p.n12) == rhs).all()
        # stage 1 itself against the schoolbook product u*y
        uy = schoolbook_mul(words_to_bits(W["u"][i], p.n), support_to_bits(W["y"][i][: p.w], p.n))
        assert (words_to_bits(r, p.n12) == (words_to_bits(W["v"][i], p.n12) ^ uy[: p.n12])).all()


def test_zero_ciphertext():
    for level in (1, 3, 5):
        p = oracle.params(level)
        u = np.zeros(p.words, np.uint64)
        v = np.zeros(p.vwords, np.uint64)
        y = np.arange(p.w, dtype=np.uint32) * 7
        assert (oracle.decrypt(p, u, v, y) == 0).all()


def test_pad_bits_of_u_ignored():
    p = oracle.params(1)
    W = valid_batch(1, 10, 1)
    u = W["u"][0].copy()
    u[p.words - 1] |= np.uint64(0xFFFFFFFFFFFFFFFF) << np.uint64(p.n % 64)
    assert (oracle.decrypt(p, u, W["v"][0], W["y"][0]) == W["m"][0]).all()


def test_printed_ciphertext_size():
    p = oracle.params(1)
    assert (p.n + 7) // 8 + p.n12 // 8 == int(printed()["ciphertext_bytes_hqc1"])


def test_shape_matches_params():
    for level in (1, 3, 5):
        p = oracle.params(level)
        sh = shape_for(level)
        assert sh.n == p.n and sh.v_words == p.vwords and sh.u_stride >= p.words
