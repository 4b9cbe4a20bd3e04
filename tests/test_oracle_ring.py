"""Pins for the oracle's ring product (oracle/ring.c, Eq. 1) against the SCHOOLBOOK product —
the polynomial-multiplication definition (convolution then X^n = 1), a different computation from
Eq. 1's rotate-and-XOR — plus special cases and algebraic invariants."""
import numpy as np
import pytest

import oracle
from bitutil import bits_to_words, schoolbook_mul, support_to_bits, words_to_bits
from golden_values import printed
from paper_2512_12904_b200 import gen

SEED = 0x5EED0001


def _rand_elem(n, idx):
    return gen.dense(SEED, gen.TAG_TEST, idx, 1, n, (n + 63) // 64)[0]


def _rand_supp(n, w, idx):
    return gen.support(SEED, gen.TAG_TEST + 1, idx, 1, n, w, w)[0]


@pytest.mark.parametrize("level", [1, 3, 5])
def test_sparse_equals_schoolbook_real_sizes(level):
    p = oracle.params(level)
    for t, w in enumerate((p.w, p.wr, 1, 2)):
        a = _rand_elem(p.n, 10 * level + t)
        s = _rand_supp(p.n, w, 10 * level + t)
        got = words_to_bits(oracle.ring_mul_sparse(a, p.n, s), p.n)
        ref = schoolbook_mul(words_to_bits(a, p.n), support_to_bits(s, p.n))
        assert (got == ref).all()


@pytest.mark.parametrize("n", [8, 63, 64, 65, 127, 257, 1024, 1031])
def test_small_rings_exhaustive_shifts(n):
    a = _rand_elem(n, n)
    ab = words_to_bits(a, n)
    for i in range(n):  # every rotation against the bit-level definition of X^i * a
        got = words_to_bits(oracle.ring_rotate(a, n, i), n)
        assert (got == np.roll(ab, i)).all()


def test_spec_example_n8():
    # n = 8, input X^5, shift 7 -> X^4
    a = bits_to_words(support_to_bits([5], 8), 1)
    assert (words_to_bits(oracle.ring_rotate(a, 8, 7), 8) == support_to_bits([4], 8)).all()


@pytest.mark.parametrize("level", [1, 5])
def test_identity_and_empty(level):
    p = oracle.params(level)
    a = _rand_elem(p.n, 99)
    assert (oracle.ring_mul_sparse(a, p.n, [0]) == a).all()      # X^0 * a = a
    assert (oracle.ring_mul_sparse(a, p.n, []) == 0).all()       # empty support


def test_linearity_commutativity_composition():
    n = 257
    a, b = _rand_elem(n, 1), _rand_elem(n, 2)
    s = _rand_supp(n, 30, 3)
    # y*(a+b) = y*a + y*b
    assert (oracle.ring_mul_sparse(a ^ b, n, s) == oracle.ring_mul_sparse(a, n, s) ^ oracle.ring_mul_sparse(b, n, s)).all()
    # commutativity a*b = b*a with dense operands written as supports
    sa = np.nonzero(words_to_bits(a, n))[0]
    sb = np.nonzero(words_to_bits(b, n))[0]
    assert (oracle.ring_mul_sparse(a, n, sb) == oracle.ring_mul_sparse(b, n, sa)).all()
    # shift composition
    for i, j in [(3, 250), (100, 200), (256, 256)]:
        lhs = oracle.ring_rotate(oracle.ring_rotate(a, n, i), n, j)
        assert (lhs == oracle.ring_rotate(a, n, (i + j) % n)).all()


def test_truncation_drops_printed_bits():
    p = oracle.params(1)
    assert p.n - p.n12 == int(printed()["truncated_bits_hqc1"])
