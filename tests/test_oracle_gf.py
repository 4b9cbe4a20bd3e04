"""Pins for the oracle's GF(2^8) (oracle/gf256.c) — not the oracle against itself:
field axioms exhaustively (a multiplication that is commutative, associative, distributive over XOR
with identity and inverses on 256 elements is a field of order 256), multiplication by x = 0x02 is
the polynomial shift, and the printed value mul(0x02, 0x80) = 0x1D fixes the modulus
x^8+x^4+x^3+x^2+1 (R#4). Together these determine every product."""
import numpy as np
import pytest

import oracle
from golden_values import printed


@pytest.fixture(scope="module")
def T():
    lib = oracle.lib()
    t = np.zeros((256, 256), dtype=np.uint8)
    for a in range(256):
        for b in range(256):
            t[a, b] = lib.orc_gf_mul(a, b)
    return t


def test_printed_value():
    assert oracle.gf_mul(0x02, 0x80) == int(printed()["gf_mul_02_80"], 16)


def test_mul_by_x_is_shift(T):
    for a in range(128):
        assert T[2, a] == a << 1  # no reduction below degree 8
    # x * x^7 = x^8 = x^4 + x^3 + x^2 + 1 under 0x11D
    assert T[2, 0x80] == 0x1D


def test_axioms_exhaustive(T):
    a = np.arange(256)
    assert (T == T.T).all(), "commutative"
    assert (T[1] == a).all() and (T[0] == 0).all(), "identity / zero"
    # distributive over XOR: a*(b^c) = a*b ^ a*c  for all a, b, c
    for x in range(256):
        lhs = T[x][np.bitwise_xor.outer(a, a)]
        rhs = np.bitwise_xor.outer(T[x], T[x])
        assert (lhs == rhs).all()
    # associativity over all triples
    ab = T  # ab[a, b]
    for c in range(256):
        assert (T[ab, c] == T[a[:, None], T[:, c][None, :]]).all()
    # every nonzero element has exactly one inverse
    for x in range(1, 256):
        assert (T[x] == 1).sum() == 1


def test_alpha_generates_group():
    seen = set()
    x = 1
    for _ in range(255):
        seen.add(x)
        x = oracle.gf_mul(x, 2)
    assert len(seen) == 255 and x == 1, "alpha = 0x02 has order 255"


def test_inverse_and_pow():
    for a in range(1, 256):
        assert oracle.gf_mul(a, oracle.gf_inv(a)) == 1
    for e in range(0, 600, 7):
        x = 1
        for _ in range(e):
            x = oracle.gf_mul(x, 0x02)
        assert oracle.gf_pow(2, e) == x
