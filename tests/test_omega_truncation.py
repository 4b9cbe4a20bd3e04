"""The RS decoders of the CUDA path form only delta coefficients of Omega = S Lambda mod x^{2 delta}
(csrc/stage3.cuh RS_OMEGA_TERMS); the oracle (oracle/rs.c) forms all 2 delta. This pins, on
the oracle's own (S, L, Lambda) and outputs and without a GPU, the two facts that make the shortcut exact:

  (1) for every received word, Omega_i = sum_{t <= L} Lambda_t S_{i+1-t} = 0 for L <= i < 2 delta whenever
      L <= delta (the final connection polynomial generates S_{L+1..2 delta}: these are BM's discrepancies);
  (2) Forney's values computed from Omega_0..Omega_{delta-1} only reproduce the oracle's corrected message
      bytes on every word the oracle accepts (ok), at the three levels' codes and on tiny codes.

Words: clean, 1..delta symbol errors, delta+1..2 delta errors (mostly rejected, some miscorrected: ok is
then still true and the claim must still hold) and uniformly random words.
"""
import numpy as np
import pytest

import oracle

CODES = [(46, 16, 15), (56, 24, 16), (90, 32, 29), (9, 1, 4), (7, 3, 2)]  # (n1, k, delta): Table I + tiny


def _tables():
    exp, log = [0] * 510, [0] * 256
    x = 1
    for e in range(255):
        exp[e] = exp[e + 255] = x
        log[x] = e
        x = oracle.gf_mul(x, 2)
    return exp, log


EXP, LOG = _tables()


def mul(a, b):
    return 0 if a == 0 or b == 0 else EXP[LOG[a] + LOG[b]]


def inv(a):
    return EXP[255 - LOG[a]]


def omega_full(S, lam, delta):
    om = []
    for i in range(2 * delta):
        v = 0
        for t in range(min(i, 2 * delta) + 1):
            v ^= mul(int(lam[t]), int(S[i - t]))
        om.append(v)
    return om


def words(n1, k, delta, rng, count):
    for c in range(count):
        msg = rng.integers(0, 256, k, dtype=np.uint8)
        w = oracle.rs_encode(msg, n1, k).copy()
        kind = c % 4
        if kind == 1:
            ne = int(rng.integers(1, delta + 1))
        elif kind == 2:
            ne = int(rng.integers(delta + 1, min(2 * delta, n1) + 1))
        else:
            ne = 0
        pos = rng.choice(n1, ne, replace=False)
        w[pos] ^= rng.integers(1, 256, ne, dtype=np.uint8)
        if kind == 3:
            w = rng.integers(0, 256, n1, dtype=np.uint8)
        yield w


@pytest.mark.parametrize("n1,k,delta", CODES)
def test_omega_vanishes_from_L_and_truncated_forney_equals_the_oracle(n1, k, delta):
    rng = np.random.default_rng(n1 * 1000 + delta)
    accepted = corrected = 0
    for w in words(n1, k, delta, rng, 240 if n1 > 9 else 400):
        out, ok, L, lam = oracle.rs_decode(w, n1, k, delta, full=True)
        S = oracle.rs_syndromes(w, n1, delta)
        if L > delta:
            assert not ok
            continue
        assert not lam[L + 1:].any()
        om = omega_full(S, lam, delta)
        assert not any(om[L:]), (L, om)  # (1): in particular nothing at i >= delta
        if not ok:
            assert (out == w[:k]).all()  # no correction applied: Omega is not used
            continue
        accepted += 1
        # (2) Forney (b = 1) at the message positions from delta coefficients only
        got = w[:k].copy()
        for j in range(k):
            xi = EXP[(255 - j) % 255]  # alpha^-j
            lam_x = 0
            for t in range(L, -1, -1):
                lam_x = mul(lam_x, xi) ^ int(lam[t])
            if lam_x:
                continue
            num = 0
            for i in range(delta - 1, -1, -1):
                num = mul(num, xi) ^ om[i]
            odd = 0  # x Lambda'(x) = Lambda_odd(x) in characteristic 2
            for t in range(1, L + 1, 2):
                odd ^= mul(int(lam[t]), EXP[(t * (255 - j)) % 255])
            got[j] ^= mul(mul(num, inv(EXP[j % 255])), inv(odd))
        assert (got == out).all()
        corrected += int((out != w[:k]).any())
    assert accepted > 50 and corrected > 10
