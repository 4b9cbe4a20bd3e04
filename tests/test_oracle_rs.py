"""Pins for the oracle's shortened RS code (oracle/rs.c):
 * tiny shortened codes over GF(2^8): the decoder equals BRUTE-FORCE bounded-distance decoding
   (search every codeword for one within distance delta; else output r[0..k) unchanged, R#7) on random
   words, exactly-delta-error words and beyond-capacity words;
 * encodings are codewords by the code's definition (every c(alpha^i) = 0, evaluated here in numpy from
   the pinned multiplication table) and systematic message-first (R#5, R#6);
 * real sizes: exactly-delta-error round trips, random words never decode, syndrome linearity, the MDS
   distance n1 - k + 1 = d of Table I and the printed 2delta(n1-1) = 1350 of P:227."""
import itertools

import numpy as np
import pytest

import oracle
from golden_values import printed, table1


@pytest.fixture(scope="module")
def T():
    lib = oracle.lib()
    return np.array([[lib.orc_gf_mul(a, b) for b in range(256)] for a in range(256)], dtype=np.uint8)


def _alpha_pows(T):
    p = [1]
    for _ in range(600):
        p.append(int(T[p[-1], 2]))
    return p


def _eval(T, c, x):
    acc = 0
    for coef in reversed(list(c)):
        acc = int(T[acc, x]) ^ int(coef)
    return acc


TINY = [(5, 1, 2), (6, 2, 2), (7, 1, 3), (9, 1, 4), (7, 3, 2)]


@pytest.mark.parametrize("n1,k,delta", TINY)
def test_tiny_codes_brute_force_bounded_distance(n1, k, delta, T):
    assert n1 - k == 2 * delta
    ap = _alpha_pows(T)
    msgs = list(itertools.product(range(256), repeat=k)) if k <= 2 else \
        [tuple(np.random.default_rng(i).integers(0, 256, k)) for i in range(3000)]
    cws = np.stack([oracle.rs_encode(m, n1, k) for m in msgs])
    # encodings are codewords (roots alpha^1..alpha^{2 delta}) and systematic
    for c, m in list(zip(cws, msgs))[:: max(1, len(msgs) // 300)]:
        assert all(_eval(T, c, ap[i]) == 0 for i in range(1, 2 * delta + 1))
        assert tuple(c[:k]) == tuple(m)
    rng = np.random.default_rng(n1 * 100 + k)
    exhaustive = k <= 2
    for trial in range(900):
        kind = trial % 3
        base = cws[rng.integers(len(cws))].copy()
        if kind == 0:
            r = rng.integers(0, 256, n1).astype(np.uint8)
        else:
            ne = delta if kind == 1 else int(rng.integers(delta + 1, 2 * delta + 1))
            pos = rng.choice(n1, ne, replace=False)
            r = base.copy()
            r[pos] ^= rng.integers(1, 256, ne).astype(np.uint8)
        dist = (cws != r[None, :]).sum(axis=1)
        out, ok = oracle.rs_decode(r, n1, k, delta)
        close = np.nonzero(dist <= delta)[0]
        if exhaustive:
            if close.size:
                assert ok and tuple(out) == tuple(cws[close[0]][:k])
            else:
                assert not ok and tuple(out) == tuple(r[:k])
        else:  # sampled codebook: only the positive direction is exhaustive
            if kind == 1:
                assert ok and tuple(out) == tuple(base[:k])
            if ok:
                pass
            else:
                assert tuple(out) == tuple(r[:k])


@pytest.mark.parametrize("level", [1, 3, 5])
def test_real_sizes(level, T):
    p = oracle.params(level)
    t1 = table1()[level]
    assert p.n1 - p.k + 1 == t1["d"], "shortened RS is MDS: d = n1 - k + 1 (Table I)"
    assert p.delta == (t1["d"] - 1) // 2
    ap = _alpha_pows(T)
    rng = np.random.default_rng(level)
    for trial in range(60):
        m = rng.integers(0, 256, p.k).astype(np.uint8)
        c = oracle.rs_encode(m, p.n1, p.k)
        assert (c[: p.k] == m).all()
        if trial < 5:
            assert all(_eval(T, c, ap[i]) == 0 for i in range(1, 2 * p.delta + 1))
        assert (oracle.rs_syndromes(c, p.n1, p.delta) == 0).all()
        r = c.copy()
        pos = rng.choice(p.n1, p.delta, replace=False)
        r[pos] ^= rng.integers(1, 256, p.delta).astype(np.uint8)
        out, ok = oracle.rs_decode(r, p.n1, p.k, p.delta)
        assert ok and (out == m).all()
        # a uniformly random word is (overwhelmingly) not within delta of any codeword
        g = rng.integers(0, 256, p.n1).astype(np.uint8)
        out, ok = oracle.rs_decode(g, p.n1, p.k, p.delta)
        assert not ok and (out == g[: p.k]).all()
        # syndrome linearity
        a, b = rng.integers(0, 256, p.n1).astype(np.uint8), rng.integers(0, 256, p.n1).astype(np.uint8)
        assert (oracle.rs_syndromes(a ^ b, p.n1, p.delta) ==
                (oracle.rs_syndromes(a, p.n1, p.delta) ^ oracle.rs_syndromes(b, p.n1, p.delta))).all()
        # syndromes by definition S_i = r(alpha^i)
        if trial < 3:
            S = oracle.rs_syndromes(a, p.n1, p.delta)
            assert all(int(S[i - 1]) == _eval(T, a, ap[i]) for i in range(1, 2 * p.delta + 1))


def test_printed_counts():
    p = oracle.params(1)
    assert 2 * p.delta * (p.n1 - 1) == int(printed()["rs_syndrome_mults_hqc1"])
    assert 2 * p.delta * 256 == int(printed()["rs_encode_table_bytes_hqc1"])


def test_zero_word():
    for level in (1, 3, 5):
        p = oracle.params(level)
        out, ok = oracle.rs_decode(np.zeros(p.n1, np.uint8), p.n1, p.k, p.delta)
        assert ok and (out == 0).all()
