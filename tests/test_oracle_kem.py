"""Pins for the oracle's KEM row (oracle/shake.c, oracle/kem.c, readings R#20-R#23):
SHAKE256 against Python's hashlib (a library implementation) and the SPEC S:102 vector; the sampler's
output contract; coins / K derivations recomputed with hashlib from their definitions; HHK round trip
and implicit rejection."""
import hashlib

import numpy as np
import pytest

import oracle
from workloads import keys, shape_for
from paper_2512_12904_b200 import gen


def test_shake256_spec_vector():
    assert oracle.shake256(b"", 32).hex() == "46b9dd2b0ba88d13233b3feb743eeb243fcd52ea62b81b82b50c27646ed5762f"


@pytest.mark.parametrize("mlen", [0, 1, 31, 135, 136, 137, 271, 272, 273, 1000, 4417])
@pytest.mark.parametrize("olen", [0, 1, 32, 64, 136, 137, 600])
def test_shake256_vs_hashlib(mlen, olen):
    msg = np.random.default_rng(mlen * 7 + olen).integers(0, 256, mlen, dtype=np.uint8).tobytes()
    assert oracle.shake256(msg, olen) == hashlib.shake_256(msg).digest(olen)


def test_keccak_permutation_consistency():
    # one absorbed block of zeros then squeeze == the permutation of the padded state (definition)
    st = np.zeros(25, np.uint64)
    st[0] ^= np.uint64(0x1F)
    st[16] ^= np.uint64(0x80) << np.uint64(56)
    out = oracle.keccak_f1600(st)
    got = b"".join(int(x).to_bytes(8, "little") for x in out[:17])
    assert got == hashlib.shake_256(b"").digest(136)


@pytest.mark.parametrize("n,w", [(17669, 75), (35851, 114), (57637, 149), (100, 99), (10, 1)])
def test_sampler_contract(n, w):
    rng = np.random.default_rng(n + w)
    for _ in range(200):
        rnd = rng.integers(0, 256, 4 * w, dtype=np.uint8).tobytes()
        s = oracle.sample_fixed_weight(rnd, n, w)
        assert len(set(s.tolist())) == w and (s < n).all()
        assert (oracle.sample_fixed_weight(rnd, n, w) == s).all()
    # a forced collision: all random words zero -> p_i = i, all distinct already
    assert (oracle.sample_fixed_weight(bytes(4 * w), n, w) == np.arange(w)).all()


def _kem_key(level, idx=0):
    p = oracle.params(level)
    h, x, y, s = keys(level, idx, 1, 0x4B454D)
    sigma = gen.rand_bytes(0x4B454D, gen.TAG_TEST, idx, 1, p.k)[0]
    hpk = oracle.kem_hpk(p, h[0], s[0])
    return p, h[0], s[0], y[0], sigma, hpk


def _ser(p, u, v):
    ub = u[: p.words].astype("<u8").tobytes()[: (p.n + 7) // 8]
    vb = v[: p.vwords].astype("<u8").tobytes()[: p.n12 // 8]
    return ub + vb


@pytest.mark.parametrize("level", [1, 3, 5])
def test_hpk_coins_and_kdf_definitions(level):
    p, h, s, y, sigma, hpk = _kem_key(level)
    nb = (p.n + 7) // 8
    pk = h[: p.words].astype("<u8").tobytes()[:nb] + s[: p.words].astype("<u8").tobytes()[:nb]
    assert hpk == hashlib.shake_256(pk + b"\x02").digest(32)
    m = np.arange(p.k, dtype=np.uint8) * 7
    theta = hashlib.shake_256(hpk + m.tobytes() + b"\x01").digest(32)
    rnd = hashlib.shake_256(theta + b"\x04").digest(12 * p.wr)
    r1, r2, e = oracle.kem_coins(p, hpk, m)
    assert (r1 == oracle.sample_fixed_weight(rnd[: 4 * p.wr], p.n, p.wr)).all()
    assert (r2 == oracle.sample_fixed_weight(rnd[4 * p.wr: 8 * p.wr], p.n, p.wr)).all()
    assert (e == oracle.sample_fixed_weight(rnd[8 * p.wr:], p.n, p.wr)).all()
    u, v, K = oracle.kem_encaps(p, h, s, hpk, m)
    assert K == hashlib.shake_256(m.tobytes() + _ser(p, u, v) + b"\x03").digest(64)
    uu, vv = oracle.encrypt(p, h, s, m, r1, r2, e)
    assert (uu == u).all() and (vv == v).all()


@pytest.mark.parametrize("level", [1, 3, 5])
def test_round_trip_and_implicit_rejection(level):
    p, h, s, y, sigma, hpk = _kem_key(level, 3)
    rng = np.random.default_rng(level)
    for t in range(4):
        m = rng.integers(0, 256, p.k, dtype=np.uint8)
        u, v, K = oracle.kem_encaps(p, h, s, hpk, m)
        K2, ok = oracle.kem_decaps(p, h, s, hpk, y, sigma, u, v)
        assert ok and K2 == K
        # tamper one bit of u or v: rejected, K = SHAKE256(sigma || c || K)
        u2, v2 = u.copy(), v.copy()
        if t % 2:
            u2[rng.integers(p.words - 1)] ^= np.uint64(1) << np.uint64(int(rng.integers(64)))
        else:
            v2[rng.integers(p.vwords)] ^= np.uint64(1) << np.uint64(int(rng.integers(64)))
        K3, ok3 = oracle.kem_decaps(p, h, s, hpk, y, sigma, u2, v2)
        assert not ok3
        assert K3 == hashlib.shake_256(sigma.tobytes() + _ser(p, u2, v2) + b"\x03").digest(64)
        assert K3 == oracle.kem_decaps(p, h, s, hpk, y, sigma, u2, v2)[0]  # deterministic
        # a bit of u in [n, 8 ceil(n/8)) is inside the serialized c, so c' != c byte-wise:
        # rejected, and K hashes the received bytes
        b = p.n + t % (8 * ((p.n + 7) // 8) - p.n)
        u4 = u.copy()
        u4[b // 64] ^= np.uint64(1) << np.uint64(b % 64)
        K4, ok4 = oracle.kem_decaps(p, h, s, hpk, y, sigma, u4, v)
        assert not ok4 and _ser(p, u4, v) != _ser(p, u, v)
        assert K4 == hashlib.shake_256(sigma.tobytes() + _ser(p, u4, v) + b"\x03").digest(64)


def test_decaps_batch_matches_single():
    level = 1
    p = oracle.params(level)
    h, x, y, s0 = keys(level, 0, 2, 0x4B)
    sh = shape_for(level)
    s = np.zeros_like(h)
    s[:, : p.words] = s0
    hpk = np.stack([np.frombuffer(oracle.kem_hpk(p, h[i], s[i]), np.uint8) for i in range(2)])
    sigma = gen.rand_bytes(0x4B, gen.TAG_TEST, 0, 2, p.k)
    key = np.array([0, 1, 1, 0, 1], np.int64)
    U = np.zeros((5, sh.u_stride), np.uint64)
    V = np.zeros((5, p.vwords), np.uint64)
    for i, kk in enumerate(key):
        m = np.full(p.k, i, np.uint8)
        u, v, _ = oracle.kem_encaps(p, h[kk], s[kk], hpk[kk].tobytes(), m)
        U[i, : p.words] = u
        V[i] = v
    V[2, 0] ^= np.uint64(1)
    K, acc = oracle.kem_decaps_batch(p, h, s, hpk, sigma, key, y[key], U, V)
    for i, kk in enumerate(key):
        Ki, oki = oracle.kem_decaps(p, h[kk], s[kk], hpk[kk].tobytes(), y[kk], sigma[kk], U[i], V[i])
        assert K[i].tobytes() == Ki and acc[i] == oki
    assert acc.tolist() == [1, 1, 0, 1, 1]


def _words_le(b: bytes, nwords: int) -> np.ndarray:
    return np.frombuffer(b + bytes(8 * nwords - len(b)), "<u8").astype(np.uint64)


@pytest.mark.parametrize("level", [1, 3, 5])
def test_keygen_from_seed_definition(level):
    """R#24 recomputed from its definition with hashlib; s = x + h*y through the (schoolbook-pinned)
    keygen product; sample_dense masks bits >= n and has weight ~ n/2."""
    p = oracle.params(level)
    nb = (p.n + 7) // 8
    for t in range(3):
        seed = bytes(np.random.default_rng(1000 * level + t).integers(0, 256, 32, dtype=np.uint8))
        h, x, y, s, sigma = oracle.kem_keygen(p, seed)
        seeds = hashlib.shake_256(seed + b"\x04").digest(64)
        hb = bytearray(hashlib.shake_256(seeds[32:] + b"\x04").digest(nb))
        if p.n % 8:
            hb[-1] &= (1 << (p.n % 8)) - 1
        assert (h == _words_le(bytes(hb), p.words)).all()
        r = hashlib.shake_256(seeds[:32] + b"\x04").digest(8 * p.w + p.k)
        assert (x == oracle.sample_fixed_weight(r[: 4 * p.w], p.n, p.w)).all()
        assert (y == oracle.sample_fixed_weight(r[4 * p.w: 8 * p.w], p.n, p.w)).all()
        assert sigma.tobytes() == r[8 * p.w:]
        assert (s == oracle.keygen(p, h, x, y)).all()
        assert len(set(x.tolist())) == p.w and len(set(y.tolist())) == p.w
        wt = sum(bin(int(v)).count("1") for v in h)
        assert abs(wt - p.n / 2) < 4 * (p.n / 4) ** 0.5
        again = oracle.kem_keygen(p, seed)
        assert all((a == b).all() for a, b in zip(again, (h, x, y, s, sigma)))


@pytest.mark.parametrize("level", [1, 5])
def test_kem_round_trip_with_seeded_keys(level):
    p = oracle.params(level)
    h, x, y, s, sigma = oracle.kem_keygen(p, bytes(range(32)))
    hpk = oracle.kem_hpk(p, h, s)
    m = np.arange(p.k, dtype=np.uint8)
    u, v, K = oracle.kem_encaps(p, h, s, hpk, m)
    K2, ok = oracle.kem_decaps(p, h, s, hpk, y, sigma, u, v)
    assert ok and K2 == K


@pytest.mark.parametrize("n,w", [(5, 2), (6, 3), (7, 3), (8, 4)])
def test_sampler_is_uniform_over_subsets(n, w):
    """R#22's fixed-weight sampler pinned by what it must achieve, not by its formula: over EVERY tuple of
    reduced draws o_i in [0, n-i) (rand_i chosen as the smallest 32-bit word with floor(rand_i (n-i) / 2^32)
    = o_i), the outputs are w distinct positions < n and each of the C(n, w) subsets appears exactly w!
    times — a uniform draw of a w-subset (the property the paper's "fixed-weight sampling", P:60, P:145,
    needs). A variant that fixes a collision against EARLIER entries produces duplicates and skewed counts."""
    import itertools
    import math
    from collections import Counter

    cnt = Counter()
    for offs in itertools.product(*[range(n - i) for i in range(w)]):
        rnd = b"".join(int(-(-o * 2**32 // (n - i))).to_bytes(4, "little") for i, o in enumerate(offs))
        pos = oracle.sample_fixed_weight(rnd, n, w)
        assert len(set(pos.tolist())) == w and int(pos.max()) < n
        cnt[tuple(sorted(pos.tolist()))] += 1
    assert len(cnt) == math.comb(n, w)
    assert set(cnt.values()) == {math.factorial(w)}
