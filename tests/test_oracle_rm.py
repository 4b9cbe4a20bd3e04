"""Pins for the oracle's duplicated RM(1,7) (oracle/rm.c): the decoder against BRUTE-FORCE
maximum-likelihood decoding over all 256 duplicated codewords (Hamming distance, ties to the smallest
b & 0x7F, R#11), on uniformly random blocks where ~20-24% of blocks tie; the encoder against the code's
printed parameters (Table I [n2, 8, d'], S:406 weights) and linearity."""
import numpy as np
import pytest

import oracle
from bitutil import words_to_bits
from golden_values import printed, table1
from paper_2512_12904_b200 import gen


def _codebook(mult):
    return np.stack([words_to_bits(oracle.rm_encode(b, mult), 128 * mult) for b in range(256)])


@pytest.mark.parametrize("level", [1, 3])
def test_code_parameters(level):
    p = oracle.params(level)
    t1 = table1()[level]
    cb = _codebook(p.mult)
    assert cb.shape[1] == t1["n2"] == p.n2
    wts = cb.sum(axis=1)
    assert wts[0] == 0
    assert wts[1:].min() == t1["dprime"], "minimum distance of a linear code = min nonzero weight (Table I d')"
    assert len({tuple(r) for r in cb}) == 256, "dimension 8"
    if level == 1:
        assert sorted(set(wts[1:].tolist())) == [int(x) for x in printed()["rm_weights_hqc1"].split(",")]
    for a in range(0, 256, 17):  # linearity
        for b in range(0, 256, 13):
            assert (cb[a] ^ cb[b] == cb[a ^ b]).all()
    assert (cb[0x80] == 1).all(), "bit 7 is the all-ones row (R#9)"


def _ml_decode(block_bits, cb):
    dist = (cb != block_bits[None, :]).sum(axis=1)
    best = dist.min()
    cands = [b for b in range(256) if dist[b] == best]
    return min(cands, key=lambda b: (b & 0x7F))


@pytest.mark.parametrize("mult", [3, 5])
def test_decode_equals_brute_force_ml_random_blocks(mult):
    cb = _codebook(mult)
    nw = 2 * mult
    blocks = gen.dense(0xAB, gen.TAG_TEST, 1000 * mult, 600, 128 * mult, nw)
    ties = 0
    for blk in blocks:
        bits = words_to_bits(blk, 128 * mult)
        dist = (cb != bits[None, :]).sum(axis=1)
        ties += (dist == dist.min()).sum() > 1
        assert oracle.rm_decode(blk, mult) == _ml_decode(bits, cb)
    assert ties > 60, "random blocks must exercise the tie rule"


@pytest.mark.parametrize("mult", [3, 5])
def test_round_trip_and_correction_radius(mult):
    rng = np.random.default_rng(mult)
    dprime = 64 * mult
    for b in range(256):
        cw = oracle.rm_encode(b, mult)
        assert oracle.rm_decode(cw, mult) == b
        bits = words_to_bits(cw, 128 * mult)
        flips = rng.choice(128 * mult, size=dprime // 2 - 1, replace=False)  # < d'/2 flips
        bits[flips] ^= 1
        w = np.packbits(bits, bitorder="little").view("<u8")
        assert oracle.rm_decode(w, mult) == b


def test_transform_definition_small_cases():
    # all-zero block: s_p = mult for every p, so F(0) = 128*mult and F(a != 0) = 0  -> byte 0x00
    z = np.zeros(6, dtype=np.uint64)
    F = oracle.rm_transform(z, 3)
    assert F[0] == 384 and (F[1:] == 0).all()
    assert oracle.rm_decode(z, 3) == 0
    # Parseval: sum_a F(a)^2 = 128 * sum_p s_p^2 on a random block
    blk = gen.dense(7, gen.TAG_TEST, 5, 1, 384, 6)[0]
    bits = words_to_bits(blk, 384).reshape(3, 128)
    s = (1 - 2 * bits.astype(np.int64)).sum(axis=0)
    F = oracle.rm_transform(blk, 3).astype(np.int64)
    assert (F ** 2).sum() == 128 * (s ** 2).sum()


@pytest.mark.parametrize("level", [1, 3, 5])
def test_code_encode_block_layout(level):
    """R#12 pinned without the oracle's decoder: in code_encode(m), block j (bits
    [j n2, (j+1) n2)) consists of mult identical 128-bit copies, and that copy is the codeword of RS symbol
    j in the codebook above (whose parameters are pinned by Table I) — so symbol j lands in block j, in
    order, copy c at +128c; and the RS symbols are rs_encode(m), message first (R#6)."""
    p = oracle.params(level)
    cb = np.stack([words_to_bits(oracle.rm_encode(b, 1), 128) for b in range(256)])
    rng = np.random.default_rng(700 + level)
    for _ in range(3):
        m = rng.integers(0, 256, p.k).astype(np.uint8)
        cw = oracle.rs_encode(m, p.n1, p.k)
        assert (cw[: p.k] == m).all()
        bits = words_to_bits(oracle.code_encode(p, m), p.n1 * p.n2)
        for j in range(p.n1):
            blk = bits[j * p.n2:(j + 1) * p.n2].reshape(p.mult, 128)
            assert (blk == blk[0]).all(), f"copies of block {j} differ"
            match = np.nonzero((cb == blk[0]).all(axis=1))[0]
            assert match.tolist() == [int(cw[j])], f"block {j} is not the codeword of RS symbol {j}"
