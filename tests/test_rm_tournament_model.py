"""Register model of stage 2's argmax tournament (csrc/stage2.cuh, HQC_RM_TOURNAMENT) against the
oracle's RM decision (oracle/rm.c, R#11: smallest a with maximal |F(a)|, bit 7 = [F(a) = -M]).

The model follows the kernel's layout: register i (0..63) holds F at a = 32 (i >> 4) + (i & 15) in its low
half and a + 16 in its high half; a node joins the adjacent register ranges [i, i+s) | [i+s, i+2s) per
half and keeps the left winner unless |right| > |left|; the two halves' winners are compared last (tie ->
smaller a). Inputs are chosen so that ties are common (random blocks and codewords with a few flips), so a
wrong pairing order or tie rule fails here before it can fail on the GPU."""
import numpy as np
import pytest

import oracle


def tournament_model(F):
    lo = np.array([F[32 * (i >> 4) + (i & 15)] for i in range(64)])
    hi = np.array([F[32 * (i >> 4) + (i & 15) + 16] for i in range(64)])

    def half(vals):
        v = list(vals)
        ix = list(range(64))
        while len(v) > 1:
            nv, nix = [], []
            for k in range(len(v) // 2):
                take_right = abs(v[2 * k + 1]) > abs(v[2 * k])
                nv.append(v[2 * k + 1] if take_right else v[2 * k])
                nix.append(ix[2 * k + 1] if take_right else ix[2 * k])
            v, ix = nv, nix
        return v[0], ix[0]

    flo, ilo = half(lo)
    fhi, ihi = half(hi)
    alo = 32 * (ilo >> 4) + (ilo & 15)
    ahi = 32 * (ihi >> 4) + (ihi & 15) + 16
    take_hi = abs(fhi) > abs(flo) or (abs(fhi) == abs(flo) and ahi < alo)
    a, f = (ahi, fhi) if take_hi else (alo, flo)
    return a | ((1 if f < 0 else 0) << 7)


@pytest.mark.parametrize("mult", [3, 5])
def test_tournament_model_matches_oracle(mult):
    rng = np.random.default_rng(77 + mult)
    words = 2 * mult
    ties = 0
    for trial in range(600):
        if trial % 3 == 0:
            block = rng.integers(0, 2**63, words, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, words, dtype=np.uint64)
        else:
            block = oracle.rm_encode(int(rng.integers(0, 256)), mult).copy()
            for _ in range(int(rng.integers(0, 80 * mult))):  # flip bits: heavy noise -> many ties
                b = int(rng.integers(0, 128 * mult))
                block[b // 64] ^= np.uint64(1) << np.uint64(b % 64)
        F = oracle.rm_transform(block, mult)
        M = np.abs(F).max()
        ties += int((np.abs(F) == M).sum() > 1)
        assert tournament_model(F) == oracle.rm_decode(block, mult), trial
    assert ties > 30  # the tie rule was exercised (47 / 600 blocks at mult 5, more at mult 3)
