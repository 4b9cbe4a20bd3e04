"""Lane model of the warp RS decoder's reformulated inversionless Berlekamp–Massey (riBM,
csrc/stage3_warp.cuh, HQC_BM_RIBM) against the oracle's plain BM (oracle/rs.c, R#7).

The model mirrors the kernel's register layout (element i on lane i mod 32, slot i / 32, values kept as
logs with the 511 sentinel for zero, the neighbour delta_{i+1} taken from lane+1 or, on lane 31, from
lane 0's next slot) so that an index or wrap mistake in that layout fails here. Claimed: same L as the
oracle on every word, and when L <= delta the same connection polynomial up to a nonzero scale
(Lambda / Lambda_0 equals the oracle's Lambda), the property the kernel's Chien / Forney steps rely on.
"""
import numpy as np
import pytest

import oracle

LOG0 = 511


def _tables():
    exp = np.zeros(1024, dtype=np.int64)
    log = np.full(256, LOG0, dtype=np.int64)
    x = 1
    for e in range(255):
        exp[e] = exp[e + 255] = x
        log[x] = e
        x <<= 1
        if x & 0x100:
            x ^= 0x11D
    return exp, log


EXP, LOG = _tables()


def ribm_model(S, delta):
    """S: syndromes S_1..S_2delta (bytes). Returns (L, Lambda[0..delta])."""
    TD, NE = 2 * delta, 3 * delta + 1
    NS = (NE + 31) // 32
    ld = np.full((NS, 32), LOG0, dtype=np.int64)  # [slot, lane]
    for s in range(NS):
        for lane in range(32):
            i = lane + 32 * s
            ld[s, lane] = LOG[S[i]] if i < TD else (0 if i == 3 * delta else LOG0)
    lt = ld.copy()
    lg, L = 0, 0
    for r in range(TD):
        ld0 = ld[0, 0]
        y = np.roll(ld, -1, axis=1)  # y[s, lane] = ld[s, (lane + 1) & 31]
        grow = ld0 != LOG0 and 2 * L <= r
        nb = y.copy()
        for s in range(NS):
            nb[s, 31] = y[s + 1, 31] if s + 1 < NS else LOG0
        val = EXP[lg + nb] ^ EXP[ld0 + lt]
        if grow:
            lt = nb
            lg = ld0
            L = r + 1 - L
        ld = LOG[val]
    flat = ld.reshape(-1)  # index s * 32 + lane = element i
    lam = np.array([EXP[flat[delta + t]] for t in range(delta + 1)], dtype=np.int64)
    return L, lam


def _gf_div(a, b):
    return 0 if a == 0 else int(EXP[(LOG[a] - LOG[b]) % 255])


@pytest.mark.parametrize("level", [1, 3, 5])
def test_ribm_model_matches_oracle_bm(level):
    p = oracle.params(level)
    n1, k, delta = p.n1, p.k, p.delta
    rng = np.random.default_rng(1000 + level)
    cases = 0
    for trial in range(160):
        msg = rng.integers(0, 256, k, dtype=np.uint8)
        cw = oracle.rs_encode(msg, n1, k)
        if trial % 8 == 7:
            r = rng.integers(0, 256, n1, dtype=np.uint8)  # garbage word
        else:
            ne = trial % (delta + 4)  # 0..delta+3 symbol errors
            r = cw.copy()
            pos = rng.choice(n1, ne, replace=False)
            r[pos] ^= rng.integers(1, 256, ne, dtype=np.uint8)
        S = oracle.rs_syndromes(r, n1, delta)
        _, ok, L_ref, lam_ref = oracle.rs_decode(r, n1, k, delta, full=True)
        L, lam = ribm_model(S, delta)
        assert L == L_ref, (trial, L, L_ref)
        if L <= delta:
            assert lam[0] != 0
            norm = [_gf_div(int(c), int(lam[0])) for c in lam]
            assert norm == [int(c) for c in lam_ref[: delta + 1]], trial
            assert not lam_ref[delta + 1:].any()
            cases += 1
    assert cases > 100
