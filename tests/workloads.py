"""Seeded workloads for the tests: generator draws (paper_2512_12904_b200.gen) encrypted by the ORACLE.
Rows are laid out in the C-ABI layout (include/hqc_gpu.h): u rows of u_stride uint64, v rows of
v_words uint64, y rows of y_stride uint32. Recipe: DESIGN.md §5 (BASELINE.json configs 1-4)."""
from functools import lru_cache

import numpy as np

import oracle
from paper_2512_12904_b200 import gen

CONFIG_SEED = {1: 0xC0F1_0001, 2: 0xC0F1_0002, 3: 0xC0F1_0003, 4: 0xC0F1_0004, 5: 0xC0F1_0005}
LEVEL_SEED = {1: CONFIG_SEED[1], 3: CONFIG_SEED[2], 5: CONFIG_SEED[3]}


def _r4(x):
    return (x + 3) // 4 * 4


def shape_for(level: int) -> gen.Shape:
    p = oracle.params(level)
    return gen.Shape(n=p.n, w=p.w, wr=p.wr, n1=p.n1, k=p.k, n2=p.n2, delta=p.delta,
                     u_stride=p.words + (p.words & 1), v_words=p.vwords, y_stride=_r4(p.w),
                     sup_stride=_r4(p.wr))


@lru_cache(maxsize=64)
def keys(level: int, key0: int, nkeys: int, seed: int):
    p = oracle.params(level)
    sh = shape_for(level)
    h, x, y = gen.key_draws(seed, sh, key0, nkeys)
    s = np.stack([oracle.keygen(p, h[i], x[i], y[i]) for i in range(nkeys)])
    return h, x, y, s


def valid_batch(level: int, i0: int, rows: int, seed: int | None = None, nthreads=None):
    seed = LEVEL_SEED[level] if seed is None else seed
    p = oracle.params(level)
    sh = shape_for(level)
    key = gen.key_of(i0, rows)
    k0 = int(key.min()) if rows else 0
    nk = int(key.max()) - k0 + 1 if rows else 1
    h, x, y, s = keys(level, k0, nk, seed)
    m, r1, r2, e = gen.ct_draws(seed, sh, i0, rows, nthreads)
    u, v = oracle.encrypt_batch(p, h, s, key - k0, m, r1, r2, e, nthreads)
    U = np.zeros((rows, sh.u_stride), np.uint64)
    U[:, : p.words] = u
    Y = np.ascontiguousarray(y[key - k0])
    return dict(u=U, v=v, y=Y, m=m, r1=r1, r2=r2, e=e, key=key - k0, x=x, h=h, s=s, shape=sh, params=p)


def adversarial_batch(i0: int, rows: int, batch: int, seed: int | None = None, nthreads=None):
    """BASELINE configs[3] (HQC-1): quarters Q0 valid, Q1 delta blocks randomised, Q2 delta+1..2delta
    blocks randomised, Q3 uniformly random u and v with y from the key (R#17)."""
    seed = CONFIG_SEED[4] if seed is None else seed
    W = valid_batch(1, i0, rows, seed, nthreads)
    p, sh = W["params"], W["shape"]
    q = gen.quarter_of(np.arange(i0, i0 + rows), batch)
    v = W["v"]
    t = np.zeros(rows, np.uint8)
    for quarter, (tmin, tmax) in ((1, (p.delta, p.delta)), (2, (p.delta + 1, 2 * p.delta))):
        mask = q == quarter
        if mask.any():
            tq = gen.randomise_blocks(v, i0, seed + quarter, sh, tmin, tmax, row_mask=mask, nthreads=nthreads)
            t = np.where(mask, tq, t)
    mask = q == 3
    if mask.any():
        idx = np.nonzero(mask)[0]
        j0, cnt = int(idx[0]), idx.size
        assert idx[-1] == j0 + cnt - 1, "quarters are contiguous"
        # uniformly random u (n bits, pad zero) and v (n1*n2 bits), stream index = ciphertext index
        W["u"][j0:j0 + cnt] = gen.dense(seed, gen.TAG_U_RAND, i0 + j0, cnt, p.n, sh.u_stride, nthreads)
        v[j0:j0 + cnt] = gen.dense(seed, gen.TAG_V_RAND, i0 + j0, cnt, p.n12, sh.v_words, nthreads)
    W["quarter"] = q
    W["t_blocks"] = t
    return W
