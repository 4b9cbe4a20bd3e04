"""GPU KEM (readings R#20-R#23) through the C ABI, bit-exact against
hashlib (H_pk) and the oracle (oracle/kem.c: Encaps, Decaps with implicit rejection). Ciphertexts fed
to the GPU Decaps are made by the oracle, so no expected value comes from the CUDA path."""
import hashlib

import numpy as np
import pytest

import oracle
from paper_2512_12904_b200 import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2512_12904_b200 import hqc  # noqa: E402
from workloads import keys  # noqa: E402

DEV = torch.device("cuda:0")
SEED = 0x4B454D5F475055


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1)).to(DEV)


def host(t, dtype, cols):
    return t.cpu().numpy().view(dtype).reshape(-1, cols)


def empty(nbytes):
    return torch.empty(max(nbytes, 16), dtype=torch.uint8, device=DEV)


def _keyset(level, nk):
    """nk oracle keys padded to the ABI rows, with sigma and the oracle's H_pk."""
    p, g = oracle.params(level), hqc.params(level)
    h, x, y, s = keys(level, 0, nk, SEED)
    H = np.zeros((nk, g.u_stride), np.uint64)
    H[:, : p.words] = h[:, : p.words]
    S = np.zeros_like(H)
    S[:, : p.words] = s
    sigma = gen.rand_bytes(SEED, gen.TAG_TEST, 0, nk, p.k)
    hpk = np.stack([np.frombuffer(oracle.kem_hpk(p, H[i], S[i]), np.uint8) for i in range(nk)])
    return p, g, H, S, y, sigma, hpk


@pytest.mark.parametrize("level", [1, 3, 5])
def test_hpk_matches_hashlib(level):
    g = hqc.params(level)
    nk = 131  # two 128-lane blocks, ragged tail
    rng = np.random.default_rng(level)
    H = rng.integers(0, 2**63, (nk, g.u_stride), dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    S = rng.integers(0, 2**63, (nk, g.u_stride), dtype=np.uint64)
    out = empty(nk * 32)
    hqc.hqc_kem_hpk_batch(level, dev(H), dev(S), out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(nk, 32)
    nb = (g.n + 7) // 8
    for i in range(nk):
        ref = hashlib.shake_256(H[i].tobytes()[:nb] + S[i].tobytes()[:nb] + b"\x02").digest(32)
        assert got[i].tobytes() == ref, i


@pytest.mark.parametrize("level", [1, 3, 5])
def test_encaps_matches_oracle(level):
    nk, B = 3, 70
    p, g, H, S, y, sigma, hpk = _keyset(level, nk)
    key = (np.arange(B) * 7 % nk).astype(np.uint32)
    m = gen.rand_bytes(SEED, gen.TAG_TEST, 1000, B, p.k)
    u, v, K = empty(B * g.u_stride * 8), empty(B * g.v_words * 8), empty(B * 64)
    ws = empty(hqc.hqc_kem_workspace_bytes(level, B))
    hqc.hqc_kem_encaps_batch(level, dev(H), dev(S), dev(hpk), dev(key), dev(m), u, v, K, ws)
    torch.cuda.synchronize()
    gu, gv = host(u, np.uint64, g.u_stride), host(v, np.uint64, g.v_words)
    gK = K.cpu().numpy().reshape(B, 64)
    for i in range(B):
        ru, rv, rK = oracle.kem_encaps(p, H[key[i]], S[key[i]], hpk[key[i]].tobytes(), m[i])
        assert (gu[i, : p.words] == ru).all() and (gu[i, p.words:] == 0).all(), i
        assert (gv[i] == rv).all(), i
        assert gK[i].tobytes() == rK, i


def _oracle_ciphertexts(p, g, H, S, hpk, key, m):
    B = len(key)
    U = np.zeros((B, g.u_stride), np.uint64)
    V = np.zeros((B, g.v_words), np.uint64)
    for i in range(B):
        u, v, _ = oracle.kem_encaps(p, H[key[i]], S[key[i]], hpk[key[i]].tobytes(), m[i])
        U[i, : p.words] = u
        V[i] = v
    return U, V


@pytest.mark.parametrize("level", [1, 3, 5])
def test_decaps_matches_oracle_with_implicit_rejection(level):
    nk, B = 4, 101
    p, g, H, S, y, sigma, hpk = _keyset(level, nk)
    key = (np.arange(B) * 5 % nk).astype(np.uint32)
    m = gen.rand_bytes(SEED, gen.TAG_TEST, 2000, B, p.k)
    U, V = _oracle_ciphertexts(p, g, H, S, hpk, key, m)
    rng = np.random.default_rng(100 + level)
    kind = np.arange(B) % 6
    for i in range(B):
        if kind[i] == 1:  # one bit of u below n: rejected
            b = int(rng.integers(p.n))
            U[i, b // 64] ^= np.uint64(1) << np.uint64(b % 64)
        elif kind[i] == 2:  # one bit of v: rejected
            b = int(rng.integers(p.n12))
            V[i, b // 64] ^= np.uint64(1) << np.uint64(b % 64)
        elif kind[i] == 3:  # a bit of u in [n, 8*ceil(n/8)) (inside the serialized bytes: rejected)
            ub = 8 * ((p.n + 7) // 8)  # or beyond them in the row's padding (not part of c: accepted)
            b = p.n + int(rng.integers(ub - p.n)) if (i // 6) % 2 == 0 else ub + int(rng.integers(64 * g.u_stride - ub))
            U[i, b // 64] ^= np.uint64(1) << np.uint64(b % 64)
        elif kind[i] == 4:  # uniformly random ciphertext
            U[i, : p.words] = rng.integers(0, 2**63, p.words, dtype=np.uint64)
            V[i] = rng.integers(0, 2**63, p.vwords, dtype=np.uint64)
        elif kind[i] == 5:  # decrypts to another message (wrong key's v with this u): rejected
            V[i] = V[(i + 1) % B]
    Kref, accref = oracle.kem_decaps_batch(p, H, S, hpk, sigma, key.astype(np.int64), y[key], U, V)
    assert accref[kind == 0].all() and not accref[(kind == 1) | (kind == 2) | (kind == 4)].any()
    k3 = np.nonzero(kind == 3)[0]
    assert not accref[k3[(k3 // 6) % 2 == 0]].any() and accref[k3[(k3 // 6) % 2 == 1]].all()
    K, acc = empty(B * 64), empty(B)
    ws = empty(hqc.hqc_kem_workspace_bytes(level, B))
    Y = np.zeros((nk, g.y_stride), np.uint32)
    Y[:, : p.w] = y[:, : p.w]
    hqc.hqc_kem_decaps_batch(level, dev(H), dev(S), dev(hpk), dev(sigma), dev(key), dev(Y), dev(U), dev(V), K, acc,
                             ws)
    torch.cuda.synchronize()
    assert (acc.cpu().numpy()[:B] == accref).all()
    assert (K.cpu().numpy()[: B * 64].reshape(B, 64) == Kref).all()


@pytest.mark.parametrize("level,B", [(1, 16384), (5, 4096)])
def test_encaps_decaps_round_trip_at_scale(level, B):
    """GPU Encaps -> GPU Decaps over many warps and one key per 256 rows (KEY_SHARE): every row is
    accepted with the same K (a property at any size); a sample is checked against the oracle."""
    nk = (B + 255) // 256
    p, g, H, S, y, sigma, hpk = _keyset(level, nk)
    key = gen.key_of(0, B).astype(np.uint32)
    m = gen.rand_bytes(SEED, gen.TAG_TEST, 5000, B, p.k)
    dH, dS, dhpk, dkey = dev(H), dev(S), dev(hpk), dev(key)
    u, v, K1, K2, acc = empty(B * g.u_stride * 8), empty(B * g.v_words * 8), empty(B * 64), empty(B * 64), empty(B)
    ws = empty(hqc.hqc_kem_workspace_bytes(level, B))
    hqc.hqc_kem_encaps_batch(level, dH, dS, dhpk, dkey, dev(m), u, v, K1, ws)
    Y = np.zeros((nk, g.y_stride), np.uint32)
    Y[:, : p.w] = y[:, : p.w]
    hqc.hqc_kem_decaps_batch(level, dH, dS, dhpk, dev(sigma), dkey, dev(Y), u, v, K2, acc, ws)
    torch.cuda.synchronize()
    assert int(acc[:B].sum()) == B
    assert torch.equal(K1[: B * 64], K2[: B * 64])
    gK = K1.cpu().numpy()[: B * 64].reshape(B, 64)
    for i in np.random.default_rng(level).choice(B, 12, replace=False):
        _, _, rK = oracle.kem_encaps(p, H[key[i]], S[key[i]], hpk[key[i]].tobytes(), m[i])
        assert gK[i].tobytes() == rK, i


def test_decaps_without_key_index():
    level, B = 3, 5
    p, g, H, S, y, sigma, hpk = _keyset(level, B)
    key = np.arange(B, dtype=np.uint32)
    m = gen.rand_bytes(SEED, gen.TAG_TEST, 9000, B, p.k)
    U, V = _oracle_ciphertexts(p, g, H, S, hpk, key, m)
    V[2, 7] ^= np.uint64(1 << 40)
    Kref, accref = oracle.kem_decaps_batch(p, H, S, hpk, sigma, key.astype(np.int64), y, U, V)
    K, acc = empty(B * 64), empty(B)
    Y = np.zeros((B, g.y_stride), np.uint32)
    Y[:, : p.w] = y[:, : p.w]
    ws = empty(hqc.hqc_kem_workspace_bytes(level, B))
    hqc.hqc_kem_decaps_batch(level, dev(H), dev(S), dev(hpk), dev(sigma), None, dev(Y), dev(U), dev(V), K, acc, ws)
    torch.cuda.synchronize()
    assert acc.cpu().numpy()[:B].tolist() == accref.tolist() == [1, 1, 0, 1, 1]
    assert (K.cpu().numpy()[: B * 64].reshape(B, 64) == Kref).all()


@pytest.mark.parametrize("level", [1, 3, 5])
def test_keygen_from_seed_matches_oracle(level):
    """hqc_kem_keygen_batch (R#24) against oracle.kem_keygen (pinned against hashlib and the schoolbook-
    pinned keygen product in tests/test_oracle_kem.py) and oracle.kem_hpk, over a ragged 128-lane tail."""
    p, g = oracle.params(level), hqc.params(level)
    nk = 133
    seeds = gen.rand_bytes(SEED, gen.TAG_TEST, 7000 + level, nk, 32)
    h, x, y, s = empty(nk * g.u_stride * 8), empty(nk * g.y_stride * 4), empty(nk * g.y_stride * 4), \
        empty(nk * g.u_stride * 8)
    sigma, hpk = empty(nk * p.k), empty(nk * 32)
    for t in (h, x, y, s):
        t.fill_(0xA5)  # padding must be written, not inherited
    hqc.hqc_kem_keygen_batch(level, dev(seeds), h, x, y, s, sigma, hpk)
    torch.cuda.synchronize()
    gh, gs = host(h, np.uint64, g.u_stride), host(s, np.uint64, g.u_stride)
    gx, gy = host(x, np.uint32, g.y_stride), host(y, np.uint32, g.y_stride)
    gsig, ghpk = sigma.cpu().numpy()[: nk * p.k].reshape(nk, p.k), hpk.cpu().numpy()[: nk * 32].reshape(nk, 32)
    for i in list(range(0, nk, 7)) + [nk - 1]:
        rh, rx, ry, rs, rsig = oracle.kem_keygen(p, seeds[i].tobytes())
        assert (gh[i, : p.words] == rh).all() and (gh[i, p.words:] == 0).all(), i
        assert (gs[i, : p.words] == rs).all() and (gs[i, p.words:] == 0).all(), i
        assert (gx[i, : p.w] == rx).all() and (gx[i, p.w:] == 0).all(), i
        assert (gy[i, : p.w] == ry).all() and (gy[i, p.w:] == 0).all(), i
        assert (gsig[i] == rsig).all(), i
        assert ghpk[i].tobytes() == oracle.kem_hpk(p, gh[i], gs[i]), i
    # properties on every key: distinct positions < n
    for arr in (gx, gy):
        a = arr[:, : p.w]
        assert (a < p.n).all()
        srt = np.sort(a, axis=1)
        assert (np.diff(srt.astype(np.int64), axis=1) > 0).all()


def test_kem_round_trip_with_seeded_gpu_keys():
    """Seeds -> GPU KeyGen -> GPU Encaps -> GPU Decaps: all accepted, equal keys; one tampered row rejected
    with the oracle's implicit-rejection key."""
    level, nk, B = 3, 4, 130
    p, g = oracle.params(level), hqc.params(level)
    seeds = gen.rand_bytes(SEED, gen.TAG_TEST, 7100, nk, 32)
    h, x, y, s = empty(nk * g.u_stride * 8), empty(nk * g.y_stride * 4), empty(nk * g.y_stride * 4), \
        empty(nk * g.u_stride * 8)
    sigma, hpk = empty(nk * p.k), empty(nk * 32)
    hqc.hqc_kem_keygen_batch(level, dev(seeds), h, x, y, s, sigma, hpk)
    key = (np.arange(B) % nk).astype(np.uint32)
    m = gen.rand_bytes(SEED, gen.TAG_TEST, 7200, B, p.k)
    u, v, K1, K2, acc = empty(B * g.u_stride * 8), empty(B * g.v_words * 8), empty(B * 64), empty(B * 64), empty(B)
    ws = empty(hqc.hqc_kem_workspace_bytes(level, B))
    dkey = dev(key)
    hqc.hqc_kem_encaps_batch(level, h, s, hpk, dkey, dev(m), u, v, K1, ws)
    v64 = v.view(torch.int64)
    v64[5 * g.v_words + 3] ^= 1 << 20
    hqc.hqc_kem_decaps_batch(level, h, s, hpk, sigma, dkey, y, u, v, K2, acc, ws)
    torch.cuda.synchronize()
    a = acc.cpu().numpy()[:B]
    assert a[5] == 0 and a.sum() == B - 1
    k1, k2 = K1.cpu().numpy()[: B * 64].reshape(B, 64), K2.cpu().numpy()[: B * 64].reshape(B, 64)
    ok = np.arange(B) != 5
    assert (k1[ok] == k2[ok]).all() and (k1[5] != k2[5]).any()
    rh, rx, ry, rs, rsig = oracle.kem_keygen(p, seeds[key[5]].tobytes())
    U = host(u, np.uint64, g.u_stride)[5:6]
    V = host(v, np.uint64, g.v_words)[5:6]
    Kref, accref = oracle.kem_decaps_batch(p, rh[None], rs[None], np.frombuffer(oracle.kem_hpk(p, rh, rs), np.uint8)[None],
                                           rsig[None], np.zeros(1, np.int64), ry[None], U, V)
    assert accref[0] == 0 and (k2[5] == Kref[0]).all()
