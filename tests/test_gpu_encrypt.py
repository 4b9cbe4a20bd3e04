"""GPU KeyGen product and Encrypt against the oracle, bit-exact, on
generator draws; plus the GPU encrypt -> GPU decrypt round trip at a full BASELINE size."""
import numpy as np
import pytest

import oracle
from paper_2512_12904_b200 import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2512_12904_b200 import hqc  # noqa: E402
from workloads import shape_for, valid_batch  # noqa: E402

DEV = torch.device("cuda:0")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).to(DEV)


def host(t, dtype, cols):
    return t.cpu().numpy().view(dtype).reshape(-1, cols)


@pytest.mark.parametrize("level", [1, 3, 5])
def test_keygen_matches_oracle(level):
    p = oracle.params(level)
    g = hqc.params(level)
    sh = shape_for(level)
    h, x, y = gen.key_draws(0xABC, sh, 0, 9)
    h[3, p.words - 1] |= np.uint64(0xFFFF) << np.uint64(p.n % 64)  # pad bits of h are ignored
    ref = np.stack([oracle.keygen(p, h[i, : p.words] & _mask(p), x[i], y[i]) for i in range(9)])
    s = torch.empty(9 * g.u_stride * 8, dtype=torch.uint8, device=DEV)
    hqc.hqc_keygen_batch(level, dev(h), dev(x), dev(y), s)
    torch.cuda.synchronize()
    got = host(s, np.uint64, g.u_stride)
    assert (got[:, : p.words] == ref).all()
    assert (got[:, p.words:] == 0).all()


def _mask(p):
    m = np.full(p.words, np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    m[-1] = np.uint64((1 << (p.n % 64)) - 1)
    return m


@pytest.mark.parametrize("level", [1, 3, 5])
def test_encrypt_matches_oracle(level):
    W = valid_batch(level, 20_000, 70)
    p, g = W["params"], hqc.params(level)
    B = 70
    # pad the key rows to u_stride
    H = np.zeros((W["h"].shape[0], g.u_stride), np.uint64)
    H[:, : W["h"].shape[1]] = W["h"]
    S = np.zeros_like(H)
    S[:, : p.words] = W["s"]
    key = W["key"].astype(np.uint32)
    u = torch.empty(B * g.u_stride * 8, dtype=torch.uint8, device=DEV)
    v = torch.empty(B * g.v_words * 8, dtype=torch.uint8, device=DEV)
    hqc.hqc_encrypt_batch(level, dev(H), dev(S), dev(key), dev(W["m"]), dev(W["r1"]), dev(W["r2"]), dev(W["e"]), u, v)
    torch.cuda.synchronize()
    gu = host(u, np.uint64, g.u_stride)
    gv = host(v, np.uint64, g.v_words)
    assert (gu == W["u"]).all()
    assert (gv == W["v"]).all()


def _edge_rows(sup, n, w):
    """Supports that reach the top of the doubled operand: position 0 (rotation d = n), n - 1 (d = 1), the
    run n-1, n-2, ... and the run 0, 1, ...; the other rows keep their generator draws."""
    sup = sup.copy()
    for i in range(sup.shape[0]):
        kind = i % 5
        row = np.sort(sup[i, :w])
        if kind == 0:
            row[0] = 0 if 0 not in row else row[0]
        elif kind == 1:
            row[-1] = n - 1 if n - 1 not in row else row[-1]
        elif kind == 2:
            row = (n - 1 - np.arange(w)).astype(np.uint32)
        elif kind == 3:
            row = np.arange(w, dtype=np.uint32)
        else:
            row[0], row[-1] = (0 if 0 not in row else row[0]), (n - 1 if n - 1 not in row else row[-1])
        assert len(set(row.tolist())) == w
        sup[i, :w] = row
    return sup


@pytest.mark.parametrize("kernel", ["1", "2"])
@pytest.mark.parametrize("level", [1, 3, 5])
def test_encrypt_and_keygen_edge_supports(level, kernel, monkeypatch):
    """Encrypt (both kernels: HQC_ENC_KERNEL, read per call) with r1, r2, e supports containing 0, n-1 and
    the runs at either end, and the KeyGen product with such x, y: the windows that reach the top word of
    the doubled operand. Bit-exact against the oracle."""
    monkeypatch.setenv("HQC_ENC_KERNEL", kernel)
    p, g, sh = oracle.params(level), hqc.params(level), shape_for(level)
    W = valid_batch(level, 30_000, 40)
    for key in ("r1", "r2", "e"):
        W[key] = _edge_rows(W[key], p.n, p.wr)
    H = np.zeros((W["h"].shape[0], g.u_stride), np.uint64)
    H[:, : W["h"].shape[1]] = W["h"]
    S = np.zeros_like(H)
    S[:, : p.words] = W["s"]
    key = W["key"].astype(np.uint32)
    B = 40
    u = torch.empty(B * g.u_stride * 8, dtype=torch.uint8, device=DEV)
    v = torch.empty(B * g.v_words * 8, dtype=torch.uint8, device=DEV)
    hqc.hqc_encrypt_batch(level, dev(H), dev(S), dev(key), dev(W["m"]), dev(W["r1"]), dev(W["r2"]), dev(W["e"]), u, v)
    torch.cuda.synchronize()
    gu, gv = host(u, np.uint64, g.u_stride), host(v, np.uint64, g.v_words)
    for i in range(B):
        k = key[i]
        ou, ov = oracle.encrypt(p, W["h"][k], W["s"][k], W["m"][i], W["r1"][i], W["r2"][i], W["e"][i])
        assert (gu[i, : p.words] == ou).all() and (gu[i, p.words:] == 0).all() and (gv[i] == ov).all(), i
    # KeyGen product s = x + h * y with edge supports in x and y
    h, x, y = gen.key_draws(0xED6E, sh, 0, 10)
    x, y = _edge_rows(x, p.n, p.w), _edge_rows(y, p.n, p.w)
    s = torch.empty(10 * g.u_stride * 8, dtype=torch.uint8, device=DEV)
    hqc.hqc_keygen_batch(level, dev(h), dev(x), dev(y), s)
    torch.cuda.synchronize()
    ref = np.stack([oracle.keygen(p, h[i, : p.words], x[i], y[i]) for i in range(10)])
    assert (host(s, np.uint64, g.u_stride)[:, : p.words] == ref).all()


@pytest.mark.parametrize("level,B", [(3, 65536)])
def test_gpu_encrypt_decrypt_round_trip_full_size(level, B):
    """configs[1] at full size entirely on the device: GPU keygen + encrypt of generator draws, then the
    fused decrypt; every row must return its message (property at any size), and a sample of rows is
    re-encrypted by the oracle to confirm the ciphertexts themselves."""
    g = hqc.params(level)
    sh = shape_for(level)
    seed = 0x5151
    nk = (B + 255) // 256
    h, x, y = gen.key_draws(seed, sh, 0, nk)
    m, r1, r2, e = gen.ct_draws(seed, sh, 0, B)
    key = gen.key_of(0, B).astype(np.uint32)
    s = torch.empty(nk * g.u_stride * 8, dtype=torch.uint8, device=DEV)
    dh = dev(h)
    hqc.hqc_keygen_batch(level, dh, dev(x), dev(y), s)
    u = torch.empty(B * g.u_stride * 8, dtype=torch.uint8, device=DEV)
    v = torch.empty(B * g.v_words * 8, dtype=torch.uint8, device=DEV)
    hqc.hqc_encrypt_batch(level, dh, s, dev(key), dev(m), dev(r1), dev(r2), dev(e), u, v)
    yrows = dev(y[key])
    mo = torch.empty(B * g.k, dtype=torch.uint8, device=DEV)
    hqc.hqc_decrypt_batch(level, u, v, yrows, mo)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    hqc.hqc_count_mismatch(level, mo, dev(m), cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    p = oracle.params(level)
    idx = np.random.default_rng(7).choice(B, 16, replace=False)
    sh_np = host(s, np.uint64, g.u_stride)
    gu, gv = host(u, np.uint64, g.u_stride), host(v, np.uint64, g.v_words)
    for i in idx:
        k = key[i]
        ou, ov = oracle.encrypt(p, h[k], sh_np[k], m[i], r1[i], r2[i], e[i])
        assert (gu[i, : p.words] == ou).all() and (gv[i] == ov).all()


@pytest.mark.parametrize("level", [1, 3, 5])
def test_scaling_config_full_size(level):
    """BASELINE configs[4]: 4,194,304 ciphertexts per level in ONE launch (the G = 1 shard), built on the
    device exactly as bench.py builds them (generator draws -> GPU keygen + encrypt, one key per 256).
    Every row must decrypt to its generator message (on-device mismatch count); a sample of rows is
    re-encrypted and decrypted by the oracle; and the rows of shard 5 of G = 8 regenerated on their own
    are byte-identical to the same rows of the G = 1 workload (per-index seeding)."""
    import bench

    B = 4_194_304
    g = hqc.params(level)
    p = oracle.params(level)
    du, dv, dy, dref = bench.make_valid_workload(level, 0, B, g, DEV)
    mo = torch.empty(B * g.k, dtype=torch.uint8, device=DEV)
    hqc.hqc_decrypt_batch(level, du, dv, dy, mo)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    hqc.hqc_count_mismatch(level, mo, dref, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    U = du.view(B, -1)
    V = dv.view(B, -1)
    Y = dy.view(B, -1)
    M = mo.view(B, -1)
    idx = np.sort(np.random.default_rng(level).choice(B, 24, replace=False))
    ti = torch.from_numpy(idx).to(DEV)
    su = U[ti].cpu().numpy().view(np.uint64)
    sv = V[ti].cpu().numpy().view(np.uint64)
    sy = Y[ti].cpu().numpy().view(np.uint32)
    sm = M[ti].cpu().numpy()
    assert (oracle.decrypt_batch(p, su, sv, sy) == sm).all()
    sh = shape_for(level)
    seed = bench.CONFIG_SEED[level]
    for i in idx[:4]:
        i = int(i)
        key = i // 256
        h, x, y = gen.key_draws(seed, sh, key, 1)
        s = oracle.keygen(p, h[0], x[0], y[0])
        m, r1, r2, e = gen.ct_draws(seed, sh, i, 1)
        u, v = oracle.encrypt_batch(p, h, s[None], np.zeros(1, np.int64), m, r1, r2, e)
        j = int(np.nonzero(idx == i)[0][0])
        assert (su[j, : p.words] == u[0]).all() and (sv[j] == v[0]).all()
    r0 = 5 * B // 8 + 1000  # inside shard 5 of G = 8, not on a key boundary
    eu, ev, ey, em = bench.make_valid_workload(level, r0, 40, g, DEV)
    assert torch.equal(eu.view(40, -1), U[r0:r0 + 40]) and torch.equal(ev.view(40, -1), V[r0:r0 + 40])
    assert torch.equal(ey.view(40, -1), Y[r0:r0 + 40]) and torch.equal(em.view(40, -1), dref.view(B, -1)[r0:r0 + 40])
    del du, dv, dy, dref, mo, U, V, Y, M
    torch.cuda.empty_cache()


def test_one_warp_encrypt_kernel_variant():
    """HQC_ENC_KERNEL=1 selects the first (one warp per ciphertext) encrypt kernel instead of the warp-pair
    kernel with per-key cached operands; the encrypt and KEM parity tests run again under it in a
    subprocess (the switch is read once per process)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HQC_ENC_KERNEL="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_kem.py",
                        "tests/test_gpu_encrypt.py", "-k", "not scaling_config and not one_warp_encrypt"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("level", [1, 3, 5])
def test_encrypt_key_switching_and_identity_rows(level):
    """The warp-pair encrypt caches each key's doubled operands across consecutive rows of one key: rows
    that switch keys back and forth (and runs of one key), and key_index = NULL (row b uses key b), must
    all match the oracle's encryption."""
    g = hqc.params(level)
    p = oracle.params(level)
    sh = shape_for(level)
    nk, B = 5, 96
    h, x, y = gen.key_draws(0x6B6579, sh, 0, nk)
    s = np.stack([oracle.keygen(p, h[i], x[i], y[i]) for i in range(nk)])
    H = np.zeros((nk, g.u_stride), np.uint64)
    H[:, : h.shape[1]] = h
    S = np.zeros_like(H)
    S[:, : p.words] = s
    rng = np.random.default_rng(level)
    key = np.concatenate([rng.integers(0, nk, 40), np.repeat([3, 1, 3], [20, 5, 31])]).astype(np.uint32)
    m, r1, r2, e = gen.ct_draws(0x6B6579, sh, 0, B)
    ru, rv = oracle.encrypt_batch(p, h, s, key.astype(np.int64), m, r1, r2, e)
    u = torch.empty(B * g.u_stride * 8, dtype=torch.uint8, device=DEV)
    v = torch.empty(B * g.v_words * 8, dtype=torch.uint8, device=DEV)
    hqc.hqc_encrypt_batch(level, dev(H), dev(S), dev(key), dev(m), dev(r1), dev(r2), dev(e), u, v)
    torch.cuda.synchronize()
    gu, gv = host(u, np.uint64, g.u_stride), host(v, np.uint64, g.v_words)
    assert (gu[:, : p.words] == ru).all() and (gu[:, p.words:] == 0).all()
    assert (gv == rv).all()
    # key_index = NULL: per-row keys
    Hr, Sr = np.ascontiguousarray(H[key]), np.ascontiguousarray(S[key])
    hqc.hqc_encrypt_batch(level, dev(Hr), dev(Sr), None, dev(m), dev(r1), dev(r2), dev(e), u, v)
    torch.cuda.synchronize()
    assert (host(u, np.uint64, g.u_stride)[:, : p.words] == ru).all() and (host(v, np.uint64, g.v_words) == rv).all()
