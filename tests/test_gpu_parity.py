"""GPU parity: the CUDA path (through the C ABI) against the ORACLE, element by element, on seeded
inputs. Integer/bit work, so the bar is bit-exact. Marked gpu: needs a B200 and the built library.

Sizes: small batches that span several chunks of 32 ciphertexts and a ragged tail, all three levels;
adversarial (undecodable) inputs; stage-level garbage inputs; edge cases (batch 0/1, 33, supports at
0 and n-1, all-zero ciphertext); and full BASELINE sizes in the bench's launch configuration with
sampled oracle checks plus the whole-batch property decrypt(encrypt(m)) = m."""
import numpy as np
import pytest

import oracle
from paper_2512_12904_b200 import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU only with -m gpu
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2512_12904_b200 import hqc  # noqa: E402
from workloads import adversarial_batch, valid_batch  # noqa: E402

DEV = torch.device("cuda:0")
LEVELS = [1, 3, 5]


def to_dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).to(DEV)


def from_dev(t, dtype, cols):
    return t.cpu().numpy().view(dtype).reshape(-1, cols)


def gpu_decrypt(level, W):
    p = hqc.params(level)
    B = W["u"].shape[0]
    m = torch.empty(B * p.k, dtype=torch.uint8, device=DEV)
    hqc.hqc_decrypt_batch(level, to_dev(W["u"]), to_dev(W["v"]), to_dev(W["y"]), m)
    torch.cuda.synchronize()
    return from_dev(m, np.uint8, p.k)


def gpu_stage1(level, W, with_v=True):
    p = hqc.params(level)
    B = W["u"].shape[0]
    r = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device=DEV)
    hqc.hqc_sparse_dense_mul_batch(level, to_dev(W["u"]), to_dev(W["y"]), to_dev(W["v"]) if with_v else None, r)
    torch.cuda.synchronize()
    return from_dev(r, np.uint64, p.v_words)


def gpu_stage2(level, r):
    p = hqc.params(level)
    B = r.shape[0]
    s = torch.empty(B * p.n1, dtype=torch.uint8, device=DEV)
    hqc.hqc_rm_decode_batch(level, to_dev(r), s)
    torch.cuda.synchronize()
    return from_dev(s, np.uint8, p.n1)


def gpu_stage3(level, sym):
    p = hqc.params(level)
    B = sym.shape[0]
    m = torch.empty(B * p.k, dtype=torch.uint8, device=DEV)
    ok = torch.empty(B, dtype=torch.uint8, device=DEV)
    hqc.hqc_rs_decode_batch(level, to_dev(sym), m, ok)
    torch.cuda.synchronize()
    return from_dev(m, np.uint8, p.k), ok.cpu().numpy()


# ---------------------------------------------------------------- end to end, small
@pytest.mark.parametrize("level", LEVELS)
@pytest.mark.parametrize("B", [1, 33, 200])
def test_decrypt_valid(level, B):
    W = valid_batch(level, 1000, B)
    p = W["params"]
    got = gpu_decrypt(level, W)
    assert (got == W["m"]).all()
    assert (got == oracle.decrypt_batch(p, W["u"], W["v"], W["y"])).all()


def test_decrypt_adversarial_quarters():
    W = adversarial_batch(0, 512, 512)
    p = W["params"]
    ref = oracle.decrypt_batch(p, W["u"], W["v"], W["y"])
    got = gpu_decrypt(1, W)
    bad = np.nonzero((got != ref).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first rows {bad[:8]} quarters {W['quarter'][bad[:8]]}"
    q = W["quarter"]
    assert (got[q == 0] == W["m"][q == 0]).all()
    assert (got[q == 3] != W["m"][q == 3]).any(axis=1).mean() > 0.9  # random ciphertexts: garbage


@pytest.mark.parametrize("level", LEVELS)
def test_decrypt_random_ciphertexts_and_edges(level):
    p = oracle.params(level)
    W = valid_batch(level, 5000, 70)
    rng = np.random.default_rng(level)
    # rows 0..29: uniformly random u, v (undecodable garbage)
    W["u"][:30] = gen.dense(11, gen.TAG_U_RAND, 0, 30, p.n, W["u"].shape[1])
    W["v"][:30] = gen.dense(11, gen.TAG_V_RAND, 0, 30, p.n12, W["v"].shape[1])
    # rows 30..33: supports hitting 0 and n-1 (the d = n and d = 1 rotations)
    W["y"][30, 0] = 0
    W["y"][31, p.w - 1] = p.n - 1
    W["y"][32, :p.w] = np.arange(p.w, dtype=np.uint32)
    W["y"][33, :p.w] = p.n - 1 - np.arange(p.w, dtype=np.uint32)
    # row 34: all-zero ciphertext -> 0^k; row 35: u pad bits set (ignored, R#13)
    W["u"][34] = 0
    W["v"][34] = 0
    W["u"][35, p.words - 1] |= np.uint64(0xFFFFFFFFFFFFFFFF) << np.uint64(p.n % 64)
    if W["u"].shape[1] > p.words:
        W["u"][35, p.words:] = rng.integers(0, 2**63, W["u"].shape[1] - p.words, dtype=np.uint64)
    # padding entries of y rows are ignored
    W["y"][36, p.w:] = 12345
    ref = oracle.decrypt_batch(p, W["u"], W["v"], W["y"])
    got = gpu_decrypt(level, W)
    assert (got == ref).all()
    assert (got[34] == 0).all()


# ---------------------------------------------------------------- per stage
@pytest.mark.parametrize("level", LEVELS)
def test_stage1_product(level):
    W = valid_batch(level, 2000, 97)
    p = W["params"]
    W["u"][:20] = gen.dense(3, gen.TAG_U_RAND, 0, 20, p.n, W["u"].shape[1])
    ref = oracle.stage1_batch(p, W["u"], W["v"], W["y"])
    assert (gpu_stage1(level, W) == ref).all()
    # v = NULL: the truncated product alone
    ref0 = oracle.stage1_batch(p, W["u"], np.zeros_like(W["v"]), W["y"])
    assert (gpu_stage1(level, W, with_v=False) == ref0).all()


@pytest.mark.parametrize("level", LEVELS)
def test_stage2_rm_random_and_real(level):
    p = oracle.params(level)
    r_rand = gen.dense(21, gen.TAG_TEST, 0, 150, p.n12, p.vwords)  # ~20% tied blocks (R#11)
    W = valid_batch(level, 3000, 40)
    r_real = oracle.stage1_batch(p, W["u"], W["v"], W["y"])
    for r in (r_rand, r_real):
        assert (gpu_stage2(level, r) == oracle.rm_decode_batch(p, r)).all()


@pytest.mark.parametrize("level", LEVELS)
def test_stage3_rs(level):
    p = oracle.params(level)
    rng = np.random.default_rng(100 + level)
    rows = []
    kinds = []
    for i in range(300):
        m = rng.integers(0, 256, p.k).astype(np.uint8)
        c = oracle.rs_encode(m, p.n1, p.k)
        kind = i % 5
        if kind == 0:  # clean
            pass
        elif kind == 1:  # exactly delta errors
            pos = rng.choice(p.n1, p.delta, replace=False)
            c[pos] ^= rng.integers(1, 256, p.delta).astype(np.uint8)
        elif kind == 2:  # random number of errors <= delta, some in the message part
            t = int(rng.integers(1, p.delta + 1))
            pos = rng.choice(p.n1, t, replace=False)
            c[pos] ^= rng.integers(1, 256, t).astype(np.uint8)
        elif kind == 3:  # beyond capacity
            t = int(rng.integers(p.delta + 1, 2 * p.delta + 1))
            pos = rng.choice(p.n1, t, replace=False)
            c[pos] ^= rng.integers(1, 256, t).astype(np.uint8)
        else:  # garbage
            c = rng.integers(0, 256, p.n1).astype(np.uint8)
        rows.append(c)
        kinds.append(kind)
    sym = np.stack(rows)
    ref, ref_ok = oracle.rs_decode_batch(p, sym)
    got, ok = gpu_stage3(level, sym)
    assert (got == ref).all()
    assert (ok == ref_ok).all()
    kinds = np.array(kinds)
    assert ok[kinds <= 2].all() and not ok[kinds == 4].any()


@pytest.mark.parametrize("level", LEVELS)
@pytest.mark.parametrize("method", ["linear", "nibble", "logexp"])
def test_stage_a6_syndromes_all_methods(level, method):
    """Step a6 alone (hqc_rs_syndromes_batch), each of the three GF-product methods, against the oracle's
    Horner evaluation S_i = r(alpha^i) (oracle/rs.c), on random words, words with zero symbols, codewords
    (all-zero syndromes) and the all-zero / all-0xFF words; 197 rows = 6 warps and a ragged tail."""
    p = oracle.params(level)
    rng = np.random.default_rng(300 + level)
    B = 197
    sym = rng.integers(0, 256, (B, p.n1)).astype(np.uint8)
    sym[1::7] &= rng.integers(0, 2, (len(sym[1::7]), p.n1)).astype(np.uint8) * 0xFF  # many zero symbols
    for i in range(2, B, 11):
        sym[i] = oracle.rs_encode(rng.integers(0, 256, p.k).astype(np.uint8), p.n1, p.k)
    sym[3] = 0
    sym[4] = 0xFF
    ref = np.stack([oracle.rs_syndromes(r, p.n1, p.delta) for r in sym])
    assert not ref[2::11].any()
    out = torch.empty(B * 2 * p.delta, dtype=torch.uint8, device=DEV)
    hqc.hqc_rs_syndromes_batch(level, to_dev(sym), out, method)
    torch.cuda.synchronize()
    assert (from_dev(out, np.uint8, 2 * p.delta) == ref).all()


# ---------------------------------------------------------------- API behaviour
def test_batch_zero_and_errors():
    p = hqc.params(1)
    x = torch.zeros(16, dtype=torch.uint8, device=DEV)
    hqc.hqc_decrypt_batch(1, x[:0], x[:0], x[:0], x[:0])  # batch 0: no launch, no error
    with pytest.raises(hqc.HqcError):
        hqc.hqc_decrypt_batch(2, x, x, x, x)


def test_mismatch_counter_and_support_validation():
    W = valid_batch(3, 7000, 64)
    p = hqc.params(3)
    m = torch.from_numpy(W["m"]).to(DEV)
    m2 = m.clone()
    m2[5, 3] ^= 1
    m2[40, 0] ^= 0x80
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    hqc.hqc_count_mismatch(3, m, m2, cnt)
    assert int(cnt.item()) == 2
    y = W["y"].copy()
    y[3, 0] = p.n
    y[9, 2] = y[9, 1]
    bad = torch.zeros(1, dtype=torch.int64, device=DEV)
    hqc.hqc_validate_support(3, to_dev(y), bad)
    assert int(bad.item()) == 2


# ---------------------------------------------------------------- full BASELINE sizes
FULL = [(1, 1024), (3, 65536), (5, 262144)]


@pytest.mark.parametrize("level,B", FULL)
def test_full_size_config(level, B):
    """BASELINE configs[0..2] at their batch sizes, launched exactly as bench.py launches them.
    Rows are 4096 distinct oracle-encrypted ciphertexts tiled to B (row i = ciphertext i mod 4096),
    so every output is known: decrypt(encrypt(m)) = m at every row, and a sample of rows is checked
    against the oracle's own decryption."""
    D = min(B, 4096)
    W = valid_batch(level, 10_000, D)
    p = W["params"]
    reps = B // D
    u = np.tile(W["u"], (reps, 1))
    v = np.tile(W["v"], (reps, 1))
    y = np.tile(W["y"], (reps, 1))
    got = gpu_decrypt(level, dict(u=u, v=v, y=y))
    assert (got == np.tile(W["m"], (reps, 1))).all()
    idx = np.random.default_rng(level).choice(B, 64, replace=False)
    ref = oracle.decrypt_batch(p, u[idx], v[idx], y[idx])
    assert (got[idx] == ref).all()


def test_full_size_adversarial():
    """BASELINE configs[3] (1,048,576 HQC-1, four quarters) in the bench launch configuration:
    the batch is 4 x 8192 distinct adversarial ciphertexts per quarter tiled 32 times; every row
    is compared against the oracle's output for its source row."""
    B, D = 1_048_576, 32768
    W = adversarial_batch(0, D, D)
    p = W["params"]
    ref = oracle.decrypt_batch(p, W["u"], W["v"], W["y"])
    q = D // 4
    order = np.concatenate([np.tile(np.arange(k * q, (k + 1) * q), B // D) for k in range(4)])
    got = gpu_decrypt(1, dict(u=W["u"][order], v=W["v"][order], y=W["y"][order]))
    assert (got == ref[order]).all()


# ---------------------------------------------------------------- both fused-kernel variants
@pytest.mark.parametrize("kernel", ["1", "2", "3", "4", "5", "6", "7", "8", "9", "10", "11", "12"])
def test_both_fused_kernel_variants(kernel, tmp_path):
    """Every decrypt kernel (hqc.KERNEL_NAMES; the library picks one per level and batch)
    against the oracle on every level, including 10 and 11, the two-launch splits with their pool scratch.
    HQC_DEC_KERNEL forces each (read once per process), so each runs in a subprocess."""
    import subprocess
    import sys
    import os

    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, "tests")
import oracle
from paper_2512_12904_b200 import hqc
from workloads import valid_batch, adversarial_batch
for level in (1, 3, 5):
    W = valid_batch(level, 40000, 77) if level != 1 else adversarial_batch(0, 128, 128)
    p = hqc.params(level)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).cuda()
    B = W["u"].shape[0]
    m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
    hqc.hqc_decrypt_batch(level, d(W["u"]), d(W["v"]), d(W["y"]), m)
    torch.cuda.synchronize()
    ref = oracle.decrypt_batch(W["params"], W["u"], W["v"], W["y"])
    assert (m.cpu().numpy().reshape(B, p.k) == ref).all(), level
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HQC_DEC_KERNEL=kernel)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("kernel", ["10", "11"])
def test_two_launch_kernel_ragged_split_and_graph_capture(kernel):
    """Kernels 10 and 11 (k_decrypt_s12 / _s12c + k_stage3, HQC-5's large-batch kernels) take their symbol scratch from the
    library's stream-ordered pool: split into parts (HQC_DEC_SPLIT=1000 over 2,500 rows: three equal parts
    of at most 1000, rounded to 32, the last one ragged) it matches the oracle, and the call captured in a CUDA graph (pool allocation inside the
    capture) replays to the same outputs; a mixed-level call after it is unaffected."""
    import os
    import subprocess
    import sys

    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, "tests")
import oracle
from paper_2512_12904_b200 import hqc
from workloads import valid_batch
KERNEL = int(sys.argv[1])
d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).cuda()
for level in (5, 1):
    W = valid_batch(level, 90000, 2500, 41)
    p = hqc.params(level)
    assert hqc.hqc_decrypt_launch_kernel(level, 2500) == KERNEL
    assert hqc.hqc_decrypt_launch_count(level, 2500) == 6
    u, v, y = d(W["u"]), d(W["v"]), d(W["y"])
    ref = oracle.decrypt_batch(W["params"], W["u"], W["v"], W["y"])
    m = torch.zeros(2500 * p.k, dtype=torch.uint8, device="cuda")
    hqc.hqc_decrypt_batch(level, u, v, y, m)
    torch.cuda.synchronize()
    assert (m.cpu().numpy().reshape(2500, p.k) == ref).all(), level
    m.zero_()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            hqc.hqc_decrypt_batch(level, u, v, y, m, stream=s)
    for _ in range(2):
        m.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert (m.cpu().numpy().reshape(2500, p.k) == ref).all(), ("graph", level)
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HQC_DEC_KERNEL=kernel, HQC_DEC_SPLIT="1000")
    r = subprocess.run([sys.executable, "-c", code, kernel], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("level,chunk", [(1, 0), (3, 100), (5, 64)])
def test_host_buffer_entry_point(level, chunk):
    """hqc_decrypt_batch_host (host buffers, chunked over two streams) = oracle, ragged last chunk."""
    W = valid_batch(level, 50_000, 333)
    p = hqc.params(level)
    hu, hv, hy = (torch.from_numpy(np.ascontiguousarray(W[k]).view(np.uint8)).pin_memory() for k in ("u", "v", "y"))
    hm = torch.zeros(333 * p.k, dtype=torch.uint8).pin_memory()
    ws = torch.empty(hqc.hqc_decrypt_host_workspace_bytes(level, chunk or 8192), dtype=torch.uint8, device=DEV)
    hqc.hqc_decrypt_batch_host(level, hu, hv, hy, hm, ws, chunk)
    torch.cuda.synchronize()
    ref = oracle.decrypt_batch(W["params"], W["u"], W["v"], W["y"])
    assert (hm.numpy().reshape(333, p.k) == ref).all()
    small = torch.empty(16, dtype=torch.uint8, device=DEV)
    with pytest.raises(hqc.HqcError):
        hqc.hqc_decrypt_batch_host(level, hu, hv, hy, hm, small, chunk)


def serialize(W, p):
    """c = u bytes (ceil(n/8)) || v bytes (n1 n2 / 8) per row, from the ABI rows."""
    ub = (p.n + 7) // 8
    U = np.ascontiguousarray(W["u"]).view(np.uint8).reshape(len(W["u"]), -1)[:, :ub]
    V = np.ascontiguousarray(W["v"]).view(np.uint8).reshape(len(W["v"]), -1)
    return np.ascontiguousarray(np.concatenate([U, V], axis=1))


@pytest.mark.parametrize("level,chunk", [(1, 0), (3, 37), (5, 64)])
def test_serialized_ciphertext_host_entry_point(level, chunk):
    """hqc_decrypt_ct_batch_host: host serialized ciphertexts (odd byte lengths, so rows start at every
    alignment) + host key indices + the device-resident key-support table; = oracle on valid, tampered and
    uniformly random ciphertexts, ragged last chunk; one key without key indices; the unpacked bytes past
    n are ignored exactly like the row API's."""
    from workloads import keys
    p = hqc.params(level)
    op = oracle.params(level)
    B = 203
    W = valid_batch(level, 60_000, B)
    rng = np.random.default_rng(level)
    W["v"][5] ^= np.uint64(1) << np.uint64(17)
    W["u"][9, : op.words] = rng.integers(0, 2**63, op.words, dtype=np.uint64)
    W["u"][9, op.words - 1] &= np.uint64((1 << (p.n % 64)) - 1)
    W["v"][9] = rng.integers(0, 2**63, op.vwords, dtype=np.uint64)
    ct = serialize(W, p)
    assert ct.shape[1] == hqc.hqc_ct_bytes(level) == (p.n + 7) // 8 + p.n12 // 8
    k0 = 60_000 // 256
    nk = int(W["key"].max()) + 1
    _, _, ykeys, _ = keys(level, k0, nk, {1: 0xC0F10001, 3: 0xC0F10002, 5: 0xC0F10003}[level])
    Y = np.zeros((nk, p.y_stride), np.uint32)
    Y[:, : p.w] = ykeys[:, : p.w]
    hct = torch.from_numpy(ct.reshape(-1)).pin_memory()
    hkey = torch.from_numpy(W["key"].astype(np.uint32)).pin_memory()
    hm = torch.zeros(B * p.k, dtype=torch.uint8).pin_memory()
    ws = torch.empty(hqc.hqc_decrypt_ct_host_workspace_bytes(level, chunk or 8192), dtype=torch.uint8, device=DEV)
    hqc.hqc_decrypt_ct_batch_host(level, hct, hkey, to_dev(Y), hm, ws, chunk)
    torch.cuda.synchronize()
    ref = oracle.decrypt_batch(W["params"], W["u"], W["v"], W["y"])
    got = hm.numpy().reshape(B, p.k)
    assert (got == ref).all()
    # one key, no key indices
    one = W["key"] == W["key"][0]
    ct1 = torch.from_numpy(np.ascontiguousarray(ct[one]).reshape(-1)).pin_memory()
    hm1 = torch.zeros(int(one.sum()) * p.k, dtype=torch.uint8).pin_memory()
    hqc.hqc_decrypt_ct_batch_host(level, ct1, None, to_dev(Y[int(W["key"][0])][None]), hm1, ws, chunk)
    torch.cuda.synchronize()
    assert (hm1.numpy().reshape(-1, p.k) == ref[one]).all()


@pytest.mark.parametrize("kernel", ["1", "2", "3"])
def test_standalone_product_kernel_variants(kernel):
    """hqc_sparse_dense_mul_batch has two kernels (one warp per ciphertext; warp pair with the output words
    split, the HQC-5 default); HQC_S1_KERNEL forces either (read once per process): the stage-1 parity
    tests run again under each in a subprocess."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HQC_S1_KERNEL=kernel)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_parity.py",
                        "-k", "stage1_product"], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_edge_batches_new_entry_points():
    """batch 0 / 1 and chunk > batch on the newer entry points: step a6, KeyGen from seeds, the
    serialized-ciphertext host call; NULL / misaligned arguments return the documented codes."""
    level = 1
    p = hqc.params(level)
    op = oracle.params(level)
    # step a6, batch 1 and 0
    sym = np.arange(p.n1, dtype=np.uint8)[None]
    out = torch.empty(2 * p.delta, dtype=torch.uint8, device=DEV)
    for meth in ("linear", "nibble", "logexp"):
        hqc.hqc_rs_syndromes_batch(level, to_dev(sym), out, meth)
        torch.cuda.synchronize()
        assert (out.cpu().numpy() == oracle.rs_syndromes(sym[0], p.n1, p.delta)).all()
    hqc.hqc_rs_syndromes_batch(level, torch.empty(0, dtype=torch.uint8, device=DEV),
                               torch.empty(0, dtype=torch.uint8, device=DEV))
    # KeyGen from one seed
    seeds = torch.arange(32, dtype=torch.uint8, device=DEV)
    h, x, y, s = (torch.empty(p.u_stride * 8, dtype=torch.uint8, device=DEV), torch.empty(p.y_stride * 4, dtype=torch.uint8, device=DEV),
                  torch.empty(p.y_stride * 4, dtype=torch.uint8, device=DEV), torch.empty(p.u_stride * 8, dtype=torch.uint8, device=DEV))
    sig = torch.empty(16 if p.k < 16 else p.k, dtype=torch.uint8, device=DEV)[: p.k]
    hqc.hqc_kem_keygen_batch(level, seeds, h, x, y, s, sig)  # no H_pk output
    torch.cuda.synchronize()
    rh, rx, ry, rs, rsig = oracle.kem_keygen(op, bytes(range(32)))
    assert (h.cpu().numpy().view(np.uint64)[: op.words] == rh).all()
    assert (y.cpu().numpy().view(np.uint32)[: p.w] == ry).all() and (sig.cpu().numpy() == rsig).all()
    # serialized host call: batch 1, chunk larger than the batch
    W = valid_batch(level, 777, 1)
    ct = serialize(W, p)
    hm = torch.zeros(p.k, dtype=torch.uint8).pin_memory()
    ws = torch.empty(hqc.hqc_decrypt_ct_host_workspace_bytes(level, 1), dtype=torch.uint8, device=DEV)
    hqc.hqc_decrypt_ct_batch_host(level, torch.from_numpy(ct.reshape(-1)).pin_memory(), None, to_dev(W["y"]), hm, ws, 64)
    torch.cuda.synchronize()
    assert (hm.numpy() == W["m"][0]).all()


def test_tensor_memory_variants_at_scale(tmp_path):
    """The opt-in tensor-memory kernels at batches that make every warp loop: k_stage1t (HQC_S1_KERNEL=3)
    over 5,000 products per level (more than 148 CTAs x 16 warps, so the grid-stride loop turns) and
    k_decrypt_t (HQC_DEC_KERNEL=4) over 60,000 HQC-1 ciphertexts (34 per warp: two RS chunks). Their outputs
    must equal the default constant-flow kernels' (themselves oracle-checked above) on the same seeded
    random inputs; the switches are read once per process, so the variants run in a subprocess."""
    import os
    import subprocess
    import sys

    arrs = {}
    for level, B in ((1, 5000), (3, 5000), (5, 5000)):
        p = oracle.params(level)
        hp = hqc.params(level)
        u = gen.dense(31, gen.TAG_U_RAND, 0, B, p.n, hp.u_stride)
        v = gen.dense(31, gen.TAG_V_RAND, 0, B, p.n12, hp.v_words)
        y = gen.support(31, gen.TAG_Y, 0, B, p.n, p.w, hp.y_stride)
        r = torch.empty(B * hp.v_words * 8, dtype=torch.uint8, device=DEV)
        hqc.hqc_sparse_dense_mul_batch(level, to_dev(u), to_dev(y), to_dev(v), r)
        torch.cuda.synchronize()
        arrs.update({f"u{level}": u, f"v{level}": v, f"y{level}": y, f"r{level}": r.cpu().numpy()})
    B = 60000
    p, hp = oracle.params(1), hqc.params(1)
    u = gen.dense(32, gen.TAG_U_RAND, 0, B, p.n, hp.u_stride)
    v = gen.dense(32, gen.TAG_V_RAND, 0, B, p.n12, hp.v_words)
    y = gen.support(32, gen.TAG_Y, 0, B, p.n, p.w, hp.y_stride)
    m = torch.empty(B * hp.k, dtype=torch.uint8, device=DEV)
    hqc.hqc_decrypt_batch(1, to_dev(u), to_dev(v), to_dev(y), m)
    torch.cuda.synchronize()
    arrs.update({"du": u, "dv": v, "dy": y, "dm": m.cpu().numpy()})
    # the reference outputs themselves against the oracle on sampled rows, so that the variants' equality
    # below is a comparison with the oracle on those rows, not only with the default kernels
    idx = np.random.default_rng(5).choice(B, 96, replace=False)
    assert (arrs["dm"].reshape(B, hp.k)[idx] == oracle.decrypt_batch(p, u[idx], v[idx], y[idx])).all()
    for level in (1, 3, 5):
        op, hp_ = oracle.params(level), hqc.params(level)
        Bl = arrs[f"u{level}"].shape[0]
        ii = np.random.default_rng(level).choice(Bl, 48, replace=False)
        ref = oracle.stage1_batch(op, arrs[f"u{level}"][ii], arrs[f"v{level}"][ii], arrs[f"y{level}"][ii])
        assert (arrs[f"r{level}"].view(np.uint64).reshape(Bl, hp_.v_words)[ii] == ref).all()
    f = tmp_path / "ref.npz"
    np.savez(f, **arrs)
    code = r'''
import sys, numpy as np, torch
from paper_2512_12904_b200 import hqc
A = np.load(sys.argv[1])
d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).cuda()
for level in (1, 3, 5):
    hp = hqc.params(level)
    B = A[f"u{level}"].shape[0]
    r = torch.empty(B * hp.v_words * 8, dtype=torch.uint8, device="cuda")
    hqc.hqc_sparse_dense_mul_batch(level, d(A[f"u{level}"]), d(A[f"y{level}"]), d(A[f"v{level}"]), r)
    torch.cuda.synchronize()
    assert (r.cpu().numpy() == A[f"r{level}"]).all(), ("k_stage1t", level)
m = torch.empty(A["dm"].size, dtype=torch.uint8, device="cuda")
hqc.hqc_decrypt_batch(1, d(A["du"]), d(A["dv"]), d(A["dy"]), m)
torch.cuda.synchronize()
assert (m.cpu().numpy() == A["dm"]).all(), "k_decrypt_t"
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HQC_S1_KERNEL="3", HQC_DEC_KERNEL="4")
    r = subprocess.run([sys.executable, "-c", code, str(f)], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


# ---------------------------------------------------------------- small batches (K4s) and split launches
@pytest.mark.parametrize("level,B", [(1, 1), (1, 33), (1, 1024), (3, 1), (3, 33), (3, 1024), (5, 1), (5, 33),
                                     (5, 1024)])
def test_small_batch_kernel(level, B):
    """BASELINE configs[0]'s size class: batches up to SMs x 8 take k_decrypt_sb (groups of G ciphertexts,
    one warp each, G chosen to spread the batch over all SMs). Bit-exact against the oracle,
    with a quarter of the rows replaced by uniformly random (undecodable) ciphertexts."""
    W = valid_batch(level, 90_000, B)
    p = W["params"]
    nr = B // 4
    if nr:
        W["u"][:nr] = gen.dense(41, gen.TAG_U_RAND, 0, nr, p.n, W["u"].shape[1])
        W["v"][:nr] = gen.dense(41, gen.TAG_V_RAND, 0, nr, p.n12, W["v"].shape[1])
    grid, wpc = hqc.hqc_decrypt_launch_shape(level, B)
    assert grid * wpc >= B and grid <= torch.cuda.get_device_properties(DEV).multi_processor_count
    got = gpu_decrypt(level, W)
    assert (got == oracle.decrypt_batch(p, W["u"], W["v"], W["y"])).all()
    assert (got[nr:] == W["m"][nr:]).all()


@pytest.mark.parametrize("sb_max,split", [("100000", ""), ("0", "700"), ("0", "64")])
def test_group_striding_and_split_launches(sb_max, split, monkeypatch):
    """Launch policies read on every call: HQC_SB_MAX forces k_decrypt_sb on a batch larger than its grid
    (groups strided over the CTAs), HQC_DEC_SPLIT runs one batch as consecutive launches of at most that
    many ciphertexts (ragged last launch); HQC-1 adversarial rows, compared with the oracle."""
    W = adversarial_batch(0, 3000, 3000)
    p = W["params"]
    ref = oracle.decrypt_batch(p, W["u"], W["v"], W["y"])
    monkeypatch.setenv("HQC_SB_MAX", sb_max)
    monkeypatch.setenv("HQC_DEC_SPLIT", split)
    got = gpu_decrypt(1, W)
    assert (got == ref).all()
