"""CPU-side checks of the C ABI (no compute calls without a GPU): the library loads, exports every
function include/hqc_gpu.h declares, hqc_get_params agrees with the oracle's independent Table I copy,
and host-side argument validation returns the documented status codes before touching CUDA."""
import ctypes
import os
import re

import pytest

import oracle
from paper_2512_12904_b200 import build as gpubuild
from paper_2512_12904_b200 import hqc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    gpubuild.build()
    return hqc.lib()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "hqc_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hqc_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/hqc_gpu.h but not exported"


@pytest.mark.parametrize("level", [1, 3, 5])
def test_params_match_oracle(level, L):
    g = hqc.params(level)
    o = oracle.params(level)
    for f in ("n", "n1", "n2", "mult", "k", "delta", "w", "wr", "n12"):
        assert getattr(g, f) == getattr(o, f), f
    assert g.u_words == o.words and g.v_words == o.vwords
    assert g.u_stride % 2 == 0 and g.u_stride >= g.u_words
    assert g.y_stride % 4 == 0 and g.y_stride >= g.w
    assert g.e_stride % 4 == 0 and g.e_stride >= g.wr


def test_host_validation(L):
    P = hqc._Params
    p = P()
    assert L.hqc_get_params(1, ctypes.byref(p)) == 0
    assert L.hqc_get_params(2, ctypes.byref(p)) == -1
    assert L.hqc_get_params(1, None) == -2
    L.hqc_get_params(1, ctypes.byref(p))
    a16 = ctypes.c_void_p(0x1000)
    a8 = ctypes.c_void_p(0x1008)
    # serialized-ciphertext host call: argument checks before any CUDA work
    assert L.hqc_ct_bytes(ctypes.byref(p)) == (p.n + 7) // 8 + p.n12 // 8 == 4417  # S:534 (HQC-1)
    ws = L.hqc_decrypt_ct_host_workspace_bytes(ctypes.byref(p), 64)
    assert L.hqc_decrypt_ct_batch_host(ctypes.byref(p), a16, None, a16, 0, a16, 4, a16, ws, 64, None) == -4
    assert L.hqc_decrypt_ct_batch_host(ctypes.byref(p), a16, None, a16, 2, a16, 4, a16, ws, 64, None) == -4
    assert L.hqc_decrypt_ct_batch_host(ctypes.byref(p), None, None, a16, 1, a16, 4, a16, ws, 64, None) == -2
    assert L.hqc_decrypt_ct_batch_host(ctypes.byref(p), a16, None, a8, 1, a16, 4, a16, ws, 64, None) == -3
    assert L.hqc_decrypt_ct_batch_host(ctypes.byref(p), a16, None, a16, 1, a16, 100, a16, ws - 1, 64, None) == -4
    assert L.hqc_decrypt_ct_batch_host(ctypes.byref(p), None, None, None, 0, None, 0, None, 0, 0, None) == 0
    # KeyGen from seeds: nkeys 0 is a no-op; NULL / misaligned arguments
    assert L.hqc_kem_keygen_batch(ctypes.byref(p), None, None, None, None, None, None, None, 0, None) == 0
    assert L.hqc_kem_keygen_batch(ctypes.byref(p), None, a16, a16, a16, a16, a16, None, 3, None) == -2
    assert L.hqc_kem_keygen_batch(ctypes.byref(p), a16, a16, a16, a16, a16, a16, a8, 3, None) == -3
    # unknown syndrome method
    assert L.hqc_rs_syndromes_batch(ctypes.byref(p), None, None, 0, 3, None) == -4
    assert L.hqc_rs_syndromes_batch(ctypes.byref(p), None, None, 0, 1, None) == 0
    # batch 0 is a no-op even with NULL pointers
    assert L.hqc_decrypt_batch(ctypes.byref(p), None, None, None, None, 0, None) == 0
    assert L.hqc_decrypt_batch(ctypes.byref(p), None, a16, a16, a16, 4, None) == -2
    assert L.hqc_decrypt_batch(ctypes.byref(p), a8, a16, a16, a16, 4, None) == -3
    assert L.hqc_decrypt_batch(ctypes.byref(p), a16, a16, a16, a16, (1 << 31) + 1, None) == -4
    bad = P()
    ctypes.memmove(ctypes.byref(bad), ctypes.byref(p), ctypes.sizeof(P))
    bad.level = 4
    assert L.hqc_decrypt_batch(ctypes.byref(bad), a16, a16, a16, a16, 4, None) == -1
    assert L.hqc_sparse_dense_mul_batch(ctypes.byref(p), a16, a16, a8, a16, 4, None) == -3
    assert L.hqc_rm_decode_batch(ctypes.byref(p), a16, None, 4, None) == -2
    assert L.hqc_rs_decode_batch(ctypes.byref(p), a16, a8, 4, None) == -3
    assert L.hqc_status_str(-5) == b"CUDA launch error"
    # KEM: workspace size is checked before anything is launched
    ws = L.hqc_kem_workspace_bytes(ctypes.byref(p), 4)
    assert ws >= 4 * (p.y_stride * 4 + p.k + 3 * p.e_stride * 4 + 1)
    assert L.hqc_kem_workspace_bytes(ctypes.byref(bad), 4) == 0
    args = [a16] * 10
    assert L.hqc_kem_decaps_batch(ctypes.byref(p), *args[:5], *args[5:9], None, 4, a16, ws - 1, None) == -4
    assert L.hqc_kem_decaps_batch(ctypes.byref(p), *args[:4], a8, *args[5:9], None, 4, a16, ws, None) == -3
    assert L.hqc_kem_encaps_batch(ctypes.byref(p), a16, a16, a16, None, a16, a16, a16, None, 4, a16, ws, None) == -2
    assert L.hqc_kem_encaps_batch(ctypes.byref(p), a16, a16, a16, None, a16, a16, a16, a16, 0, None, 0, None) == 0
    assert L.hqc_kem_hpk_batch(ctypes.byref(p), a16, None, a16, 2, None) == -2


def test_binding_refuses_cpu_tensors(L):
    torch = pytest.importorskip("torch")
    x = torch.zeros(64, dtype=torch.uint8)
    with pytest.raises(hqc.HqcError):
        hqc.hqc_rm_decode_batch(1, x, x)


def test_helper_and_key_index_validation(L):
    """ABI checks added in round 2: the helpers check pointer alignment like
    every entry point; the serialized-ciphertext call rejects a HOST key index >= nkeys with HQC_ERR_SIZE
    before anything is enqueued (it used to clamp it); the binding raises HqcError (not assert) on
    mismatched row counts, so python -O keeps the checks."""
    P = hqc._Params
    p = P()
    L.hqc_get_params(1, ctypes.byref(p))
    a16, a8 = ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1008)
    cnt = ctypes.c_void_p(0x2000)
    assert L.hqc_count_mismatch(ctypes.byref(p), a8, a16, 4, cnt, None) == -3
    assert L.hqc_count_mismatch(ctypes.byref(p), a16, a16, 4, ctypes.c_void_p(0x2008), None) == -3
    assert L.hqc_count_mismatch(ctypes.byref(p), a16, None, 4, cnt, None) == -2
    assert L.hqc_validate_support(ctypes.byref(p), a8, 4, cnt, None) == -3
    assert L.hqc_validate_support(ctypes.byref(p), a16, 4, None, None) == -2
    keys = (ctypes.c_uint32 * 4)(0, 1, 2, 1)
    ws = L.hqc_decrypt_ct_host_workspace_bytes(ctypes.byref(p), 4)
    assert L.hqc_decrypt_ct_batch_host(ctypes.byref(p), a16, keys, a16, 2, a16, 4, a16, ws, 4, None) == -4
    torch = pytest.importorskip("torch")
    ct = torch.zeros(2 * 4417, dtype=torch.uint8)
    m = torch.zeros(3 * 16, dtype=torch.uint8)
    with pytest.raises(hqc.HqcError):  # 2 ciphertexts, 3 output rows: refused before the C call
        hqc.hqc_decrypt_ct_batch_host(1, ct, None, torch.zeros(4 * p.y_stride, dtype=torch.uint8), m,
                                      torch.zeros(16, dtype=torch.uint8))
    with pytest.raises(hqc.HqcError):  # host key index out of range
        hqc.hqc_decrypt_ct_batch_host(1, ct, torch.tensor([0, 5], dtype=torch.int32).view(torch.uint8),
                                      torch.zeros(4 * p.y_stride, dtype=torch.uint8), m[:32],
                                      torch.zeros(16, dtype=torch.uint8))
