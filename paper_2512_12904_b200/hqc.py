"""Thin Python binding of libhqcgpu.so (include/hqc_gpu.h): argument marshalling only.

Every function takes torch CUDA tensors (any dtype view of the documented layout), passes their
device pointers and the current torch stream to the C ABI, and raises on a nonzero status. All
compute happens in the library's sm_100a kernels; there is no CPU or PyTorch fallback — a missing
library raises ImportError-like RuntimeError at first use.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhqcgpu.so")


class HqcError(RuntimeError):
    pass


class _Params(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32)] + [
        (f, ctypes.c_uint32)
        for f in ("n", "n1", "n2", "mult", "k", "delta", "w", "wr", "n12", "u_words", "u_stride", "v_words",
                  "y_stride", "e_stride")
    ]


@dataclass(frozen=True)
class Params:
    level: int
    n: int
    n1: int
    n2: int
    mult: int
    k: int
    delta: int
    w: int
    wr: int
    n12: int
    u_words: int
    u_stride: int
    v_words: int
    y_stride: int
    e_stride: int


_lib = None
_cparams: dict[int, _Params] = {}


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise HqcError(f"{LIB_PATH} is missing: build it with `python -m paper_2512_12904_b200.build` "
                           "(or __graft_entry__.build()); there is no fallback path")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
        P = ctypes.POINTER(_Params)
        sigs = {
            "hqc_get_params": [i32, P],
            "hqc_decrypt_batch": [P, vp, vp, vp, vp, sz, vp],
            "hqc_sparse_dense_mul_batch": [P, vp, vp, vp, vp, sz, vp],
            "hqc_rm_decode_batch": [P, vp, vp, sz, vp],
            "hqc_rs_decode_batch": [P, vp, vp, sz, vp],
            "hqc_rs_decode_batch_ex": [P, vp, vp, vp, sz, vp],
            "hqc_rs_syndromes_batch": [P, vp, vp, sz, i32, vp],
            "hqc_count_mismatch": [P, vp, vp, sz, vp, vp],
            "hqc_validate_support": [P, vp, sz, vp, vp],
            "hqc_decrypt_launch_shape": [P, sz, ctypes.POINTER(i32), ctypes.POINTER(i32)],
            "hqc_decrypt_launch_kernel": [P, sz],
            "hqc_keygen_batch": [P, vp, vp, vp, vp, sz, vp],
            "hqc_encrypt_batch": [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp],
            "hqc_kem_hpk_batch": [P, vp, vp, vp, sz, vp],
            "hqc_kem_keygen_batch": [P, vp, vp, vp, vp, vp, vp, vp, sz, vp],
            "hqc_kem_encaps_batch": [P, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, sz, vp],
            "hqc_kem_decaps_batch": [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, sz, vp],
        }
        for name, args in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = i32
        L.hqc_kem_workspace_bytes.argtypes = [P, sz]
        L.hqc_kem_workspace_bytes.restype = sz
        L.hqc_decrypt_host_workspace_bytes.argtypes = [P, sz]
        L.hqc_decrypt_host_workspace_bytes.restype = sz
        L.hqc_decrypt_batch_host.argtypes = [P, vp, vp, vp, vp, sz, vp, sz, sz, vp]
        L.hqc_decrypt_batch_host.restype = i32
        L.hqc_ct_bytes.argtypes = [P]
        L.hqc_ct_bytes.restype = sz
        L.hqc_decrypt_ct_host_workspace_bytes.argtypes = [P, sz]
        L.hqc_decrypt_ct_host_workspace_bytes.restype = sz
        L.hqc_decrypt_ct_batch_host.argtypes = [P, vp, vp, vp, sz, vp, sz, vp, sz, sz, vp]
        L.hqc_decrypt_ct_batch_host.restype = i32
        L.hqc_decrypt_launch_count.argtypes = [P, sz]
        L.hqc_decrypt_launch_count.restype = ctypes.c_longlong
        L.hqc_status_str.argtypes = [i32]
        L.hqc_status_str.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _cp(level: int) -> _Params:
    if level not in _cparams:
        p = _Params()
        _check(lib().hqc_get_params(level, ctypes.byref(p)))
        _cparams[level] = p
    return _cparams[level]


def params(level: int) -> Params:
    p = _cp(level)
    return Params(*[getattr(p, f) for f, _ in _Params._fields_])


def _check(status: int):
    if status != 0:
        raise HqcError(f"libhqcgpu: {lib().hqc_status_str(status).decode()} (status {status})")


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise HqcError("libhqcgpu entry points take CUDA tensors (device pointers)")
    if not t.is_contiguous():
        raise HqcError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need(cond: bool, msg: str) -> None:
    """Argument check that survives python -O (unlike assert)."""
    if not cond:
        raise HqcError(msg)


def _keys_in_range(key_index, nkeys: int, batch: int, check: bool) -> None:
    """key_index (None: row i uses key i) must address rows of the per-key tables: the kernels index them
    without a bound (the C ABI has no key count), so an out-of-range index would read out of bounds. On a
    CUDA tensor the check costs one reduction and a synchronisation; check=False skips it."""
    if key_index is None:
        _need(batch <= nkeys, f"no key_index: {batch} rows need {batch} keys, got {nkeys}")
        return
    _need(_rows(key_index, 4, "key_index") == batch, "key_index: one uint32 per row")
    if check and batch:
        import torch

        k = key_index.view(torch.int32) if key_index.dtype != torch.int32 else key_index
        lo, hi = int(k.min().item()), int(k.max().item())
        _need(0 <= lo and hi < nkeys, f"key_index out of range [0, {nkeys}): min {lo}, max {hi}")


def _rows(t, row_bytes: int, name: str) -> int:
    nbytes = t.numel() * t.element_size()
    if nbytes % row_bytes:
        raise HqcError(f"{name}: {nbytes} bytes is not a whole number of {row_bytes}-byte rows")
    return nbytes // row_bytes


def hqc_decrypt_batch(level: int, u, v, y_support, m_out, stream=None) -> None:
    """m_out[b] = C.Decode(v[b] ^ trunc(u[b] * y[b])) — the fused kernel."""
    p = params(level)
    B = _rows(u, 8 * p.u_stride, "u")
    _need(_rows(v, 8 * p.v_words, "v") == B and _rows(y_support, 4 * p.y_stride, "y") == B, "row counts of the arguments disagree")
    _need(_rows(m_out, p.k, "m_out") == B, "row counts of the arguments disagree")
    _check(lib().hqc_decrypt_batch(ctypes.byref(_cp(level)), _ptr(u), _ptr(v), _ptr(y_support), _ptr(m_out), B,
                                   _stream(stream)))


def hqc_sparse_dense_mul_batch(level: int, u, y_support, v, r_out, stream=None) -> None:
    p = params(level)
    B = _rows(u, 8 * p.u_stride, "u")
    _need(_rows(r_out, 8 * p.v_words, "r_out") == B, "row counts of the arguments disagree")
    _check(lib().hqc_sparse_dense_mul_batch(ctypes.byref(_cp(level)), _ptr(u), _ptr(y_support), _ptr(v),
                                            _ptr(r_out), B, _stream(stream)))


def hqc_rm_decode_batch(level: int, r, sym_out, stream=None) -> None:
    p = params(level)
    B = _rows(r, 8 * p.v_words, "r")
    _need(_rows(sym_out, p.n1, "sym_out") == B, "row counts of the arguments disagree")
    _check(lib().hqc_rm_decode_batch(ctypes.byref(_cp(level)), _ptr(r), _ptr(sym_out), B, _stream(stream)))


def hqc_rs_decode_batch(level: int, sym, m_out, ok_out=None, stream=None) -> None:
    p = params(level)
    B = _rows(sym, p.n1, "sym")
    _need(_rows(m_out, p.k, "m_out") == B, "row counts of the arguments disagree")
    _check(lib().hqc_rs_decode_batch_ex(ctypes.byref(_cp(level)), _ptr(sym), _ptr(m_out), _ptr(ok_out), B,
                                        _stream(stream)))


SYN_METHODS = {"linear": 0, "nibble": 1, "logexp": 2}


def hqc_rs_syndromes_batch(level: int, sym, syn_out, method: str = "linear", stream=None) -> None:
    """S_1..S_2delta of each received word (step a6); method: linear | nibble | logexp."""
    p = params(level)
    B = _rows(sym, p.n1, "sym")
    _need(_rows(syn_out, 2 * p.delta, "syn_out") == B, "row counts of the arguments disagree")
    _check(lib().hqc_rs_syndromes_batch(ctypes.byref(_cp(level)), _ptr(sym), _ptr(syn_out), B, SYN_METHODS[method],
                                        _stream(stream)))


def hqc_count_mismatch(level: int, m_out, m_ref, d_count, stream=None) -> None:
    p = params(level)
    B = _rows(m_out, p.k, "m_out")
    _check(lib().hqc_count_mismatch(ctypes.byref(_cp(level)), _ptr(m_out), _ptr(m_ref), B, _ptr(d_count),
                                    _stream(stream)))


def hqc_validate_support(level: int, y_support, d_bad, stream=None) -> None:
    p = params(level)
    B = _rows(y_support, 4 * p.y_stride, "y")
    _check(lib().hqc_validate_support(ctypes.byref(_cp(level)), _ptr(y_support), B, _ptr(d_bad),
                                      _stream(stream)))


def hqc_decrypt_launch_shape(level: int, batch: int) -> tuple[int, int]:
    g, w = ctypes.c_int(0), ctypes.c_int(0)
    _check(lib().hqc_decrypt_launch_shape(ctypes.byref(_cp(level)), batch, ctypes.byref(g), ctypes.byref(w)))
    return g.value, w.value


KERNEL_NAMES = {1: "k_decrypt_w1 (fused, one warp per ciphertext range, lane-per-word RS)",
                2: "k_decrypt (fused, warp pair)", 3: "k_decrypt_ws (fused, warp-specialised)",
                4: "k_decrypt_t (fused, tensor-memory product)",
                5: "k_decrypt_sb (fused, one warp per ciphertext, warp-parallel RS)",
                6: "k_decrypt_wd (fused, chunks of 32 per warp, CTA-shared work counter, lane-per-word RS)",
                7: "k_decrypt_sp (fused, warp pair per ciphertext, small batches)",
                8: "k_decrypt_wl (fused, compact warps: v above u in E, chunks of 32, lane-per-word RS)",
                9: "k_decrypt_wl<static> (fused, compact warps, per-warp contiguous ranges)",
                10: "k_decrypt_s12 + k_stage3 (stages 1+2, symbols via HBM, lane-per-word RS: two launches)",
                11: "k_decrypt_s12c + k_stage3 (compact stages 1+2: r above u in E, v from L2; symbols via HBM, "
                    "lane-per-word RS: two launches)",
                12: "k_decrypt_wc (fused, compact warps, RS chunks of 32 consecutive ciphertexts shared by the CTA, "
                    "lane-per-word RS)"}


def hqc_decrypt_launch_kernel(level: int, batch: int) -> int:
    """Which fused kernel hqc_decrypt_batch launches for `batch` (KERNEL_NAMES)."""
    k = int(lib().hqc_decrypt_launch_kernel(ctypes.byref(_cp(level)), batch))
    _check(min(k, 0))
    return k


def hqc_decrypt_launch_count(level: int, batch: int) -> int:
    """How many kernel launches hqc_decrypt_batch makes for `batch`."""
    n = int(lib().hqc_decrypt_launch_count(ctypes.byref(_cp(level)), batch))
    _check(min(n, 0))
    return n


def hqc_keygen_batch(level: int, h, x, y, s_out, stream=None) -> None:
    """s = x + h*y per key (Alg. 3)."""
    p = params(level)
    K = _rows(h, 8 * p.u_stride, "h")
    _need(_rows(x, 4 * p.y_stride, "x") == K and _rows(y, 4 * p.y_stride, "y") == K, "row counts of the arguments disagree")
    _need(_rows(s_out, 8 * p.u_stride, "s_out") == K, "row counts of the arguments disagree")
    _check(lib().hqc_keygen_batch(ctypes.byref(_cp(level)), _ptr(h), _ptr(x), _ptr(y), _ptr(s_out), K,
                                  _stream(stream)))


def hqc_encrypt_batch(level: int, h, s, key_index, m, r1, r2, e, u_out, v_out, stream=None,
                      check_keys: bool = True) -> None:
    """u = r1 + h*r2, v = trunc(mG + s*r2 + e) per ciphertext (Alg. 1); key_index may be None."""
    p = params(level)
    B = _rows(m, p.k, "m")
    nk = _rows(h, 8 * p.u_stride, "h")
    _need(_rows(s, 8 * p.u_stride, "s") == nk, "h and s: one row per key each")
    _keys_in_range(key_index, nk, B, check_keys)
    for t, nm in ((r1, "r1"), (r2, "r2"), (e, "e")):
        _need(_rows(t, 4 * p.e_stride, nm) == B, "row counts of the arguments disagree")
    _need(_rows(u_out, 8 * p.u_stride, "u_out") == B and _rows(v_out, 8 * p.v_words, "v_out") == B, "row counts of the arguments disagree")
    _check(lib().hqc_encrypt_batch(ctypes.byref(_cp(level)), _ptr(h), _ptr(s), _ptr(key_index), _ptr(m), _ptr(r1),
                                   _ptr(r2), _ptr(e), _ptr(u_out), _ptr(v_out), B, _stream(stream)))


def hqc_kem_workspace_bytes(level: int, batch: int) -> int:
    return int(lib().hqc_kem_workspace_bytes(ctypes.byref(_cp(level)), batch))


def _nbytes(t) -> int:
    return t.numel() * t.element_size()


def hqc_kem_hpk_batch(level: int, h, s, hpk_out, stream=None) -> None:
    """H_pk = SHAKE256(h bytes || s bytes || 0x02, 32) per key (R#20-R#21)."""
    p = params(level)
    K = _rows(h, 8 * p.u_stride, "h")
    _need(_rows(s, 8 * p.u_stride, "s") == K and _rows(hpk_out, 32, "hpk_out") == K, "row counts of the arguments disagree")
    _check(lib().hqc_kem_hpk_batch(ctypes.byref(_cp(level)), _ptr(h), _ptr(s), _ptr(hpk_out), K, _stream(stream)))


def hqc_kem_keygen_batch(level: int, seeds, h_out, x_out, y_out, s_out, sigma_out, hpk_out=None, stream=None) -> None:
    """KeyGen from 32-byte seeds (R#24): h, x, y, sigma by SHAKE256 expansion, s = x + h*y, H_pk."""
    p = params(level)
    K = _rows(seeds, 32, "seeds")
    _need(_rows(h_out, 8 * p.u_stride, "h_out") == K and _rows(s_out, 8 * p.u_stride, "s_out") == K, "row counts of the arguments disagree")
    _need(_rows(x_out, 4 * p.y_stride, "x_out") == K and _rows(y_out, 4 * p.y_stride, "y_out") == K, "row counts of the arguments disagree")
    _need(_rows(sigma_out, p.k, "sigma_out") == K, "row counts of the arguments disagree")
    if hpk_out is not None:
        _need(_rows(hpk_out, 32, "hpk_out") == K, "row counts of the arguments disagree")
    _check(lib().hqc_kem_keygen_batch(ctypes.byref(_cp(level)), _ptr(seeds), _ptr(h_out), _ptr(x_out), _ptr(y_out),
                                      _ptr(s_out), _ptr(sigma_out), _ptr(hpk_out), K, _stream(stream)))


def hqc_kem_encaps_batch(level: int, h, s, hpk, key_index, m, u_out, v_out, K_out, workspace, stream=None,
                         check_keys: bool = True) -> None:
    """HHK Encaps with caller-drawn messages m: coins(H_pk, m) -> Encrypt -> K (R#20-R#23)."""
    p = params(level)
    B = _rows(m, p.k, "m")
    nk = _rows(h, 8 * p.u_stride, "h")
    _need(_rows(s, 8 * p.u_stride, "s") == nk and _rows(hpk, 32, "hpk") == nk, "h, s, hpk: one row per key each")
    _keys_in_range(key_index, nk, B, check_keys)
    _need(_rows(u_out, 8 * p.u_stride, "u_out") == B and _rows(v_out, 8 * p.v_words, "v_out") == B, "row counts of the arguments disagree")
    _need(_rows(K_out, 64, "K_out") == B, "row counts of the arguments disagree")
    _check(lib().hqc_kem_encaps_batch(ctypes.byref(_cp(level)), _ptr(h), _ptr(s), _ptr(hpk), _ptr(key_index), _ptr(m),
                                      _ptr(u_out), _ptr(v_out), _ptr(K_out), B, _ptr(workspace), _nbytes(workspace),
                                      _stream(stream)))


def hqc_kem_decaps_batch(level: int, h, s, hpk, sigma, key_index, y_support, u, v, K_out, accepted_out, workspace,
                         stream=None, check_keys: bool = True) -> None:
    """HHK Decaps with implicit rejection: Decrypt -> coins -> re-encrypt and compare -> K (R#20-R#23).
    h, s, hpk, sigma, y_support are per KEY; key_index (None = identity) maps rows to keys."""
    p = params(level)
    B = _rows(u, 8 * p.u_stride, "u")
    nk = _rows(h, 8 * p.u_stride, "h")
    _need(_rows(s, 8 * p.u_stride, "s") == nk and _rows(hpk, 32, "hpk") == nk and _rows(sigma, p.k, "sigma") >= nk
          and _rows(y_support, 4 * p.y_stride, "y_support") == nk, "h, s, hpk, sigma, y_support: one row per key each")
    _keys_in_range(key_index, nk, B, check_keys)
    _need(_rows(v, 8 * p.v_words, "v") == B and _rows(K_out, 64, "K_out") == B, "row counts of the arguments disagree")
    _check(lib().hqc_kem_decaps_batch(ctypes.byref(_cp(level)), _ptr(h), _ptr(s), _ptr(hpk), _ptr(sigma),
                                      _ptr(key_index), _ptr(y_support), _ptr(u), _ptr(v), _ptr(K_out),
                                      _ptr(accepted_out), B, _ptr(workspace), _nbytes(workspace), _stream(stream)))


def hqc_decrypt_host_workspace_bytes(level: int, chunk: int) -> int:
    return int(lib().hqc_decrypt_host_workspace_bytes(ctypes.byref(_cp(level)), chunk))


def _hptr(t):
    if t.is_cuda:
        raise HqcError("hqc_decrypt_batch_host takes host (CPU) tensors for u, v, y, m")
    if not t.is_contiguous():
        raise HqcError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def hqc_decrypt_batch_host(level: int, u, v, y_support, m_out, workspace, chunk: int = 0, stream=None) -> None:
    """The end-to-end call: host (ideally pinned) u, v, y in, host m out; the library pipelines the
    copies and the fused kernel over two internal streams. workspace: a CUDA tensor of at least
    hqc_decrypt_host_workspace_bytes(level, chunk) bytes."""
    p = params(level)
    B = _rows(u, 8 * p.u_stride, "u")
    _need(_rows(v, 8 * p.v_words, "v") == B and _rows(y_support, 4 * p.y_stride, "y") == B, "row counts of the arguments disagree")
    _need(_rows(m_out, p.k, "m_out") == B, "row counts of the arguments disagree")
    wb = workspace.numel() * workspace.element_size()
    _check(lib().hqc_decrypt_batch_host(ctypes.byref(_cp(level)), _hptr(u), _hptr(v), _hptr(y_support), _hptr(m_out),
                                        B, _ptr(workspace), wb, chunk, _stream(stream)))


def hqc_ct_bytes(level: int) -> int:
    """Serialized ciphertext size: ceil(n/8) + n1*n2/8 bytes."""
    return int(lib().hqc_ct_bytes(ctypes.byref(_cp(level))))


def hqc_decrypt_ct_host_workspace_bytes(level: int, chunk: int) -> int:
    return int(lib().hqc_decrypt_ct_host_workspace_bytes(ctypes.byref(_cp(level)), chunk))


def hqc_decrypt_ct_batch_host(level: int, ct, key_index, y_keys, m_out, workspace, chunk: int = 0,
                              stream=None) -> None:
    """The server-side end-to-end call: host serialized ciphertexts (+ host key indices, None when there
    is one key) in, host m out; y_keys is the device-resident [nkeys][y_stride] key-support table."""
    p = params(level)
    B = _rows(ct, hqc_ct_bytes(level), "ct")
    _need(_rows(m_out, p.k, "m_out") == B, "row counts of the arguments disagree")
    nk = _rows(y_keys, 4 * p.y_stride, "y_keys")
    _keys_in_range(key_index, nk, B, True) if key_index is not None else _need(nk >= 1, "y_keys: at least one key")
    wb = workspace.numel() * workspace.element_size()
    _check(lib().hqc_decrypt_ct_batch_host(ctypes.byref(_cp(level)), _hptr(ct),
                                           None if key_index is None else _hptr(key_index), _ptr(y_keys), nk,
                                           _hptr(m_out), B, _ptr(workspace), wb, chunk, _stream(stream)))
