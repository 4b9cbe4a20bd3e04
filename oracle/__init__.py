"""ORACLE — test infrastructure only (see oracle/oracle.h for the full header).

A plain, slow CPU implementation of HQC.PKE (Encrypt/Decrypt, the concatenated RS/RM code and the
Eq. 1 ring product) written from /root/reference/PAPER.md, compiled from the C sources in this
directory with plain ``gcc -O2`` into ``oracle/liboracle.so`` and called through ctypes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package. It shares no code with ``paper_2512_12904_b200`` (the CUDA path).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SOURCES = ["params.c", "gf256.c", "ring.c", "rm.c", "rs.c", "pke.c", "shake.c", "kem.c", "batch.c"]


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no -march=native, no vector intrinsics)."""
    srcs = [os.path.join(_HERE, s) for s in _SOURCES] + [os.path.join(_HERE, "oracle.h")]
    if not force and os.path.exists(_SO):
        so_m = os.path.getmtime(_SO)
        if all(os.path.getmtime(s) <= so_m for s in srcs):
            return _SO
    tmp = _SO + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-Wall", "-Wextra", "-o", tmp]
    cmd += [os.path.join(_HERE, s) for s in _SOURCES] + ["-lpthread"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _SO)
    return _SO


class _Params(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32)] + [
        (f, ctypes.c_uint32)
        for f in ("n", "w", "wr", "n1", "k", "d", "delta", "n2", "mult", "dprime", "n12", "words", "vwords")
    ]


@dataclass(frozen=True)
class Params:
    level: int
    n: int
    w: int
    wr: int
    n1: int
    k: int
    d: int
    delta: int
    n2: int
    mult: int
    dprime: int
    n12: int
    words: int
    vwords: int

    def _c(self) -> _Params:
        return _Params(*[getattr(self, f) for f, _ in _Params._fields_])


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        c_p = ctypes.c_void_p
        u8, u32, sz, i32 = ctypes.c_uint8, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_int
        sigs = {
            "orc_get_params": (i32, [i32, P(_Params)]),
            "orc_gf_mul": (u8, [u8, u8]),
            "orc_gf_pow": (u8, [u8, u32]),
            "orc_gf_inv": (u8, [u8]),
            "orc_ring_rotate": (None, [c_p, u32, u32, c_p]),
            "orc_ring_mul_sparse": (None, [c_p, u32, c_p, u32, c_p]),
            "orc_rm_encode": (None, [u8, u32, c_p, u32]),
            "orc_rm_decode": (u8, [c_p, u32, u32]),
            "orc_rm_transform": (None, [c_p, u32, u32, c_p]),
            "orc_rs_encode": (None, [c_p, u32, u32, c_p]),
            "orc_rs_syndromes": (None, [c_p, u32, u32, c_p]),
            "orc_rs_decode": (i32, [c_p, u32, u32, u32, c_p]),
            "orc_rs_decode_ex": (i32, [c_p, u32, u32, u32, c_p, c_p, c_p]),
            "orc_code_encode": (None, [P(_Params), c_p, c_p]),
            "orc_code_decode": (None, [P(_Params), c_p, c_p, c_p]),
            "orc_keygen": (None, [P(_Params), c_p, c_p, c_p, c_p]),
            "orc_encrypt": (None, [P(_Params), c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
            "orc_decrypt_stage1": (None, [P(_Params), c_p, c_p, c_p, c_p]),
            "orc_decrypt": (None, [P(_Params), c_p, c_p, c_p, c_p]),
            "orc_decrypt_batch": (None, [P(_Params), c_p, sz, c_p, sz, c_p, sz, c_p, sz, sz, i32]),
            "orc_stage1_batch": (None, [P(_Params), c_p, sz, c_p, sz, c_p, sz, c_p, sz, sz, i32]),
            "orc_rm_decode_batch": (None, [P(_Params), c_p, sz, c_p, sz, sz, i32]),
            "orc_rs_decode_batch": (None, [P(_Params), c_p, sz, c_p, sz, c_p, sz, i32]),
            "orc_keccak_f1600": (None, [c_p]),
            "orc_shake256": (None, [c_p, sz, c_p, sz]),
            "orc_sample_fixed_weight": (None, [c_p, u32, u32, c_p]),
            "orc_kem_hpk": (None, [P(_Params), c_p, c_p, c_p]),
            "orc_kem_coins": (None, [P(_Params), c_p, c_p, c_p, c_p, c_p]),
            "orc_kem_encaps": (None, [P(_Params), c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
            "orc_kem_keygen": (None, [P(_Params), c_p, c_p, c_p, c_p, c_p, c_p]),
            "orc_kem_decaps": (i32, [P(_Params), c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
            "orc_kem_decaps_batch": (None, [P(_Params), c_p, c_p, sz, c_p, c_p, c_p, c_p, sz, c_p, sz, c_p, sz, c_p,
                                            c_p, sz, i32]),
            "orc_encrypt_batch": (
                None,
                [P(_Params), c_p, sz, c_p, sz, c_p, c_p, sz, c_p, c_p, c_p, sz, c_p, sz, c_p, sz, sz, i32],
            ),
        }
        for name, (res, args) in sigs.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def params(level: int) -> Params:
    p = _Params()
    if lib().orc_get_params(level, ctypes.byref(p)) != 0:
        raise ValueError(f"unknown HQC level {level}")
    return Params(*[getattr(p, f) for f, _ in _Params._fields_])


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the oracle must be C-contiguous"
    return a.ctypes.data


def _threads(n: int | None) -> int:
    return int(n) if n else (os.cpu_count() or 1)


# ---------------- GF(2^8) ----------------
def gf_mul(a: int, b: int) -> int:
    return lib().orc_gf_mul(a, b)


def gf_pow(a: int, e: int) -> int:
    return lib().orc_gf_pow(a, e)


def gf_inv(a: int) -> int:
    return lib().orc_gf_inv(a)


# ---------------- ring ----------------
def ring_rotate(a: np.ndarray, n: int, i: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.zeros((n + 63) // 64, dtype=np.uint64)
    lib().orc_ring_rotate(_ptr(a), n, i, _ptr(out))
    return out


def ring_mul_sparse(a: np.ndarray, n: int, supp) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    s = np.ascontiguousarray(np.asarray(supp, dtype=np.uint32))
    out = np.zeros((n + 63) // 64, dtype=np.uint64)
    lib().orc_ring_mul_sparse(_ptr(a), n, _ptr(s) if s.size else None, s.size, _ptr(out))
    return out


# ---------------- RM ----------------
def rm_encode(b: int, mult: int) -> np.ndarray:
    out = np.zeros(2 * mult, dtype=np.uint64)
    lib().orc_rm_encode(b, mult, _ptr(out), 0)
    return out


def rm_decode(block: np.ndarray, mult: int, off: int = 0) -> int:
    block = np.ascontiguousarray(block, dtype=np.uint64)
    return lib().orc_rm_decode(_ptr(block), off, mult)


def rm_transform(block: np.ndarray, mult: int, off: int = 0) -> np.ndarray:
    block = np.ascontiguousarray(block, dtype=np.uint64)
    F = np.zeros(128, dtype=np.int32)
    lib().orc_rm_transform(_ptr(block), off, mult, _ptr(F))
    return F


# ---------------- RS ----------------
def rs_encode(msg, n1: int, k: int) -> np.ndarray:
    m = np.ascontiguousarray(np.asarray(msg, dtype=np.uint8))
    assert m.size == k
    cw = np.zeros(n1, dtype=np.uint8)
    lib().orc_rs_encode(_ptr(m), n1, k, _ptr(cw))
    return cw


def rs_syndromes(r, n1: int, delta: int) -> np.ndarray:
    r = np.ascontiguousarray(np.asarray(r, dtype=np.uint8))
    S = np.zeros(2 * delta, dtype=np.uint8)
    lib().orc_rs_syndromes(_ptr(r), n1, delta, _ptr(S))
    return S


def rs_decode(r, n1: int, k: int, delta: int, full: bool = False):
    r = np.ascontiguousarray(np.asarray(r, dtype=np.uint8))
    out = np.zeros(k, dtype=np.uint8)
    L = ctypes.c_uint32(0)
    lam = np.zeros(2 * delta + 1, dtype=np.uint8)
    ok = lib().orc_rs_decode_ex(_ptr(r), n1, k, delta, _ptr(out), ctypes.byref(L), _ptr(lam))
    if full:
        return out, bool(ok), int(L.value), lam
    return out, bool(ok)


# ---------------- code / PKE (single) ----------------
def code_encode(p: Params, msg) -> np.ndarray:
    m = np.ascontiguousarray(np.asarray(msg, dtype=np.uint8))
    out = np.zeros(p.vwords, dtype=np.uint64)
    lib().orc_code_encode(ctypes.byref(p._c()), _ptr(m), _ptr(out))
    return out


def code_decode(p: Params, vec: np.ndarray):
    vec = np.ascontiguousarray(vec, dtype=np.uint64)
    m = np.zeros(p.k, dtype=np.uint8)
    sym = np.zeros(p.n1, dtype=np.uint8)
    lib().orc_code_decode(ctypes.byref(p._c()), _ptr(vec), _ptr(m), _ptr(sym))
    return m, sym


def keygen(p: Params, h: np.ndarray, x, y) -> np.ndarray:
    h = np.ascontiguousarray(h[: p.words], dtype=np.uint64)
    x = np.ascontiguousarray(np.asarray(x, dtype=np.uint32)[: p.w])
    y = np.ascontiguousarray(np.asarray(y, dtype=np.uint32)[: p.w])
    s = np.zeros(p.words, dtype=np.uint64)
    lib().orc_keygen(ctypes.byref(p._c()), _ptr(h), _ptr(x), _ptr(y), _ptr(s))
    return s


def encrypt(p: Params, h, s, m, r1, r2, e):
    args = [
        np.ascontiguousarray(h[: p.words], dtype=np.uint64),
        np.ascontiguousarray(s[: p.words], dtype=np.uint64),
        np.ascontiguousarray(np.asarray(m, dtype=np.uint8)[: p.k]),
        np.ascontiguousarray(np.asarray(r1, dtype=np.uint32)[: p.wr]),
        np.ascontiguousarray(np.asarray(r2, dtype=np.uint32)[: p.wr]),
        np.ascontiguousarray(np.asarray(e, dtype=np.uint32)[: p.wr]),
    ]
    u = np.zeros(p.words, dtype=np.uint64)
    v = np.zeros(p.vwords, dtype=np.uint64)
    lib().orc_encrypt(ctypes.byref(p._c()), *[_ptr(a) for a in args], _ptr(u), _ptr(v))
    return u, v


def decrypt_stage1(p: Params, u, v, y) -> np.ndarray:
    u = np.ascontiguousarray(u[: p.words], dtype=np.uint64)
    v = np.ascontiguousarray(v[: p.vwords], dtype=np.uint64)
    y = np.ascontiguousarray(np.asarray(y, dtype=np.uint32)[: p.w])
    r = np.zeros(p.vwords, dtype=np.uint64)
    lib().orc_decrypt_stage1(ctypes.byref(p._c()), _ptr(u), _ptr(v), _ptr(y), _ptr(r))
    return r


def decrypt(p: Params, u, v, y) -> np.ndarray:
    u = np.ascontiguousarray(u[: p.words], dtype=np.uint64)
    v = np.ascontiguousarray(v[: p.vwords], dtype=np.uint64)
    y = np.ascontiguousarray(np.asarray(y, dtype=np.uint32)[: p.w])
    m = np.zeros(p.k, dtype=np.uint8)
    lib().orc_decrypt(ctypes.byref(p._c()), _ptr(u), _ptr(v), _ptr(y), _ptr(m))
    return m


# ---------------- batched (row-strided 2-D arrays) ----------------
def _rows(a: np.ndarray, dtype) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=dtype)
    assert a.ndim == 2
    return a


def decrypt_batch(p: Params, u, v, y, nthreads: int | None = None) -> np.ndarray:
    u, v, y = _rows(u, np.uint64), _rows(v, np.uint64), _rows(y, np.uint32)
    B = u.shape[0]
    assert v.shape[0] == B and y.shape[0] == B
    assert u.shape[1] >= p.words and v.shape[1] >= p.vwords and y.shape[1] >= p.w
    m = np.zeros((B, p.k), dtype=np.uint8)
    lib().orc_decrypt_batch(ctypes.byref(p._c()), _ptr(u), u.shape[1], _ptr(v), v.shape[1], _ptr(y),
                            y.shape[1], _ptr(m), p.k, B, _threads(nthreads))
    return m


def stage1_batch(p: Params, u, v, y, nthreads: int | None = None) -> np.ndarray:
    u, v, y = _rows(u, np.uint64), _rows(v, np.uint64), _rows(y, np.uint32)
    B = u.shape[0]
    r = np.zeros((B, p.vwords), dtype=np.uint64)
    lib().orc_stage1_batch(ctypes.byref(p._c()), _ptr(u), u.shape[1], _ptr(v), v.shape[1], _ptr(y),
                           y.shape[1], _ptr(r), p.vwords, B, _threads(nthreads))
    return r


def rm_decode_batch(p: Params, r, nthreads: int | None = None) -> np.ndarray:
    r = _rows(r, np.uint64)
    B = r.shape[0]
    sym = np.zeros((B, p.n1), dtype=np.uint8)
    lib().orc_rm_decode_batch(ctypes.byref(p._c()), _ptr(r), r.shape[1], _ptr(sym), p.n1, B,
                              _threads(nthreads))
    return sym


def rs_decode_batch(p: Params, sym, nthreads: int | None = None):
    sym = _rows(sym, np.uint8)
    B = sym.shape[0]
    m = np.zeros((B, p.k), dtype=np.uint8)
    ok = np.zeros(B, dtype=np.uint8)
    lib().orc_rs_decode_batch(ctypes.byref(p._c()), _ptr(sym), sym.shape[1], _ptr(m), p.k, _ptr(ok), B,
                              _threads(nthreads))
    return m, ok


def encrypt_batch(p: Params, h, s, key_of_row, m, r1, r2, e, nthreads: int | None = None):
    h, s = _rows(h, np.uint64), _rows(s, np.uint64)
    key_of_row = np.ascontiguousarray(key_of_row, dtype=np.int64)
    m = _rows(m, np.uint8)
    r1, r2, e = _rows(r1, np.uint32), _rows(r2, np.uint32), _rows(e, np.uint32)
    assert r1.shape == r2.shape == e.shape
    B = m.shape[0]
    u = np.zeros((B, p.words), dtype=np.uint64)
    v = np.zeros((B, p.vwords), dtype=np.uint64)
    lib().orc_encrypt_batch(ctypes.byref(p._c()), _ptr(h), h.shape[1], _ptr(s), s.shape[1],
                            _ptr(key_of_row), _ptr(m), m.shape[1], _ptr(r1), _ptr(r2), _ptr(e),
                            r1.shape[1], _ptr(u), p.words, _ptr(v), p.vwords, B, _threads(nthreads))
    return u, v


# ---------------- KEM row (SHAKE256, sampler, HHK) ----------------
def shake256(msg: bytes, outlen: int) -> bytes:
    m = np.frombuffer(bytes(msg), dtype=np.uint8).copy() if len(msg) else np.zeros(1, np.uint8)
    out = np.zeros(max(outlen, 1), np.uint8)
    lib().orc_shake256(_ptr(m), len(msg), _ptr(out), outlen)
    return out[:outlen].tobytes()


def keccak_f1600(state) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(state, dtype=np.uint64).copy())
    lib().orc_keccak_f1600(_ptr(a))
    return a


def sample_fixed_weight(rnd: bytes, n: int, w: int) -> np.ndarray:
    r = np.frombuffer(bytes(rnd), dtype=np.uint8).copy()
    assert r.size >= 4 * w
    out = np.zeros(w, np.uint32)
    lib().orc_sample_fixed_weight(_ptr(r), n, w, _ptr(out))
    return out


def kem_hpk(p: Params, h, s) -> bytes:
    h = np.ascontiguousarray(h[: p.words], dtype=np.uint64)
    s = np.ascontiguousarray(s[: p.words], dtype=np.uint64)
    out = np.zeros(32, np.uint8)
    lib().orc_kem_hpk(ctypes.byref(p._c()), _ptr(h), _ptr(s), _ptr(out))
    return out.tobytes()


def kem_coins(p: Params, hpk: bytes, m):
    hp = np.frombuffer(hpk, np.uint8).copy()
    m = np.ascontiguousarray(np.asarray(m, dtype=np.uint8)[: p.k])
    r = np.zeros((3, p.wr), np.uint32)
    lib().orc_kem_coins(ctypes.byref(p._c()), _ptr(hp), _ptr(m), _ptr(r[0]), _ptr(r[1]), _ptr(r[2]))
    return r[0], r[1], r[2]


def kem_encaps(p: Params, h, s, hpk: bytes, m):
    h = np.ascontiguousarray(h[: p.words], dtype=np.uint64)
    s = np.ascontiguousarray(s[: p.words], dtype=np.uint64)
    hp = np.frombuffer(hpk, np.uint8).copy()
    m = np.ascontiguousarray(np.asarray(m, dtype=np.uint8)[: p.k])
    u = np.zeros(p.words, np.uint64)
    v = np.zeros(p.vwords, np.uint64)
    K = np.zeros(64, np.uint8)
    lib().orc_kem_encaps(ctypes.byref(p._c()), _ptr(h), _ptr(s), _ptr(hp), _ptr(m), _ptr(u), _ptr(v), _ptr(K))
    return u, v, K.tobytes()


def kem_keygen(p: Params, seed: bytes):
    """KeyGen from a 32-byte seed (R#24): returns h (words), x, y (w positions), s (words), sigma (k bytes)."""
    sd = np.frombuffer(bytes(seed), np.uint8).copy()
    assert sd.size == 32
    h = np.zeros(p.words, np.uint64)
    s = np.zeros(p.words, np.uint64)
    x = np.zeros(p.w, np.uint32)
    y = np.zeros(p.w, np.uint32)
    sigma = np.zeros(p.k, np.uint8)
    lib().orc_kem_keygen(ctypes.byref(p._c()), _ptr(sd), _ptr(h), _ptr(x), _ptr(y), _ptr(s), _ptr(sigma))
    return h, x, y, s, sigma


def kem_decaps(p: Params, h, s, hpk: bytes, y, sigma, u, v):
    h = np.ascontiguousarray(h[: p.words], dtype=np.uint64)
    s = np.ascontiguousarray(s[: p.words], dtype=np.uint64)
    hp = np.frombuffer(hpk, np.uint8).copy()
    y = np.ascontiguousarray(np.asarray(y, dtype=np.uint32)[: p.w])
    sg = np.ascontiguousarray(np.asarray(sigma, dtype=np.uint8)[: p.k])
    u = np.ascontiguousarray(u[: p.words], dtype=np.uint64)
    v = np.ascontiguousarray(v[: p.vwords], dtype=np.uint64)
    K = np.zeros(64, np.uint8)
    ok = lib().orc_kem_decaps(ctypes.byref(p._c()), _ptr(h), _ptr(s), _ptr(hp), _ptr(y), _ptr(sg), _ptr(u), _ptr(v),
                              _ptr(K))
    return K.tobytes(), bool(ok)


def kem_decaps_batch(p: Params, h, s, hpk, sigma, key_of_row, y, u, v, nthreads=None):
    h, s = _rows(h, np.uint64), _rows(s, np.uint64)
    assert h.shape == s.shape
    hpk = np.ascontiguousarray(hpk, dtype=np.uint8)
    sigma = np.ascontiguousarray(sigma, dtype=np.uint8)
    assert sigma.shape[1] == p.k and hpk.shape[1] == 32
    key_of_row = np.ascontiguousarray(key_of_row, dtype=np.int64)
    y, u, v = _rows(y, np.uint32), _rows(u, np.uint64), _rows(v, np.uint64)
    B = u.shape[0]
    K = np.zeros((B, 64), np.uint8)
    acc = np.zeros(B, np.uint8)
    lib().orc_kem_decaps_batch(ctypes.byref(p._c()), _ptr(h), _ptr(s), h.shape[1], _ptr(hpk), _ptr(sigma),
                               _ptr(key_of_row), _ptr(y), y.shape[1], _ptr(u), u.shape[1], _ptr(v), v.shape[1],
                               _ptr(K), _ptr(acc), B, _threads(nthreads))
    return K, acc
