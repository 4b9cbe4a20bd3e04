"""Seeded synthetic input generator, shared by the tests and bench.py.

Holds none of the method's arithmetic: only counter-based draws (hqcgen.c) plus plain array
bookkeeping (which key a ciphertext uses, overwriting whole RM blocks of v with random words for
the adversarial config). Sizes (n, w, ...) are passed in by the caller; this module keeps no
parameter tables.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libhqcgen.so")

# stream tags: one independent stream family per kind of draw
TAG_H, TAG_X, TAG_Y, TAG_R1, TAG_R2, TAG_E, TAG_M = 1, 2, 3, 4, 5, 6, 7
TAG_ADV_BLOCKS, TAG_ADV_BITS, TAG_U_RAND, TAG_V_RAND = 8, 9, 10, 11
TAG_TEST = 100  # free-form test draws

KEY_SHARE = 256  # one keypair per 256 ciphertexts (BASELINE configs 2-3; R#16 for all configs)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "hqcgen.c")
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(src):
        return _SO
    tmp = _SO + f".tmp{os.getpid()}"
    subprocess.run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-Wall", "-o", tmp, src, "-lpthread"],
                   check=True)
    os.replace(tmp, _SO)
    return _SO


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        c_p, u64, u32, sz, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_int
        _lib.hqcgen_u64.restype = u64
        _lib.hqcgen_u64.argtypes = [u64, u32, u64, u64]
        _lib.hqcgen_dense.argtypes = [u64, u32, u64, sz, u32, u32, c_p, i32]
        _lib.hqcgen_support.argtypes = [u64, u32, u64, sz, u32, u32, u32, c_p, i32]
        _lib.hqcgen_bytes.argtypes = [u64, u32, u64, sz, u32, u32, c_p, i32]
        _lib.hqcgen_blocks.argtypes = [u64, u32, u64, sz, u32, u32, u32, u32, c_p, c_p, i32]
        _lib.hqcgen_dense_idx.argtypes = [u64, u32, c_p, sz, u32, u32, c_p, i32]
        for f in ("hqcgen_dense", "hqcgen_support", "hqcgen_bytes", "hqcgen_blocks", "hqcgen_dense_idx"):
            getattr(_lib, f).restype = None
    return _lib


def _nt(n):
    return int(n) if n else (os.cpu_count() or 1)


def dense(seed: int, tag: int, idx0: int, rows: int, nbits: int, stride: int, nthreads=None) -> np.ndarray:
    """rows x stride uint64 words; bits >= nbits are zero."""
    out = np.empty((rows, stride), dtype=np.uint64)
    _L().hqcgen_dense(seed, tag, idx0, rows, nbits, stride, out.ctypes.data, _nt(nthreads))
    return out


def support(seed: int, tag: int, idx0: int, rows: int, n: int, w: int, stride: int, nthreads=None) -> np.ndarray:
    """rows x stride uint32; the first w entries of each row are distinct positions in [0, n), sorted."""
    assert stride >= w and 0 < w < n
    out = np.empty((rows, stride), dtype=np.uint32)
    _L().hqcgen_support(seed, tag, idx0, rows, n, w, stride, out.ctypes.data, _nt(nthreads))
    return out


def rand_bytes(seed: int, tag: int, idx0: int, rows: int, k: int, stride: int | None = None, nthreads=None):
    stride = stride or k
    out = np.empty((rows, stride), dtype=np.uint8)
    _L().hqcgen_bytes(seed, tag, idx0, rows, k, stride, out.ctypes.data, _nt(nthreads))
    return out


def blocks(seed: int, tag: int, idx0: int, rows: int, n1: int, tmin: int, tmax: int, nthreads=None):
    """For each row: t ~ U{tmin..tmax} and t distinct block indices in [0, n1), sorted (pad 0xFF)."""
    t = np.empty(rows, dtype=np.uint8)
    idx = np.empty((rows, tmax), dtype=np.uint8)
    _L().hqcgen_blocks(seed, tag, idx0, rows, n1, tmin, tmax, tmax, t.ctypes.data, idx.ctypes.data,
                       _nt(nthreads))
    return t, idx


@dataclass(frozen=True)
class Shape:
    """The sizes a workload needs; filled by the caller from its own parameter table."""

    n: int
    w: int
    wr: int
    n1: int
    k: int
    n2: int
    delta: int
    u_stride: int  # words per u row (>= ceil(n/64))
    v_words: int   # words per v row (= n1*n2/64)
    y_stride: int  # uint32 per support row (>= w)
    sup_stride: int  # uint32 per r1/r2/e row (>= wr)


def key_of(i0: int, rows: int) -> np.ndarray:
    return (np.arange(i0, i0 + rows, dtype=np.int64) // KEY_SHARE)


def key_draws(seed: int, sh: Shape, key0: int, nkeys: int, nthreads=None):
    h = dense(seed, TAG_H, key0, nkeys, sh.n, sh.u_stride, nthreads)
    x = support(seed, TAG_X, key0, nkeys, sh.n, sh.w, sh.y_stride, nthreads)
    y = support(seed, TAG_Y, key0, nkeys, sh.n, sh.w, sh.y_stride, nthreads)
    return h, x, y


def ct_draws(seed: int, sh: Shape, i0: int, rows: int, nthreads=None):
    m = rand_bytes(seed, TAG_M, i0, rows, sh.k, sh.k, nthreads)
    r1 = support(seed, TAG_R1, i0, rows, sh.n, sh.wr, sh.sup_stride, nthreads)
    r2 = support(seed, TAG_R2, i0, rows, sh.n, sh.wr, sh.sup_stride, nthreads)
    e = support(seed, TAG_E, i0, rows, sh.n, sh.wr, sh.sup_stride, nthreads)
    return m, r1, r2, e


def quarter_of(i: np.ndarray, batch: int) -> np.ndarray:
    """Adversarial config (BASELINE configs[3]): four equal quarters Q0..Q3 of the batch."""
    q = batch // 4
    return np.minimum(np.asarray(i) // max(q, 1), 3)


def block_patches(i0: int, rows: int, seed: int, sh: Shape, tmin: int, tmax: int, row_mask=None, nthreads=None):
    """The draws of randomise_blocks without applying them: per row t ~ U{tmin..tmax} (0 where row_mask
    is False) and a list of (row indices, block indices, bits[len, n2/64] uint64), one entry per slot."""
    assert sh.n2 % 64 == 0
    bw = sh.n2 // 64
    t, idx = blocks(seed, TAG_ADV_BLOCKS, i0, rows, sh.n1, tmin, tmax, nthreads)
    if row_mask is None:
        row_mask = np.ones(rows, dtype=bool)
    t = np.where(row_mask, t, 0).astype(np.uint8)
    sel = np.nonzero(row_mask)[0]
    patches = []
    for slot in range(tmax if sel.size else 0):
        rr = sel[t[sel] > slot]
        if rr.size == 0:
            continue
        # random words for (row, slot): stream index = global row * 256 + slot
        sidx = np.ascontiguousarray((i0 + rr.astype(np.uint64)) * np.uint64(256) + np.uint64(slot))
        bits = np.empty((rr.size, bw), dtype=np.uint64)
        _L().hqcgen_dense_idx(seed, TAG_ADV_BITS, sidx.ctypes.data, rr.size, sh.n2, bw, bits.ctypes.data,
                              _nt(nthreads))
        patches.append((rr, idx[rr, slot].astype(np.int64), bits))
    return t, patches


def randomise_blocks(v: np.ndarray, i0: int, seed: int, sh: Shape, tmin: int, tmax: int, row_mask=None,
                     nthreads=None):
    """Overwrite t ~ U{tmin..tmax} distinct RM blocks of each selected row of v (rows = ciphertexts
    i0..i0+len(v)) with uniform random bits (R#17). n2 is a multiple of 64, so a block is whole words.
    Returns the per-row block count t (0 where row_mask is False)."""
    bw = sh.n2 // 64
    t, patches = block_patches(i0, v.shape[0], seed, sh, tmin, tmax, row_mask, nthreads)
    for rr, b, bits in patches:
        cols = b[:, None] * bw + np.arange(bw)[None, :]
        v[rr[:, None], cols] = bits
    return t
