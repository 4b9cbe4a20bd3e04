"""Plain bit-array helpers for tests (little-endian bit order)."""
import numpy as np


def words_to_bits(w: np.ndarray, nbits: int) -> np.ndarray:
    b = np.unpackbits(np.ascontiguousarray(w, dtype="<u8").view(np.uint8), bitorder="little")
    return b[:nbits].astype(np.uint8)


def bits_to_words(b: np.ndarray, nwords: int) -> np.ndarray:
    b = np.asarray(b, dtype=np.uint8)
    pad = np.zeros(nwords * 64, dtype=np.uint8)
    pad[: b.size] = b
    return np.packbits(pad, bitorder="little").view("<u8").astype(np.uint64)


def support_to_bits(supp, n: int) -> np.ndarray:
    b = np.zeros(n, dtype=np.uint8)
    b[np.asarray(supp, dtype=np.int64)] = 1
    return b


def schoolbook_mul(a_bits: np.ndarray, b_bits: np.ndarray) -> np.ndarray:
    """The ring product by its definition: the polynomial product sum_i sum_j a_i b_j X^{i+j}
    (a linear convolution of the coefficient sequences, counted exactly in float64 via FFT — counts
    stay far below 2^52), then reduction by X^n = 1 (fold the top half) and mod 2."""
    n = a_bits.size
    assert b_bits.size == n
    L = 1
    while L < 2 * n:
        L *= 2
    fa = np.fft.rfft(a_bits.astype(np.float64), L)
    fb = np.fft.rfft(b_bits.astype(np.float64), L)
    c = np.rint(np.fft.irfft(fa * fb, L)[: 2 * n - 1]).astype(np.int64)
    full = np.zeros(2 * n, dtype=np.int64)
    full[: 2 * n - 1] = c
    return ((full[:n] + full[n:]) % 2).astype(np.uint8)
