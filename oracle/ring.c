/* ORACLE (test infrastructure only) — the ring R = GF(2)[X]/(X^n - 1).
 *
 * Eq. 1 (§III.B):  a1(X)·a2(X) mod (X^N - 1) = XOR_{i in Supp(a1)} X^i · a2(X).
 * "Each rotation corresponds to a cyclic shift by a support index followed by XOR accumulation"
 * (P:166). "Each cyclic shift decomposes into a coarse word rotation and a fine intra-word bit
 * rotation ... A final masking step enforces the (X^N - 1) modulus" (§III.B.1).
 *
 * orc_ring_rotate computes X^i·a as (a << i) mod X^n  XOR  (a >> (n - i)): bit (t+i) mod n of the
 * result is bit t of a. The two multi-word shifts are written out word by word (word part q, bit
 * part s, carries between adjacent words), then bits >= n are masked off.
 * Pins (tests/test_oracle_ring.py): equality with the schoolbook (convolution) product at all three
 * n and on small rings; supp={0} gives a; supp={} gives 0; linearity; commutativity on n=257;
 * shift composition; bit-level definition of the rotation. */
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

static uint32_t nwords(uint32_t n) { return (n + 63) / 64; }

/* out = a << sh, as a W-word vector (bits shifted past word W-1 are dropped). */
static void shl_words(const uint64_t *a, uint32_t W, uint32_t sh, uint64_t *out) {
  uint32_t q = sh / 64, s = sh % 64;
  for (uint32_t k = 0; k < W; k++) {
    uint64_t lo = (k >= q) ? a[k - q] : 0;
    uint64_t carry = (s != 0 && k >= q + 1) ? (a[k - q - 1] >> (64 - s)) : 0;
    out[k] = (s ? (lo << s) : lo) | carry;
  }
}

/* out = a >> sh, as a W-word vector. */
static void shr_words(const uint64_t *a, uint32_t W, uint32_t sh, uint64_t *out) {
  uint32_t q = sh / 64, s = sh % 64;
  for (uint32_t k = 0; k < W; k++) {
    uint64_t hi = (k + q < W) ? a[k + q] : 0;
    uint64_t carry = (s != 0 && k + q + 1 < W) ? (a[k + q + 1] << (64 - s)) : 0;
    out[k] = (s ? (hi >> s) : hi) | carry;
  }
}

static void mask_to_n(uint64_t *v, uint32_t n) {
  uint32_t W = nwords(n);
  if (n % 64) v[W - 1] &= (~0ull) >> (64 - n % 64);
}

void orc_ring_rotate(const uint64_t *a, uint32_t n, uint32_t i, uint64_t *out) {
  uint32_t W = nwords(n);
  i %= n;
  uint64_t *t1 = (uint64_t *)malloc(sizeof(uint64_t) * W);
  uint64_t *t2 = (uint64_t *)malloc(sizeof(uint64_t) * W);
  shl_words(a, W, i, t1); /* X^i * a before reduction: bits >= n must wrap around ... */
  mask_to_n(t1, n);
  if (i) shr_words(a, W, n - i, t2); /* ... to position (t + i) - n: that is a >> (n - i) */
  else memset(t2, 0, sizeof(uint64_t) * W);
  for (uint32_t k = 0; k < W; k++) out[k] = t1[k] ^ t2[k];
  mask_to_n(out, n);
  free(t1);
  free(t2);
}

void orc_ring_mul_sparse(const uint64_t *a, uint32_t n, const uint32_t *supp, uint32_t wt,
                         uint64_t *out) {
  uint32_t W = nwords(n);
  uint64_t *rot = (uint64_t *)malloc(sizeof(uint64_t) * W);
  memset(out, 0, sizeof(uint64_t) * W);
  for (uint32_t j = 0; j < wt; j++) { /* XOR over i in Supp(a1) of X^i * a2 (Eq. 1) */
    orc_ring_rotate(a, n, supp[j], rot);
    for (uint32_t k = 0; k < W; k++) out[k] ^= rot[k];
  }
  free(rot);
}
