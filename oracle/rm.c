/* ORACLE (test infrastructure only) — the inner duplicated Reed–Muller code RM(1,7) x mult.
 *
 * Table I: RM [384,8,192] for HQC-1 (3 copies of RM(1,7) = [128,8,64]) and
 * [640,8,320] for HQC-3/5 (5 copies). The paper names only a "byte-parallel Reed–Muller decoder"
 * and gives no algorithm; the readings used here are DESIGN.md R#9-R#12:
 *   R#9  encoding: codeword bit p (p = 0..127) of byte b is b7 XOR parity(b & 0x7F & p);
 *   R#12 block j occupies bits [j*n2, (j+1)*n2); copy c of the block occupies +128c;
 *   R#10 decoding: soft values s_p = sum over copies of (1 - 2*bit), Hadamard coefficients
 *        F(a) = sum_p s_p * (-1)^popcount(a & p), a = 0..127, written here as the definition
 *        (a double loop over a and p, not a fast transform);
 *   R#11 decision: a* = the SMALLEST a with |F(a)| maximal; byte = a* | 0x80 if F(a*) < 0.
 * This equals maximum-likelihood decoding over the 256 duplicated codewords with ties broken
 * toward the smallest (b & 0x7F); tests/test_oracle_rm.py pins it to that brute force. */
#include "oracle.h"

static int get_bit(const uint64_t *v, uint32_t t) { return (int)((v[t / 64] >> (t % 64)) & 1); }
static void put_bit(uint64_t *v, uint32_t t, int b) {
  uint64_t m = 1ull << (t % 64);
  if (b) v[t / 64] |= m; else v[t / 64] &= ~m;
}
static int parity8(uint32_t x) { return __builtin_parity(x & 0xFFu); } /* XOR of the 8 low bits */

void orc_rm_encode(uint8_t b, uint32_t mult, uint64_t *vec, uint32_t off) {
  for (uint32_t c = 0; c < mult; c++)
    for (uint32_t p = 0; p < 128; p++)
      put_bit(vec, off + 128 * c + p, ((b >> 7) & 1) ^ parity8((uint32_t)(b & 0x7F) & p));
}

void orc_rm_transform(const uint64_t *vec, uint32_t off, uint32_t mult, int32_t F[128]) {
  int32_t s[128];
  for (uint32_t p = 0; p < 128; p++) {
    s[p] = 0;
    for (uint32_t c = 0; c < mult; c++) s[p] += 1 - 2 * get_bit(vec, off + 128 * c + p);
  }
  for (uint32_t a = 0; a < 128; a++) {
    int32_t acc = 0;
    for (uint32_t p = 0; p < 128; p++) acc += parity8(a & p) ? -s[p] : s[p];
    F[a] = acc;
  }
}

uint8_t orc_rm_decode(const uint64_t *vec, uint32_t off, uint32_t mult) {
  int32_t F[128];
  orc_rm_transform(vec, off, mult, F);
  uint32_t best = 0;
  int32_t bestabs = -1;
  for (uint32_t a = 0; a < 128; a++) { /* strict '>' keeps the smallest a among equal maxima */
    int32_t m = F[a] < 0 ? -F[a] : F[a];
    if (m > bestabs) { bestabs = m; best = a; }
  }
  return (uint8_t)(best | (F[best] < 0 ? 0x80u : 0u));
}
