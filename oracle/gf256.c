/* ORACLE (test infrastructure only) — GF(2^8) arithmetic.
 * The paper never states the field (R#4): GF(2)[x]/(x^8+x^4+x^3+x^2+1) = 0x11D with alpha = x = 0x02,
 * as in SPEC S:236. Multiplication here is the definition — a carry-less (shift-and-XOR) product
 * followed by reduction modulo 0x11D — with no tables. The paper's lookup tables
 * are an implementation technique for the same products.
 * Pins (tests/test_oracle_gf.py): mul(0x02,0x80)=0x1D, alpha has order 255, field axioms
 * exhaustive over all pairs, a * a^254 = 1, agreement with a polynomial-arithmetic model in Python. */
#include "oracle.h"

uint8_t orc_gf_mul(uint8_t a, uint8_t b) {
  /* carry-less product of two degree-<8 polynomials: degree <= 14 */
  uint32_t prod = 0;
  for (int i = 0; i < 8; i++)
    if ((b >> i) & 1) prod ^= (uint32_t)a << i;
  /* reduce modulo x^8 + x^4 + x^3 + x^2 + 1 from the top bit down */
  for (int deg = 14; deg >= 8; deg--)
    if ((prod >> deg) & 1) prod ^= 0x11Du << (deg - 8);
  return (uint8_t)prod;
}

uint8_t orc_gf_pow(uint8_t a, uint32_t e) {
  uint8_t r = 1;
  for (uint32_t i = 0; i < e; i++) r = orc_gf_mul(r, a);
  return r;
}

/* Fermat: a^(2^8 - 2) = a^{-1} for a != 0. */
uint8_t orc_gf_inv(uint8_t a) { return orc_gf_pow(a, 254); }
