/* ORACLE (test infrastructure only) — concatenated code and HQC.PKE.
 *
 * Concatenated code C: outer shortened RS, inner duplicated RM. Encoding RS-encodes the k
 * message bytes, then RM-encodes symbol j into bits [j*n2, (j+1)*n2). C.Decode (Alg. 2,
 * P:83; "applies Reed–Muller then Reed–Solomon decoding") RM-decodes each block, then
 * RS-decodes the n1 symbols.
 *
 * KeyGen  (Alg. 3): s = x + h*y.
 * Encrypt (Alg. 1):  u = r1 + h*r2,  v = mG + s*r2 + e, truncated to n1*n2 bits (R#3).
 * Decrypt (Alg. 2):  m' = C.Decode(v - u*y)  — with the SECRET y as multiplicand (R#1)
 *                             and "-"/"+" = XOR (R#2), on the low n1*n2 bits (R#3).
 * Every product is a sparse x dense product by Eq. 1 (orc_ring_mul_sparse), since h*r2, s*r2, h*y
 * and u*y all have a fixed-weight factor.
 * Pins (tests/test_oracle_pke.py): decrypt(encrypt(m)) = m; all-zero ciphertext -> 0^k; the
 * algebraic identity v + u*y = mG + x*r2 + r1*y + e (truncated); stage-1 vs a schoolbook product. */
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

static void set_bit(uint64_t *v, uint32_t t) { v[t / 64] |= 1ull << (t % 64); }

static void to_dense(const uint32_t *supp, uint32_t wt, uint32_t words, uint64_t *out) {
  memset(out, 0, sizeof(uint64_t) * words);
  for (uint32_t j = 0; j < wt; j++) set_bit(out, supp[j]);
}

/* keep bits [0, nbits) of a, zero the rest of the first vwords words */
static void truncate_to(const uint64_t *a, uint32_t nbits, uint32_t vwords, uint64_t *out) {
  for (uint32_t k = 0; k < vwords; k++) out[k] = a[k];
  if (nbits % 64) out[vwords - 1] &= (~0ull) >> (64 - nbits % 64);
}

void orc_code_encode(const orc_params *p, const uint8_t *msg, uint64_t *vec) {
  uint8_t *cw = (uint8_t *)malloc(p->n1);
  orc_rs_encode(msg, p->n1, p->k, cw);
  memset(vec, 0, sizeof(uint64_t) * p->vwords);
  for (uint32_t j = 0; j < p->n1; j++) orc_rm_encode(cw[j], p->mult, vec, j * p->n2);
  free(cw);
}

void orc_code_decode(const orc_params *p, const uint64_t *vec, uint8_t *msg, uint8_t *sym_out) {
  uint8_t *sym = (uint8_t *)malloc(p->n1);
  for (uint32_t j = 0; j < p->n1; j++) sym[j] = orc_rm_decode(vec, j * p->n2, p->mult);
  orc_rs_decode(sym, p->n1, p->k, p->delta, msg);
  if (sym_out) memcpy(sym_out, sym, p->n1);
  free(sym);
}

void orc_keygen(const orc_params *p, const uint64_t *h, const uint32_t *x, const uint32_t *y,
                uint64_t *s) {
  uint64_t *hy = (uint64_t *)malloc(sizeof(uint64_t) * p->words);
  uint64_t *xd = (uint64_t *)malloc(sizeof(uint64_t) * p->words);
  orc_ring_mul_sparse(h, p->n, y, p->w, hy); /* h * y */
  to_dense(x, p->w, p->words, xd);
  for (uint32_t k = 0; k < p->words; k++) s[k] = xd[k] ^ hy[k]; /* s = x + h*y */
  free(hy);
  free(xd);
}

void orc_encrypt(const orc_params *p, const uint64_t *h, const uint64_t *s, const uint8_t *m,
                 const uint32_t *r1, const uint32_t *r2, const uint32_t *e, uint64_t *u,
                 uint64_t *v) {
  const uint32_t W = p->words;
  uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * W);
  uint64_t *d = (uint64_t *)malloc(sizeof(uint64_t) * W);
  uint64_t *mg = (uint64_t *)calloc(W, sizeof(uint64_t));
  /* u = r1 + h * r2 */
  orc_ring_mul_sparse(h, p->n, r2, p->wr, t);
  to_dense(r1, p->wr, W, d);
  for (uint32_t k = 0; k < W; k++) u[k] = d[k] ^ t[k];
  /* v = trunc(mG + s * r2 + e) */
  orc_code_encode(p, m, mg); /* fills the first vwords words; the rest stay zero */
  orc_ring_mul_sparse(s, p->n, r2, p->wr, t);
  to_dense(e, p->wr, W, d);
  for (uint32_t k = 0; k < W; k++) t[k] ^= mg[k] ^ d[k];
  truncate_to(t, p->n12, p->vwords, v);
  free(t);
  free(d);
  free(mg);
}

void orc_decrypt_stage1(const orc_params *p, const uint64_t *u, const uint64_t *v,
                        const uint32_t *y, uint64_t *r) {
  const uint32_t W = p->words;
  uint64_t *um = (uint64_t *)malloc(sizeof(uint64_t) * W);
  uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * W);
  memcpy(um, u, sizeof(uint64_t) * W);
  if (p->n % 64) um[W - 1] &= (~0ull) >> (64 - p->n % 64); /* bits >= n are not part of u (R#13) */
  orc_ring_mul_sparse(um, p->n, y, p->w, t);                /* u * y (Eq. 1) */
  truncate_to(t, p->n12, p->vwords, t);
  for (uint32_t k = 0; k < p->vwords; k++) r[k] = v[k] ^ t[k]; /* v - u*y */
  if (p->n12 % 64) r[p->vwords - 1] &= (~0ull) >> (64 - p->n12 % 64);
  free(um);
  free(t);
}

void orc_decrypt(const orc_params *p, const uint64_t *u, const uint64_t *v, const uint32_t *y,
                 uint8_t *m) {
  uint64_t *r = (uint64_t *)malloc(sizeof(uint64_t) * p->vwords);
  orc_decrypt_stage1(p, u, v, y, r);
  orc_code_decode(p, r, m, NULL);
  free(r);
}
