/* ORACLE (test infrastructure only) — HQC.KEM with the HHK transform and implicit rejection
 * (SURVEY §8(f) row 2). The paper describes it in prose only ("In Decap, the receiver
 * decrypts the ciphertext (calling Decrypt), and then re-encrypts to verify correctness, and securely
 * rejects invalid ciphertexts"); the concrete hash inputs follow DESIGN.md readings R#20-R#23:
 *   R#20 domain tags G = 0x01, H = 0x02, K = 0x03, PRNG = 0x04 appended to the hashed bytes;
 *   R#21 pk serialised as h bytes || s bytes (ceil(n/8) each); H_pk = H(pk) (32 bytes), so that
 *        theta = G(H_pk || m) (32 bytes) does not re-hash the whole key per message;
 *   R#22 coins: SHAKE256(theta || PRNG) read as little-endian 32-bit words, w_r words each for r1,
 *        r2, e, each mapped to distinct positions by the fixed-weight sampler below;
 *   R#23 K = SHAKE256(m' || c || K, 64) when the re-encryption equals c, else SHAKE256(sigma || c || K, 64),
 *        with c = u bytes (ceil(n/8)) || v bytes (n1 n2 / 8).
 *   R#24 KeyGen from a 32-byte seed: (seed_sk || seed_pk) = SHAKE256(seed || PRNG, 64);
 *        h = SHAKE256(seed_pk || PRNG, ceil(n/8)) with bits >= n cleared ("sample_dense");
 *        SHAKE256(seed_sk || PRNG, 8w + k) -> x = sample(words 0..w), y = sample(words w..2w),
 *        sigma = bytes [8w, 8w + k); s = x + h*y (Alg. 3).
 * Fixed-weight sampler (R#22): p_i = i + floor(rand_i (n - i) / 2^32); then for i = w-1 down to 0,
 * p_i = i if p_i repeats a later entry. Every position is then distinct: p_i >= i for the
 * untouched entries and the replaced ones take the still-unused index i. */
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

void orc_sample_fixed_weight(const uint8_t *rnd, uint32_t n, uint32_t w, uint32_t *out) {
  for (uint32_t i = 0; i < w; i++) {
    uint32_t x = (uint32_t)rnd[4 * i] | ((uint32_t)rnd[4 * i + 1] << 8) | ((uint32_t)rnd[4 * i + 2] << 16) |
                 ((uint32_t)rnd[4 * i + 3] << 24);
    out[i] = i + (uint32_t)(((uint64_t)x * (uint64_t)(n - i)) >> 32);
  }
  for (int64_t i = (int64_t)w - 1; i >= 0; i--) {
    int dup = 0;
    for (uint32_t j = (uint32_t)i + 1; j < w; j++) dup |= out[j] == out[i];
    if (dup) out[i] = (uint32_t)i;
  }
}

static size_t nbytes(uint32_t bits) { return (bits + 7) / 8; }

static void put_words_le(const uint64_t *w, size_t nb, uint8_t *out) {
  for (size_t i = 0; i < nb; i++) out[i] = (uint8_t)(w[i / 8] >> (8 * (i % 8)));
}

void orc_kem_hpk(const orc_params *p, const uint64_t *h, const uint64_t *s, uint8_t hpk[32]) {
  const size_t nb = nbytes(p->n);
  uint8_t *buf = (uint8_t *)malloc(2 * nb + 1);
  put_words_le(h, nb, buf);
  put_words_le(s, nb, buf + nb);
  buf[2 * nb] = 0x02; /* H */
  orc_shake256(buf, 2 * nb + 1, hpk, 32);
  free(buf);
}

void orc_kem_coins(const orc_params *p, const uint8_t hpk[32], const uint8_t *m, uint32_t *r1, uint32_t *r2,
                   uint32_t *e) {
  uint8_t in[32 + 64 + 1], theta[33];
  memcpy(in, hpk, 32);
  memcpy(in + 32, m, p->k);
  in[32 + p->k] = 0x01; /* G */
  orc_shake256(in, 32 + p->k + 1, theta, 32);
  theta[32] = 0x04; /* PRNG */
  uint8_t *rnd = (uint8_t *)malloc(12 * (size_t)p->wr);
  orc_shake256(theta, 33, rnd, 12 * (size_t)p->wr);
  orc_sample_fixed_weight(rnd, p->n, p->wr, r1);
  orc_sample_fixed_weight(rnd + 4 * p->wr, p->n, p->wr, r2);
  orc_sample_fixed_weight(rnd + 8 * p->wr, p->n, p->wr, e);
  free(rnd);
}

static void kdf(const orc_params *p, const uint8_t *first, const uint64_t *u, const uint64_t *v, uint8_t K[64]) {
  const size_t ub = nbytes(p->n), vb = p->n12 / 8;
  uint8_t *buf = (uint8_t *)malloc(p->k + ub + vb + 1);
  memcpy(buf, first, p->k);
  put_words_le(u, ub, buf + p->k);
  put_words_le(v, vb, buf + p->k + ub);
  buf[p->k + ub + vb] = 0x03; /* K */
  orc_shake256(buf, p->k + ub + vb + 1, K, 64);
  free(buf);
}

void orc_kem_encaps(const orc_params *p, const uint64_t *h, const uint64_t *s, const uint8_t hpk[32],
                    const uint8_t *m, uint64_t *u, uint64_t *v, uint8_t K[64]) {
  uint32_t *r = (uint32_t *)malloc(sizeof(uint32_t) * 3 * p->wr);
  orc_kem_coins(p, hpk, m, r, r + p->wr, r + 2 * p->wr);
  orc_encrypt(p, h, s, m, r, r + p->wr, r + 2 * p->wr, u, v);
  kdf(p, m, u, v, K);
  free(r);
}

int orc_kem_decaps(const orc_params *p, const uint64_t *h, const uint64_t *s, const uint8_t hpk[32],
                   const uint32_t *y, const uint8_t *sigma, const uint64_t *u, const uint64_t *v, uint8_t K[64]) {
  uint8_t *m = (uint8_t *)malloc(p->k);
  orc_decrypt(p, u, v, y, m);
  uint32_t *r = (uint32_t *)malloc(sizeof(uint32_t) * 3 * p->wr);
  orc_kem_coins(p, hpk, m, r, r + p->wr, r + 2 * p->wr);
  uint64_t *u2 = (uint64_t *)malloc(sizeof(uint64_t) * p->words);
  uint64_t *v2 = (uint64_t *)malloc(sizeof(uint64_t) * p->vwords);
  orc_encrypt(p, h, s, m, r, r + p->wr, r + 2 * p->wr, u2, v2);
  /* compare c' with c byte-wise over the full serialised length: the ceil(n/8) u bytes (u' has
     zero bits in [n, 8 ceil(n/8)), so a received u with any of those bits set differs) and the n1 n2 / 8
     v bytes; the row's words beyond the u bytes are not part of c */
  uint64_t *um = (uint64_t *)malloc(sizeof(uint64_t) * p->words);
  memcpy(um, u, sizeof(uint64_t) * p->words);
  const uint32_t ubits = 8 * (uint32_t)nbytes(p->n);
  if (ubits % 64) um[p->words - 1] &= (~0ull) >> (64 - ubits % 64);
  int eq = memcmp(um, u2, sizeof(uint64_t) * p->words) == 0 && memcmp(v, v2, sizeof(uint64_t) * p->vwords) == 0;
  kdf(p, eq ? m : sigma, u, v, K);
  free(m); free(r); free(u2); free(v2); free(um);
  return eq;
}

void orc_kem_keygen(const orc_params *p, const uint8_t seed[32], uint64_t *h, uint32_t *x, uint32_t *y,
                    uint64_t *s, uint8_t *sigma) {
  uint8_t in[33], seeds[64];
  memcpy(in, seed, 32);
  in[32] = 0x04; /* PRNG */
  orc_shake256(in, 33, seeds, 64);
  /* h from seed_pk */
  const size_t nb = nbytes(p->n);
  uint8_t *hb = (uint8_t *)calloc(8 * (size_t)p->words, 1);
  memcpy(in, seeds + 32, 32);
  orc_shake256(in, 33, hb, nb);
  for (uint32_t i = 0; i < p->words; i++) {
    uint64_t w = 0;
    for (int b = 0; b < 8; b++) w |= (uint64_t)hb[8 * i + b] << (8 * b);
    h[i] = w;
  }
  if (p->n % 64) h[p->words - 1] &= (~0ull) >> (64 - p->n % 64);
  free(hb);
  /* x, y, sigma from seed_sk */
  uint8_t *r = (uint8_t *)malloc(8 * (size_t)p->w + p->k);
  memcpy(in, seeds, 32);
  orc_shake256(in, 33, r, 8 * (size_t)p->w + p->k);
  orc_sample_fixed_weight(r, p->n, p->w, x);
  orc_sample_fixed_weight(r + 4 * p->w, p->n, p->w, y);
  memcpy(sigma, r + 8 * p->w, p->k);
  free(r);
  orc_keygen(p, h, x, y, s);
}
