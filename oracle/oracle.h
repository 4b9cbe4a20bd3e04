/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the batched HQC.PKE.Decrypt hot path
 * computes, written from PAPER.md (arxiv 2512.12904, "OptHQC") and the readings listed in
 * DESIGN.md §3. It exists to define "correct" for the CUDA path and is pinned, by the CPU tests in
 * tests/test_oracle_*.py, to things other than itself (brute-force ML / bounded-distance decoding,
 * schoolbook products, closed forms, Table I of the paper).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 * or call this library. It shares no code, header, table or constant generator with the CUDA path
 * (paper_2512_12904_b200/), and neither side includes the other.
 *
 * Citation convention: "P:n" = /root/reference/PAPER.md line n (section / algorithm / table named),
 * "S:n" = /root/reference/SPEC.md line n. DESIGN.md §3 "R#k" = reading #k of an ambiguous passage.
 *
 * Parity status: every function below is pinned by at least one CPU test;
 * none is "parity unpinned".
 *
 * Bit order: element bit t lives in 64-bit word t/64 at bit t%64; bits >= n are zero.
 */
#ifndef HQC_ORACLE_H
#define HQC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Table I "HQC parameter sets" plus the derived quantities of R#3, R#15. */
typedef struct {
  int32_t level;    /* 1, 3, 5 */
  uint32_t n;       /* ring length N (Table I) */
  uint32_t w;       /* omega: weight of x, y (Table I) */
  uint32_t wr;      /* omega_r = omega_e (Table I) */
  uint32_t n1;      /* RS length (Table I "[n1,k,d]") */
  uint32_t k;       /* RS dimension = message bytes */
  uint32_t d;       /* RS minimum distance */
  uint32_t delta;   /* (d-1)/2, R#15 */
  uint32_t n2;      /* duplicated RM length (Table I "[n2,8,d']") */
  uint32_t mult;    /* n2 / 128 copies of RM(1,7) */
  uint32_t dprime;  /* duplicated RM minimum distance */
  uint32_t n12;     /* n1*n2: truncation length, R#3 */
  uint32_t words;   /* ceil(n/64): words of a ring element */
  uint32_t vwords;  /* ceil(n12/64): words of a truncated element */
} orc_params;

int orc_get_params(int level, orc_params *out); /* 0 ok, -1 unknown level */

/* ---- GF(2^8) = GF(2)[x]/(x^8+x^4+x^3+x^2+1), alpha = 0x02 (R#4) ---- */
uint8_t orc_gf_mul(uint8_t a, uint8_t b);
uint8_t orc_gf_pow(uint8_t a, uint32_t e);
uint8_t orc_gf_inv(uint8_t a); /* a^254; a must be nonzero (returns 0 for 0) */

/* ---- Ring R = GF(2)[X]/(X^n - 1) (Eq. 1) ---- */
void orc_ring_rotate(const uint64_t *a, uint32_t n, uint32_t i, uint64_t *out);
void orc_ring_mul_sparse(const uint64_t *a, uint32_t n, const uint32_t *supp, uint32_t wt,
                         uint64_t *out);

/* ---- Duplicated RM(1,7) (Table I; R#9-#12) ---- */
/* Writes the mult*128 bits of the encoding of byte b into bits [off, off + mult*128) of vec. */
void orc_rm_encode(uint8_t b, uint32_t mult, uint64_t *vec, uint32_t off);
/* Decodes the block at bits [off, off + mult*128) of vec. */
uint8_t orc_rm_decode(const uint64_t *vec, uint32_t off, uint32_t mult);
/* The Hadamard coefficients F(a), a = 0..127, of that block (by definition, R#10). */
void orc_rm_transform(const uint64_t *vec, uint32_t off, uint32_t mult, int32_t F[128]);

/* ---- Shortened RS [n1, k, 2*delta+1] over GF(2^8) (R#5-#7) ---- */
void orc_rs_encode(const uint8_t *msg, uint32_t n1, uint32_t k, uint8_t *cw);
void orc_rs_syndromes(const uint8_t *r, uint32_t n1, uint32_t delta, uint8_t *S /* 2*delta */);
/* Returns ok (1) when a codeword within distance delta was found and corrected, else 0.
   msg_out receives k bytes (corrected, or r[0..k) unchanged on failure). */
int orc_rs_decode(const uint8_t *r, uint32_t n1, uint32_t k, uint32_t delta, uint8_t *msg_out);
/* Same, exposing the BM linear complexity L and the locator Lambda[0..2*delta]. */
int orc_rs_decode_ex(const uint8_t *r, uint32_t n1, uint32_t k, uint32_t delta, uint8_t *msg_out,
                     uint32_t *L_out, uint8_t *lambda_out);

/* ---- Concatenated code C ---- */
void orc_code_encode(const orc_params *p, const uint8_t *msg, uint64_t *vec /* p->vwords */);
void orc_code_decode(const orc_params *p, const uint64_t *vec, uint8_t *msg, uint8_t *sym_out);

/* ---- PKE (Alg. 1-3); R#1 decrypt multiplies by the secret y ---- */
void orc_keygen(const orc_params *p, const uint64_t *h, const uint32_t *x, const uint32_t *y,
                uint64_t *s /* p->words */);
void orc_encrypt(const orc_params *p, const uint64_t *h, const uint64_t *s, const uint8_t *m,
                 const uint32_t *r1, const uint32_t *r2, const uint32_t *e,
                 uint64_t *u /* p->words */, uint64_t *v /* p->vwords */);
/* Stage 1 alone: r = v XOR trunc_{n12}(u * y)  (R#1-#3); r has p->vwords words. */
void orc_decrypt_stage1(const orc_params *p, const uint64_t *u, const uint64_t *v,
                        const uint32_t *y, uint64_t *r);
void orc_decrypt(const orc_params *p, const uint64_t *u, const uint64_t *v, const uint32_t *y,
                 uint8_t *m);

/* ---- KEM row of SURVEY §8(f) (HHK with implicit rejection; readings R#20-R#23 in DESIGN.md) ---- */
void orc_keccak_f1600(uint64_t A[25]);
void orc_shake256(const uint8_t *msg, size_t len, uint8_t *out, size_t outlen);
/* w distinct positions in [0, n) from 4w bytes of PRNG output (R#22) */
void orc_sample_fixed_weight(const uint8_t *rnd, uint32_t n, uint32_t w, uint32_t *out);
/* serialised pk = h bytes (ceil(n/8)) || s bytes (ceil(n/8)); H_pk = SHAKE256(pk || 0x02, 32) */
void orc_kem_hpk(const orc_params *p, const uint64_t *h, const uint64_t *s, uint8_t hpk[32]);
/* theta = SHAKE256(H_pk || m || 0x01, 32); (r1, r2, e) = sample(SHAKE256(theta || 0x04, 12 wr)) */
void orc_kem_coins(const orc_params *p, const uint8_t hpk[32], const uint8_t *m, uint32_t *r1, uint32_t *r2,
                   uint32_t *e);
/* Encaps: c = Encrypt(pk, m; coins(m)), K = SHAKE256(m || c || 0x03, 64), c = u bytes || v bytes */
void orc_kem_encaps(const orc_params *p, const uint64_t *h, const uint64_t *s, const uint8_t hpk[32],
                    const uint8_t *m, uint64_t *u, uint64_t *v, uint8_t K[64]);
/* KeyGen from a 32-byte seed (R#24): h (p->words, bits >= n zero), x, y (w positions each), s, sigma (k bytes) */
void orc_kem_keygen(const orc_params *p, const uint8_t seed[32], uint64_t *h, uint32_t *x, uint32_t *y,
                    uint64_t *s, uint8_t *sigma);
/* Decaps: m' = Decrypt; c' = Encrypt(pk, m'; coins(m')); K = SHAKE256((c' == c ? m' : sigma) || c || 0x03, 64).
   Returns 1 if the ciphertext was accepted (c' == c). */
int orc_kem_decaps(const orc_params *p, const uint64_t *h, const uint64_t *s, const uint8_t hpk[32],
                   const uint32_t *y, const uint8_t *sigma, const uint64_t *u, const uint64_t *v, uint8_t K[64]);

/* ---- Batched drivers (strided rows; nthreads POSIX threads, static partition) ---- */
void orc_decrypt_batch(const orc_params *p, const uint64_t *u, size_t u_stride,
                       const uint64_t *v, size_t v_stride, const uint32_t *y, size_t y_stride,
                       uint8_t *m, size_t m_stride, size_t batch, int nthreads);
void orc_encrypt_batch(const orc_params *p, const uint64_t *h, size_t h_stride,
                       const uint64_t *s, size_t s_stride, const int64_t *key_of_row,
                       const uint8_t *m, size_t m_stride, const uint32_t *r1, const uint32_t *r2,
                       const uint32_t *e, size_t sup_stride, uint64_t *u, size_t u_stride,
                       uint64_t *v, size_t v_stride, size_t batch, int nthreads);
void orc_rm_decode_batch(const orc_params *p, const uint64_t *r, size_t r_stride, uint8_t *sym,
                         size_t sym_stride, size_t batch, int nthreads);
void orc_rs_decode_batch(const orc_params *p, const uint8_t *sym, size_t sym_stride,
                         uint8_t *m, size_t m_stride, uint8_t *ok, size_t batch, int nthreads);
void orc_kem_decaps_batch(const orc_params *p, const uint64_t *h, const uint64_t *s, size_t key_stride,
                          const uint8_t *hpk, const uint8_t *sigma, const int64_t *key_of_row,
                          const uint32_t *y, size_t y_stride, const uint64_t *u, size_t u_stride,
                          const uint64_t *v, size_t v_stride, uint8_t *K, uint8_t *acc, size_t batch,
                          int nthreads);
void orc_stage1_batch(const orc_params *p, const uint64_t *u, size_t u_stride, const uint64_t *v,
                      size_t v_stride, const uint32_t *y, size_t y_stride, uint64_t *r,
                      size_t r_stride, size_t batch, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
