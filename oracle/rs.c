/* ORACLE (test infrastructure only) — the outer shortened Reed–Solomon code over GF(2^8).
 *
 * Table I: RS [46,16,31], [56,24,33], [90,32,59]; the paper optimises only the encoder
 * (table-driven LFSR, §III.D) and the syndromes ("alpha^{i(j-1)}"), and names the
 * rest "error vector recovery". Readings:
 *   R#5  byte j (0-based) of a word is the coefficient of X^j; S_i = r(alpha^i), i = 1..2*delta;
 *        the generator has roots alpha^1..alpha^{2 delta};
 *   R#6  systematic message-first layout: c_j = m_j for j < k;
 *   R#7  decoding = syndromes -> Berlekamp–Massey (Massey 1969, full 2*delta+1 coefficients) ->
 *        Chien search over j in [0, n1) -> Forney (b = 1); ok <=> L <= delta and deg Lambda = L
 *        and #roots = L; on failure the output is r[0..k) unchanged.
 * All polynomial evaluations are Horner's rule with orc_gf_mul (no tables).
 * Pins (tests/test_oracle_rs.py): brute-force bounded-distance decoding over every codeword of tiny
 * shortened codes; zero syndromes and systematic layout of encodings; delta-error round trips at
 * the three real sizes; syndrome linearity; Table I minimum distances. */
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* p(x) = sum_i p[i] x^i, evaluated at x by Horner's rule. */
static uint8_t poly_eval(const uint8_t *p, uint32_t len, uint8_t x) {
  uint8_t acc = 0;
  for (uint32_t i = len; i-- > 0;) acc = orc_gf_mul(acc, x) ^ p[i];
  return acc;
}

void orc_rs_syndromes(const uint8_t *r, uint32_t n1, uint32_t delta, uint8_t *S) {
  for (uint32_t i = 1; i <= 2 * delta; i++) S[i - 1] = poly_eval(r, n1, orc_gf_pow(2, i));
}

void orc_rs_encode(const uint8_t *msg, uint32_t n1, uint32_t k, uint8_t *cw) {
  const uint32_t t2 = n1 - k; /* 2*delta parity symbols */
  /* g*(x) = prod_{i=1}^{2 delta} (x + alpha^{-i}): the reciprocal of g(x) = prod (x + alpha^i).
     A word c is a codeword iff c*(x) = x^{n1-1} c(1/x) is a multiple of g*(x), because
     c*(alpha^{-i}) = alpha^{-i(n1-1)} c(alpha^i). */
  uint8_t *g = (uint8_t *)calloc(t2 + 1, 1);
  g[0] = 1;
  for (uint32_t i = 1; i <= t2; i++) {
    uint8_t root = orc_gf_inv(orc_gf_pow(2, i));
    for (uint32_t t = i; t > 0; t--) g[t] = g[t - 1] ^ orc_gf_mul(g[t], root); /* g *= (x + root) */
    g[0] = orc_gf_mul(g[0], root);
  }
  /* c*(x) = M*(x) x^{2 delta} + (M*(x) x^{2 delta} mod g*(x)), with M*(x) = sum_j m_j x^{k-1-j}:
     the usual systematic division encoder, message in the top k coefficients of c*. */
  uint8_t *rem = (uint8_t *)calloc(n1, 1);
  for (uint32_t j = 0; j < k; j++) rem[t2 + (k - 1 - j)] = msg[j];
  for (int64_t deg = (int64_t)n1 - 1; deg >= (int64_t)t2; deg--) {
    uint8_t coef = rem[deg]; /* g* is monic: subtract coef * x^{deg - 2 delta} * g*(x) */
    for (uint32_t t = 0; t <= t2; t++) rem[deg - t2 + t] ^= orc_gf_mul(coef, g[t]);
  }
  /* c*_e for e < 2 delta is the remainder; e >= 2 delta is the message. Undo the reversal. */
  for (uint32_t j = 0; j < n1; j++) {
    uint32_t e = n1 - 1 - j;
    cw[j] = (j < k) ? msg[j] : rem[e];
  }
  free(rem);
  free(g);
}

int orc_rs_decode_ex(const uint8_t *r, uint32_t n1, uint32_t k, uint32_t delta, uint8_t *msg_out,
                     uint32_t *L_out, uint8_t *lambda_out) {
  const uint32_t N = 2 * delta, CAP = N + 1;
  uint8_t *S = (uint8_t *)malloc(N);
  orc_rs_syndromes(r, n1, delta, S);

  /* Berlekamp–Massey over the sequence s_0..s_{N-1} = S_1..S_N (Massey 1969). */
  uint8_t *C = (uint8_t *)calloc(CAP, 1), *B = (uint8_t *)calloc(CAP, 1),
          *T = (uint8_t *)calloc(CAP, 1);
  C[0] = 1; B[0] = 1;
  uint32_t L = 0, m = 1;
  uint8_t b = 1;
  for (uint32_t rr = 0; rr < N; rr++) {
    uint8_t d = S[rr];
    for (uint32_t i = 1; i <= L && i <= rr; i++) d ^= orc_gf_mul(C[i], S[rr - i]);
    if (d == 0) {
      m += 1;
    } else {
      uint8_t coef = orc_gf_mul(d, orc_gf_inv(b));
      memcpy(T, C, CAP);
      /* C(x) <- C(x) - coef * x^m * B(x); deg(x^m B) <= rr + 1 - L <= N, so CAP coefficients hold it */
      for (uint32_t i = m; i < CAP; i++) C[i] ^= orc_gf_mul(coef, B[i - m]);
      if (2 * L <= rr) {
        L = rr + 1 - L;
        memcpy(B, T, CAP);
        b = d;
        m = 1;
      } else {
        m += 1;
      }
    }
  }
  uint32_t deg = 0;
  for (uint32_t i = 0; i < CAP; i++)
    if (C[i]) deg = i;

  /* Chien search: position j is an error location iff Lambda(alpha^{-j}) = 0. */
  uint8_t *root = (uint8_t *)calloc(n1, 1);
  uint32_t nroots = 0;
  for (uint32_t j = 0; j < n1; j++) {
    uint8_t xinv = orc_gf_inv(orc_gf_pow(2, j));
    root[j] = poly_eval(C, CAP, xinv) == 0;
    nroots += root[j];
  }
  int ok = (L <= delta) && (deg == L) && (nroots == L);

  /* Forney (first syndrome index b = 1): e_j = Omega(X^{-1}) / Lambda'(X^{-1}), X = alpha^j,
     Omega(x) = S(x) Lambda(x) mod x^{2 delta}, S(x) = sum_{i<2 delta} S_{i+1} x^i. */
  uint8_t *Om = (uint8_t *)calloc(N, 1), *Dl = (uint8_t *)calloc(CAP, 1);
  for (uint32_t i = 0; i < N; i++)
    for (uint32_t t = 0; t <= i && t < CAP; t++) Om[i] ^= orc_gf_mul(C[t], S[i - t]);
  for (uint32_t i = 1; i < CAP; i += 2) Dl[i - 1] = C[i]; /* formal derivative in char. 2 */
  for (uint32_t j = 0; j < k; j++) {
    uint8_t out = r[j];
    if (ok && root[j]) {
      uint8_t xinv = orc_gf_inv(orc_gf_pow(2, j));
      uint8_t num = poly_eval(Om, N, xinv), den = poly_eval(Dl, CAP, xinv);
      out ^= orc_gf_mul(num, orc_gf_inv(den));
    }
    msg_out[j] = out;
  }
  if (L_out) *L_out = L;
  if (lambda_out) memcpy(lambda_out, C, CAP);
  free(S); free(C); free(B); free(T); free(root); free(Om); free(Dl);
  return ok;
}

int orc_rs_decode(const uint8_t *r, uint32_t n1, uint32_t k, uint32_t delta, uint8_t *msg_out) {
  return orc_rs_decode_ex(r, n1, k, delta, msg_out, NULL, NULL);
}
