/* ORACLE (test infrastructure only) — batched drivers: a static partition of independent rows over
 * POSIX threads (SURVEY §8(d) "oracle timed on the box's host cores"). Each row runs the plain
 * single-ciphertext functions unchanged. */
#include <pthread.h>
#include <stdlib.h>

#include "oracle.h"

typedef struct {
  int kind;
  const orc_params *p;
  const void *a0, *a1, *a2, *a3, *a4, *a5, *a6;
  size_t s0, s1, s2, s3, s4, s5, s6;
  void *o0, *o1, *o2;  /* K_DECAP passes v (input) through o2 */
  size_t os0, os1;
  size_t lo, hi;
} job_t;

enum { K_DEC, K_ENC, K_RM, K_RS, K_ST1, K_DECAP };

static void *worker(void *arg) {
  job_t *j = (job_t *)arg;
  const orc_params *p = j->p;
  for (size_t i = j->lo; i < j->hi; i++) {
    switch (j->kind) {
      case K_DEC:
        orc_decrypt(p, (const uint64_t *)j->a0 + i * j->s0, (const uint64_t *)j->a1 + i * j->s1,
                    (const uint32_t *)j->a2 + i * j->s2, (uint8_t *)j->o0 + i * j->os0);
        break;
      case K_ST1:
        orc_decrypt_stage1(p, (const uint64_t *)j->a0 + i * j->s0,
                           (const uint64_t *)j->a1 + i * j->s1, (const uint32_t *)j->a2 + i * j->s2,
                           (uint64_t *)j->o0 + i * j->os0);
        break;
      case K_RM: {
        const uint64_t *r = (const uint64_t *)j->a0 + i * j->s0;
        uint8_t *sym = (uint8_t *)j->o0 + i * j->os0;
        for (uint32_t b = 0; b < p->n1; b++) sym[b] = orc_rm_decode(r, b * p->n2, p->mult);
        break;
      }
      case K_RS: {
        int ok = orc_rs_decode((const uint8_t *)j->a0 + i * j->s0, p->n1, p->k, p->delta,
                               (uint8_t *)j->o0 + i * j->os0);
        if (j->o1) ((uint8_t *)j->o1)[i] = (uint8_t)ok;
        break;
      }
      case K_DECAP: {
        int64_t key = ((const int64_t *)j->a4)[i];
        int acc = orc_kem_decaps(p, (const uint64_t *)j->a0 + key * j->s0, (const uint64_t *)j->a1 + key * j->s0,
                                 (const uint8_t *)j->a2 + key * 32, (const uint32_t *)j->a5 + i * j->s5,
                                 (const uint8_t *)j->a3 + key * p->k, (const uint64_t *)j->a6 + i * j->s6,
                                 (const uint64_t *)j->o2 + i * j->os1, (uint8_t *)j->o0 + i * 64);
        if (j->o1) ((uint8_t *)j->o1)[i] = (uint8_t)acc;
        break;
      }
      case K_ENC: {
        int64_t key = ((const int64_t *)j->a2)[i];
        orc_encrypt(p, (const uint64_t *)j->a0 + key * j->s0, (const uint64_t *)j->a1 + key * j->s1,
                    (const uint8_t *)j->a3 + i * j->s3, (const uint32_t *)j->a4 + i * j->s4,
                    (const uint32_t *)j->a5 + i * j->s4, (const uint32_t *)j->a6 + i * j->s4,
                    (uint64_t *)j->o0 + i * j->os0, (uint64_t *)j->o1 + i * j->os1);
        break;
      }
    }
  }
  return NULL;
}

static void run(job_t *tmpl, size_t batch, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if ((size_t)nthreads > batch) nthreads = batch ? (int)batch : 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
  job_t *jobs = (job_t *)malloc(sizeof(job_t) * nthreads);
  for (int t = 0; t < nthreads; t++) {
    jobs[t] = *tmpl;
    jobs[t].lo = batch * t / nthreads;
    jobs[t].hi = batch * (t + 1) / nthreads;
    pthread_create(&th[t], NULL, worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}

void orc_decrypt_batch(const orc_params *p, const uint64_t *u, size_t u_stride,
                       const uint64_t *v, size_t v_stride, const uint32_t *y, size_t y_stride,
                       uint8_t *m, size_t m_stride, size_t batch, int nthreads) {
  job_t j = {0};
  j.kind = K_DEC; j.p = p;
  j.a0 = u; j.s0 = u_stride; j.a1 = v; j.s1 = v_stride; j.a2 = y; j.s2 = y_stride;
  j.o0 = m; j.os0 = m_stride;
  run(&j, batch, nthreads);
}

void orc_stage1_batch(const orc_params *p, const uint64_t *u, size_t u_stride, const uint64_t *v,
                      size_t v_stride, const uint32_t *y, size_t y_stride, uint64_t *r,
                      size_t r_stride, size_t batch, int nthreads) {
  job_t j = {0};
  j.kind = K_ST1; j.p = p;
  j.a0 = u; j.s0 = u_stride; j.a1 = v; j.s1 = v_stride; j.a2 = y; j.s2 = y_stride;
  j.o0 = r; j.os0 = r_stride;
  run(&j, batch, nthreads);
}

void orc_rm_decode_batch(const orc_params *p, const uint64_t *r, size_t r_stride, uint8_t *sym,
                         size_t sym_stride, size_t batch, int nthreads) {
  job_t j = {0};
  j.kind = K_RM; j.p = p;
  j.a0 = r; j.s0 = r_stride; j.o0 = sym; j.os0 = sym_stride;
  run(&j, batch, nthreads);
}

void orc_rs_decode_batch(const orc_params *p, const uint8_t *sym, size_t sym_stride, uint8_t *m,
                         size_t m_stride, uint8_t *ok, size_t batch, int nthreads) {
  job_t j = {0};
  j.kind = K_RS; j.p = p;
  j.a0 = sym; j.s0 = sym_stride; j.o0 = m; j.os0 = m_stride; j.o1 = ok;
  run(&j, batch, nthreads);
}

void orc_encrypt_batch(const orc_params *p, const uint64_t *h, size_t h_stride,
                       const uint64_t *s, size_t s_stride, const int64_t *key_of_row,
                       const uint8_t *m, size_t m_stride, const uint32_t *r1, const uint32_t *r2,
                       const uint32_t *e, size_t sup_stride, uint64_t *u, size_t u_stride,
                       uint64_t *v, size_t v_stride, size_t batch, int nthreads) {
  job_t j = {0};
  j.kind = K_ENC; j.p = p;
  j.a0 = h; j.s0 = h_stride; j.a1 = s; j.s1 = s_stride; j.a2 = key_of_row;
  j.a3 = m; j.s3 = m_stride; j.a4 = r1; j.a5 = r2; j.a6 = e; j.s4 = sup_stride;
  j.o0 = u; j.os0 = u_stride; j.o1 = v; j.os1 = v_stride;
  run(&j, batch, nthreads);
}

void orc_kem_decaps_batch(const orc_params *p, const uint64_t *h, const uint64_t *s, size_t key_stride,
                          const uint8_t *hpk, const uint8_t *sigma, const int64_t *key_of_row,
                          const uint32_t *y, size_t y_stride, const uint64_t *u, size_t u_stride,
                          const uint64_t *v, size_t v_stride, uint8_t *K, uint8_t *acc, size_t batch,
                          int nthreads) {
  job_t j = {0};
  j.kind = K_DECAP; j.p = p;
  j.a0 = h; j.a1 = s; j.s0 = key_stride; j.a2 = hpk; j.a3 = sigma; j.a4 = key_of_row;
  j.a5 = y; j.s5 = y_stride; j.a6 = u; j.s6 = u_stride;
  j.o2 = (void *)v; j.os1 = v_stride; j.o0 = K; j.o1 = acc;
  run(&j, batch, nthreads);
}
