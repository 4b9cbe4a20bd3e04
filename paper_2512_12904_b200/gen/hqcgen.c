/* Seeded synthetic input generator (DESIGN.md §5 "input recipe").
 *
 * Shared by the tests (which feed the draws to the oracle) and bench.py (which feeds them to the GPU
 * keygen/encrypt kernels). It holds NONE of the method's arithmetic: only counter-based random
 * draws — dense random words, fixed-weight supports (distinct sorted positions), random bytes, and
 * "t distinct block indices" for the adversarial configs. Every row is a pure function of
 * (seed, tag, row index), so any shard of any batch regenerates identically for any GPU count.
 *
 * PRNG: SplitMix64 (Steele, Lea, Flood 2014) with a per-(seed, tag, index) starting state.
 * Position draws map a 32-bit value x to floor(x * n / 2^32) (multiply-shift), then reject
 * duplicates ("draws uniform positions by rejection and rejects duplicates until
 * w distinct indices exist, then sorts them"). */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct { uint64_t s; } rng_t;

static inline rng_t rng_make(uint64_t seed, uint32_t tag, uint64_t idx) {
  rng_t r;
  r.s = mix64(mix64(seed ^ ((uint64_t)(tag + 1) * 0x9E3779B97F4A7C15ull)) ^ idx);
  return r;
}
static inline uint64_t rng_next(rng_t *r) {
  r->s += 0x9E3779B97F4A7C15ull;
  return mix64(r->s);
}
static inline uint32_t rng_below(rng_t *r, uint32_t n) {
  return (uint32_t)(((rng_next(r) >> 32) * (uint64_t)n) >> 32);
}

uint64_t hqcgen_u64(uint64_t seed, uint32_t tag, uint64_t idx, uint64_t ctr) {
  rng_t r = rng_make(seed, tag, idx);
  uint64_t x = 0;
  for (uint64_t i = 0; i <= ctr; i++) x = rng_next(&r);
  return x;
}

/* ---- row generators ---- */

static void dense_row(uint64_t seed, uint32_t tag, uint64_t idx, uint32_t nbits, uint32_t stride,
                      uint64_t *out) {
  rng_t r = rng_make(seed, tag, idx);
  uint32_t nw = (nbits + 63) / 64;
  for (uint32_t k = 0; k < stride; k++) out[k] = (k < nw) ? rng_next(&r) : 0;
  if (nbits % 64) out[nw - 1] &= (~0ull) >> (64 - nbits % 64);
}

static int cmp_u32(const void *a, const void *b) {
  uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return (x > y) - (x < y);
}

/* w distinct positions in [0, n), sorted ascending; bitmap = scratch of ceil(n/64) zeroed words */
static void support_row(uint64_t seed, uint32_t tag, uint64_t idx, uint32_t n, uint32_t w,
                        uint32_t stride, uint32_t *out, uint64_t *bitmap) {
  rng_t r = rng_make(seed, tag, idx);
  uint32_t got = 0;
  while (got < w) {
    uint32_t pos = rng_below(&r, n);
    uint64_t m = 1ull << (pos % 64);
    if (bitmap[pos / 64] & m) continue;
    bitmap[pos / 64] |= m;
    out[got++] = pos;
  }
  for (uint32_t j = 0; j < w; j++) bitmap[out[j] / 64] = 0;
  qsort(out, w, sizeof(uint32_t), cmp_u32);
  for (uint32_t j = w; j < stride; j++) out[j] = 0;
}

static void bytes_row(uint64_t seed, uint32_t tag, uint64_t idx, uint32_t k, uint32_t stride,
                      uint8_t *out) {
  rng_t r = rng_make(seed, tag, idx);
  uint64_t x = 0;
  for (uint32_t j = 0; j < stride; j++) {
    if (j >= k) { out[j] = 0; continue; }
    if (j % 8 == 0) x = rng_next(&r);
    out[j] = (uint8_t)(x >> (8 * (j % 8)));
  }
}

/* t ~ U{tmin..tmax}, then t distinct indices in [0, n1) sorted; out_idx row padded with 0xFF */
static void blocks_row(uint64_t seed, uint32_t tag, uint64_t idx, uint32_t n1, uint32_t tmin,
                       uint32_t tmax, uint32_t stride, uint8_t *out_t, uint8_t *out_idx) {
  rng_t r = rng_make(seed, tag, idx);
  uint32_t t = tmin + rng_below(&r, tmax - tmin + 1);
  uint32_t tmp[256];
  uint8_t used[256];
  memset(used, 0, sizeof used);
  uint32_t got = 0;
  while (got < t) {
    uint32_t b = rng_below(&r, n1);
    if (used[b]) continue;
    used[b] = 1;
    tmp[got++] = b;
  }
  qsort(tmp, t, sizeof(uint32_t), cmp_u32);
  *out_t = (uint8_t)t;
  for (uint32_t j = 0; j < stride; j++) out_idx[j] = (j < t) ? (uint8_t)tmp[j] : 0xFF;
}

/* ---- threaded batch front-ends ---- */

typedef struct {
  int kind;
  uint64_t seed, idx0;
  uint32_t tag, a, b, c, stride;
  void *out, *out2;
  size_t lo, hi;
} gjob_t;

enum { G_DENSE, G_SUPPORT, G_BYTES, G_BLOCKS, G_DENSE_IDX };

static void *gworker(void *arg) {
  gjob_t *j = (gjob_t *)arg;
  uint64_t *bitmap = NULL;
  if (j->kind == G_SUPPORT) bitmap = (uint64_t *)calloc((j->a + 63) / 64 + 1, sizeof(uint64_t));
  for (size_t i = j->lo; i < j->hi; i++) {
    uint64_t idx = (j->kind == G_DENSE_IDX) ? ((const uint64_t *)j->out2)[i] : j->idx0 + i;
    switch (j->kind) {
      case G_DENSE_IDX:
      case G_DENSE: dense_row(j->seed, j->tag, idx, j->a, j->stride, (uint64_t *)j->out + i * j->stride); break;
      case G_SUPPORT:
        support_row(j->seed, j->tag, idx, j->a, j->b, j->stride, (uint32_t *)j->out + i * j->stride, bitmap);
        break;
      case G_BYTES: bytes_row(j->seed, j->tag, idx, j->a, j->stride, (uint8_t *)j->out + i * j->stride); break;
      case G_BLOCKS:
        blocks_row(j->seed, j->tag, idx, j->a, j->b, j->c, j->stride, (uint8_t *)j->out2 + i,
                   (uint8_t *)j->out + i * j->stride);
        break;
    }
  }
  free(bitmap);
  return NULL;
}

static void grun(gjob_t *tmpl, size_t rows, int nthreads) {
  if (rows == 0) return;
  if (nthreads < 1) nthreads = 1;
  if ((size_t)nthreads * 64 > rows) nthreads = (int)((rows + 63) / 64);
  pthread_t th[256];
  gjob_t jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; t++) {
    jobs[t] = *tmpl;
    jobs[t].lo = rows * t / nthreads;
    jobs[t].hi = rows * (t + 1) / nthreads;
    pthread_create(&th[t], NULL, gworker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
}

void hqcgen_dense(uint64_t seed, uint32_t tag, uint64_t idx0, size_t rows, uint32_t nbits,
                  uint32_t stride, uint64_t *out, int nthreads) {
  gjob_t j = {G_DENSE, seed, idx0, tag, nbits, 0, 0, stride, out, NULL, 0, 0};
  grun(&j, rows, nthreads);
}

void hqcgen_support(uint64_t seed, uint32_t tag, uint64_t idx0, size_t rows, uint32_t n,
                    uint32_t w, uint32_t stride, uint32_t *out, int nthreads) {
  gjob_t j = {G_SUPPORT, seed, idx0, tag, n, w, 0, stride, out, NULL, 0, 0};
  grun(&j, rows, nthreads);
}

void hqcgen_bytes(uint64_t seed, uint32_t tag, uint64_t idx0, size_t rows, uint32_t k,
                  uint32_t stride, uint8_t *out, int nthreads) {
  gjob_t j = {G_BYTES, seed, idx0, tag, k, 0, 0, stride, out, NULL, 0, 0};
  grun(&j, rows, nthreads);
}

void hqcgen_blocks(uint64_t seed, uint32_t tag, uint64_t idx0, size_t rows, uint32_t n1,
                   uint32_t tmin, uint32_t tmax, uint32_t stride, uint8_t *out_t, uint8_t *out_idx,
                   int nthreads) {
  gjob_t j = {G_BLOCKS, seed, idx0, tag, n1, tmin, tmax, stride, out_idx, out_t, 0, 0};
  grun(&j, rows, nthreads);
}

/* dense rows for an explicit list of stream indices (adversarial block bits) */
void hqcgen_dense_idx(uint64_t seed, uint32_t tag, const uint64_t *idx, size_t rows, uint32_t nbits,
                      uint32_t stride, uint64_t *out, int nthreads) {
  gjob_t j = {G_DENSE_IDX, seed, 0, tag, nbits, 0, 0, stride, out, (void *)idx, 0, 0};
  grun(&j, rows, nthreads);
}
