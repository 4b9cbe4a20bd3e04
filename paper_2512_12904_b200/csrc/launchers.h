// Per-level host launchers (defined in hqc_l1.cu, hqc_l3.cu, hqc_l5.cu; dispatched by hqc_gpu.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#define HQC_LEVEL_API(L)                                                                                        \
  int decrypt_l##L(const uint64_t *u, const uint64_t *v, const uint32_t *y, uint8_t *m, size_t batch,            \
                   cudaStream_t st);                                                                            \
  int stage1_l##L(const uint64_t *u, const uint32_t *y, const uint64_t *v, uint64_t *r, size_t batch,            \
                  cudaStream_t st);                                                                             \
  int stage2_l##L(const uint64_t *r, uint8_t *sym, size_t batch, cudaStream_t st);                              \
  int stage3_l##L(const uint8_t *sym, uint8_t *m, uint8_t *ok, size_t batch, cudaStream_t st);                  \
  int keygen_l##L(const uint64_t *h, const uint32_t *x, const uint32_t *y, uint64_t *s, size_t nkeys,           \
                  cudaStream_t st);                                                                             \
  int encrypt_l##L(const uint64_t *h, const uint64_t *s, const uint32_t *key, const uint8_t *m,                \
                   const uint32_t *r1, const uint32_t *r2, const uint32_t *e, uint64_t *u, uint64_t *v,        \
                   size_t batch, cudaStream_t st);                                                              \
  int shape_l##L(size_t batch, int *grid, int *wpc);                                                            \
  int kind_l##L(size_t batch);                                                                                  \
  long long nlaunch_l##L(size_t batch);                                                                         \
  int syndromes_l##L(const uint8_t *sym, uint8_t *syn, size_t batch, int method, cudaStream_t st);              \
  size_t kem_ws_l##L(size_t batch);                                                                             \
  int kem_keygen_l##L(const uint8_t *seeds, uint64_t *h, uint32_t *x, uint32_t *y, uint64_t *s, uint8_t *sigma,    \
                      uint8_t *hpk, size_t nkeys, cudaStream_t st);                                             \
  int kem_hpk_l##L(const uint64_t *h, const uint64_t *s, uint8_t *hpk, size_t nkeys, cudaStream_t st);          \
  int kem_encaps_l##L(const uint64_t *h, const uint64_t *s, const uint8_t *hpk, const uint32_t *key,            \
                      const uint8_t *m, uint64_t *u, uint64_t *v, uint8_t *K, size_t batch, void *ws,           \
                      cudaStream_t st);                                                                         \
  int kem_decaps_l##L(const uint64_t *h, const uint64_t *s, const uint8_t *hpk, const uint8_t *sigma,           \
                      const uint32_t *key, const uint32_t *y, const uint64_t *u, const uint64_t *v, uint8_t *K, \
                      uint8_t *acc, size_t batch, void *ws, cudaStream_t st);

namespace hqc {
HQC_LEVEL_API(1)
HQC_LEVEL_API(3)
HQC_LEVEL_API(5)
}  // namespace hqc
