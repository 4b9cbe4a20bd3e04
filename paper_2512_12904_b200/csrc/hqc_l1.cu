// Level-1 instantiation of the kernels (own translation unit: own constant bank).
#define HQC_THIS_LEVEL 1
#include "kernels.cuh"
#include "kem.cuh"
#include "syndromes.cuh"
#include "launchers.h"

namespace hqc {
using PL = Lv<1>;
int decrypt_l1(const uint64_t *u, const uint64_t *v, const uint32_t *y, uint8_t *m, size_t batch, cudaStream_t st) {
  return launch_decrypt<PL>(u, v, y, m, batch, st);
}
int stage1_l1(const uint64_t *u, const uint32_t *y, const uint64_t *v, uint64_t *r, size_t batch, cudaStream_t st) {
  return launch_stage1<PL>(u, y, v, r, batch, st);
}
int stage2_l1(const uint64_t *r, uint8_t *sym, size_t batch, cudaStream_t st) { return launch_stage2<PL>(r, sym, batch, st); }
int stage3_l1(const uint8_t *sym, uint8_t *m, uint8_t *ok, size_t batch, cudaStream_t st) {
  return launch_stage3<PL>(sym, m, ok, batch, st);
}
int keygen_l1(const uint64_t *h, const uint32_t *x, const uint32_t *y, uint64_t *s, size_t nkeys, cudaStream_t st) {
  return launch_keygen<PL>(h, x, y, s, nkeys, st);
}
int encrypt_l1(const uint64_t *h, const uint64_t *s, const uint32_t *key, const uint8_t *m, const uint32_t *r1,
                const uint32_t *r2, const uint32_t *e, uint64_t *u, uint64_t *v, size_t batch, cudaStream_t st) {
  return launch_encrypt<PL>(h, s, key, m, r1, r2, e, u, v, batch, st);
}
int syndromes_l1(const uint8_t *sym, uint8_t *syn, size_t batch, int method, cudaStream_t st) {
  return launch_syndromes<PL>(sym, syn, batch, method, st);
}
int shape_l1(size_t batch, int *grid, int *wpc) { return shape_impl<PL>(batch, grid, wpc); }
int kind_l1(size_t batch) { return kind_impl<PL>(batch); }
long long nlaunch_l1(size_t batch) { return nlaunch_impl<PL>(batch); }
size_t kem_ws_l1(size_t batch) { return kem_ws_bytes<PL>(batch); }
int kem_keygen_l1(const uint8_t *seeds, uint64_t *h, uint32_t *x, uint32_t *y, uint64_t *s, uint8_t *sigma,
                   uint8_t *hpk, size_t nkeys, cudaStream_t st) {
  return launch_kem_keygen<PL>(seeds, h, x, y, s, sigma, hpk, nkeys, st);
}
int kem_hpk_l1(const uint64_t *h, const uint64_t *s, uint8_t *hpk, size_t nkeys, cudaStream_t st) {
  return launch_kem_hpk<PL>(h, s, hpk, nkeys, st);
}
int kem_encaps_l1(const uint64_t *h, const uint64_t *s, const uint8_t *hpk, const uint32_t *key, const uint8_t *m,
                   uint64_t *u, uint64_t *v, uint8_t *K, size_t batch, void *ws, cudaStream_t st) {
  return launch_kem_encaps<PL>(h, s, hpk, key, m, u, v, K, batch, ws, st);
}
int kem_decaps_l1(const uint64_t *h, const uint64_t *s, const uint8_t *hpk, const uint8_t *sigma, const uint32_t *key,
                   const uint32_t *y, const uint64_t *u, const uint64_t *v, uint8_t *K, uint8_t *acc, size_t batch,
                   void *ws, cudaStream_t st) {
  return launch_kem_decaps<PL>(h, s, hpk, sigma, key, y, u, v, K, acc, batch, ws, st);
}
}  // namespace hqc
