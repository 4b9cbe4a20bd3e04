// libhqcgpu.so — C ABI (include/hqc_gpu.h): validation and per-level dispatch. The kernels live in
// kernels.cuh and are instantiated per level in hqc_l1.cu / hqc_l3.cu / hqc_l5.cu.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "../../include/hqc_gpu.h"
#include "launchers.h"
#include "levels.cuh"

namespace hqc {
__global__ void k_count_mismatch(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, uint32_t k,
                                 size_t batch, unsigned long long *count) {
  unsigned long long local = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < batch; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t diff = 0;
    for (uint32_t j = 0; j < k; j++) diff |= a[i * k + j] ^ b[i * k + j];
    local += diff != 0;
  }
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

__global__ void k_validate_support(const uint32_t *__restrict__ y, uint32_t n, uint32_t w, uint32_t stride,
                                   size_t batch, unsigned long long *bad) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < batch; i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t *row = y + i * stride;
    bool b = false;
    for (uint32_t j = 0; j < w; j++) {
      const uint32_t x = row[j];
      b |= x >= n;
      for (uint32_t t = 0; t < j; t++) b |= row[t] == x;
    }
    if (b) atomicAdd(bad, 1ull);
  }
}

// Serialized ciphertexts (c = u bytes (ceil(n/8)) || v bytes (n1 n2 / 8)) -> the ABI rows of
// hqc_decrypt_batch: u [u_stride] and v [v_words] 64-bit words, and the ciphertext's key support row
// from the device-resident key table. One warp per ciphertext; the byte stream has arbitrary alignment,
// so each 32-bit word is a funnel shift of two aligned source words.
__global__ void k_unpack_ct(const uint8_t *__restrict__ ct, size_t ct_bytes, uint32_t ub, uint32_t vb,
                            uint32_t u_words32, uint32_t v_words32, const uint32_t *__restrict__ key,
                            const uint32_t *__restrict__ y_keys, uint32_t nkeys, uint32_t y_stride,
                            uint32_t *__restrict__ u_out, uint32_t *__restrict__ v_out, uint32_t *__restrict__ y_out,
                            size_t n) {
  const int lane = threadIdx.x & 31;
  const size_t nw = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t stride = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t c = nw; c < n; c += stride) {
    const size_t b0 = c * ct_bytes;
    auto row = [&](size_t off, uint32_t nbytes, uint32_t nwords, uint32_t *dst) {
      const size_t a = b0 + off;
      const uint32_t *src = reinterpret_cast<const uint32_t *>(ct + (a & ~(size_t)3));
      const uint32_t sh = 8u * (uint32_t)(a & 3);
      const uint32_t last = (nbytes + 3) / 4;  // source words that carry row bytes
      for (uint32_t q = lane; q < nwords; q += 32) {
        uint32_t w = 0;
        if (q < last) {
          const uint32_t lo = src[q];
          const uint32_t hi = (4 * (q + 1) < nbytes + (sh >> 3)) ? src[q + 1] : 0u;
          w = __funnelshift_r(lo, hi, sh);
          if (4 * (q + 1) > nbytes) w &= 0xFFFFFFFFu >> (8 * (4 * (q + 1) - nbytes));  // bytes past the row
        }
        dst[q] = w;
      }
    };
    row(0, ub, u_words32, u_out + c * u_words32);
    row(ub, vb, v_words32, v_out + c * v_words32);
    uint32_t k = key ? key[c] : 0u;
    k = k < nkeys ? k : nkeys - 1;  // checked on the host before the launch; clamped for memory safety only
    for (uint32_t q = lane; q < y_stride; q += 32) y_out[c * y_stride + q] = y_keys[(size_t)k * y_stride + q];
  }
}

}  // namespace hqc

// ================================================================================================
// C ABI
using namespace hqc;

template <int L> static void fill_params(hqc_params *o) {
  using P = Lv<L>;
  o->level = L;
  o->n = P::N; o->n1 = P::N1; o->n2 = P::N2; o->mult = P::MULT; o->k = P::K; o->delta = P::DELTA;
  o->w = P::W; o->wr = P::WR; o->n12 = P::N12; o->u_words = P::U_WORDS; o->u_stride = P::U_STRIDE;
  o->v_words = P::V_WORDS; o->y_stride = P::Y_STRIDE; o->e_stride = P::E_STRIDE;
}

extern "C" int hqc_get_params(int level, hqc_params *out) {
  if (!out) return HQC_ERR_NULL;
  switch (level) {
    case 1: fill_params<1>(out); return HQC_OK;
    case 3: fill_params<3>(out); return HQC_OK;
    case 5: fill_params<5>(out); return HQC_OK;
    default: return HQC_ERR_LEVEL;
  }
}

extern "C" const char *hqc_status_str(int s) {
  switch (s) {
    case HQC_OK: return "ok";
    case HQC_ERR_LEVEL: return "unknown parameter level";
    case HQC_ERR_NULL: return "null pointer";
    case HQC_ERR_ALIGN: return "pointer not 16-byte aligned";
    case HQC_ERR_SIZE: return "batch too large";
    case HQC_ERR_CUDA: return "CUDA launch error";
    default: return "unknown status";
  }
}

static int check_level(const hqc_params *p) {
  if (!p) return HQC_ERR_NULL;
  if (p->level != 1 && p->level != 3 && p->level != 5) return HQC_ERR_LEVEL;
  return HQC_OK;
}
static bool misaligned(const void *q) { return (reinterpret_cast<uintptr_t>(q) & 15u) != 0; }

#define HQC_CHECK_PTR(q)                 \
  do {                                   \
    if (!(q)) return HQC_ERR_NULL;       \
    if (misaligned(q)) return HQC_ERR_ALIGN; \
  } while (0)

// Clear a launch error left pending by earlier, unrelated work, so that the cudaGetLastError after this
// call's launches reports this call only (a sticky error, i.e. a dead context, persists and is reported).
#define HQC_DISPATCH(p, fn, ...)                                 \
  (void)cudaGetLastError();                                      \
  switch ((p)->level) {                                          \
    case 1: return fn##_l1(__VA_ARGS__);                         \
    case 3: return fn##_l3(__VA_ARGS__);                         \
    default: return fn##_l5(__VA_ARGS__);                        \
  }

extern "C" int hqc_decrypt_batch(const hqc_params *p, const uint64_t *u, const uint64_t *v,
                                 const uint32_t *y, uint8_t *m, size_t batch, void *stream) {
  int s = check_level(p);
  if (s) return s;
  if (batch == 0) return HQC_OK;
  if (batch > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(u); HQC_CHECK_PTR(v); HQC_CHECK_PTR(y); HQC_CHECK_PTR(m);
  HQC_DISPATCH(p, decrypt, u, v, y, m, batch, (cudaStream_t)stream);
}

extern "C" int hqc_sparse_dense_mul_batch(const hqc_params *p, const uint64_t *u, const uint32_t *y,
                                          const uint64_t *v, uint64_t *r, size_t batch, void *stream) {
  int s = check_level(p);
  if (s) return s;
  if (batch == 0) return HQC_OK;
  if (batch > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(u); HQC_CHECK_PTR(y); HQC_CHECK_PTR(r);
  if (v && misaligned(v)) return HQC_ERR_ALIGN;
  HQC_DISPATCH(p, stage1, u, y, v, r, batch, (cudaStream_t)stream);
}

extern "C" int hqc_rm_decode_batch(const hqc_params *p, const uint64_t *r, uint8_t *sym, size_t batch,
                                   void *stream) {
  int s = check_level(p);
  if (s) return s;
  if (batch == 0) return HQC_OK;
  if (batch > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(r); HQC_CHECK_PTR(sym);
  HQC_DISPATCH(p, stage2, r, sym, batch, (cudaStream_t)stream);
}

extern "C" int hqc_rs_decode_batch_ex(const hqc_params *p, const uint8_t *sym, uint8_t *m, uint8_t *ok,
                                      size_t batch, void *stream) {
  int s = check_level(p);
  if (s) return s;
  if (batch == 0) return HQC_OK;
  if (batch > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(sym); HQC_CHECK_PTR(m);
  if (ok && misaligned(ok)) return HQC_ERR_ALIGN;
  HQC_DISPATCH(p, stage3, sym, m, ok, batch, (cudaStream_t)stream);
}

extern "C" int hqc_rs_decode_batch(const hqc_params *p, const uint8_t *sym, uint8_t *m, size_t batch,
                                   void *stream) {
  return hqc_rs_decode_batch_ex(p, sym, m, nullptr, batch, stream);
}

extern "C" int hqc_rs_syndromes_batch(const hqc_params *p, const uint8_t *sym, uint8_t *syn_out, size_t batch,
                                      int method, void *stream) {
  int s = check_level(p);
  if (s) return s;
  if (method < 0 || method > 2) return HQC_ERR_SIZE;
  if (batch == 0) return HQC_OK;
  if (batch > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(sym); HQC_CHECK_PTR(syn_out);
  HQC_DISPATCH(p, syndromes, sym, syn_out, batch, method, (cudaStream_t)stream);
}

extern "C" int hqc_count_mismatch(const hqc_params *p, const uint8_t *a, const uint8_t *b, size_t batch,
                                  unsigned long long *count, void *stream) {
  int s = check_level(p);
  if (s) return s;
  if (batch == 0) return HQC_OK;
  HQC_CHECK_PTR(a); HQC_CHECK_PTR(b); HQC_CHECK_PTR(count);
  (void)cudaGetLastError();
  size_t grid = (batch + 255) / 256;
  if (grid > 4096) grid = 4096;
  k_count_mismatch<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a, b, p->k, batch, count);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

extern "C" int hqc_validate_support(const hqc_params *p, const uint32_t *y, size_t batch,
                                    unsigned long long *bad, void *stream) {
  int s = check_level(p);
  if (s) return s;
  if (batch == 0) return HQC_OK;
  HQC_CHECK_PTR(y); HQC_CHECK_PTR(bad);
  (void)cudaGetLastError();
  size_t grid = (batch + 255) / 256;
  if (grid > 4096) grid = 4096;
  k_validate_support<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(y, p->n, p->w, p->y_stride, batch, bad);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

extern "C" int hqc_decrypt_launch_shape(const hqc_params *p, size_t batch, int *grid, int *wpc) {
  int s = check_level(p);
  if (s) return s;
  if (!grid || !wpc) return HQC_ERR_NULL;
  HQC_DISPATCH(p, shape, batch, grid, wpc);
}

extern "C" int hqc_decrypt_launch_kernel(const hqc_params *p, size_t batch) {
  int s = check_level(p);
  if (s) return s;
  HQC_DISPATCH(p, kind, batch);
}

extern "C" long long hqc_decrypt_launch_count(const hqc_params *p, size_t batch) {
  int s = check_level(p);
  if (s) return s;
  HQC_DISPATCH(p, nlaunch, batch);
}

extern "C" int hqc_keygen_batch(const hqc_params *p, const uint64_t *h, const uint32_t *x, const uint32_t *y,
                                uint64_t *s_out, size_t nkeys, void *stream) {
  int st = check_level(p);
  if (st) return st;
  if (nkeys == 0) return HQC_OK;
  if (nkeys > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(h); HQC_CHECK_PTR(x); HQC_CHECK_PTR(y); HQC_CHECK_PTR(s_out);
  HQC_DISPATCH(p, keygen, h, x, y, s_out, nkeys, (cudaStream_t)stream);
}

extern "C" int hqc_encrypt_batch(const hqc_params *p, const uint64_t *h, const uint64_t *s,
                                 const uint32_t *key_index, const uint8_t *m, const uint32_t *r1,
                                 const uint32_t *r2, const uint32_t *e, uint64_t *u_out, uint64_t *v_out,
                                 size_t batch, void *stream) {
  int st = check_level(p);
  if (st) return st;
  if (batch == 0) return HQC_OK;
  if (batch > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(h); HQC_CHECK_PTR(s); HQC_CHECK_PTR(m); HQC_CHECK_PTR(r1); HQC_CHECK_PTR(r2);
  HQC_CHECK_PTR(e); HQC_CHECK_PTR(u_out); HQC_CHECK_PTR(v_out);
  if (key_index && misaligned(key_index)) return HQC_ERR_ALIGN;
  HQC_DISPATCH(p, encrypt, h, s, key_index, m, r1, r2, e, u_out, v_out, batch, (cudaStream_t)stream);
}

// ---- KEM row: kem.cuh
extern "C" size_t hqc_kem_workspace_bytes(const hqc_params *p, size_t batch) {
  if (check_level(p)) return 0;
  switch (p->level) {
    case 1: return kem_ws_l1(batch);
    case 3: return kem_ws_l3(batch);
    default: return kem_ws_l5(batch);
  }
}

extern "C" int hqc_kem_hpk_batch(const hqc_params *p, const uint64_t *h, const uint64_t *s, uint8_t *hpk_out,
                                 size_t nkeys, void *stream) {
  int st = check_level(p);
  if (st) return st;
  if (nkeys == 0) return HQC_OK;
  if (nkeys > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(h); HQC_CHECK_PTR(s); HQC_CHECK_PTR(hpk_out);
  HQC_DISPATCH(p, kem_hpk, h, s, hpk_out, nkeys, (cudaStream_t)stream);
}

extern "C" int hqc_kem_keygen_batch(const hqc_params *p, const uint8_t *seeds, uint64_t *h_out, uint32_t *x_out,
                                    uint32_t *y_out, uint64_t *s_out, uint8_t *sigma_out, uint8_t *hpk_out,
                                    size_t nkeys, void *stream) {
  int st = check_level(p);
  if (st) return st;
  if (nkeys == 0) return HQC_OK;
  if (nkeys > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(seeds); HQC_CHECK_PTR(h_out); HQC_CHECK_PTR(x_out); HQC_CHECK_PTR(y_out); HQC_CHECK_PTR(s_out);
  HQC_CHECK_PTR(sigma_out);
  if (hpk_out && misaligned(hpk_out)) return HQC_ERR_ALIGN;
  HQC_DISPATCH(p, kem_keygen, seeds, h_out, x_out, y_out, s_out, sigma_out, hpk_out, nkeys, (cudaStream_t)stream);
}

extern "C" int hqc_kem_encaps_batch(const hqc_params *p, const uint64_t *h, const uint64_t *s, const uint8_t *hpk,
                                    const uint32_t *key_index, const uint8_t *m, uint64_t *u_out, uint64_t *v_out,
                                    uint8_t *K_out, size_t batch, void *d_work, size_t work_bytes, void *stream) {
  int st = check_level(p);
  if (st) return st;
  if (batch == 0) return HQC_OK;
  if (batch > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(h); HQC_CHECK_PTR(s); HQC_CHECK_PTR(hpk); HQC_CHECK_PTR(m); HQC_CHECK_PTR(u_out);
  HQC_CHECK_PTR(v_out); HQC_CHECK_PTR(K_out); HQC_CHECK_PTR(d_work);
  if (key_index && misaligned(key_index)) return HQC_ERR_ALIGN;
  if (work_bytes < hqc_kem_workspace_bytes(p, batch)) return HQC_ERR_SIZE;
  HQC_DISPATCH(p, kem_encaps, h, s, hpk, key_index, m, u_out, v_out, K_out, batch, d_work, (cudaStream_t)stream);
}

extern "C" int hqc_kem_decaps_batch(const hqc_params *p, const uint64_t *h, const uint64_t *s, const uint8_t *hpk,
                                    const uint8_t *sigma, const uint32_t *key_index, const uint32_t *y_support,
                                    const uint64_t *u, const uint64_t *v, uint8_t *K_out, uint8_t *accepted_out,
                                    size_t batch, void *d_work, size_t work_bytes, void *stream) {
  int st = check_level(p);
  if (st) return st;
  if (batch == 0) return HQC_OK;
  if (batch > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  HQC_CHECK_PTR(h); HQC_CHECK_PTR(s); HQC_CHECK_PTR(hpk); HQC_CHECK_PTR(sigma); HQC_CHECK_PTR(y_support);
  HQC_CHECK_PTR(u); HQC_CHECK_PTR(v); HQC_CHECK_PTR(K_out); HQC_CHECK_PTR(d_work);
  if (key_index && misaligned(key_index)) return HQC_ERR_ALIGN;
  if (work_bytes < hqc_kem_workspace_bytes(p, batch)) return HQC_ERR_SIZE;
  HQC_DISPATCH(p, kem_decaps, h, s, hpk, sigma, key_index, y_support, u, v, K_out, accepted_out, batch, d_work,
               (cudaStream_t)stream);
}

// ---- the host-buffer entry points' internal streams and events, created once per device (on first use)
// and kept for the process: a per-call create/destroy costs driver calls on every request.
struct HostPipe {
  cudaStream_t st[2] = {nullptr, nullptr};
  cudaEvent_t start = nullptr, done[2] = {nullptr, nullptr};
  bool ready = false;
};
static std::mutex g_pipe_mu;
static HostPipe g_pipe[16];

// The device's pipe, or null if it cannot be created. The two streams are used by one call at a time:
// g_pipe_mu is held for the whole enqueue of a call (the enqueue is asynchronous and short).
static HostPipe *host_pipe(int *dev_out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  HostPipe &hp = g_pipe[dev];
  if (!hp.ready) {
    if (cudaStreamCreateWithFlags(&hp.st[0], cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&hp.st[1], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&hp.start, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&hp.done[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&hp.done[1], cudaEventDisableTiming) != cudaSuccess)
      return nullptr;
    hp.ready = true;
  }
  *dev_out = dev;
  return &hp;
}

// ---- host-buffer entry point: chunked, double-buffered H2D / decrypt / D2H on two internal streams
static size_t host_row_in(const hqc_params *p) {
  return (size_t)p->u_stride * 8 + (size_t)p->v_words * 8 + (size_t)p->y_stride * 4;
}

extern "C" size_t hqc_decrypt_host_workspace_bytes(const hqc_params *p, size_t chunk) {
  if (check_level(p)) return 0;
  const size_t per = ((size_t)p->u_stride * 8 + 15) / 16 * 16 + ((size_t)p->v_words * 8 + 15) / 16 * 16 +
                     ((size_t)p->y_stride * 4 + 15) / 16 * 16 + ((size_t)p->k + 15) / 16 * 16;
  return 2 * per * chunk + 4 * 256;
}

extern "C" int hqc_decrypt_batch_host(const hqc_params *p, const uint64_t *u_h, const uint64_t *v_h,
                                      const uint32_t *y_h, uint8_t *m_h, size_t batch, void *d_work,
                                      size_t work_bytes, size_t chunk, void *stream) {
  int s = check_level(p);
  if (s) return s;
  if (batch == 0) return HQC_OK;
  if (batch > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  if (!u_h || !v_h || !y_h || !m_h || !d_work) return HQC_ERR_NULL;
  if (misaligned(d_work)) return HQC_ERR_ALIGN;
  if (chunk == 0) chunk = 8192;
  if (chunk > batch) chunk = batch;
  if (work_bytes < hqc_decrypt_host_workspace_bytes(p, chunk)) return HQC_ERR_SIZE;
  (void)host_row_in;
  const size_t ub = (size_t)p->u_stride * 8, vb = (size_t)p->v_words * 8, yb = (size_t)p->y_stride * 4;
  auto r16 = [](size_t x) { return (x + 15) / 16 * 16; };
  uint8_t *base = static_cast<uint8_t *>(d_work);
  uint8_t *buf[2][4];
  for (int b = 0; b < 2; b++) {
    uint8_t *q = base + b * (r16(ub) + r16(vb) + r16(yb) + r16(p->k)) * chunk;
    buf[b][0] = q;
    buf[b][1] = q + r16(ub) * chunk;
    buf[b][2] = buf[b][1] + r16(vb) * chunk;
    buf[b][3] = buf[b][2] + r16(yb) * chunk;
  }
  cudaStream_t caller = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  int dev = 0;
  HostPipe *hp = host_pipe(&dev);
  if (!hp) return HQC_ERR_CUDA;
  (void)cudaGetLastError();
  cudaStream_t *st = hp->st;
  cudaEvent_t start = hp->start, *done = hp->done;
  int rc = HQC_OK;
  {
    cudaEventRecord(start, caller);
    cudaStreamWaitEvent(st[0], start, 0);
    cudaStreamWaitEvent(st[1], start, 0);
    size_t c = 0;
    for (size_t off = 0; off < batch && rc == HQC_OK; off += chunk, c++) {
      const size_t n = batch - off < chunk ? batch - off : chunk;
      const int b = (int)(c & 1);
      cudaStream_t sb = st[b];
      if (cudaMemcpyAsync(buf[b][0], reinterpret_cast<const uint8_t *>(u_h) + off * ub, n * ub,
                          cudaMemcpyHostToDevice, sb) != cudaSuccess ||
          cudaMemcpyAsync(buf[b][1], reinterpret_cast<const uint8_t *>(v_h) + off * vb, n * vb,
                          cudaMemcpyHostToDevice, sb) != cudaSuccess ||
          cudaMemcpyAsync(buf[b][2], reinterpret_cast<const uint8_t *>(y_h) + off * yb, n * yb,
                          cudaMemcpyHostToDevice, sb) != cudaSuccess) {
        rc = HQC_ERR_CUDA;
        break;
      }
      rc = hqc_decrypt_batch(p, reinterpret_cast<const uint64_t *>(buf[b][0]),
                             reinterpret_cast<const uint64_t *>(buf[b][1]),
                             reinterpret_cast<const uint32_t *>(buf[b][2]), buf[b][3], n, (void *)sb);
      if (rc == HQC_OK && cudaMemcpyAsync(m_h + off * p->k, buf[b][3], n * p->k, cudaMemcpyDeviceToHost, sb) !=
                              cudaSuccess)
        rc = HQC_ERR_CUDA;
    }
    cudaEventRecord(done[0], st[0]);
    cudaEventRecord(done[1], st[1]);
    cudaStreamWaitEvent(caller, done[0], 0);
    cudaStreamWaitEvent(caller, done[1], 0);
  }
  return rc;
}

// ---- serialized-ciphertext host entry point (the server-side call): host c bytes + key indices in,
//      host m out; the keys' supports stay resident on the device
extern "C" size_t hqc_ct_bytes(const hqc_params *p) {
  if (check_level(p)) return 0;
  return ((size_t)p->n + 7) / 8 + (size_t)p->n12 / 8;
}

extern "C" size_t hqc_decrypt_ct_host_workspace_bytes(const hqc_params *p, size_t chunk) {
  if (check_level(p)) return 0;
  auto r16 = [](size_t x) { return (x + 15) / 16 * 16; };
  const size_t per = r16(hqc_ct_bytes(p) * chunk + 8) + r16(4 * chunk) + r16((size_t)p->u_stride * 8 * chunk) +
                     r16((size_t)p->v_words * 8 * chunk) + r16((size_t)p->y_stride * 4 * chunk) +
                     r16((size_t)p->k * chunk);
  return 2 * per;
}

extern "C" int hqc_decrypt_ct_batch_host(const hqc_params *p, const uint8_t *ct_h, const uint32_t *key_h,
                                         const uint32_t *y_keys, size_t nkeys, uint8_t *m_h, size_t batch,
                                         void *d_work, size_t work_bytes, size_t chunk, void *stream) {
  int s = check_level(p);
  if (s) return s;
  if (batch == 0) return HQC_OK;
  if (batch > HQC_MAX_BATCH) return HQC_ERR_SIZE;
  if (!ct_h || !y_keys || !m_h || !d_work) return HQC_ERR_NULL;
  if (nkeys == 0 || (!key_h && nkeys != 1)) return HQC_ERR_SIZE;
  if (misaligned(d_work) || misaligned(y_keys)) return HQC_ERR_ALIGN;
  if (chunk == 0) chunk = 8192;
  if (chunk > batch) chunk = batch;
  if (work_bytes < hqc_decrypt_ct_host_workspace_bytes(p, chunk)) return HQC_ERR_SIZE;
  auto r16 = [](size_t x) { return (x + 15) / 16 * 16; };
  const size_t cb = hqc_ct_bytes(p), ub = ((size_t)p->n + 7) / 8, vb = (size_t)p->n12 / 8;
  const size_t sz[6] = {r16(cb * chunk + 8), r16(4 * chunk), r16((size_t)p->u_stride * 8 * chunk),
                        r16((size_t)p->v_words * 8 * chunk), r16((size_t)p->y_stride * 4 * chunk),
                        r16((size_t)p->k * chunk)};
  uint8_t *buf[2][6];
  uint8_t *q = static_cast<uint8_t *>(d_work);
  for (int b = 0; b < 2; b++)
    for (int i = 0; i < 6; i++) {
      buf[b][i] = q;
      q += sz[i];
    }
  if (key_h)  // key indices are host data here: checked before anything is enqueued
    for (size_t i = 0; i < batch; i++)
      if (key_h[i] >= nkeys) return HQC_ERR_SIZE;
  cudaStream_t caller = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  int dev = 0, sms = 148;
  HostPipe *hp = host_pipe(&dev);
  if (!hp) return HQC_ERR_CUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  (void)cudaGetLastError();
  cudaStream_t *st = hp->st;
  cudaEvent_t start = hp->start, *done = hp->done;
  int rc = HQC_OK;
  {
    cudaEventRecord(start, caller);
    cudaStreamWaitEvent(st[0], start, 0);
    cudaStreamWaitEvent(st[1], start, 0);
    size_t c = 0;
    for (size_t off = 0; off < batch && rc == HQC_OK; off += chunk, c++) {
      const size_t n = batch - off < chunk ? batch - off : chunk;
      const int b = (int)(c & 1);
      cudaStream_t sb = st[b];
      if (cudaMemcpyAsync(buf[b][0], ct_h + off * cb, n * cb, cudaMemcpyHostToDevice, sb) != cudaSuccess ||
          (key_h && cudaMemcpyAsync(buf[b][1], key_h + off, n * 4, cudaMemcpyHostToDevice, sb) != cudaSuccess)) {
        rc = HQC_ERR_CUDA;
        break;
      }
      size_t grid = (n * 32 + 255) / 256;
      if (grid > (size_t)sms * 8) grid = (size_t)sms * 8;
      k_unpack_ct<<<(unsigned)grid, 256, 0, sb>>>(buf[b][0], cb, (uint32_t)ub, (uint32_t)vb, 2 * p->u_stride,
                                                  2 * p->v_words, key_h ? reinterpret_cast<const uint32_t *>(buf[b][1])
                                                                        : nullptr,
                                                  y_keys, (uint32_t)nkeys, p->y_stride,
                                                  reinterpret_cast<uint32_t *>(buf[b][2]),
                                                  reinterpret_cast<uint32_t *>(buf[b][3]),
                                                  reinterpret_cast<uint32_t *>(buf[b][4]), n);
      if (cudaGetLastError() != cudaSuccess) {
        rc = HQC_ERR_CUDA;
        break;
      }
      rc = hqc_decrypt_batch(p, reinterpret_cast<const uint64_t *>(buf[b][2]),
                             reinterpret_cast<const uint64_t *>(buf[b][3]),
                             reinterpret_cast<const uint32_t *>(buf[b][4]), buf[b][5], n, (void *)sb);
      if (rc == HQC_OK && cudaMemcpyAsync(m_h + off * p->k, buf[b][5], n * p->k, cudaMemcpyDeviceToHost, sb) !=
                              cudaSuccess)
        rc = HQC_ERR_CUDA;
    }
    cudaEventRecord(done[0], st[0]);
    cudaEventRecord(done[1], st[1]);
    cudaStreamWaitEvent(caller, done[0], 0);
    cudaStreamWaitEvent(caller, done[1], 0);
  }
  return rc;
}
