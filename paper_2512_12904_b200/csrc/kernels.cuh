// Kernel templates + host launchers of libhqcgpu.so, instantiated once per parameter level in
// hqc_l1.cu / hqc_l3.cu / hqc_l5.cu (each level has its own constant bank for its GF(2)-linear tables).
// DESIGN.md §6 describes each kernel.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "../../include/hqc_gpu.h"
#include "async_copy.cuh"
#include "encrypt.cuh"
#include "gf256.cuh"
#include "levels.cuh"
#include "stage1.cuh"
#include "stage2.cuh"
#include "stage3.cuh"

namespace hqc {

// ------------------------------------------------------------------------------------------------
// Shared-memory carve-up of the fused / stage-1 kernels (per warp), 16-byte aligned pieces.
template <class P> struct WarpSmem {
  static constexpr uint32_t E_BYTES = round_up(
      (DecShape<P>::E_WORDS * 4 > S3Scratch<P>::BYTES ? DecShape<P>::E_WORDS * 4 : S3Scratch<P>::BYTES), 16);
  static constexpr uint32_t UB = P::U_STRIDE * 8, VB = P::V_WORDS * 8, YB = P::Y_STRIDE * 4;
  static_assert(UB % 16 == 0 && VB % 16 == 0 && YB % 16 == 0, "TMA bulk copies move 16-byte multiples");
  static constexpr uint32_t STG_UV_BYTES = round_up(UB > VB ? UB : VB, 16);
  static constexpr uint32_t STG_BYTES = STG_UV_BYTES + round_up(YB, 16);
  static constexpr uint32_t D_BYTES = round_up(DecShape<P>::WPAD * 4, 16);
  static constexpr uint32_t SYM_BYTES = round_up(P::N1 * 32, 16);
  static constexpr uint32_t BAR_BYTES = 16;
  static constexpr uint32_t S1_BYTES = E_BYTES + STG_BYTES + D_BYTES + BAR_BYTES;  // stage-1 kernel
  static constexpr uint32_t BYTES = S1_BYTES + SYM_BYTES;                          // fused kernel
};

// Per-warp stage-1 pipeline: rows of ciphertext i+1 are fetched by TMA while ciphertext i is
// computed (u and y during stage 2/3 of ciphertext i, v during its product loop).
template <class P> struct S1Pipe {
  uint32_t *E, *stg_u, *stg_y, *dsm;
  uint64_t *bar;
  uint32_t phase;
  const uint64_t *u, *v;
  const uint32_t *y;

  __device__ __forceinline__ S1Pipe(uint8_t *ws, const uint64_t *u_, const uint64_t *v_, const uint32_t *y_, int lane)
      : u(u_), v(v_), y(y_) {
    using S = WarpSmem<P>;
    E = reinterpret_cast<uint32_t *>(ws);
    stg_u = reinterpret_cast<uint32_t *>(ws + S::E_BYTES);
    stg_y = reinterpret_cast<uint32_t *>(ws + S::E_BYTES + S::STG_UV_BYTES);
    dsm = reinterpret_cast<uint32_t *>(ws + S::E_BYTES + S::STG_BYTES);
    bar = reinterpret_cast<uint64_t *>(ws + S::E_BYTES + S::STG_BYTES + S::D_BYTES);
    phase = 0;
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
  }
  __device__ __forceinline__ void wait() {
    mbar_wait(bar, phase);
    phase ^= 1u;
  }
  __device__ __forceinline__ void issue_uy(size_t ct, int lane) {
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar, WarpSmem<P>::UB + WarpSmem<P>::YB);
      tma_load_1d(stg_u, u + ct * P::U_STRIDE, WarpSmem<P>::UB, bar);
      tma_load_1d(stg_y, y + ct * P::Y_STRIDE, WarpSmem<P>::YB, bar);
    }
  }
  __device__ __forceinline__ void issue_v(size_t ct, int lane) {
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar, WarpSmem<P>::VB);
      tma_load_1d(stg_u, v + ct * P::V_WORDS, WarpSmem<P>::VB, bar);
    }
  }
  // Stage 1 of ciphertext ct (its u, y already requested); leaves r in E; requests next's u, y.
  __device__ __forceinline__ void run(size_t ct, bool has_next, size_t next, int lane) {
    wait();
    using S = DecShape<P>;
    s1_stage_d<P, S>(stg_y, dsm, lane);
    s1_build_E<P, S>(stg_u, E, lane);
    __syncwarp();
    if (v) issue_v(ct, lane);
    uint32_t acc[S::R];
    s1_product<P, S>(E, dsm, acc, lane);
    __syncwarp();  // every lane is done reading E: r overwrites it
    if (v) {
      wait();  // v has landed in the staging buffer during the product loop
      s1_store_r_xor<S>(acc, E, stg_u, lane);
    } else {
      s1_store_r<S>(acc, E, lane);
    }
    __syncwarp();
    if (has_next) issue_uy(next, lane);
  }
};

constexpr uint32_t GF_BYTES = round_up(sizeof(GfTables), 16);

// ------------------------------------------------------------------------------------------------
// K1: stage 1 alone. One warp per ciphertext (grid-stride over warps).
template <class P>
__global__ void __launch_bounds__(128) k_stage1(const uint64_t *__restrict__ u, const uint32_t *__restrict__ y,
                                                const uint64_t *__restrict__ v, uint64_t *__restrict__ r_out,
                                                size_t batch) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  S1Pipe<P> pipe(smem + (size_t)wib * WarpSmem<P>::S1_BYTES, u, v, y, lane);
  const size_t nwarps = (size_t)gridDim.x * (blockDim.x >> 5);
  size_t ct = (size_t)blockIdx.x * (blockDim.x >> 5) + wib;
  if (ct < batch) pipe.issue_uy(ct, lane);
  for (; ct < batch; ct += nwarps) {
    pipe.run(ct, ct + nwarps < batch, ct + nwarps, lane);
    uint4 *dst = reinterpret_cast<uint4 *>(r_out + ct * P::V_WORDS);
    const uint4 *src = reinterpret_cast<const uint4 *>(pipe.E);
    for (uint32_t c = lane; c < P::NW / 4; c += 32) dst[c] = src[c];
    __syncwarp();
  }
}

// K2: stage 2 alone. One thread per RM block.
template <class P>
__global__ void __launch_bounds__(128) k_stage2(const uint64_t *__restrict__ r, uint8_t *__restrict__ sym,
                                                size_t nblocks) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nblocks) return;
  const size_t ct = t / P::N1, j = t % P::N1;
  const uint4 *src = reinterpret_cast<const uint4 *>(r + ct * P::V_WORDS) + j * (P::N2 / 128);
  uint32_t X[P::MULT * 4];
#pragma unroll
  for (int c = 0; c < (int)P::MULT; c++) {
    const uint4 x = __ldg(src + c);
    X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
  }
  sym[t] = (uint8_t)rm_decode_block<P::MULT>(X);
}

// K3: stage 3 alone. One thread per ciphertext; a warp stages its 32 rows of symbols into shared
// memory as [j][lane] so every later access is conflict-free.
template <class P>
__global__ void __launch_bounds__(128) k_stage3(const uint8_t *__restrict__ sym, uint8_t *__restrict__ m_out,
                                                uint8_t *__restrict__ ok_out, size_t batch) {
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  gf_tables_to_smem(gf);
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t *ws = smem + GF_BYTES + (size_t)wib * (S3Scratch<P>::BYTES + round_up(P::N1 * 32, 16));
  uint16_t *scr = reinterpret_cast<uint16_t *>(ws);
  uint8_t *sb = ws + S3Scratch<P>::BYTES;
  const size_t nwarps = (size_t)gridDim.x * (blockDim.x >> 5);
  for (size_t base = ((size_t)blockIdx.x * (blockDim.x >> 5) + wib) * 32; base < batch; base += nwarps * 32) {
    const size_t rows = batch - base < 32 ? batch - base : 32;
    for (uint32_t e = lane; e < 32 * P::N1; e += 32) {  // e = row*N1 + j (coalesced read)
      const uint32_t row = e / P::N1, j = e % P::N1;
      sb[j * 32 + row] = row < rows ? sym[(base + row) * P::N1 + j] : 0;
    }
    __syncwarp();
    const bool act = (size_t)lane < rows;
    auto sym_at = [&](int j) -> uint32_t { return sb[j * 32 + lane]; };
    const uint32_t ok = rs_decode_lane<P>(sym_at, gf, scr, lane, act ? m_out + (base + lane) * P::K : nullptr);
    if (act && ok_out) ok_out[base + lane] = (uint8_t)ok;
    __syncwarp();
  }
}

// K4: fused decrypt, one warp PAIR (one 64-thread CTA) per ciphertext at a time. The pair shares the
// ciphertext's doubled-u copy E: both warps build it, each warp runs the rotate-and-XOR over half of
// the support indices, warp 1 hands its accumulators to warp 0 through shared memory, warp 0 adds v
// and writes r. Stage 2 spreads the n1 RM blocks over the 64 threads; stage 3 decodes a chunk of 64
// ciphertexts, one per thread. Rows of the next ciphertext are fetched by TMA during stage 2/3.
// Sharing E halves the shared memory per warp (more resident warps to hide latency) and lets the two
// warps finish a ciphertext's stage 2 in one round for n1 <= 64.
template <class P> struct PairSmem {
  using S = DecShape<P>;
  static constexpr uint32_t XOFF = round_up(P::NW, 4);  // warp-1 accumulator image, above r in E
  static_assert(XOFF + P::NW <= S::E_WORDS, "the accumulator image fits in E above r");
  static constexpr uint32_t E_BYTES = round_up(
      S::E_WORDS * 4 > 2 * S3Scratch<P>::BYTES ? S::E_WORDS * 4 : 2 * S3Scratch<P>::BYTES, 16);
  static constexpr uint32_t UB = P::U_STRIDE * 8, VB = P::V_WORDS * 8, YB = P::Y_STRIDE * 4;
  static constexpr uint32_t STG_UV_BYTES = round_up(UB > VB ? UB : VB, 16);
  static constexpr uint32_t STG_BYTES = STG_UV_BYTES + round_up(YB, 16);
  static constexpr uint32_t D_BYTES = round_up(S::WPAD * 4, 16);
  static constexpr uint32_t SYM_BYTES = round_up(P::N1 * 64, 16);
  static constexpr uint32_t BYTES = E_BYTES + STG_BYTES + D_BYTES + SYM_BYTES + 16;
  static constexpr uint32_t W0 = (P::W / 2) & ~1u;  // warp 0 takes indices [0, W0), warp 1 [W0, W)
};

template <class P>
__global__ void __launch_bounds__(64) k_decrypt(const uint64_t *__restrict__ u, const uint64_t *__restrict__ v,
                                                const uint32_t *__restrict__ y, uint8_t *__restrict__ m_out,
                                                size_t batch, size_t per) {
  using S = DecShape<P>;
  using M = PairSmem<P>;
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  uint8_t *base_p = smem + GF_BYTES;
  uint32_t *E = reinterpret_cast<uint32_t *>(base_p);
  uint32_t *stg_u = reinterpret_cast<uint32_t *>(base_p + M::E_BYTES);
  uint32_t *stg_y = reinterpret_cast<uint32_t *>(base_p + M::E_BYTES + M::STG_UV_BYTES);
  uint32_t *dsm = reinterpret_cast<uint32_t *>(base_p + M::E_BYTES + M::STG_BYTES);
  uint8_t *sym = base_p + M::E_BYTES + M::STG_BYTES + M::D_BYTES;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sym + M::SYM_BYTES);
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  gf_tables_to_smem(gf);
  if (tid == 0) mbar_init(bar, 1);
  __syncthreads();
  uint32_t phase = 0;
  auto issue_uy = [&](size_t ct) {
    fence_proxy_async_smem();
    mbar_expect_tx(bar, M::UB + M::YB);
    tma_load_1d(stg_u, u + ct * P::U_STRIDE, M::UB, bar);
    tma_load_1d(stg_y, y + ct * P::Y_STRIDE, M::YB, bar);
  };
  const size_t lo = (size_t)blockIdx.x * per;
  const size_t hi = lo + per < batch ? lo + per : batch;
  if (lo < hi && tid == 0) issue_uy(lo);
  const uint32_t j0 = wid ? M::W0 : 0u, j1 = wid ? P::W : M::W0;
  for (size_t base = lo; base < hi; base += 64) {
    const uint32_t rows = (uint32_t)(hi - base < 64 ? hi - base : 64);
    for (uint32_t s = 0; s < rows; s++) {
      const size_t ct = base + s;
      mbar_wait(bar, phase);  // u, y of ct
      phase ^= 1u;
      s1_stage_d<P, S, 64>(stg_y, dsm, tid);
      s1_build_E<P, S, 64>(stg_u, E, tid);
      __syncthreads();
      if (tid == 0) {  // v lands in the staging buffer while the product runs
        fence_proxy_async_smem();
        mbar_expect_tx(bar, M::VB);
        tma_load_1d(stg_u, v + ct * P::V_WORDS, M::VB, bar);
      }
      uint32_t acc[S::R];
      s1_product_range<P, S>(E, dsm, acc, lane, j0, j1);
      __syncthreads();  // both warps are done reading E
      if (wid == 1) s1_store_r<S>(acc, E + M::XOFF, lane);
      __syncthreads();
      mbar_wait(bar, phase);  // v of ct
      phase ^= 1u;
      if (wid == 0) s1_store_r_xor2<S>(acc, E, E + M::XOFF, stg_u, lane);
      __syncthreads();
      if (tid == 0 && ct + 1 < hi) issue_uy(ct + 1);
#ifndef HQC_EXP_SKIP
#define HQC_EXP_SKIP 0  // experiments only (scripts/exp_variants.py): 1 = skip stage 2, 2 = skip stage 3
#endif
      if (!(HQC_EXP_SKIP & 1))
      for (uint32_t j = tid; j < P::N1; j += 64) {  // stage 2: one RM block per thread
        const uint4 *src = reinterpret_cast<const uint4 *>(E) + j * (P::N2 / 128);
        uint32_t X[P::MULT * 4];
#pragma unroll
        for (int c = 0; c < (int)P::MULT; c++) {
          const uint4 x = src[c];
          X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
        }
        sym[j * 64 + s] = (uint8_t)rm_decode_block<P::MULT>(X);
      }
      __syncthreads();
    }
    for (uint32_t e = tid; e < P::N1 * 64; e += 64)
      if ((e & 63) >= rows) sym[e] = 0;
    __syncthreads();
    const uint32_t slot = 32 * wid + lane;
    const bool act = slot < rows;
    auto sym_at = [&](int j) -> uint32_t { return sym[j * 64 + slot]; };
    if (!(HQC_EXP_SKIP & 2))
      rs_decode_lane<P>(sym_at, gf, reinterpret_cast<uint16_t *>(base_p + wid * S3Scratch<P>::BYTES), lane,
                        act ? m_out + (base + slot) * P::K : nullptr);
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------------
// host side
struct DevInfo {
  int sms = 0;
  int cap_decrypt[6] = {0};  // resident CTAs/SM of k_decrypt per level
  int cap_stage1[6] = {0};
  bool ready[6] = {false};
};

static std::mutex g_mu;
static DevInfo g_dev[16];

constexpr int WARPS_PER_CTA = 1;  // stage-1 kernel: one warp per CTA (fine-grained SM balance)
constexpr int DEC_THREADS = 64;   // fused kernel: one warp pair per CTA

template <class P> static uint32_t decrypt_smem() { return GF_BYTES + PairSmem<P>::BYTES; }
template <class P> static uint32_t stage1_smem() { return WARPS_PER_CTA * WarpSmem<P>::S1_BYTES; }
template <class P> static uint32_t stage3_smem(int warps) {
  return GF_BYTES + warps * (S3Scratch<P>::BYTES + round_up(P::N1 * 32, 16));
}

template <class P> static cudaError_t prepare(int dev, DevInfo &di) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (di.ready[P::level]) return cudaSuccess;
  cudaError_t e;
  if ((e = cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_decrypt<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, decrypt_smem<P>())) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_stage1<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, stage1_smem<P>())) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_stage3<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, stage3_smem<P>(4))) != cudaSuccess) return e;
  int c = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_decrypt<P>, DEC_THREADS, decrypt_smem<P>())) != cudaSuccess) return e;
  di.cap_decrypt[P::level] = c > 0 ? c : 1;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_stage1<P>, 32 * WARPS_PER_CTA, stage1_smem<P>())) != cudaSuccess) return e;
  di.cap_stage1[P::level] = c > 0 ? c : 1;
  di.ready[P::level] = true;
  return cudaSuccess;
}

static int cur_device(DevInfo **out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return -1;
  *out = &g_dev[dev];
  return dev;
}

// Work split of the fused kernel: every resident CTA (warp pair) gets an equal contiguous range of at
// least MIN_PER ciphertexts (the lane-per-ciphertext RS stage wants full chunks).
constexpr size_t MIN_PER = 32;
template <class P> static void decrypt_shape(DevInfo &di, size_t batch, int *grid, size_t *per) {
  const size_t cap = (size_t)di.sms * di.cap_decrypt[P::level];
  size_t ctas = (batch + MIN_PER - 1) / MIN_PER;
  if (ctas > cap) ctas = cap;
  if (ctas == 0) ctas = 1;
  *per = (batch + ctas - 1) / ctas;
  *grid = (int)((batch + *per - 1) / *per);
}

template <class P>
static int launch_decrypt(const uint64_t *u, const uint64_t *v, const uint32_t *y, uint8_t *m, size_t batch,
                          cudaStream_t st) {
  DevInfo *di;
  const int dev = cur_device(&di);
  if (dev < 0 || prepare<P>(dev, *di) != cudaSuccess) return HQC_ERR_CUDA;
  int grid;
  size_t per;
  decrypt_shape<P>(*di, batch, &grid, &per);
  k_decrypt<P><<<grid, DEC_THREADS, decrypt_smem<P>(), st>>>(u, v, y, m, batch, per);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P>
static int launch_stage1(const uint64_t *u, const uint32_t *y, const uint64_t *v, uint64_t *r, size_t batch,
                         cudaStream_t st) {
  DevInfo *di;
  const int dev = cur_device(&di);
  if (dev < 0 || prepare<P>(dev, *di) != cudaSuccess) return HQC_ERR_CUDA;
  const size_t cap = (size_t)di->sms * di->cap_stage1[P::level];
  size_t grid = (batch + WARPS_PER_CTA - 1) / WARPS_PER_CTA;
  if (grid > cap) grid = cap;
  k_stage1<P><<<(unsigned)grid, 32 * WARPS_PER_CTA, stage1_smem<P>(), st>>>(u, y, v, r, batch);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P> static int launch_stage2(const uint64_t *r, uint8_t *sym, size_t batch, cudaStream_t st) {
  const size_t nb = batch * P::N1;
  const size_t grid = (nb + 127) / 128;
  k_stage2<P><<<(unsigned)grid, 128, 0, st>>>(r, sym, nb);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P>
static int launch_stage3(const uint8_t *sym, uint8_t *m, uint8_t *ok, size_t batch, cudaStream_t st) {
  DevInfo *di;
  const int dev = cur_device(&di);
  if (dev < 0 || prepare<P>(dev, *di) != cudaSuccess) return HQC_ERR_CUDA;
  const int warps = 4;
  size_t grid = (batch + 32 * warps - 1) / (32 * warps);
  const size_t cap = (size_t)di->sms * 16;
  if (grid > cap) grid = cap;
  k_stage3<P><<<(unsigned)grid, 32 * warps, stage3_smem<P>(warps), st>>>(sym, m, ok, batch);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P>
static int launch_keygen(const uint64_t *h, const uint32_t *x, const uint32_t *y, uint64_t *s, size_t nkeys,
                         cudaStream_t st) {
  const uint32_t smem = EncSmem<P>::BYTES;
  if (cudaFuncSetAttribute(k_keygen<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return HQC_ERR_CUDA;
  size_t grid = nkeys < 65535 ? nkeys : 65535;
  k_keygen<P><<<(unsigned)grid, 32, smem, st>>>(h, x, y, s, nkeys);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P>
static int launch_encrypt(const uint64_t *h, const uint64_t *s, const uint32_t *key, const uint8_t *m,
                          const uint32_t *r1, const uint32_t *r2, const uint32_t *e, uint64_t *u, uint64_t *v,
                          size_t batch, cudaStream_t st) {
  const uint32_t smem = EncSmem<P>::BYTES;
  if (cudaFuncSetAttribute(k_encrypt<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return HQC_ERR_CUDA;
  DevInfo *di;
  if (cur_device(&di) < 0) return HQC_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t grid = batch;
  const size_t cap = (size_t)(sms > 0 ? sms : 148) * 16;
  if (grid > cap) grid = cap;
  k_encrypt<P><<<(unsigned)grid, 32, smem, st>>>(h, s, key, m, r1, r2, e, u, v, batch);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P> static int shape_impl(size_t batch, int *grid, int *wpc) {
  DevInfo *di;
  const int dev = cur_device(&di);
  if (dev < 0 || prepare<P>(dev, *di) != cudaSuccess) return HQC_ERR_CUDA;
  size_t per;
  decrypt_shape<P>(*di, batch, grid, &per);
  *wpc = DEC_THREADS / 32;
  return HQC_OK;
}

}  // namespace hqc
