// Kernel templates + host launchers of libhqcgpu.so, instantiated once per parameter level in
// hqc_l1.cu / hqc_l3.cu / hqc_l5.cu (each level has its own constant bank for its GF(2)-linear tables).
// DESIGN.md §6 describes each kernel.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "../../include/hqc_gpu.h"
#include "async_copy.cuh"
#include "exp_timing.cuh"
#include "encrypt.cuh"
#include "gf256.cuh"
#include "levels.cuh"
#include "stage1.cuh"
#include "stage1_tmem.cuh"
#include "stage2.cuh"
#include "stage3.cuh"
#include "stage3_warp.cuh"

namespace hqc {

#ifdef HQC_EXP_TIMING  // experiments only: per-phase cycle counters (exp_timing.cuh)
#define HQC_CAT2(a, b) a##b
#define HQC_CAT(a, b) HQC_CAT2(a, b)
extern "C" int HQC_CAT(hqc_exp_warp_span_l, HQC_THIS_LEVEL)(unsigned long long *host, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, g_warp_span, sizeof(unsigned long long) * 2 * (n < 8192 ? n : 8192)) ==
                 cudaSuccess ? 0 : -5;
}
extern "C" int HQC_CAT(hqc_exp_phases_l, HQC_THIS_LEVEL)(unsigned long long *host8) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host8, g_phase_cycles, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {0};
  return cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z)) == cudaSuccess ? 0 : -5;
}
#endif


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
  // symbol rows [j][slot] with a 36-byte pitch: 9 words per row (odd), so the stage-2 byte stores of one
  // slot by the lanes j = 0..31 fall in 32 distinct banks (a 32-byte pitch made them 8-way conflicts)
  static constexpr uint32_t SYM_PITCH = 36;
  static constexpr uint32_t SYM_BYTES = round_up(P::N1 * SYM_PITCH, 16);
  static constexpr uint32_t BAR_BYTES = 16;
  static constexpr uint32_t S1_BYTES = E_BYTES + STG_BYTES + D_BYTES + BAR_BYTES;  // stage-1 kernel
  // RM stage over two ciphertexts at a time when n1 leaves a mostly idle last round of 32 lanes
  // (HQC-1: 46 blocks = 32 + 14; 92 = 3 x 32 - 4): the even ciphertext's r waits in R2
#ifndef HQC_PAIR_S2
#define HQC_PAIR_S2 (P::level == 1)
#endif
  static constexpr bool PAIR_S2 = HQC_PAIR_S2;
  static constexpr uint32_t R2_BYTES = PAIR_S2 ? round_up(P::NW * 4, 16) : 0u;
  static constexpr uint32_t BYTES = S1_BYTES + SYM_BYTES + R2_BYTES;               // fused kernel
};

// The one-warp products of S1Pipe with shifted lane windows (stage1.cuh: one SHFL.UP instead of the
// (R+1)-th LDS per index and lane). Measured SLOWER (profiles/r02/ab_shfl.log: standalone product -1.5..-3%,
// fused -0.6..-2.5%): the shuffle is served by the same shared-memory data path it was meant to spare.
// Off; kept as an experiment switch.
#ifndef HQC_S1_SHFL
#define HQC_S1_SHFL 0
#endif

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
  // Stage 1 of ciphertext ct (its u, y already requested); leaves r in rout (default: E, which it may
  // overwrite); requests next's u, y.
  __device__ __forceinline__ void run(size_t ct, bool has_next, size_t next, int lane, uint32_t *rout = nullptr) {
    if (rout == nullptr) rout = E;
    PHASE_T0();
    wait();
    PHASE(1);
    using S = DecShape<P>;    // E and the staged rows
#if HQC_S1_SHFL
    using ST = DecShapeSh<P>;  // shifted lane windows (s1_product_range_sh); words [ST::NOUT, NW) by the tail
    constexpr uint32_t TW = ST::TW;
    static_assert(ST::E_WORDS <= S::E_WORDS, "the shifted windows stay inside E");
#else
    using ST = DecShapeT<P>;  // the lanes' product; words [ST::NOUT, NW) by s1_tail_words
    constexpr uint32_t TW = dec_tail_words<P>();
#endif
    s1_stage_d<P, S>(stg_y, dsm, lane);
    s1_build_E<P, S>(stg_u, E, lane);
    __syncwarp();
    PHASE(2);
    if (v) issue_v(ct, lane);
    else if (has_next) issue_uy(next, lane);  // no v to stage: the next rows land during this product
#if HQC_S1_SEG && !HQC_S1_SHFL
    using G = DecSeg<P>;
    static_assert(S::E_WORDS >= G::E_NEED, "the segmented windows stay inside E");
    uint32_t acc[G::LMAX], top;
    s1_seg_product<P, G, s1_unroll_dec<P>()>(E, dsm, acc, top, lane);
    __syncwarp();  // every lane is done reading E: r overwrites it
    PHASE(3);
    if (v) {
      wait();  // v has landed in the staging buffer during the product loop
      s1_seg_store_xor<G>(acc, top, rout, stg_u, lane);
    } else {
      s1_seg_store<G>(acc, top, rout, lane);
    }
#else
    uint32_t acc[ST::R];
#if HQC_S1_SHFL
    s1_product_range_sh<P, ST>(E, dsm, acc, lane, 0, P::W);
#else
    s1_product<P, ST>(E, dsm, acc, lane);
#endif
    uint32_t mine = 0;  // lane i < TW: word ST::NOUT + i
    if constexpr (TW > 0) {
      uint32_t t[TW];
      s1_tail_words<P, ST, ST::NOUT, TW>(E, dsm, lane, t);
#pragma unroll
      for (uint32_t i = 0; i < TW; i++) mine = (uint32_t)lane == i ? t[i] : mine;
    }
    __syncwarp();  // every lane is done reading E: r overwrites it
    PHASE(3);
    if (v) {
      wait();  // v has landed in the staging buffer during the product loop
#if HQC_S1_SHFL
      s1_store_r_xor_sh<ST>(acc, rout, stg_u, lane);
#else
      s1_store_r_xor<ST>(acc, rout, stg_u, lane);
#endif
      if (TW > 0 && (uint32_t)lane < TW) rout[ST::NOUT + lane] = mine ^ stg_u[ST::NOUT + lane];
    } else {
#if HQC_S1_SHFL
      s1_store_r_sh<ST>(acc, rout, lane);
#else
      s1_store_r<ST>(acc, rout, lane);
#endif
      if (TW > 0 && (uint32_t)lane < TW) rout[ST::NOUT + lane] = mine;
    }
#endif
    __syncwarp();
    PHASE(4);
    if (v && has_next) issue_uy(next, lane);
  }
};

constexpr uint32_t GF_BYTES = round_up(sizeof(GfTables), 16);

constexpr int WARPS_PER_CTA_S1 = 1;  // stage-1 kernel CTA size (warps)

// ------------------------------------------------------------------------------------------------
// K1: stage 1 alone. One warp per ciphertext at a time, on the pipe of k_decrypt_sb (SbPipe, defined with
// it below): u lands by TMA in E's lower half, r is formed in the staging buffer and leaves by a TMA bulk
// store, and the next u is fetched into E as soon as the product has read it. One CTA of G warps per SM
// owns a contiguous range and its warps take products from it through a shared-memory counter (the
// one-warp CTAs of round 1 with strided ranges left each SM a tail of few warps).
#ifndef HQC_S1K_MINB
#define HQC_S1K_MINB 1
#endif
template <class P> struct SbPipe;
template <class P> struct SbPipeSmem;
template <class P> struct S1kSmem {
  static constexpr uint32_t bytes(uint32_t g);
  static constexpr uint32_t fit(uint32_t g);
};
template <class P>
__global__ void __launch_bounds__(512, HQC_S1K_MINB) k_stage1(const uint64_t *__restrict__ u, const uint32_t *__restrict__ y,
                                                const uint64_t *__restrict__ v, uint64_t *__restrict__ r_out,
                                                size_t batch) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t G = blockDim.x >> 5;
  unsigned int *next_item = reinterpret_cast<unsigned int *>(smem);
  SbPipe<P> pipe(smem + 16 + (size_t)wib * SbPipeSmem<P>::BYTES, u, v, y, lane);
  const size_t per_cta = (batch + gridDim.x - 1) / gridDim.x;
  const size_t c0 = (size_t)blockIdx.x * per_cta;
  const size_t c1 = c0 + per_cta < batch ? c0 + per_cta : batch;
  size_t ct = c0 + wib;
  if (ct < c1) pipe.issue_uy(ct, lane);
  if (threadIdx.x == 0) *next_item = G;
  __syncthreads();
  while (ct < c1) {
    uint32_t nx = 0;
    if (lane == 0) nx = atomicAdd(next_item, 1u);
    const size_t nct = c0 + __shfl_sync(0xffffffffu, nx, 0);
    if (lane == 0) tma_store_wait_read();  // the previous r (in the staging buffer) has been read by its store
    __syncwarp();
    pipe.template run<s1_unroll_s1<P>()>(ct, nct < c1, nct, lane);
    fence_proxy_async_smem();  // r -> HBM by a TMA bulk store, asynchronous to the next product
    __syncwarp();
    if (lane == 0) tma_store_1d(r_out + ct * P::V_WORDS, pipe.stg, P::V_WORDS * 8);
    ct = nct;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// E built up to E_WORDS words (an E-build shape with the pair's E size)
template <class P, uint32_t EW> struct EBuildShape {
  static constexpr uint32_t E_WORDS = EW;
};

// K1p: stage 1 alone, WARP PAIR per CTA sharing one E, each warp computing HALF of the output words
// over all support indices (no accumulator hand-off; R = odd ceil(n12/64)). Halving the shared memory
// per warp doubles the resident warps of this shared-memory-bound kernel. The result goes to HBM
// through E (both warps done reading it) with coalesced 16-byte stores.
template <class P> struct S1PairSmem {
  static constexpr uint32_t NWH = P::NW / 2;
  static_assert(P::NW % 2 == 0 && (NWH % 4) == 0, "each half of r is whole 16-byte chunks");
  using S = ProdShape<P, NWH, P::W>;
  static constexpr uint32_t E_WORDS = round_up(P::Q0 + NWH + 32 * S::R + 2, 4);
  static constexpr uint32_t E_BYTES = round_up(E_WORDS * 4, 16);
  static constexpr uint32_t UB = P::U_STRIDE * 8, VB = P::V_WORDS * 8, YB = P::Y_STRIDE * 4;
  static constexpr uint32_t STG_UV_BYTES = round_up(UB > VB ? UB : VB, 16);
  static constexpr uint32_t STG_BYTES = STG_UV_BYTES + round_up(YB, 16);
  static constexpr uint32_t D_BYTES = round_up(S::WPAD * 4, 16);
  static constexpr uint32_t BYTES = E_BYTES + STG_BYTES + D_BYTES + 16;
};

template <class P>
__global__ void __launch_bounds__(64, 1) k_stage1p(const uint64_t *__restrict__ u, const uint32_t *__restrict__ y,
                                                   const uint64_t *__restrict__ v, uint64_t *__restrict__ r_out,
                                                   size_t batch) {
  using M = S1PairSmem<P>;
  using S = typename M::S;
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t *E = reinterpret_cast<uint32_t *>(smem);
  uint32_t *stg_u = reinterpret_cast<uint32_t *>(smem + M::E_BYTES);
  uint32_t *stg_y = reinterpret_cast<uint32_t *>(smem + M::E_BYTES + M::STG_UV_BYTES);
  uint32_t *dsm = reinterpret_cast<uint32_t *>(smem + M::E_BYTES + M::STG_BYTES);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + M::E_BYTES + M::STG_BYTES + M::D_BYTES);
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) mbar_init(bar, 1);
  __syncthreads();
  uint32_t phase = 0;
  auto issue_uy = [&](size_t ct) {
    fence_proxy_async_smem();
    mbar_expect_tx(bar, M::UB + M::YB);
    tma_load_1d(stg_u, u + ct * P::U_STRIDE, M::UB, bar);
    tma_load_1d(stg_y, y + ct * P::Y_STRIDE, M::YB, bar);
  };
  size_t ct = blockIdx.x;
  if (ct < batch && tid == 0) issue_uy(ct);
  for (; ct < batch; ct += gridDim.x) {
    const size_t next = ct + gridDim.x;
    mbar_wait(bar, phase);
    phase ^= 1u;
    s1_stage_d<P, S, 64>(stg_y, dsm, tid);
    s1_build_E<P, EBuildShape<P, M::E_WORDS>, 64>(stg_u, E, tid);
    __syncthreads();
    if (tid == 0) {
      if (v) {  // v lands in the staging buffer during the product
        fence_proxy_async_smem();
        mbar_expect_tx(bar, M::VB);
        tma_load_1d(stg_u, v + ct * P::V_WORDS, M::VB, bar);
      } else if (next < batch) {
        issue_uy(next);
      }
    }
    uint32_t acc[S::R];
    s1_product_range<P, S>(E + wid * M::NWH, dsm, acc, lane, 0, P::W);
    __syncthreads();  // both warps are done reading E
    if (v) {
      mbar_wait(bar, phase);
      phase ^= 1u;
      s1_store_r_xor<S>(acc, E + wid * M::NWH, stg_u + wid * M::NWH, lane);
    } else {
      s1_store_r<S>(acc, E + wid * M::NWH, lane);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {  // r (in E) -> HBM by a TMA bulk store; E is rebuilt only after it has been read
      tma_store_1d(r_out + ct * P::V_WORDS, E, P::V_WORDS * 8);
      if (v && next < batch) issue_uy(next);
      tma_store_wait_read();
    }
    __syncthreads();  // E and the staging buffer are free again
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
// k_stage3's register cap: 4 CTAs of 128 threads per SM (<= 128 registers, no spills; uncapped it took 158
// and 3 CTAs): HQC-5 stage 3 alone 0.84 -> 0.77 ms per 262,144 (profiles/r02/ab_s3.log); 5 CTAs spill.
#ifndef HQC_S3_MINB
#define HQC_S3_MINB 4
#endif
// Experiment: k_stage3's antilog lookups from a lane-replicated table (rs_decode_lane REPL): two CTAs of 8
// warps per SM instead of four of 4 (the 16 KB copy is per CTA).
#ifndef HQC_S3_REPL
#define HQC_S3_REPL 0
#endif
constexpr uint32_t S3_REPL_BYTES = HQC_S3_REPL ? 16384u : 0u;
template <class P>
__global__ void __launch_bounds__(HQC_S3_REPL ? 256 : 128, HQC_S3_REPL ? 2 : HQC_S3_MINB)
    k_stage3(const uint8_t *__restrict__ sym, uint8_t *__restrict__ m_out, uint8_t *__restrict__ ok_out, size_t batch) {
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  gf_tables_to_smem(gf);
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
#if HQC_S3_REPL
  uint8_t *rexp = smem + GF_BYTES;  // EXPT[0..512) replicated per lane: word (e / 4) * 32 + lane
  for (uint32_t w = threadIdx.x; w < 128 * 32; w += blockDim.x)
    reinterpret_cast<uint32_t *>(rexp)[w] = reinterpret_cast<const uint32_t *>(gf->exp)[w >> 5];
  __syncthreads();
#endif
  uint8_t *ws = smem + GF_BYTES + S3_REPL_BYTES + (size_t)wib * (S3Scratch<P>::BYTES + round_up(P::N1 * 32, 16));
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
#if HQC_S3_REPL
    const uint32_t ok = rs_decode_lane<P, decltype(sym_at), true>(sym_at, gf, scr, lane,
                                                                   act ? m_out + (base + lane) * P::K : nullptr, rexp);
#else
    const uint32_t ok = rs_decode_lane<P>(sym_at, gf, scr, lane, act ? m_out + (base + lane) * P::K : nullptr);
#endif
    if (act && ok_out) ok_out[base + lane] = (uint8_t)ok;
    __syncwarp();
  }
}

#ifndef HQC_DEC_MINCTAS  // min resident CTAs (register cap) of the pair kernel, swept in scripts/exp_occ.py
#define HQC_DEC_MINCTAS (P::level == 5 ? 6 : (P::level == 1 ? 14 : 8))
#endif
#ifndef HQC_DEC_MINCTAS_W1
// (HQC-5: shared memory holds 8 one-warp CTAs per SM anyway; a cap of 14 forced 128 registers and spills,
// 8 lets it keep 239: +0.2-0.3%, profiles/r02/ab_w1m.log)
#define HQC_DEC_MINCTAS_W1 (P::level == 5 ? 8 : (P::level == 1 ? 16 : 12))
#endif

// K4a: fused decrypt, one warp per ciphertext (the pair-free variant). Warp g owns ciphertexts
// [g*per, (g+1)*per) in chunks of 32: stage 1 + stage 2 per ciphertext (symbols parked as [j][slot]),
// then stage 3 with one lane per ciphertext of the chunk. Chosen per level by DecPolicy below.
template <class P>
__global__ void __launch_bounds__(32, HQC_DEC_MINCTAS_W1) k_decrypt_w1(const uint64_t *__restrict__ u,
                                                                     const uint64_t *__restrict__ v,
                                                                     const uint32_t *__restrict__ y,
                                                                     uint8_t *__restrict__ m_out, size_t batch,
                                                                     size_t per) {
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  gf_tables_to_smem(gf);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint8_t *ws = smem + GF_BYTES;
  S1Pipe<P> pipe(ws, u, v, y, lane);
  uint8_t *sb = ws + WarpSmem<P>::S1_BYTES;
  uint32_t *R2 = reinterpret_cast<uint32_t *>(sb + WarpSmem<P>::SYM_BYTES);
  const size_t lo = (size_t)blockIdx.x * per;
  const size_t hi = lo + per < batch ? lo + per : batch;
  if (lo < hi) pipe.issue_uy(lo, lane);
  // stage 2 of ciphertexts' RM blocks: t < N1 -> block t of (r0, slot s0); else block t - N1 of (r1, s1)
  auto stage2 = [&](const uint32_t *r0, uint32_t s0, const uint32_t *r1, uint32_t s1, uint32_t nblk) {
    for (uint32_t t = lane; t < nblk; t += 32) {
      const bool second = t >= P::N1;
      const uint32_t j = second ? t - P::N1 : t;
      const uint4 *src = reinterpret_cast<const uint4 *>(second ? r1 : r0) + j * (P::N2 / 128);
      uint32_t X[P::MULT * 4];
#pragma unroll
      for (int c = 0; c < (int)P::MULT; c++) {
        const uint4 x = src[c];
        X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
      }
      sb[j * WarpSmem<P>::SYM_PITCH + (second ? s1 : s0)] = (uint8_t)rm_decode_block<P::MULT>(X);
    }
  };
  for (size_t base = lo; base < hi; base += 32) {
    const uint32_t rows = (uint32_t)(hi - base < 32 ? hi - base : 32);
    for (uint32_t s = 0; s < rows; s++) {
      const size_t ct = base + s;
      if constexpr (WarpSmem<P>::PAIR_S2) {
        if ((s & 1) == 0 && s + 1 < rows) {  // park r in R2; decoded together with the next one
          pipe.run(ct, ct + 1 < hi, ct + 1, lane, R2);
          continue;
        }
        pipe.run(ct, ct + 1 < hi, ct + 1, lane);
        if (s & 1) stage2(R2, s - 1, pipe.E, s, 2 * P::N1);
        else stage2(pipe.E, s, pipe.E, s, P::N1);
      } else {
        pipe.run(ct, ct + 1 < hi, ct + 1, lane);
        stage2(pipe.E, s, pipe.E, s, P::N1);
      }
      __syncwarp();
    }
    for (uint32_t s = rows; s < 32; s++)
      for (uint32_t j = lane; j < P::N1; j += 32) sb[j * WarpSmem<P>::SYM_PITCH + s] = 0;
    __syncwarp();
    const bool act = (uint32_t)lane < rows;
    auto sym_at = [&](int j) -> uint32_t { return sb[j * WarpSmem<P>::SYM_PITCH + lane]; };
    rs_decode_lane<P>(sym_at, gf, reinterpret_cast<uint16_t *>(pipe.E), lane,
                      act ? m_out + (base + lane) * P::K : nullptr);
    __syncwarp();
  }
}


// K4d: K4a (chunks of 32 decryptions per warp, paired RM stage for HQC-1, lane-per-word RS) with the
// warps of a CTA sharing the work: the CTA owns a contiguous range and its G warps take decryptions from it
// one at a time through a shared-memory counter (claimed one ahead for the TMA prefetch), each warp filling
// its own chunk of symbol rows and decoding it when it holds 32 or the range runs out. K4a's one-warp CTAs
// own fixed ranges, and on HQC-1 the SM averaged 13.1 active warps of the 15.8 resident
// (profiles/r02/ncu_fused.md): warps sharing an SM progress at different rates and the early finishers idle.
template <class P> struct WdSmem {
  static constexpr uint32_t IDX_BYTES = 32 * 4;  // the chunk's decryption indices
  static constexpr uint32_t WARP_BYTES = WarpSmem<P>::BYTES + IDX_BYTES;
  static constexpr uint32_t bytes(uint32_t g) { return GF_BYTES + 16 + g * WARP_BYTES; }
  // warps per CTA: at most 16 (512 threads, <= 128 registers), fewer where shared memory runs out
  // (HQC-3: 13 of 16.4 KB, HQC-5: 8 of 26 KB)
  static constexpr uint32_t fit(uint32_t g) { return g > 1 && bytes(g) > 227u * 1024u ? fit(g - 1) : g; }
#ifndef HQC_WD_G
#define HQC_WD_G 16
#endif
  static constexpr uint32_t MAX_G = fit(HQC_WD_G);
};

template <class P>
__global__ void __launch_bounds__(32 * WdSmem<P>::MAX_G, 1) k_decrypt_wd(const uint64_t *__restrict__ u,
                                                                        const uint64_t *__restrict__ v,
                                                                        const uint32_t *__restrict__ y,
                                                                        uint8_t *__restrict__ m_out,
                                                                        size_t batch) {
  using M = WdSmem<P>;
  using W = WarpSmem<P>;
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  unsigned int *next_item = reinterpret_cast<unsigned int *>(smem + GF_BYTES);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t G = blockDim.x >> 5;
  uint8_t *ws = smem + GF_BYTES + 16 + (size_t)wib * M::WARP_BYTES;
  S1Pipe<P> pipe(ws, u, v, y, lane);
  uint8_t *sb = ws + W::S1_BYTES;
  uint32_t *R2 = reinterpret_cast<uint32_t *>(sb + W::SYM_BYTES);
  uint32_t *cidx = reinterpret_cast<uint32_t *>(ws + W::BYTES);
  const size_t per_cta = (batch + gridDim.x - 1) / gridDim.x;
  const size_t c0 = (size_t)blockIdx.x * per_cta;
  const size_t c1 = c0 + per_cta < batch ? c0 + per_cta : batch;
  size_t ct = c0 + wib;
  if (ct < c1) pipe.issue_uy(ct, lane);
  if (threadIdx.x == 0) *next_item = G;
  gf_tables_to_smem(gf);
  __syncthreads();
  auto stage2 = [&](const uint32_t *r0, uint32_t s0, const uint32_t *r1, uint32_t s1, uint32_t nblk) {
    for (uint32_t t = lane; t < nblk; t += 32) {
      const bool second = t >= P::N1;
      const uint32_t j = second ? t - P::N1 : t;
      const uint4 *src = reinterpret_cast<const uint4 *>(second ? r1 : r0) + j * (P::N2 / 128);
      uint32_t X[P::MULT * 4];
#pragma unroll
      for (int c = 0; c < (int)P::MULT; c++) {
        const uint4 x = src[c];
        X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
      }
      sb[j * W::SYM_PITCH + (second ? s1 : s0)] = (uint8_t)rm_decode_block<P::MULT>(X);
    }
  };
  uint32_t s = 0;  // slot of ct in the warp's current chunk
  while (ct < c1) {
    uint32_t nx = 0;
    if (lane == 0) nx = atomicAdd(next_item, 1u);
    const size_t nct = c0 + __shfl_sync(0xffffffffu, nx, 0);
    const bool more = nct < c1;
    if (lane == 0) cidx[s] = (uint32_t)(ct - c0);
    if constexpr (W::PAIR_S2) {
      if ((s & 1) == 0 && s + 1 < 32 && more) {  // park r in R2; decoded together with the next one
        pipe.run(ct, true, nct, lane, R2);
      } else {
        pipe.run(ct, more, nct, lane);
        if (s & 1) stage2(R2, s - 1, pipe.E, s, 2 * P::N1);
        else stage2(pipe.E, s, pipe.E, s, P::N1);
      }
    } else {
      pipe.run(ct, more, nct, lane);
      stage2(pipe.E, s, pipe.E, s, P::N1);
    }
    __syncwarp();
    s++;
    if (s == 32 || !more) {  // the chunk is full, or this warp's last decryption: stage 3, lane per word
      for (uint32_t q = s; q < 32; q++)
        for (uint32_t j = lane; j < P::N1; j += 32) sb[j * W::SYM_PITCH + q] = 0;
      __syncwarp();
      const bool act = (uint32_t)lane < s;
      auto sym_at = [&](int j) -> uint32_t { return sb[j * W::SYM_PITCH + lane]; };
      rs_decode_lane<P>(sym_at, gf, reinterpret_cast<uint16_t *>(pipe.E), lane,
                        act ? m_out + (c0 + cidx[lane]) * P::K : nullptr);
      __syncwarp();
      s = 0;
    }
    ct = nct;
  }
}


// K4l: the lane-per-word RS decoder of K4a/K4d in a COMPACT per-warp layout. K4s (one warp per decryption,
// warp RS) needs a staging buffer for v next to E; K4d (chunks of 32, lane RS) needs the symbol chunk on top
// of K4a's staging buffers — neither leaves room for 16 warps per SM at HQC-3. Here v is not staged: it is
// fetched (TMA) after the product, into the part of E above u's row, which the product no longer needs,
// r is formed there in place, stage 2 reads it there, and the chunk's RS scratch reuses it; meanwhile the
// next u lands below it. Per warp: E, the support row, the rotation amounts, the symbol chunk — HQC-3
// 11.8 KB (16 warps per SM), HQC-5 19.3 KB (11). The CTA's warps share its range through a counter (K4d).
// The v fetch is not hidden behind this warp's product (it cannot land earlier); other warps hide it.
// K4l's v: 1 = not staged — prefetched into L2 when the product starts and XORed into each RM block by
// stage 2 straight from global memory (as in K4c); 0 = fetched by TMA after the product into the region
// above u's row, where r is then formed in place. Measured (profiles/r02/ab_vl2.log): 65,536 +0.2%,
// 262,144 +0.8%, 4,194,304 -1.2% with 1 — no clear gain, so 0 (an experiment switch).
#ifndef HQC_WL_VL2
#define HQC_WL_VL2 0
#endif
template <class P> struct WlSmem {
  using S = DecShape<P>;
  static constexpr uint32_t UB = P::U_STRIDE * 8, VB = P::V_WORDS * 8, YB = P::Y_STRIDE * 4;
  static constexpr uint32_t RB = VB > S3Scratch<P>::BYTES ? VB : S3Scratch<P>::BYTES;  // v, r, RS scratch
  static constexpr uint32_t E_BYTES = round_up(S::E_WORDS * 4 > UB + RB ? S::E_WORDS * 4 : UB + RB, 16);
  static constexpr uint32_t Y_BYTES = round_up(YB, 16);
  static constexpr uint32_t D_BYTES = round_up(S::WPAD * 4, 16);
  static constexpr uint32_t SYM_PITCH = 36;
  static constexpr uint32_t SYM_BYTES = round_up(P::N1 * SYM_PITCH, 16);
  static constexpr uint32_t IDX_BYTES = 32 * 4;
  static constexpr uint32_t WARP_BYTES = E_BYTES + Y_BYTES + D_BYTES + SYM_BYTES + IDX_BYTES + 16;
  static constexpr uint32_t bytes(uint32_t g) { return GF_BYTES + 16 + g * WARP_BYTES; }
  static constexpr uint32_t fit(uint32_t g) { return g > 1 && bytes(g) > 227u * 1024u ? fit(g - 1) : g; }
  static constexpr uint32_t MAX_G = fit(16);
  static_assert(UB % 16 == 0, "the v / r region starts 16-byte aligned above u's row");
};

// DYNAMIC = false: each warp owns a contiguous share of the CTA's range instead (warps stay in phase, as in
// K4a — what HQC-5's 8.6k-instruction kernel prefers, profiles/r02/ab_wd5.log).
template <class P, bool DYNAMIC = true>
__global__ void __launch_bounds__(32 * WlSmem<P>::MAX_G, 1) k_decrypt_wl(const uint64_t *__restrict__ u,
                                                                        const uint64_t *__restrict__ v,
                                                                        const uint32_t *__restrict__ y,
                                                                        uint8_t *__restrict__ m_out,
                                                                        size_t batch) {
  using M = WlSmem<P>;
  using S = DecShape<P>;
  using ST = DecShapeT<P>;
  constexpr uint32_t TW = dec_tail_words<P>();
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  unsigned int *next_item = reinterpret_cast<unsigned int *>(smem + GF_BYTES);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t G = blockDim.x >> 5;
  uint8_t *ws = smem + GF_BYTES + 16 + (size_t)wib * M::WARP_BYTES;
  uint32_t *E = reinterpret_cast<uint32_t *>(ws);
  uint32_t *Rv = reinterpret_cast<uint32_t *>(ws + M::UB);  // v, then r, then the RS scratch
  uint32_t *stg_y = reinterpret_cast<uint32_t *>(ws + M::E_BYTES);
  uint32_t *dsm = reinterpret_cast<uint32_t *>(ws + M::E_BYTES + M::Y_BYTES);
  uint8_t *sb = ws + M::E_BYTES + M::Y_BYTES + M::D_BYTES;
  uint32_t *cidx = reinterpret_cast<uint32_t *>(sb + M::SYM_BYTES);
  uint64_t *bar = reinterpret_cast<uint64_t *>(sb + M::SYM_BYTES + M::IDX_BYTES);  // [0] u, y  [1] v
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncwarp();
  auto issue_uy = [&](size_t c) {
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar, M::UB + M::YB);
      tma_load_1d(E, u + c * P::U_STRIDE, M::UB, bar);
      tma_load_1d(stg_y, y + c * P::Y_STRIDE, M::YB, bar);
    }
  };
  const size_t per_cta = (batch + gridDim.x - 1) / gridDim.x;
  size_t c0 = (size_t)blockIdx.x * per_cta;
  size_t c1 = c0 + per_cta < batch ? c0 + per_cta : batch;
  const size_t cbase = c0;  // chunk indices are relative to the CTA's range
  if constexpr (!DYNAMIC) {  // this warp's contiguous share
    const size_t n = c1 > c0 ? c1 - c0 : 0, pw = (n + G - 1) / G;
    const size_t w0 = c0 + (size_t)wib * pw;
    c0 = w0 < c1 ? w0 : c1;
    c1 = c0 + pw < c1 ? c0 + pw : c1;
  }
  size_t ct = DYNAMIC ? c0 + wib : c0;
  if (ct < c1) issue_uy(ct);
  if (threadIdx.x == 0) *next_item = G;
  gf_tables_to_smem(gf);
  __syncthreads();
  uint32_t ph_uy = 0, ph_v = 0, slot = 0;
  while (ct < c1) {
    size_t nct = ct + 1;
    if constexpr (DYNAMIC) {
      uint32_t nx = 0;
      if (lane == 0) nx = atomicAdd(next_item, 1u);
      nct = c0 + __shfl_sync(0xffffffffu, nx, 0);
    }
    const bool more = nct < c1;
    mbar_wait(bar, ph_uy);
    ph_uy ^= 1u;
    s1_stage_d<P, S>(stg_y, dsm, lane);
    s1_build_E_upper<P, S>(E, lane);  // the shifted upper copy of E from u's row in its lower half
    __syncwarp();
#if HQC_WL_VL2
    if (lane == 0) tma_prefetch_l2(v + ct * P::V_WORDS, M::VB);  // v reaches L2 during the product
#endif
#if HQC_S1_SEG
    using G = DecSeg<P>;
    static_assert(S::E_WORDS >= G::E_NEED, "the segmented windows stay inside E");
    uint32_t acc[G::LMAX], top;
    s1_seg_product<P, G, s1_unroll_dec<P>()>(E, dsm, acc, top, lane);
#else
    uint32_t acc[ST::R];
    s1_product<P, ST>(E, dsm, acc, lane);
    uint32_t mine = 0;
    if constexpr (TW > 0) {
      uint32_t t[TW];
      s1_tail_words<P, ST, ST::NOUT, TW>(E, dsm, lane, t);
#pragma unroll
      for (uint32_t i = 0; i < TW; i++) mine = (uint32_t)lane == i ? t[i] : mine;
    }
#endif
    __syncwarp();  // E is read: v may land above u's row, the next u in it
#if HQC_WL_VL2 && HQC_S1_SEG
    if (more) issue_uy(nct);
    if (lane == 0) cidx[slot] = (uint32_t)(ct - cbase);
    s1_seg_store<G>(acc, top, Rv, lane);  // u*y above u's row; stage 2 adds v from L2
    (void)ph_v;
#else
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar + 1, M::VB);
      tma_load_1d(Rv, v + ct * P::V_WORDS, M::VB, bar + 1);
    }
    if (more) issue_uy(nct);
    if (lane == 0) cidx[slot] = (uint32_t)(ct - cbase);
    mbar_wait(bar + 1, ph_v);
    ph_v ^= 1u;
#endif
#if HQC_S1_SEG && HQC_WL_VL2
#elif HQC_S1_SEG
    s1_seg_store_xor<G>(acc, top, Rv, Rv, lane);  // r = acc ^ v in place
#else
    s1_store_r_xor<ST>(acc, Rv, Rv, lane);  // r = acc ^ v in place
    if (TW > 0 && (uint32_t)lane < TW) Rv[ST::NOUT + lane] = mine ^ Rv[ST::NOUT + lane];
#endif
    __syncwarp();
#if HQC_WL_VL2 && HQC_S1_SEG
    const uint4 *vg = reinterpret_cast<const uint4 *>(v + ct * P::V_WORDS);
#endif
    for (uint32_t j = lane; j < P::N1; j += 32) {  // stage 2 into the chunk's slot
      const uint4 *src = reinterpret_cast<const uint4 *>(Rv) + j * (P::N2 / 128);
      uint32_t X[P::MULT * 4];
#pragma unroll
      for (int c = 0; c < (int)P::MULT; c++) {
        uint4 x = src[c];
#if HQC_WL_VL2 && HQC_S1_SEG
        const uint4 w = __ldg(vg + j * (P::N2 / 128) + c);
        x.x ^= w.x; x.y ^= w.y; x.z ^= w.z; x.w ^= w.w;
#endif
        X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
      }
      sb[j * M::SYM_PITCH + slot] = (uint8_t)rm_decode_block<P::MULT>(X);
    }
    __syncwarp();
    slot++;
    if (slot == 32 || !more) {  // stage 3, lane per word, scratch above u's row
      for (uint32_t q = slot; q < 32; q++)
        for (uint32_t j = lane; j < P::N1; j += 32) sb[j * M::SYM_PITCH + q] = 0;
      __syncwarp();
      const bool act = (uint32_t)lane < slot;
      auto sym_at = [&](int j) -> uint32_t { return sb[j * M::SYM_PITCH + lane]; };
      rs_decode_lane<P>(sym_at, gf, reinterpret_cast<uint16_t *>(Rv), lane,
                        act ? m_out + (cbase + cidx[lane]) * P::K : nullptr);
      __syncwarp();
      slot = 0;
    }
    ct = nct;
  }
}


// K4w (round 2, session 3; opt-in, HQC_DEC_KERNEL=12): K4l with the RS chunks SHARED by the CTA. Measured
// against K4l (profiles/r02/ab_wc.log, ab_wc2.log): HQC-3 65,536 1.081 vs 1.046 ms (slower), 262,144 4.08
// vs 4.24 (faster), 4,194,304 equal; HQC-1 12% slower than K4d. Neither BASELINE size gains, so not a default. K4l decodes a warp's own chunk of 32
// when it is full or the warp's work runs out; at 65,536 HQC-3 ciphertexts a warp gets ~28, so every chunk
// is decoded at the very end of the launch, all 16 warps of an SM at once with no product left to overlap
// (~40 us of a 1.05 ms launch; 4,194,304 runs at 0.86 of the roofline against 0.83). Here a chunk is 32
// CONSECUTIVE ciphertexts of the CTA's range, whichever warps decrypt them: stage 2 writes each symbol row
// into a ring of R chunk buffers shared by the CTA, a per-buffer counter counts the rows in, and the warp
// that completes a chunk decodes it at once (lane per word, its outputs contiguous), while the other warps
// keep multiplying. Only the CTA's last chunk is decoded at the end. A warp about to write into a buffer
// first waits (rarely) until the chunk R places earlier has been decoded out of it; the oldest chunk
// always completes, so no warp waits forever. The instruction stream is the same for every ciphertext.
#ifndef HQC_WC_RING
#define HQC_WC_RING 4
#endif
// The CTA's last chunk decoded word by word by the warp decoder of every idle warp (1) or by one lane decode
// (0). Measured (profiles/r02/ab_wc2.log): no change at 65,536, slower at 262,144 (4.13 vs 4.08 ms): 0.
#ifndef HQC_WC_WARPTAIL
#define HQC_WC_WARPTAIL 0
#endif
template <class P> struct WcSmem {
  using S = DecShape<P>;
  static constexpr uint32_t UB = P::U_STRIDE * 8, VB = P::V_WORDS * 8, YB = P::Y_STRIDE * 4;
  static constexpr uint32_t RB = VB > S3Scratch<P>::BYTES ? VB : S3Scratch<P>::BYTES;  // v, r, RS scratch
  static constexpr uint32_t E_BYTES = round_up(S::E_WORDS * 4 > UB + RB ? S::E_WORDS * 4 : UB + RB, 16);
  static constexpr uint32_t Y_BYTES = round_up(YB, 16);
  static constexpr uint32_t D_BYTES = round_up(S::WPAD * 4, 16);
  static constexpr uint32_t WARP_BYTES = E_BYTES + Y_BYTES + D_BYTES + 16;
  static constexpr uint32_t RING = HQC_WC_RING;
  static constexpr uint32_t SYM_PITCH = 36;  // odd word pitch: the 32 lanes' stage-2 byte stores hit 32 banks
  static constexpr uint32_t BUF_BYTES = round_up(P::N1 * SYM_PITCH, 16);
  static constexpr uint32_t CTL_BYTES = round_up(2 * RING * 4, 16);  // done[RING], gen[RING]
  static constexpr uint32_t HEAD = GF_BYTES + 16 + CTL_BYTES + RING * BUF_BYTES;
  static constexpr uint32_t bytes(uint32_t g) { return HEAD + g * WARP_BYTES; }
  static constexpr uint32_t fit(uint32_t g) { return g > 1 && bytes(g) > 227u * 1024u ? fit(g - 1) : g; }
  static constexpr uint32_t MAX_G = fit(16);
  static_assert(UB % 16 == 0, "the v / r region starts 16-byte aligned above u's row");
  static_assert(RING >= 2, "a ring of at least two chunk buffers");
  static_assert(RB >= round_up(P::N1, 16) + RsWarpScratch<P>::BYTES, "the warp decoder's word and scratch fit above u");
};

template <class P>
__global__ void __launch_bounds__(32 * WcSmem<P>::MAX_G, 1) k_decrypt_wc(const uint64_t *__restrict__ u,
                                                                        const uint64_t *__restrict__ v,
                                                                        const uint32_t *__restrict__ y,
                                                                        uint8_t *__restrict__ m_out,
                                                                        size_t batch) {
  using M = WcSmem<P>;
  using S = DecShape<P>;
  using G = DecSeg<P>;
  static_assert(S::E_WORDS >= G::E_NEED, "the segmented windows stay inside E");
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  unsigned int *next_item = reinterpret_cast<unsigned int *>(smem + GF_BYTES);
  unsigned int *done = reinterpret_cast<unsigned int *>(smem + GF_BYTES + 16);  // rows in, per buffer
  volatile unsigned int *gen = done + M::RING;  // chunks decoded out of each buffer
  uint8_t *ring = smem + GF_BYTES + 16 + M::CTL_BYTES;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t NG = blockDim.x >> 5;
  uint8_t *ws = smem + M::HEAD + (size_t)wib * M::WARP_BYTES;
  uint32_t *E = reinterpret_cast<uint32_t *>(ws);
  uint32_t *Rv = reinterpret_cast<uint32_t *>(ws + M::UB);  // v, then r, then the RS scratch
  uint32_t *stg_y = reinterpret_cast<uint32_t *>(ws + M::E_BYTES);
  uint32_t *dsm = reinterpret_cast<uint32_t *>(ws + M::E_BYTES + M::Y_BYTES);
  uint64_t *bar = reinterpret_cast<uint64_t *>(ws + M::E_BYTES + M::Y_BYTES + M::D_BYTES);  // [0] u, y  [1] v
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncwarp();
  auto issue_uy = [&](size_t c) {
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar, M::UB + M::YB);
      tma_load_1d(E, u + c * P::U_STRIDE, M::UB, bar);
      tma_load_1d(stg_y, y + c * P::Y_STRIDE, M::YB, bar);
    }
  };
  const size_t per_cta = (batch + gridDim.x - 1) / gridDim.x;
  const size_t c0 = (size_t)blockIdx.x * per_cta;
  const size_t c1 = c0 + per_cta < batch ? c0 + per_cta : batch;
  size_t ct = c0 + wib;
  if (ct < c1) issue_uy(ct);
  if (threadIdx.x == 0) next_item[0] = NG, next_item[1] = 0;  // work counter, last-chunk word counter
  if (threadIdx.x < 2 * M::RING) done[threadIdx.x] = 0;  // done[] and gen[]
  gf_tables_to_smem(gf);
  __syncthreads();
  const size_t nrows = c1 > c0 ? c1 - c0 : 0;
  const uint32_t last_chunk = nrows ? (uint32_t)((nrows - 1) >> 5) : 0u;
  uint32_t ph_uy = 0, ph_v = 0;
  while (ct < c1) {
    uint32_t nx = 0;
    if (lane == 0) nx = atomicAdd(next_item, 1u);
    const size_t nct = c0 + __shfl_sync(0xffffffffu, nx, 0);
    const bool more = nct < c1;
    mbar_wait(bar, ph_uy);
    ph_uy ^= 1u;
    s1_stage_d<P, S>(stg_y, dsm, lane);
    s1_build_E_upper<P, S>(E, lane);
    __syncwarp();
    uint32_t acc[G::LMAX], top;
    s1_seg_product<P, G, s1_unroll_dec<P>()>(E, dsm, acc, top, lane);
    __syncwarp();  // E is read: v may land above u's row, the next u in it
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar + 1, M::VB);
      tma_load_1d(Rv, v + ct * P::V_WORDS, M::VB, bar + 1);
    }
    if (more) issue_uy(nct);
    mbar_wait(bar + 1, ph_v);
    ph_v ^= 1u;
    s1_seg_store_xor<G>(acc, top, Rv, Rv, lane);  // r = acc ^ v in place
    // this ciphertext's chunk, its slot and its buffer (row k of the CTA's range)
    const size_t k = ct - c0;
    const uint32_t chunk = (uint32_t)(k >> 5), slot = (uint32_t)(k & 31), b = chunk % M::RING;
    uint8_t *sb = ring + (size_t)b * M::BUF_BYTES;
    if (lane == 0)  // the chunk RING places earlier must have been decoded out of this buffer
      while (gen[b] != chunk / M::RING) __nanosleep(64);
    __syncwarp();
    for (uint32_t j = lane; j < P::N1; j += 32) {  // stage 2 into the chunk's slot
      const uint4 *src = reinterpret_cast<const uint4 *>(Rv) + j * (P::N2 / 128);
      uint32_t X[P::MULT * 4];
#pragma unroll
      for (int c = 0; c < (int)P::MULT; c++) {
        const uint4 x = src[c];
        X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
      }
      sb[j * M::SYM_PITCH + slot] = (uint8_t)rm_decode_block<P::MULT>(X);
    }
    __syncwarp();
    const size_t cstart = c0 + ((size_t)chunk << 5);
    const uint32_t csize = c1 - cstart < 32 ? (uint32_t)(c1 - cstart) : 32u;
    uint32_t last = 0;
    if (lane == 0) {
      __threadfence_block();  // the row is visible before it is counted
      last = atomicAdd(done + b, 1u) + 1u == csize;
    }
    if (__shfl_sync(0xffffffffu, last, 0) && (!HQC_WC_WARPTAIL || chunk != last_chunk)) {  // decode it now
      __threadfence_block();
      for (uint32_t q = csize; q < 32; q++)
        for (uint32_t j = lane; j < P::N1; j += 32) sb[j * M::SYM_PITCH + q] = 0;
      __syncwarp();
      auto sym_at = [&](int j) -> uint32_t { return sb[j * M::SYM_PITCH + lane]; };
      rs_decode_lane<P>(sym_at, gf, reinterpret_cast<uint16_t *>(Rv), lane,
                        (uint32_t)lane < csize ? m_out + (cstart + lane) * P::K : nullptr);
      __syncwarp();
      if (lane == 0) {
        done[b] = 0;
        __threadfence_block();
        gen[b] = chunk / M::RING + 1;  // the buffer is free for chunk + RING
      }
    }
    __syncwarp();
    ct = nct;
  }
#if HQC_WC_WARPTAIL
  // The CTA's last chunk: once its rows are all in, every warp that has run out of work takes words of it
  // one at a time and decodes each with the whole warp (stage3_warp.cuh) — ~11k cycles per word instead of
  // one lane decode of the whole chunk by a single warp (~20k dependent warp instructions).
  if (nrows) {
    const uint32_t b = last_chunk % M::RING;
    const uint32_t csize = (uint32_t)(nrows - ((size_t)last_chunk << 5));
    const uint8_t *sb = ring + (size_t)b * M::BUF_BYTES;
    volatile unsigned int *vdone = done;
    if (lane == 0)
      while (vdone[b] < csize) __nanosleep(128);
    __syncwarp();
    __threadfence_block();
    uint8_t *mysym = reinterpret_cast<uint8_t *>(Rv);
    uint16_t *scr = reinterpret_cast<uint16_t *>(reinterpret_cast<uint8_t *>(Rv) + round_up(P::N1, 16));
    while (true) {
      uint32_t w = 0;
      if (lane == 0) w = atomicAdd(next_item + 1, 1u);
      w = __shfl_sync(0xffffffffu, w, 0);
      if (w >= csize) break;
      for (uint32_t j = lane; j < P::N1; j += 32) mysym[j] = sb[j * M::SYM_PITCH + w];
      __syncwarp();
      rs_decode_warp<P>(mysym, gf, scr, lane, m_out + (c0 + ((size_t)last_chunk << 5) + w) * P::K);
      __syncwarp();
    }
  }
#endif
}


// K4s: fused decrypt for SMALL batches (BASELINE configs[0]: HQC-1 at 1,024). K4a gives every warp at
// least 16 consecutive ciphertexts, so a batch of 1,024 occupies 64 warps on 64 SMs and the launch is the
// latency of 16 products in a row plus a lane-per-word RS decode. Here every warp takes ONE ciphertext at a
// time through all three stages: stage 1 by S1Pipe as in K4a, stage 2 lane per RM block, stage 3 by the
// whole warp (stage3_warp.cuh: syndromes, Chien, Omega and Forney lane-parallel, BM over the lanes as
// coefficients; no constant-bank tables, no CTA barrier). A CTA packs G such warps to share one copy of the
// GF tables; the host picks G so that the batch spreads over all SMs (G = ceil(batch / SMs), capped by
// shared memory), and warps stride over the batch when it is larger than the grid. Constant-flow.
// The stage-1 pipe of k_decrypt_sb. Unlike S1Pipe, u lands by TMA DIRECTLY in the lower half of E
// (E[q] = u32[q] for q < Q0: the copy out of a staging row is gone, only the shifted upper half is built),
// r is formed in place over v in the staging buffer, and stages 2 and 3 work there (stage 3's scratch
// too), so E is free once the product has read it: the next ciphertext's u is fetched into E during this
// one's stages 2 and 3. Two mbarriers: u, y (bar[0]) and v (bar[1]) are in flight at the same time.
template <class P> struct SbPipeSmem {
  using S = DecShape<P>;
  static constexpr uint32_t UB = P::U_STRIDE * 8, VB = P::V_WORDS * 8, YB = P::Y_STRIDE * 4;
  static_assert(UB <= S::E_WORDS * 4, "u lands inside E");
  static constexpr uint32_t E_BYTES = round_up(S::E_WORDS * 4, 16);
  static constexpr uint32_t STG_BYTES = round_up(VB > RsWarpScratch<P>::BYTES ? VB : RsWarpScratch<P>::BYTES, 16);
  static constexpr uint32_t Y_BYTES = round_up(YB, 16);
  static constexpr uint32_t D_BYTES = round_up(S::WPAD * 4, 16);
  static constexpr uint32_t BYTES = E_BYTES + STG_BYTES + Y_BYTES + D_BYTES + 16;
};

template <class P> struct SbPipe {
  using M = SbPipeSmem<P>;
  uint32_t *E, *stg, *stg_y, *dsm;
  uint64_t *bar;  // [0]: u, y   [1]: v
  uint32_t ph_uy = 0, ph_v = 0;
  const uint64_t *u, *v;
  const uint32_t *y;

  __device__ __forceinline__ SbPipe(uint8_t *ws, const uint64_t *u_, const uint64_t *v_, const uint32_t *y_, int lane)
      : u(u_), v(v_), y(y_) {
    E = reinterpret_cast<uint32_t *>(ws);
    stg = reinterpret_cast<uint32_t *>(ws + M::E_BYTES);
    stg_y = reinterpret_cast<uint32_t *>(ws + M::E_BYTES + M::STG_BYTES);
    dsm = reinterpret_cast<uint32_t *>(ws + M::E_BYTES + M::STG_BYTES + M::Y_BYTES);
    bar = reinterpret_cast<uint64_t *>(ws + M::E_BYTES + M::STG_BYTES + M::Y_BYTES + M::D_BYTES);
    if (lane == 0) {
      mbar_init(bar, 1);
      mbar_init(bar + 1, 1);
    }
    __syncwarp();
  }
  __device__ __forceinline__ void issue_uy(size_t ct, int lane) {  // E and stg_y must be free
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar, M::UB + M::YB);
      tma_load_1d(E, u + ct * P::U_STRIDE, M::UB, bar);
      tma_load_1d(stg_y, y + ct * P::Y_STRIDE, M::YB, bar);
    }
  }
  // E from the u row already in its lower half (stage1.cuh: s1_build_E_upper)
  __device__ __forceinline__ void build_E(int lane) { s1_build_E_upper<P, DecShape<P>>(E, lane); }
  // Stage 1 of ct (its u, y requested); leaves r in stg; requests next's u, y as soon as E is read.
  // U: the product's index-pair unroll (0: the fused kernels' s1_unroll_dec; k_stage1 passes its own).
  template <int U = 0>
  __device__ __forceinline__ void run(size_t ct, bool has_next, size_t next, int lane) {
    using S = DecShape<P>;
    using ST = DecShapeT<P>;
    constexpr uint32_t TW = dec_tail_words<P>();
    PHASE_T0();
    mbar_wait(bar, ph_uy);
    ph_uy ^= 1u;
    PHASE(1);
    s1_stage_d<P, S>(stg_y, dsm, lane);
    build_E(lane);
    __syncwarp();
    PHASE(2);
    if (v && lane == 0) {  // v lands in stg during the product
      fence_proxy_async_smem();
      mbar_expect_tx(bar + 1, M::VB);
      tma_load_1d(stg, v + ct * P::V_WORDS, M::VB, bar + 1);
    }
#if HQC_S1_SEG
    using G = DecSeg<P>;
    static_assert(S::E_WORDS >= G::E_NEED, "the segmented windows stay inside E");
    uint32_t acc[G::LMAX], top;
    s1_seg_product<P, G, (U ? U : s1_unroll_dec<P>())>(E, dsm, acc, top, lane);
    __syncwarp();  // every lane is done reading E (and dsm, stg_y): the next rows may land
    PHASE(3);
    if (has_next) issue_uy(next, lane);
    if (v) {
      mbar_wait(bar + 1, ph_v);
      ph_v ^= 1u;
      s1_seg_store_xor<G>(acc, top, stg, stg, lane);  // r = acc ^ v in place (each lane its own words)
    } else {  // the standalone product: r = acc
      s1_seg_store<G>(acc, top, stg, lane);
    }
#else
    uint32_t acc[ST::R];
    s1_product<P, ST>(E, dsm, acc, lane);
    uint32_t mine = 0;  // lane i < TW: word ST::NOUT + i
    if constexpr (TW > 0) {
      uint32_t t[TW];
      s1_tail_words<P, ST, ST::NOUT, TW>(E, dsm, lane, t);
#pragma unroll
      for (uint32_t i = 0; i < TW; i++) mine = (uint32_t)lane == i ? t[i] : mine;
    }
    __syncwarp();  // every lane is done reading E (and dsm, stg_y): the next rows may land
    PHASE(3);
    if (has_next) issue_uy(next, lane);
    if (v) {
      mbar_wait(bar + 1, ph_v);
      ph_v ^= 1u;
      s1_store_r_xor<ST>(acc, stg, stg, lane);  // r = acc ^ v, word by word in place (each lane its own words)
      if (TW > 0 && (uint32_t)lane < TW) stg[ST::NOUT + lane] = mine ^ stg[ST::NOUT + lane];
    } else {  // the standalone product: r = acc
      s1_store_r<ST>(acc, stg, lane);
      if (TW > 0 && (uint32_t)lane < TW) stg[ST::NOUT + lane] = mine;
    }
#endif
    __syncwarp();
    PHASE(4);
  }
};

template <class P> struct SbSmem {
  static constexpr uint32_t MAX_G = 16;  // warps per CTA; 512 threads: <= 128 registers
  static constexpr uint32_t SYM_BYTES = round_up(P::N1, 16);  // the warp's received symbols
  static constexpr uint32_t WARP_BYTES = SbPipeSmem<P>::BYTES + SYM_BYTES;
  static constexpr uint32_t CTR_BYTES = 16;  // the CTA's work counter
  static constexpr uint32_t bytes(uint32_t g) { return GF_BYTES + CTR_BYTES + g * WARP_BYTES; }
};

template <class P> constexpr uint32_t S1kSmem<P>::bytes(uint32_t g) { return 16 + g * SbPipeSmem<P>::BYTES; }
template <class P> constexpr uint32_t S1kSmem<P>::fit(uint32_t g) {
  return g > 1 && bytes(g) > 227u * 1024u ? fit(g - 1) : g;
}

template <class P>
__global__ void __launch_bounds__(32 * SbSmem<P>::MAX_G, 1) k_decrypt_sb(const uint64_t *__restrict__ u,
                                                                        const uint64_t *__restrict__ v,
                                                                        const uint32_t *__restrict__ y,
                                                                        uint8_t *__restrict__ m_out,
                                                                        size_t batch, uint32_t stagger_ns) {
  using M = SbSmem<P>;
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  unsigned int *next_item = reinterpret_cast<unsigned int *>(smem + GF_BYTES);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t G = blockDim.x >> 5;
  uint8_t *ws = smem + GF_BYTES + M::CTR_BYTES + (size_t)wib * M::WARP_BYTES;
  uint8_t *sym = ws + SbPipeSmem<P>::BYTES;
  PHASE_T0();
  SbPipe<P> pipe(ws, u, v, y, lane);
  // The CTA owns the contiguous range [c0, c1); its warps take ciphertexts from it one at a time through a
  // shared-memory counter (claimed one ciphertext ahead, so that its rows are prefetched during the current
  // product). Statically strided warps ended up to 11% apart (HQC-3, 65,536: profiles/r02/warp_span.log):
  // warps sharing an SM progress at different rates.
  const size_t per_cta = (batch + gridDim.x - 1) / gridDim.x;
  const size_t c0 = (size_t)blockIdx.x * per_cta;
  const size_t c1 = c0 + per_cta < batch ? c0 + per_cta : batch;
  size_t ct = c0 + wib;
  WARP_SPAN(0, (size_t)blockIdx.x * G + wib);
  if (ct < c1) pipe.issue_uy(ct, lane);  // the first rows are in flight while the GF tables are copied
  if (threadIdx.x == 0) *next_item = G;
  gf_tables_to_smem(gf);
  __syncthreads();
  if (stagger_ns) __nanosleep(stagger_ns * (uint32_t)wib);  // experiments: de-phase the warps of a CTA
  PHASE(0);
  while (ct < c1) {
    uint32_t nx = 0;
    if (lane == 0) nx = atomicAdd(next_item, 1u);
    const size_t nct = c0 + __shfl_sync(0xffffffffu, nx, 0);
    pipe.run(ct, nct < c1, nct, lane);
    PHASE_T0();
    for (uint32_t j = lane; j < P::N1; j += 32) {  // stage 2: lane per RM block of r (in the staging buffer)
      const uint4 *src = reinterpret_cast<const uint4 *>(pipe.stg) + j * (P::N2 / 128);
      uint32_t X[P::MULT * 4];
#pragma unroll
      for (int c = 0; c < (int)P::MULT; c++) {
        const uint4 x = src[c];
        X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
      }
      sym[j] = (uint8_t)rm_decode_block<P::MULT>(X);
    }
    __syncwarp();  // the symbols are complete and r is consumed: the staging buffer is stage 3's scratch
    PHASE(5);
    rs_decode_warp<P>(sym, gf, reinterpret_cast<uint16_t *>(pipe.stg), lane, m_out + ct * P::K);
    __syncwarp();  // E and sym are free for the next ciphertext
    PHASE(7);
    ct = nct;
  }
  WARP_SPAN(1, (size_t)blockIdx.x * G + wib);
}

// K4x (round 2, HQC-5 at large batches): the decrypt as TWO launches — this kernel runs stages 1 and 2 on
// the pipe of k_stage1 (a CTA of up to 16 warps per SM, 128 registers, the CTA-shared work counter) and
// writes each ciphertext's n1 received symbols to a scratch row in HBM; k_stage3 then decodes them 32 per
// warp with the lane-per-word RS decoder. HQC-5's lane decoder needs ~240 registers, which held the fused
// kernels to 8 warps per SM, and its chunks left the shared-memory pipe idle while they ran; split, the
// product runs at k_stage1's occupancy and the decoder at its own (profiles/r02/time_stages.log: three
// separate stage launches already beat the fused K4a at 262,144, 9.15 vs 9.57 ms). The symbols cost
// n1 bytes per ciphertext of HBM each way.
template <class P>
__global__ void __launch_bounds__(512, 1) k_decrypt_s12(const uint64_t *__restrict__ u, const uint64_t *__restrict__ v,
                                                        const uint32_t *__restrict__ y, uint8_t *__restrict__ sym_out,
                                                        size_t batch, uint32_t stagger_ns) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t G = blockDim.x >> 5;
  unsigned int *next_item = reinterpret_cast<unsigned int *>(smem);
  SbPipe<P> pipe(smem + 16 + (size_t)wib * SbPipeSmem<P>::BYTES, u, v, y, lane);
  const size_t per_cta = (batch + gridDim.x - 1) / gridDim.x;
  const size_t c0 = (size_t)blockIdx.x * per_cta;
  const size_t c1 = c0 + per_cta < batch ? c0 + per_cta : batch;
  size_t ct = c0 + wib;
  if (ct < c1) pipe.issue_uy(ct, lane);
  if (threadIdx.x == 0) *next_item = G;
  __syncthreads();
  if (stagger_ns) __nanosleep(stagger_ns * (uint32_t)wib);  // experiments: de-phase the warps of a CTA
  while (ct < c1) {
    uint32_t nx = 0;
    if (lane == 0) nx = atomicAdd(next_item, 1u);
    const size_t nct = c0 + __shfl_sync(0xffffffffu, nx, 0);
    pipe.run(ct, nct < c1, nct, lane);
    uint8_t *dst = sym_out + ct * P::N1;
    for (uint32_t j = lane; j < P::N1; j += 32) {  // stage 2: lane per RM block of r (in the staging buffer)
      const uint4 *src = reinterpret_cast<const uint4 *>(pipe.stg) + j * (P::N2 / 128);
      uint32_t X[P::MULT * 4];
#pragma unroll
      for (int c = 0; c < (int)P::MULT; c++) {
        const uint4 x = src[c];
        X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
      }
      dst[j] = (uint8_t)rm_decode_block<P::MULT>(X);
    }
    __syncwarp();  // r is consumed: the next v may land in the staging buffer
    ct = nct;
  }
}


// K4c (round 2, HQC-5 at large batches): K4x's first launch in a COMPACT per-warp layout. k_decrypt_s12 stages
// v in a 7.2 KB buffer next to E (22.8 KB per warp: 9 warps per SM), and the warps that are in stage 2 leave
// the shared-memory pipe to the others. Here v is not staged at all: its row is prefetched into L2 (a bulk
// prefetch, no shared memory) when the product starts, r = u*y is stored above u's row in E (16-byte
// aligned; the product is done reading E), the next u lands below it by TMA during stage 2, and stage 2
// XORs v into each RM block straight from global memory (L2 hits) — 15.5 KB per warp, 14 warps per SM.
template <class P> struct CxSmem {
  using S = DecShape<P>;
  using G = DecSeg<P>;
  static constexpr uint32_t UB = P::U_STRIDE * 8, YB = P::Y_STRIDE * 4, VB = P::V_WORDS * 8;
  static constexpr uint32_t R_OFF = round_up(UB, 16) / 4;  // r's first word, above u's row
  static constexpr uint32_t EW0 = G::E_NEED > R_OFF + P::NW ? G::E_NEED : R_OFF + P::NW;
  static constexpr uint32_t E_WORDS = round_up(EW0 > 2 * P::Q0 + 2 ? EW0 : 2 * P::Q0 + 2, 4);
  static constexpr uint32_t E_BYTES = E_WORDS * 4;
  static constexpr uint32_t Y_BYTES = round_up(YB, 16);
  static constexpr uint32_t D_BYTES = round_up(S::WPAD * 4, 16);
  static constexpr uint32_t WARP_BYTES = E_BYTES + Y_BYTES + D_BYTES + 16;
  static constexpr uint32_t bytes(uint32_t g) { return 16 + g * WARP_BYTES; }
  static constexpr uint32_t fit(uint32_t g) { return g > 1 && bytes(g) > 227u * 1024u ? fit(g - 1) : g; }
  static constexpr uint32_t MAX_G = fit(16);
  static_assert(VB % 16 == 0 && (P::N2 / 8) % 16 == 0, "v rows and RM blocks are whole 16-byte chunks");
};

template <class P>
__global__ void __launch_bounds__(512, 1) k_decrypt_s12c(const uint64_t *__restrict__ u, const uint64_t *__restrict__ v,
                                                         const uint32_t *__restrict__ y, uint8_t *__restrict__ sym_out,
                                                         size_t batch) {
  using M = CxSmem<P>;
  using S = DecShape<P>;
  using G = DecSeg<P>;
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t NG = blockDim.x >> 5;
  unsigned int *next_item = reinterpret_cast<unsigned int *>(smem);
  uint8_t *ws = smem + 16 + (size_t)wib * M::WARP_BYTES;
  uint32_t *E = reinterpret_cast<uint32_t *>(ws);
  uint32_t *Rr = E + M::R_OFF;
  uint32_t *stg_y = reinterpret_cast<uint32_t *>(ws + M::E_BYTES);
  uint32_t *dsm = reinterpret_cast<uint32_t *>(ws + M::E_BYTES + M::Y_BYTES);
  uint64_t *bar = reinterpret_cast<uint64_t *>(ws + M::E_BYTES + M::Y_BYTES + M::D_BYTES);
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  auto issue_uy = [&](size_t c) {
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar, M::UB + M::YB);
      tma_load_1d(E, u + c * P::U_STRIDE, M::UB, bar);
      tma_load_1d(stg_y, y + c * P::Y_STRIDE, M::YB, bar);
    }
  };
  const size_t per_cta = (batch + gridDim.x - 1) / gridDim.x;
  const size_t c0 = (size_t)blockIdx.x * per_cta;
  const size_t c1 = c0 + per_cta < batch ? c0 + per_cta : batch;
  size_t ct = c0 + wib;
  if (ct < c1) issue_uy(ct);
  if (threadIdx.x == 0) *next_item = NG;
  __syncthreads();
  uint32_t ph = 0;
  while (ct < c1) {
    uint32_t nx = 0;
    if (lane == 0) nx = atomicAdd(next_item, 1u);
    const size_t nct = c0 + __shfl_sync(0xffffffffu, nx, 0);
    const bool more = nct < c1;
    mbar_wait(bar, ph);
    ph ^= 1u;
    if (lane == 0) tma_prefetch_l2(v + ct * P::V_WORDS, M::VB);  // v reaches L2 during the product
    s1_stage_d<P, S>(stg_y, dsm, lane);
    s1_build_E_upper<P, M>(E, lane);
    __syncwarp();
    uint32_t acc[G::LMAX], top;
    s1_seg_product<P, G, s1_unroll_dec<P>()>(E, dsm, acc, top, lane);
    __syncwarp();  // E, the support row and the rotation amounts are read
    s1_seg_store<G>(acc, top, Rr, lane);  // r above u's row
    if (more) issue_uy(nct);              // the next u lands below it during stage 2
    __syncwarp();
    uint8_t *dst = sym_out + ct * P::N1;
    const uint4 *vg = reinterpret_cast<const uint4 *>(v + ct * P::V_WORDS);
    for (uint32_t j = lane; j < P::N1; j += 32) {  // stage 2: lane per RM block of r ^ v
      const uint4 *src = reinterpret_cast<const uint4 *>(Rr) + j * (P::N2 / 128);
      uint32_t X[P::MULT * 4];
#pragma unroll
      for (int c = 0; c < (int)P::MULT; c++) {
        const uint4 x = src[c];
        const uint4 w = __ldg(vg + j * (P::N2 / 128) + c);
        X[4 * c] = x.x ^ w.x; X[4 * c + 1] = x.y ^ w.y; X[4 * c + 2] = x.z ^ w.z; X[4 * c + 3] = x.w ^ w.w;
      }
      dst[j] = (uint8_t)rm_decode_block<P::MULT>(X);
    }
    __syncwarp();  // r is consumed: the next E build may overwrite it
    ct = nct;
  }
}


// K4p: small batches with a warp PAIR per decryption (configs[0]: 1,024 decryptions are 7 per SM, and a
// launch is the latency of one decryption: product ~10k cycles — the SM's shared memory saturated by its 7
// products — stage 2 6.6k in two rounds of 32 lanes, stage 3 ~10.7k; profiles/r02/sb_phases*.log). The pair
// shares E: warp A builds it from the u row TMA put in its lower half (the SbPipe layout), both run the
// product over half of the support indices, B's accumulators meet A's and v in the staging buffer, and
// stage 2 is split between the warps (one round each for n1 <= 64); warp A runs stage 3 (stage3_warp.cuh).
// A named barrier per pair (ids 1..8) orders the steps; the pairs of a CTA share only the GF tables.
template <class P> struct SpSmem {
  using S = DecShape<P>;
  using ST = DecShapeT<P>;
  static constexpr uint32_t UB = P::U_STRIDE * 8, VB = P::V_WORDS * 8, YB = P::Y_STRIDE * 4;
  static constexpr uint32_t E_BYTES = round_up(S::E_WORDS * 4, 16);
  static constexpr uint32_t STG_BYTES = round_up(VB > RsWarpScratch<P>::BYTES ? VB : RsWarpScratch<P>::BYTES, 16);
  static constexpr uint32_t X_BYTES = round_up(P::NW * 4, 16);  // warp B's accumulator image
  static constexpr uint32_t Y_BYTES = round_up(YB, 16);
  static constexpr uint32_t D_BYTES = round_up(S::WPAD * 4, 16);
  static constexpr uint32_t SYM_BYTES = round_up(P::N1, 16);
  static constexpr uint32_t PAIR_BYTES = E_BYTES + STG_BYTES + X_BYTES + Y_BYTES + D_BYTES + SYM_BYTES + 16;
  static constexpr uint32_t MAX_PAIRS = 8;  // named barriers 1..8; 512 threads
  static constexpr uint32_t bytes(uint32_t pairs) { return GF_BYTES + pairs * PAIR_BYTES; }
  static constexpr uint32_t W0 = (P::W / 2) & ~1u;  // warp A: indices [0, W0), warp B: [W0, W)
};

__device__ __forceinline__ void pair_sync(uint32_t id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

template <class P>
__global__ void __launch_bounds__(64 * SpSmem<P>::MAX_PAIRS, 1) k_decrypt_sp(const uint64_t *__restrict__ u,
                                                                           const uint64_t *__restrict__ v,
                                                                           const uint32_t *__restrict__ y,
                                                                           uint8_t *__restrict__ m_out,
                                                                           size_t batch) {
  using M = SpSmem<P>;
  using S = typename M::S;
  using ST = typename M::ST;
  constexpr uint32_t TW = dec_tail_words<P>();
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t pr = (uint32_t)wib >> 1, wa = (uint32_t)wib & 1u;  // pair, warp of the pair (0 = A)
  const uint32_t npairs = blockDim.x >> 6;
  uint8_t *ps = smem + GF_BYTES + (size_t)pr * M::PAIR_BYTES;
  uint32_t *E = reinterpret_cast<uint32_t *>(ps);
  uint32_t *stg = reinterpret_cast<uint32_t *>(ps + M::E_BYTES);
  uint32_t *X = reinterpret_cast<uint32_t *>(ps + M::E_BYTES + M::STG_BYTES);
  uint32_t *stg_y = reinterpret_cast<uint32_t *>(ps + M::E_BYTES + M::STG_BYTES + M::X_BYTES);
  uint32_t *dsm = reinterpret_cast<uint32_t *>(ps + M::E_BYTES + M::STG_BYTES + M::X_BYTES + M::Y_BYTES);
  uint8_t *sym = ps + M::E_BYTES + M::STG_BYTES + M::X_BYTES + M::Y_BYTES + M::D_BYTES;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sym + M::SYM_BYTES);  // [0]: u, y   [1]: v
  const uint32_t bid = 1 + pr;
  if (wa == 0 && lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  const size_t step = (size_t)gridDim.x * npairs;
  size_t ct = (size_t)blockIdx.x * npairs + pr;
  auto issue_uy = [&](size_t c) {
    fence_proxy_async_smem();
    mbar_expect_tx(bar, M::UB + M::YB);
    tma_load_1d(E, u + c * P::U_STRIDE, M::UB, bar);
    tma_load_1d(stg_y, y + c * P::Y_STRIDE, M::YB, bar);
  };
  gf_tables_to_smem(gf);
  __syncthreads();  // mbarriers initialised, GF tables in place
  if (wa == 0 && lane == 0 && ct < batch) issue_uy(ct);
  uint32_t ph_uy = 0, ph_v = 0;
  for (; ct < batch; ct += step) {
    PHASE_T0();
    const bool has_next = ct + step < batch;
    if (wa == 0) {
      mbar_wait(bar, ph_uy);
      s1_stage_d<P, S>(stg_y, dsm, lane);
      s1_build_E_upper<P, S>(E, lane);  // E from the u row in its lower half
      __syncwarp();
      if (lane == 0) {  // v lands in stg during the product
        fence_proxy_async_smem();
        mbar_expect_tx(bar + 1, M::VB);
        tma_load_1d(stg, v + ct * P::V_WORDS, M::VB, bar + 1);
      }
    }
    ph_uy ^= 1u;
    pair_sync(bid);  // E and the rotation amounts are ready
    PHASE(2);
#if HQC_S1_SEG
    using G = DecSeg<P>;
    static_assert(S::E_WORDS >= G::E_NEED, "the segmented windows stay inside E");
    uint32_t acc[G::LMAX], top;
    s1_seg_product<P, G, s1_unroll_dec<P>()>(E, dsm, acc, top, lane, wa ? M::W0 : 0u, wa ? P::W : M::W0);
    if (wa) s1_seg_store<G>(acc, top, X, lane);
    pair_sync(bid);  // both warps are done with E; B's image is in X
    PHASE(3);
    if (wa == 0) {
      if (has_next && lane == 0) issue_uy(ct + step);
      mbar_wait(bar + 1, ph_v);
      s1_seg_store_xor2<G>(acc, top, stg, X, stg, lane);  // r = acc_A ^ acc_B ^ v, in place over v
    }
#else
    uint32_t acc[ST::R];
    s1_product_range<P, ST>(E, dsm, acc, lane, wa ? M::W0 : 0u, wa ? P::W : M::W0);
    uint32_t mine = 0;
    if constexpr (TW > 0) {
      if (wa == 0) {
        uint32_t t[TW];
        s1_tail_words<P, ST, ST::NOUT, TW>(E, dsm, lane, t);
#pragma unroll
        for (uint32_t i = 0; i < TW; i++) mine = (uint32_t)lane == i ? t[i] : mine;
      }
    }
    if (wa) s1_store_r<ST>(acc, X, lane);
    pair_sync(bid);  // both warps are done with E; B's image is in X
    if (wa == 0) {
      if (has_next && lane == 0) issue_uy(ct + step);
      mbar_wait(bar + 1, ph_v);
      s1_store_r_xor2<ST>(acc, stg, X, stg, lane);  // r = acc_A ^ acc_B ^ v, in place over v
      if (TW > 0 && (uint32_t)lane < TW) stg[ST::NOUT + lane] = mine ^ stg[ST::NOUT + lane];
    }
#endif
    ph_v ^= 1u;
    pair_sync(bid);  // r complete
    PHASE(4);
    constexpr uint32_t NH = (P::N1 + 1) / 2;  // stage 2: A blocks [0, NH), B [NH, n1)
    for (uint32_t j = (wa ? NH : 0u) + lane; j < (wa ? P::N1 : NH); j += 32) {
      const uint4 *src = reinterpret_cast<const uint4 *>(stg) + j * (P::N2 / 128);
      uint32_t Xv[P::MULT * 4];
#pragma unroll
      for (int c = 0; c < (int)P::MULT; c++) {
        const uint4 x = src[c];
        Xv[4 * c] = x.x; Xv[4 * c + 1] = x.y; Xv[4 * c + 2] = x.z; Xv[4 * c + 3] = x.w;
      }
      sym[j] = (uint8_t)rm_decode_block<P::MULT>(Xv);
    }
    pair_sync(bid);  // symbols complete, r consumed
    PHASE(5);
    if (wa == 0) rs_decode_warp<P>(sym, gf, reinterpret_cast<uint16_t *>(stg), lane, m_out + ct * P::K);
    pair_sync(bid);  // stg and sym free for the next decryption
    PHASE(7);
  }
}


// K4t: fused decrypt with the product's windows in TENSOR MEMORY (stage1_tmem.cuh), one CTA per SM of
// WARPS warps; warp g owns ciphertexts [g*per, (g+1)*per) in chunks of 32 like K4a: stage 1 (TmPipe) +
// stage 2 per ciphertext (symbols parked as [j][slot]), then stage 3 with one lane per ciphertext.
#ifndef HQC_DEC_T_WARPS
#define HQC_DEC_T_WARPS (P::level == 5 ? 8 : 12)
#endif
template <class P> struct TmDec {
  static constexpr int WARPS = HQC_DEC_T_WARPS;
  static constexpr uint32_t COLS = WARPS == 16 ? 128 : (WARPS == 12 ? 160 : (WARPS == 8 ? 256 : 512));
  static constexpr uint32_t SYM_PITCH = 36;  // odd word pitch: conflict-free stage-2 byte stores (WarpSmem)
  static constexpr uint32_t SYM_BYTES = round_up(P::N1 * SYM_PITCH, 16);
  using M = TmS1<P, WARPS, COLS, GF_BYTES + 16, SYM_BYTES, S3Scratch<P>::BYTES>;
};

template <class P>
__global__ void __launch_bounds__(32 * TmDec<P>::WARPS, 1) k_decrypt_t(const uint64_t *__restrict__ u,
                                                                        const uint64_t *__restrict__ v,
                                                                        const uint32_t *__restrict__ y,
                                                                        uint8_t *__restrict__ m_out, size_t batch,
                                                                        size_t per) {
  using D = TmDec<P>;
  using M = typename D::M;
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  gf_tables_to_smem(gf);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t ta = tm_cta_alloc<M>(smem, wib);  // (its CTA barrier also publishes the GF tables)
  TmPipe<P, M> pipe(smem + M::PRE + (size_t)wib * M::WARP_BYTES, ta, u, v, y, lane);
  uint8_t *sb = pipe.extra;
  const size_t gw = (size_t)blockIdx.x * D::WARPS + wib;
  const size_t lo = gw * per < batch ? gw * per : batch;
  const size_t hi = lo + per < batch ? lo + per : batch;
  if (lo < hi) pipe.fetch(lo, lane);
  for (size_t base = lo; base < hi; base += 32) {
    const uint32_t rows = (uint32_t)(hi - base < 32 ? hi - base : 32);
    for (uint32_t s = 0; s < rows; s++) {
      const size_t ct = base + s;
      pipe.run(ct, ct + 1 < hi, ct + 1, lane);
      for (uint32_t j = lane; j < P::N1; j += 32) {  // stage 2: lane per RM block of r (in E)
        const uint4 *src = reinterpret_cast<const uint4 *>(pipe.E) + j * (P::N2 / 128);
        uint32_t X[P::MULT * 4];
#pragma unroll
        for (int c = 0; c < (int)P::MULT; c++) {
          const uint4 x = src[c];
          X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
        }
        sb[j * D::SYM_PITCH + s] = (uint8_t)rm_decode_block<P::MULT>(X);
      }
      __syncwarp();
    }
    for (uint32_t s = rows; s < 32; s++)
      for (uint32_t j = lane; j < P::N1; j += 32) sb[j * D::SYM_PITCH + s] = 0;
    __syncwarp();
    const bool act = (uint32_t)lane < rows;
    auto sym_at = [&](int j) -> uint32_t { return sb[j * D::SYM_PITCH + lane]; };
    rs_decode_lane<P>(sym_at, gf, reinterpret_cast<uint16_t *>(pipe.E), lane,
                      act ? m_out + (base + lane) * P::K : nullptr);
    __syncwarp();
  }
  tm_cta_free<M>(smem, wib);
}


// K4b: fused decrypt, WARP-SPECIALISED. CTA = 4 warps:
//   warps 0-1 (product pair): per ciphertext, build E from the TMA-staged u, run the rotate-and-XOR
//     over half of the support indices each, XOR their accumulators into a ring slot that TMA has
//     pre-filled with v (slot = v ^ acc1 ^ acc0 = r), then hand the slot over (mbarrier "full"); the
//     next ciphertext's u, y are fetched right after E is built.
//   warp 2 (RM decoder): per ciphertext, stage 2 on the slot (lane per RM block), symbols into one of
//     two [n1][32] chunk buffers, slot released (mbarrier "empty").
//   warp 3 (RS decoder): per chunk of 32 ciphertexts, stage 3 (lane per ciphertext).
// The product warps never leave the shared-memory-bound loop for RM/RS work, so the LSU stays fed
// while the decoders use the ALU/FMA pipes; the two-deep rings absorb the decoders' burstiness.
template <class P> struct WsSmem {
  using S = DecShape<P>;
  static constexpr uint32_t E_BYTES = round_up(S::E_WORDS * 4, 16);
  static constexpr uint32_t UB = P::U_STRIDE * 8, VB = P::V_WORDS * 8, YB = P::Y_STRIDE * 4;
  static constexpr uint32_t STG_BYTES = round_up(UB, 16) + round_up(YB, 16);
  static constexpr uint32_t D_BYTES = round_up(S::WPAD * 4, 16);
  static constexpr uint32_t SLOT_BYTES = round_up(VB, 16);
  static constexpr uint32_t SYM_BYTES = round_up(P::N1 * 32, 16);
  static constexpr uint32_t SCR_BYTES = round_up(S3Scratch<P>::BYTES, 16);
  static constexpr uint32_t BYTES = E_BYTES + STG_BYTES + D_BYTES + 2 * SLOT_BYTES + 2 * SYM_BYTES + SCR_BYTES + 128;
  static constexpr uint32_t W0 = (P::W / 2) & ~1u;
};

#ifndef HQC_DEC_MINCTAS_WS
#define HQC_DEC_MINCTAS_WS (P::level == 5 ? 3 : 6)
#endif

template <class P>
__global__ void __launch_bounds__(128, HQC_DEC_MINCTAS_WS) k_decrypt_ws(const uint64_t *__restrict__ u,
                                                                        const uint64_t *__restrict__ v,
                                                                        const uint32_t *__restrict__ y,
                                                                        uint8_t *__restrict__ m_out, size_t batch,
                                                                        size_t per) {
  using S = DecShape<P>;
  using M = WsSmem<P>;
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  uint8_t *b0 = smem + GF_BYTES;
  uint32_t *E = reinterpret_cast<uint32_t *>(b0);
  uint32_t *stg_u = reinterpret_cast<uint32_t *>(b0 + M::E_BYTES);
  uint32_t *stg_y = reinterpret_cast<uint32_t *>(b0 + M::E_BYTES + round_up(M::UB, 16));
  uint32_t *dsm = reinterpret_cast<uint32_t *>(b0 + M::E_BYTES + M::STG_BYTES);
  uint8_t *slots = b0 + M::E_BYTES + M::STG_BYTES + M::D_BYTES;
  uint8_t *symb = slots + 2 * M::SLOT_BYTES;  // [2][n1][32]
  uint16_t *scr = reinterpret_cast<uint16_t *>(symb + 2 * M::SYM_BYTES);
  uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(scr) + M::SCR_BYTES);
  uint64_t *bar_u = bars;            // u, y of the next ciphertext
  uint64_t *bar_full = bars + 1;     // [2]: slot holds r
  uint64_t *bar_empty = bars + 3;    // [2]: slot free
  uint64_t *bar_v = bars + 5;        // [2]: v landed in the slot
  uint64_t *bar_sfull = bars + 7;    // [2]: symbol chunk complete
  uint64_t *bar_sempty = bars + 9;   // [2]: symbol chunk consumed
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  gf_tables_to_smem(gf);
  if (tid == 0) {
    mbar_init(bar_u, 1);
    for (int s = 0; s < 2; s++) {
      mbar_init(bar_full + s, 1);
      mbar_init(bar_empty + s, 1);
      mbar_init(bar_v + s, 1);
      mbar_init(bar_sfull + s, 1);
      mbar_init(bar_sempty + s, 1);
    }
  }
  __syncthreads();
  const size_t lo = (size_t)blockIdx.x * per;
  const size_t hi = lo + per < batch ? lo + per : batch;

  if (wid < 2) {
    // ------------------------------------------------------------------ product pair
    const int ptid = tid;  // 0..63
    uint32_t ph_u = 0, ph_empty[2] = {1u, 1u}, ph_v[2] = {0u, 0u};
    auto issue_uy = [&](size_t ct) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar_u, M::UB + M::YB);
      tma_load_1d(stg_u, u + ct * P::U_STRIDE, M::UB, bar_u);
      tma_load_1d(stg_y, y + ct * P::Y_STRIDE, M::YB, bar_u);
    };
    if (lo < hi && ptid == 0) issue_uy(lo);
    const uint32_t j0 = wid ? M::W0 : 0u, j1 = wid ? P::W : M::W0;
    for (size_t ct = lo; ct < hi; ct++) {
      const int s = (int)((ct - lo) & 1);
      uint32_t *slot = reinterpret_cast<uint32_t *>(slots + s * M::SLOT_BYTES);
      PHASE_T0();
      mbar_wait(bar_u, ph_u);
      ph_u ^= 1u;
      PHASE(8);
      s1_stage_d<P, S, 64>(stg_y, dsm, ptid);
      s1_build_E<P, S, 64>(stg_u, E, ptid);
      asm volatile("bar.sync 1, 64;" ::: "memory");
      PHASE(9);
      if (ptid == 0) {
        if (ct + 1 < hi) issue_uy(ct + 1);      // the staging buffer is free once E is built
        mbar_wait(bar_empty + s, ph_empty[s]);  // the RM decoder has released this slot
        fence_proxy_async_smem();
        mbar_expect_tx(bar_v + s, M::VB);
        tma_load_1d(slot, v + ct * P::V_WORDS, M::VB, bar_v + s);
      }
      ph_empty[s] ^= 1u;
      PHASE(10);
      uint32_t acc[S::R];
      s1_product_range<P, S>(E, dsm, acc, lane, j0, j1);
      PHASE(11);
      mbar_wait(bar_v + s, ph_v[s]);
      ph_v[s] ^= 1u;
      if (wid == 1) s1_xor_into<S>(acc, slot, lane);
      asm volatile("bar.sync 1, 64;" ::: "memory");  // also: both warps are done reading E
      if (wid == 0) {
        s1_xor_into<S>(acc, slot, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_full + s);  // release: the slot now holds r
      }
      PHASE(12);
    }
  } else if (wid == 2) {
    // ------------------------------------------------------------------ RM decoder (stage 2)
    uint32_t ph_full[2] = {0u, 0u}, ph_sempty[2] = {1u, 1u};
    uint32_t col = 0, b = 0;
    uint8_t *sym = symb;
    for (size_t ct = lo; ct < hi; ct++) {
      const int s = (int)((ct - lo) & 1);
      if (col == 0) {  // starting a chunk: wait until the RS decoder is done with this buffer
        mbar_wait(bar_sempty + b, ph_sempty[b]);
        ph_sempty[b] ^= 1u;
        sym = symb + b * M::SYM_BYTES;
      }
      const uint32_t *r = reinterpret_cast<const uint32_t *>(slots + s * M::SLOT_BYTES);
      PHASE_T0();
      mbar_wait(bar_full + s, ph_full[s]);
      ph_full[s] ^= 1u;
      PHASE(13);
      for (uint32_t j = lane; j < P::N1; j += 32) {
        const uint4 *src = reinterpret_cast<const uint4 *>(r) + j * (P::N2 / 128);
        uint32_t X[P::MULT * 4];
#pragma unroll
        for (int c = 0; c < (int)P::MULT; c++) {
          const uint4 x = src[c];
          X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
        }
        sym[j * 32 + col] = (uint8_t)rm_decode_block<P::MULT>(X);
      }
      __syncwarp();
      PHASE(14);
      if (lane == 0) mbar_arrive(bar_empty + s);
      if (++col == 32 || ct + 1 == hi) {
        for (uint32_t e = lane; e < P::N1 * 32; e += 32)
          if ((e & 31) >= col) sym[e] = 0;
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_sfull + b);
        col = 0;
        b ^= 1u;
      }
    }
  } else {
    // ------------------------------------------------------------------ RS decoder (stage 3)
    uint32_t ph_sfull[2] = {0u, 0u};
    uint32_t b = 0;
    for (size_t base = lo; base < hi; base += 32) {
      const uint32_t rows = (uint32_t)(hi - base < 32 ? hi - base : 32);
      PHASE_T0();
      mbar_wait(bar_sfull + b, ph_sfull[b]);
      ph_sfull[b] ^= 1u;
      PHASE(15);
      const uint8_t *sym = symb + b * M::SYM_BYTES;
      const bool act = (uint32_t)lane < rows;
      auto sym_at = [&](int j) -> uint32_t { return sym[j * 32 + lane]; };
      rs_decode_lane<P>(sym_at, gf, scr, lane, act ? m_out + (base + lane) * P::K : nullptr);
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_sempty + b);
      b ^= 1u;
    }
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
  // Work split of stage 1 between the two warps:
  //   SPLIT_WORDS: warp w computes output words [w*NW/2, (w+1)*NW/2) over all w indices (R = odd
  //     ceil(NW/64)); no hand-off. Fewer registers and wasted lanes for HQC-1/5, but measured 3% and
  //     1% slower than the index split on B200 (profiles/r01/NOTES.md), so it is off.
  //   else: warp w takes half of the support indices over all NW words (R = odd ceil(NW/32); exact
  //     35 for HQC-3), and warp 1 hands its accumulators to warp 0 through shared memory.
#ifndef HQC_SPLIT_WORDS
#define HQC_SPLIT_WORDS false
#endif
  static constexpr bool SPLIT_WORDS = HQC_SPLIT_WORDS;
  static constexpr uint32_t NWH = P::NW / 2;
  using S = typename std::conditional<SPLIT_WORDS, ProdShape<P, P::NW / 2, P::W>, DecShape<P>>::type;
  static constexpr uint32_t EW_NEED = SPLIT_WORDS ? round_up(P::Q0 + NWH + 32 * S::R + 2, 4) : S::E_WORDS;
  static constexpr uint32_t XOFF = round_up(P::NW, 4);  // warp-1 accumulator image, above r in E
  static_assert(SPLIT_WORDS || XOFF + P::NW <= S::E_WORDS, "the accumulator image fits in E above r");
  static constexpr uint32_t E_WORDS = EW_NEED;
  static constexpr uint32_t E_BYTES = round_up(
      E_WORDS * 4 > 2 * S3Scratch<P>::BYTES ? E_WORDS * 4 : 2 * S3Scratch<P>::BYTES, 16);
  static constexpr uint32_t UB = P::U_STRIDE * 8, VB = P::V_WORDS * 8, YB = P::Y_STRIDE * 4;
  static constexpr uint32_t STG_UV_BYTES = round_up(UB > VB ? UB : VB, 16);
  // DSTAGE: a second staging buffer so the next ciphertext's u, y are fetched during this one's
  // product loop (HQC-1: stage 2 alone is too short to hide the fetch; HQC-3/5 have no smem to spare
  // and hide it already — profiles/r01/NOTES.md).
  static constexpr bool DSTAGE = P::level == 1;
  static constexpr uint32_t STG_BYTES = STG_UV_BYTES + round_up(YB, 16) + (DSTAGE ? STG_UV_BYTES : 0);
  static constexpr uint32_t D_BYTES = round_up(S::WPAD * 4, 16);
#ifndef HQC_SYM_PITCH2
#define HQC_SYM_PITCH2 68
#endif
  static constexpr uint32_t SYM_PITCH = HQC_SYM_PITCH2;  // 17 words (odd): conflict-free stage-2 byte stores (see WarpSmem)
  static constexpr uint32_t SYM_BYTES = round_up(P::N1 * SYM_PITCH, 16);
#ifndef HQC_PAIR_XBUF
#define HQC_PAIR_XBUF 1
#endif
  // XBUF: warp 1's accumulator image in its own buffer (after the barriers) instead of above r in E,
  // so warp 1 can store it without waiting for warp 0 to finish reading E (one CTA barrier fewer).
  static constexpr bool XBUF = HQC_PAIR_XBUF && !SPLIT_WORDS;
#ifndef HQC_PAIR_RX
#define HQC_PAIR_RX 1
#endif
  // RX: r is combined in place in XBUF and stage 2 reads it there, so the next ciphertext's E build
  // does not have to wait for stage 2 (one CTA barrier fewer per ciphertext)
  static constexpr bool RX = HQC_PAIR_RX && XBUF;
  static constexpr uint32_t XBUF_BYTES = XBUF ? round_up(P::NW * 4, 16) : 0;
  static constexpr uint32_t BYTES = E_BYTES + STG_BYTES + D_BYTES + SYM_BYTES + 16 * 2 + XBUF_BYTES;
  static constexpr uint32_t W0 = (P::W / 2) & ~1u;  // index split: warp 0 takes [0, W0), warp 1 [W0, W)
};


// Register cap per level (minimum resident CTAs): the fused kernel is latency-bound at the occupancy
// its register count allows, so the cap trades a few registers for more resident warp pairs.
template <class P> struct DecOcc {
  static constexpr int MIN_CTAS = HQC_DEC_MINCTAS;
};

template <class P>
__global__ void __launch_bounds__(64, DecOcc<P>::MIN_CTAS) k_decrypt(const uint64_t *__restrict__ u, const uint64_t *__restrict__ v,
                                                const uint32_t *__restrict__ y, uint8_t *__restrict__ m_out,
                                                size_t batch, size_t per) {
  using M = PairSmem<P>;
  using S = typename M::S;
  extern __shared__ __align__(16) uint8_t smem[];
  GfTables *gf = reinterpret_cast<GfTables *>(smem);
  uint8_t *base_p = smem + GF_BYTES;
  uint32_t *E = reinterpret_cast<uint32_t *>(base_p);
  uint32_t *stg_u = reinterpret_cast<uint32_t *>(base_p + M::E_BYTES);
  uint32_t *stg_y = reinterpret_cast<uint32_t *>(base_p + M::E_BYTES + M::STG_UV_BYTES);
  uint32_t *dsm = reinterpret_cast<uint32_t *>(base_p + M::E_BYTES + M::STG_BYTES);
  uint8_t *sym = base_p + M::E_BYTES + M::STG_BYTES + M::D_BYTES;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sym + M::SYM_BYTES);  // u, y (and v unless DSTAGE)
  uint32_t *stg_v = M::DSTAGE ? stg_y + round_up(M::YB, 16) / 4 : stg_u;
  uint64_t *barv = M::DSTAGE ? bar + 1 : bar;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  gf_tables_to_smem(gf);
  if (tid == 0) {
    mbar_init(bar, 1);
    if (M::DSTAGE) mbar_init(barv, 1);
  }
  __syncthreads();
  uint32_t phase = 0, phasev = 0;
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
      PHASE_T0();
      mbar_wait(bar, phase);  // u, y of ct
      phase ^= 1u;
      PHASE(0);
      s1_stage_d<P, S, 64>(stg_y, dsm, tid);
      s1_build_E<P, EBuildShape<P, M::E_WORDS>, 64>(stg_u, E, tid);
      __syncthreads();
      if (tid == 0) {  // v lands in the staging buffer while the product runs
        fence_proxy_async_smem();
        mbar_expect_tx(barv, M::VB);
        tma_load_1d(stg_v, v + ct * P::V_WORDS, M::VB, barv);
        if (M::DSTAGE && ct + 1 < hi) issue_uy(ct + 1);
      }
      PHASE(1);
      uint32_t acc[S::R];
      if constexpr (M::SPLIT_WORDS) {
        const uint32_t w0 = wid * M::NWH;  // this warp's first output word
        s1_product_range<P, S>(E + w0, dsm, acc, lane, 0, P::W);
        __syncthreads();  // both warps are done reading E
        if (M::DSTAGE) {
          mbar_wait(barv, phasev);  // v of ct
          phasev ^= 1u;
        } else {
          mbar_wait(bar, phase);
          phase ^= 1u;
        }
        s1_store_r_xor<S>(acc, E + w0, stg_v + w0, lane);
      } else {
        s1_product_range<P, S>(E, dsm, acc, lane, j0, j1);
        PHASE(2);
        uint32_t *xs = M::XBUF ? reinterpret_cast<uint32_t *>(bar + 4) : E + M::XOFF;
        if (!M::XBUF) __syncthreads();  // both warps are done reading E
        PHASE(3);
        if (wid == 1) s1_store_r<S>(acc, xs, lane);
        __syncthreads();
        if (M::DSTAGE) {
          mbar_wait(barv, phasev);  // v of ct
          phasev ^= 1u;
        } else {
          mbar_wait(bar, phase);
          phase ^= 1u;
        }
        if (wid == 0) s1_store_r_xor2<S>(acc, M::RX ? xs : E, xs, stg_v, lane);
      }
      __syncthreads();
      PHASE(4);
      if (!M::DSTAGE && tid == 0 && ct + 1 < hi) issue_uy(ct + 1);
#ifndef HQC_EXP_SKIP
#define HQC_EXP_SKIP 0  // experiments only (scripts/exp_variants.py): 1 = skip stage 2, 2 = skip stage 3
#endif
      if (!(HQC_EXP_SKIP & 1))
      for (uint32_t j = tid; j < P::N1; j += 64) {  // stage 2: one RM block per thread
        const uint4 *src = reinterpret_cast<const uint4 *>(M::RX ? reinterpret_cast<uint32_t *>(bar + 4) : E) +
                           j * (P::N2 / 128);
        uint32_t X[P::MULT * 4];
#pragma unroll
        for (int c = 0; c < (int)P::MULT; c++) {
          const uint4 x = src[c];
          X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
        }
        sym[j * M::SYM_PITCH + s] = (uint8_t)rm_decode_block<P::MULT>(X);
      }
      PHASE(5);
      if (!M::RX) __syncthreads();  // (RX: the next E build writes E, not r; the barrier after it orders XBUF)
      PHASE(6);
    }
    for (uint32_t e = tid; e < P::N1 * 64; e += 64)
      if ((e & 63) >= rows) sym[(e >> 6) * M::SYM_PITCH + (e & 63)] = 0;
    __syncthreads();
    const uint32_t slot = 32 * wid + lane;
    const bool act = slot < rows;
    auto sym_at = [&](int j) -> uint32_t { return sym[j * M::SYM_PITCH + slot]; };
    PHASE_T0();
    if (!(HQC_EXP_SKIP & 2))
      rs_decode_lane<P>(sym_at, gf, reinterpret_cast<uint16_t *>(base_p + wid * S3Scratch<P>::BYTES), lane,
                        act ? m_out + (base + slot) * P::K : nullptr);
    PHASE(7);
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------------
// host side
struct DevInfo {
  int sms = 0;
  int cap_decrypt[6] = {0};     // resident CTAs/SM of k_decrypt per level
  int cap_decrypt_w1[6] = {0};  // resident CTAs/SM of k_decrypt_w1 per level
  int cap_decrypt_ws[6] = {0};  // resident CTAs/SM of k_decrypt_ws per level
  int cap_stage1[6] = {0};
  bool ready[6] = {false};
  cudaMemPool_t pool = nullptr;  // the library's stream-ordered pool for K4x's symbol scratch
};

static std::mutex g_mu;
static DevInfo g_dev[16];

constexpr int WARPS_PER_CTA = 1;  // stage-1 kernel: one warp per CTA (fine-grained SM balance)
constexpr int DEC_THREADS = 64;   // fused kernel: one warp pair per CTA

template <class P> static uint32_t decrypt_smem() { return GF_BYTES + PairSmem<P>::BYTES; }
template <class P> static uint32_t decrypt_w1_smem() { return GF_BYTES + WarpSmem<P>::BYTES; }
template <class P> static uint32_t decrypt_ws_smem() { return GF_BYTES + WsSmem<P>::BYTES; }
template <class P> static uint32_t decrypt_t_smem() { return TmDec<P>::M::SMEM_BYTES; }

// Which fused kernel a level uses (measured, profiles/r01/NOTES.md): 1 = one warp per ciphertext,
// 2 = warp pair, 3 = warp-specialised, 4 = tensor-memory product (K4t), 5 = small-batch groups (K4s),
// 6 = K4a with CTA-shared work (K4d), 7 = small batches with a warp pair per decryption (K4p),
// 8 = compact lane-RS warps (K4l), 9 = K4l with static per-warp ranges, 10 = stages 1+2 and stage 3 as two
// launches (K4x), 11 = K4x with the compact first launch (K4c), 12 = K4l with CTA-shared RS chunks (K4w).
// HQC_DEC_KERNEL=1..12 overrides.
static int dec_kernel_env() {
  static int env = [] {
    const char *s = getenv("HQC_DEC_KERNEL");
    return s ? atoi(s) : 0;
  }();
  return env >= 1 && env <= 12 ? env : 0;
}
template <class P> static int dec_kernel() {
  if (dec_kernel_env()) return dec_kernel_env();
  // above the K4s range: HQC-1 K4d (65,536: 0.526 vs 0.560 ms for K4a; 262,144: +6.7%,
  // profiles/r02/ab_wd.log), HQC-3 K4l (65,536: 1.073 vs 1.139 ms for K4s, profiles/r02/ab_wl.log; K4d fits
  // only 13 warps there), HQC-5 K4a (K4d -5.5%, K4l -2.4..-5%: its de-phased warps contend harder)
  return P::level == 1 ? 6 : P::level == 3 ? 8 : 1;
}
// Read on every call (experiments sweep them within one process): HQC_SB_MAX = the largest batch that
// takes K4s by default; HQC_DEC_SPLIT = the most ciphertexts one launch of the large-batch kernels takes.
static long env_long(const char *name, long dflt) {
  const char *s = getenv(name);
  return s && *s ? atol(s) : dflt;
}
// K4s up to this batch (scripts/sweep_launch.py small / large / cross, profiles/r02/
// sweep_*.log): HQC-3 at every batch (65,536: 5.61e7/s vs 5.41e7 for the warp pair K4; 262,144: 5.79e7 vs
// 5.53e7); HQC-1 up to ~40,000 (32,768: 1.04e8 vs 9.28e7; 49,152: 1.06e8 vs 1.10e8 — beyond, K4a's paired
// RM stage and lane-per-word RS win); HQC-5 up to ~24,000 (16,384: 2.41e7 vs 2.24e7; 32,768: 2.37e7 vs
// 2.58e7 — its shared memory allows 10 warps per SM in K4s, 8 in K4a but with the cheaper lane RS).
template <class P> static size_t sb_max_batch(int sms) {
  // HQC-3: K4s up to ~44,000, K4l beyond (32,768: 0.591 vs 0.600 ms; 65,536: 1.139 vs 1.073;
  // 4,194,304: 6.05e7 vs 6.36e7/s — profiles/r02/ab_wl*.log)
  // HQC-5: K4s up to ~16,000, K4c beyond (16,384: 0.678 vs 0.678 ms; 32,768: 1.18 vs 1.33 —
  // profiles/r02/sweep_x5.log, after the segmented layout and the unroll of 2)
  const long dflt = (long)sms * (P::level == 1 ? 270 : P::level == 3 ? 300 : 110);
  const long v = env_long("HQC_SB_MAX", dflt);
  return v < 0 ? ~(size_t)0 : (size_t)v;
}
// K4p (a warp pair per decryption) for the tiniest batches, up to 4 decryptions per SM: one decryption
// 10.7 vs 13.5 us, 148 11.7 vs 14.4, 512 13.2 vs 14.2; from 1,024 (7 per SM) K4s is faster again
// (17.7 vs 19.4 us: the SM's shared memory is saturated by the products either way and the pair's barriers
// and idle second warp in stage 3 cost more than the halved stage 2; profiles/r02/ab_sp.log).
template <class P> static size_t sp_max_batch(int sms) { return (size_t)env_long("HQC_SP_MAX", (long)sms * 4); }
// K4x (two launches) for HQC-5 from ~96,000 (131,072: 4.77 vs 4.88 ms for K4a; 262,144 9.36 vs 9.58;
// 4,194,304 in launches of 1,048,576: 2.83e7 vs 2.74e7/s; 65,536: 2.55 vs 2.53 — profiles/r02/ab_x5.log).
// Since K4c (k_decrypt_s12c) and the unroll of 2, the two-launch form wins for HQC-5 at every batch above the
// K4s range (32,768: 1.18 ms vs 1.22 for K4a and 1.24 for K4x; 262,144: 8.48 vs 9.45 / 9.01 —
// profiles/r02/sweep_x5.log). HQC-3's K4x beats K4l by 1-4% between ~131,072 and ~524,288 and loses at
// 4,194,304 (profiles/r02/sweep_x3.log); not used there (neither configs[1] nor configs[4] is in that range).
template <class P> static size_t x_min_batch(int sms) {
  const long v = env_long("HQC_X_MIN", P::level == 5 ? (long)sms * 110 : -1);
  return v < 0 ? ~(size_t)0 : (size_t)v;
}
template <class P> static int dec_kernel_for(int sms, size_t batch) {
  if (dec_kernel_env()) return dec_kernel_env();
  if (batch <= sp_max_batch<P>(sms)) return 7;
  if (batch <= sb_max_batch<P>(sms)) return 5;
  // K4c rather than K4x: 14 compact warps per SM instead of 9 (262,144: 9.10 vs 9.30 ms; 1,048,576: 36.04 vs
  // 36.84; 131,072: 4.63 vs 4.75 — profiles/r02/ab_k4c.log)
  if (batch >= x_min_batch<P>(sms)) return 11;
  // HQC-3 (session 3): K4l while a warp holds at most one RS chunk (batch <= sms x 16 x 32 = 75,776), K4w
  // from there to ~600,000, where K4l's partial chunks cost a whole RS pass each (81,920: 16.44 vs 17.28 ns
  // per decryption; 262,144: 15.69 vs 16.24; 524,288: 15.57 vs 16.05), K4l again for the largest batches
  // (4,194,304: 15.27 vs 15.42 ns) — profiles/r02/scan3*.log, split_new.log
  if (P::level == 3 && batch > (size_t)sms * 512u && batch <= (size_t)sms * 4096u) return 12;
  return dec_kernel<P>();
}
// The largest group (warps per CTA) of K4s whose shared memory fits one CTA.
template <class P> constexpr uint32_t sb_max_g() {
  uint32_t g = SbSmem<P>::MAX_G;
  while (g > 1 && SbSmem<P>::bytes(g) > 227u * 1024u) g--;
  return g;
}
template <class P> static bool use_pair() { return dec_kernel<P>() == 2; }
// Which standalone product kernel: 1 = one warp per ciphertext (k_stage1), 2 = warp pair with the output
// words split (k_stage1p), 3 = windows from tensor memory (k_stage1t, stage1_tmem.cuh). Measured (65,536,
// v = NULL, ms): HQC-1 0.370 / 0.373 / 0.380, HQC-3 0.985 / 1.046 / 0.892, HQC-5 2.42 / 2.14 / 1.89.
// The default stays constant-flow (R#8): k_stage1t buckets the support by offset range, so its
// per-range trip counts depend on y; it is opt-in (HQC_S1_KERNEL=3) for inputs whose timing may leak.
template <class P> static int stage1_kernel() {
  static int env = [] {
    const char *s = getenv("HQC_S1_KERNEL");
    return s ? atoi(s) : 0;
  }();
  if (env == 1 || env == 2 || env == 3) return env;
  // round 2: k_stage1 with the CTA-shared work counter beats the warp pair at HQC-5 too (1.847 vs 2.117 ms
  // per 65,536, profiles/r02/ab_s1_l5.log)
  return 1;
}
template <class P> static uint32_t stage1_g() { return S1kSmem<P>::fit(16); }
template <class P> static uint32_t stage1_smem() { return S1kSmem<P>::bytes(stage1_g<P>()); }
template <class P> static uint32_t stage3_smem(int warps) {
  return GF_BYTES + S3_REPL_BYTES + warps * (S3Scratch<P>::BYTES + round_up(P::N1 * 32, 16));
}

template <class P> static cudaError_t prepare(int dev, DevInfo &di) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (di.ready[P::level]) return cudaSuccess;
  cudaError_t e;
  if ((e = cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_decrypt<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, decrypt_smem<P>())) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_stage1<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, stage1_smem<P>())) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_stage3<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, stage3_smem<P>(HQC_S3_REPL ? 8 : 4))) != cudaSuccess) return e;
  int c = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_decrypt<P>, DEC_THREADS, decrypt_smem<P>())) != cudaSuccess) return e;
  di.cap_decrypt[P::level] = c > 0 ? c : 1;
  if ((e = cudaFuncSetAttribute(k_decrypt_w1<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, decrypt_w1_smem<P>())) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_decrypt_w1<P>, 32, decrypt_w1_smem<P>())) != cudaSuccess) return e;
  di.cap_decrypt_w1[P::level] = c > 0 ? c : 1;
  if ((e = cudaFuncSetAttribute(k_decrypt_ws<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, decrypt_ws_smem<P>())) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_decrypt_ws<P>, 128, decrypt_ws_smem<P>())) != cudaSuccess) return e;
  di.cap_decrypt_ws[P::level] = c > 0 ? c : 1;
  {
    uint32_t q = SpSmem<P>::MAX_PAIRS;
    while (q > 1 && SpSmem<P>::bytes(q) > 227u * 1024u) q--;
    if ((e = cudaFuncSetAttribute(k_decrypt_sp<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SpSmem<P>::bytes(q))) != cudaSuccess) return e;
  }
  if ((e = cudaFuncSetAttribute(k_decrypt_wl<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                WlSmem<P>::bytes(WlSmem<P>::MAX_G))) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_decrypt_wl<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                WlSmem<P>::bytes(WlSmem<P>::MAX_G))) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_decrypt_wc<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                WcSmem<P>::bytes(WcSmem<P>::MAX_G))) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_decrypt_wd<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                WdSmem<P>::bytes(WdSmem<P>::MAX_G))) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_decrypt_sb<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                SbSmem<P>::bytes(sb_max_g<P>()))) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_stage1<P>, 32 * stage1_g<P>(), stage1_smem<P>())) != cudaSuccess) return e;
  di.cap_stage1[P::level] = c > 0 ? c : 1;
  if ((e = cudaFuncSetAttribute(k_decrypt_s12<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, stage1_smem<P>())) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_decrypt_s12c<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                CxSmem<P>::bytes(CxSmem<P>::MAX_G))) != cudaSuccess) return e;
  if (!di.pool) {  // the library's own pool (the device's default pool and its release threshold stay the caller's)
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if ((e = cudaMemPoolCreate(&di.pool, &props)) != cudaSuccess) return e;
    uint64_t keep = ~0ull;  // keep freed scratch for the next call instead of returning it at every sync
    if ((e = cudaMemPoolSetAttribute(di.pool, cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess) return e;
  }
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
  const int kind = dec_kernel_for<P>(di.sms, batch);
  if (kind == 5) {  // groups of G ciphertexts (G warps per CTA) spread over all SMs; *per = G
    size_t g = (batch + di.sms - 1) / (size_t)di.sms;
    if (g < 1) g = 1;
    if (g > sb_max_g<P>()) g = sb_max_g<P>();
    *per = g;
    size_t groups = (batch + g - 1) / g;
    const size_t cap = (size_t)di.sms * (227u * 1024u / SbSmem<P>::bytes((uint32_t)g) > 0
                                             ? 227u * 1024u / SbSmem<P>::bytes((uint32_t)g) : 1u);
    *grid = (int)(groups < cap ? groups : cap);
    return;
  }
  if (kind == 7) {  // pairs of warps, one decryption each; *per = pairs per CTA
    constexpr uint32_t maxp = [] {
      uint32_t q = SpSmem<P>::MAX_PAIRS;
      while (q > 1 && SpSmem<P>::bytes(q) > 227u * 1024u) q--;
      return q;
    }();
    size_t g = (batch + di.sms - 1) / (size_t)di.sms;
    if (g < 1) g = 1;
    if (g > maxp) g = maxp;
    *per = g;
    const size_t groups = (batch + g - 1) / g;
    *grid = (int)(groups < (size_t)di.sms ? groups : (size_t)di.sms);
    return;
  }
  if (kind == 8 || kind == 9) {  // one CTA of up to MAX_G warps per SM; *per = warps per CTA
    size_t g = (batch + di.sms - 1) / (size_t)di.sms;
    if (g < 1) g = 1;
    if (g > WlSmem<P>::MAX_G) g = WlSmem<P>::MAX_G;
    const long eg = env_long("HQC_WL_G", 0);  // experiments: warps per CTA
    if (eg > 0 && (size_t)eg < g) g = (size_t)eg;
    *per = g;
    const size_t groups = (batch + g - 1) / g;
    *grid = (int)(groups < (size_t)di.sms ? groups : (size_t)di.sms);
    return;
  }
  if (kind == 10) {  // k_decrypt_s12: one CTA of up to stage1_g warps per SM; *per = warps per CTA
    size_t g = (batch + di.sms - 1) / (size_t)di.sms;
    if (g < 1) g = 1;
    if (g > stage1_g<P>()) g = stage1_g<P>();
    *per = g;
    const size_t groups = (batch + g - 1) / g;
    *grid = (int)(groups < (size_t)di.sms ? groups : (size_t)di.sms);
    return;
  }
  if (kind == 12) {  // k_decrypt_wc: one CTA of up to WcSmem::MAX_G warps per SM; *per = warps per CTA
    size_t g = (batch + di.sms - 1) / (size_t)di.sms;
    if (g < 1) g = 1;
    if (g > WcSmem<P>::MAX_G) g = WcSmem<P>::MAX_G;
    *per = g;
    const size_t groups = (batch + g - 1) / g;
    *grid = (int)(groups < (size_t)di.sms ? groups : (size_t)di.sms);
    return;
  }
  if (kind == 11) {  // k_decrypt_s12c: one CTA of up to CxSmem::MAX_G warps per SM; *per = warps per CTA
    size_t g = (batch + di.sms - 1) / (size_t)di.sms;
    if (g < 1) g = 1;
    if (g > CxSmem<P>::MAX_G) g = CxSmem<P>::MAX_G;
    *per = g;
    const size_t groups = (batch + g - 1) / g;
    *grid = (int)(groups < (size_t)di.sms ? groups : (size_t)di.sms);
    return;
  }
  if (kind == 6) {  // one CTA of up to MAX_G warps per SM; *per = warps per CTA
    size_t g = (batch + di.sms - 1) / (size_t)di.sms;
    if (g < 1) g = 1;
    if (g > WdSmem<P>::MAX_G) g = WdSmem<P>::MAX_G;
    *per = g;
    const size_t groups = (batch + g - 1) / g;
    *grid = (int)(groups < (size_t)di.sms ? groups : (size_t)di.sms);
    return;
  }
  if (kind == 4) {  // one CTA of WARPS warps per SM; at least 16 ciphertexts per warp
    const size_t warps = (size_t)di.sms * TmDec<P>::WARPS;
    size_t pw = (batch + warps - 1) / warps;
    if (pw < MIN_PER / 2) pw = MIN_PER / 2;
    *per = pw;
    const size_t nw = (batch + pw - 1) / pw;
    *grid = (int)((nw + TmDec<P>::WARPS - 1) / TmDec<P>::WARPS);
    if (*grid < 1) *grid = 1;
    return;
  }
  const int c = kind == 1 ? di.cap_decrypt_w1[P::level] : kind == 2 ? di.cap_decrypt[P::level] : di.cap_decrypt_ws[P::level];
  const size_t cap = (size_t)di.sms * c;
#ifndef HQC_PAIR_MIN_PER
#define HQC_PAIR_MIN_PER MIN_PER
#endif
  const size_t min_per = kind == 1 ? MIN_PER / 2 : kind == 2 ? (size_t)HQC_PAIR_MIN_PER : 2 * MIN_PER;
  size_t ctas = (batch + min_per - 1) / min_per;
  if (ctas > cap) ctas = cap;
  if (ctas == 0) ctas = 1;
  *per = (batch + ctas - 1) / ctas;
  *grid = (int)((batch + *per - 1) / *per);
}

// Largest batch of one launch of the persistent kernels (0 = unlimited): a long contiguous range per CTA
// lets the CTAs drift out of lockstep, so a big batch runs as consecutive launches.
template <class P> static size_t dec_split(int sms) {
  const long s = env_long("HQC_DEC_SPLIT", -1);
  if (s >= 0) return (size_t)s;
  // HQC-1: parts of at most 65,536, the batch cut into EQUAL parts (dec_part; session 3): a batch of 73,728
  // used to run as 65,536 + 8,192 and lost 12% (profiles/r02/scan3.log). Parts of one RS chunk per warp
  // (sms x 512 = 75,776) were measured too and lost 5% at 1,048,576 and 4,194,304 (split_new.log).
  (void)sms;
  // measured at 4,194,304 (scripts/sweep_launch.py split, profiles/r02/sweep_split.log): HQC-1 +7% at 65,536
  // per launch; HQC-5 K4a +9% at 262,144, K4x (its default there since) best at 1,048,576 (2.83e7/s against
  // 2.81e7 unsplit and at 262,144; its symbol scratch is then 94 MB, profiles/r02/ab_x5.log); HQC-3 unsplit
  return P::level == 1 ? 65536u : P::level == 5 ? 1048576u : 0u;
}
// Equal parts of at most `split` ciphertexts (the part size rounded up to 32): how many ciphertexts each
// launch of launch_decrypt takes.
// A batch at most 1/8 above the limit runs as one launch: a small second part cost more than the longer
// first one (HQC-1 73,728: 8.06 ns per decryption in one launch, 9.63 as two of 36,864, 8.64 as 65,536 +
// 8,192; 81,920: 8.70 in one, 8.52 in two — profiles/r02/split2.log).
static size_t dec_part(size_t batch, size_t split) {
  if (split == 0 || batch <= split + split / 8) return batch;
  const size_t parts = (batch + split - 1) / split;
  const size_t p = (batch + parts - 1) / parts;
  return (p + 31) / 32 * 32;
}

template <class P>
static int launch_stage3_on(DevInfo *di, const uint8_t *sym, uint8_t *m, uint8_t *ok, size_t batch, cudaStream_t st) {
  const long ew = env_long("HQC_S3_WARPS", 4);  // experiments: warps per CTA (1..4)
  const int warps = HQC_S3_REPL ? 8 : (ew >= 1 && ew <= 4 ? (int)ew : 4);
  size_t grid = (batch + 32 * warps - 1) / (32 * warps);
  const size_t cap = (size_t)di->sms * 16;
  if (grid > cap) grid = cap;
  k_stage3<P><<<(unsigned)grid, 32 * warps, stage3_smem<P>(warps), st>>>(sym, m, ok, batch);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P>
static int launch_decrypt_one(DevInfo *di, const uint64_t *u, const uint64_t *v, const uint32_t *y, uint8_t *m,
                              size_t batch, cudaStream_t st) {
  int grid;
  size_t per;
  decrypt_shape<P>(*di, batch, &grid, &per);
  switch (dec_kernel_for<P>(di->sms, batch)) {
    case 1: k_decrypt_w1<P><<<grid, 32, decrypt_w1_smem<P>(), st>>>(u, v, y, m, batch, per); break;
    case 2: k_decrypt<P><<<grid, DEC_THREADS, decrypt_smem<P>(), st>>>(u, v, y, m, batch, per); break;
    case 4:
      if (cudaFuncSetAttribute(k_decrypt_t<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, decrypt_t_smem<P>()) !=
          cudaSuccess)
        return HQC_ERR_CUDA;
      k_decrypt_t<P><<<grid, 32 * TmDec<P>::WARPS, decrypt_t_smem<P>(), st>>>(u, v, y, m, batch, per);
      break;
    case 6:
      k_decrypt_wd<P><<<grid, 32 * (unsigned)per, WdSmem<P>::bytes((uint32_t)per), st>>>(u, v, y, m, batch);
      break;
    case 7:
      k_decrypt_sp<P><<<grid, 64 * (unsigned)per, SpSmem<P>::bytes((uint32_t)per), st>>>(u, v, y, m, batch);
      break;
    case 8:
      k_decrypt_wl<P, true><<<grid, 32 * (unsigned)per, WlSmem<P>::bytes((uint32_t)per), st>>>(u, v, y, m, batch);
      break;
    case 9:
      k_decrypt_wl<P, false><<<grid, 32 * (unsigned)per, WlSmem<P>::bytes((uint32_t)per), st>>>(u, v, y, m, batch);
      break;
    case 5:
      k_decrypt_sb<P><<<grid, 32 * (unsigned)per, SbSmem<P>::bytes((uint32_t)per), st>>>(
          u, v, y, m, batch, (uint32_t)env_long("HQC_SB_STAGGER", 0));
      break;
    case 10: {  // stages 1+2 -> symbols in a pool scratch -> stage 3 (stream-ordered: freed after k_stage3)
      uint8_t *sym = nullptr;
      if (cudaMallocFromPoolAsync(reinterpret_cast<void **>(&sym), batch * P::N1, di->pool, st) != cudaSuccess)
        return HQC_ERR_CUDA;
      k_decrypt_s12<P><<<grid, 32 * (unsigned)per, S1kSmem<P>::bytes((uint32_t)per), st>>>(
          u, v, y, sym, batch, (uint32_t)env_long("HQC_S12_STAGGER", 0));
      const int rc = launch_stage3_on<P>(di, sym, m, nullptr, batch, st);
      const bool freed = cudaFreeAsync(sym, st) == cudaSuccess;
      if (rc != HQC_OK || !freed) return HQC_ERR_CUDA;
      break;
    }
    case 12:
      k_decrypt_wc<P><<<grid, 32 * (unsigned)per, WcSmem<P>::bytes((uint32_t)per), st>>>(u, v, y, m, batch);
      break;
    case 11: {  // K4c: the compact stages 1+2 -> symbols in a pool scratch -> stage 3
      uint8_t *sym = nullptr;
      if (cudaMallocFromPoolAsync(reinterpret_cast<void **>(&sym), batch * P::N1, di->pool, st) != cudaSuccess)
        return HQC_ERR_CUDA;
      k_decrypt_s12c<P><<<grid, 32 * (unsigned)per, CxSmem<P>::bytes((uint32_t)per), st>>>(u, v, y, sym, batch);
      const int rc = launch_stage3_on<P>(di, sym, m, nullptr, batch, st);
      const bool freed = cudaFreeAsync(sym, st) == cudaSuccess;
      if (rc != HQC_OK || !freed) return HQC_ERR_CUDA;
      break;
    }
    default: k_decrypt_ws<P><<<grid, 128, decrypt_ws_smem<P>(), st>>>(u, v, y, m, batch, per); break;
  }
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P>
static int launch_decrypt(const uint64_t *u, const uint64_t *v, const uint32_t *y, uint8_t *m, size_t batch,
                          cudaStream_t st) {
  DevInfo *di;
  const int dev = cur_device(&di);
  if (dev < 0 || prepare<P>(dev, *di) != cudaSuccess) return HQC_ERR_CUDA;
  const size_t split = dec_part(batch, dec_split<P>(di->sms));
  if (batch <= split) return launch_decrypt_one<P>(di, u, v, y, m, batch, st);
  for (size_t off = 0; off < batch; off += split) {
    const size_t n = batch - off < split ? batch - off : split;
    const int rc = launch_decrypt_one<P>(di, u + off * P::U_STRIDE, v + off * P::V_WORDS, y + off * P::Y_STRIDE,
                                         m + off * P::K, n, st);
    if (rc != HQC_OK) return rc;
  }
  return HQC_OK;
}

template <class P>
static int launch_stage1(const uint64_t *u, const uint32_t *y, const uint64_t *v, uint64_t *r, size_t batch,
                         cudaStream_t st) {
  DevInfo *di;
  const int dev = cur_device(&di);
  if (dev < 0 || prepare<P>(dev, *di) != cudaSuccess) return HQC_ERR_CUDA;
  if (stage1_kernel<P>() == 3) {  // windows from tensor memory (k_stage1t), one CTA of 8 warps per SM
    constexpr uint32_t smem = TmS1Std<P>::SMEM_BYTES;
    if (cudaFuncSetAttribute(k_stage1t<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return HQC_ERR_CUDA;
    size_t grid = (batch + TmS1Std<P>::WARPS - 1) / TmS1Std<P>::WARPS;
    if (grid > (size_t)di->sms) grid = di->sms;
    k_stage1t<P><<<(unsigned)grid, 32 * TmS1Std<P>::WARPS, smem, st>>>(u, y, v, r, batch);
    return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
  }
  if (stage1_kernel<P>() == 2) {  // warp pair, output words split (k_stage1p)
    const uint32_t smem = S1PairSmem<P>::BYTES;
    if (cudaFuncSetAttribute(k_stage1p<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return HQC_ERR_CUDA;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stage1p<P>, 64, smem) != cudaSuccess || per_sm < 1)
      return HQC_ERR_CUDA;
    size_t grid = batch;
    const size_t capp = (size_t)di->sms * per_sm;
    if (grid > capp) grid = capp;
    k_stage1p<P><<<(unsigned)grid, 64, smem, st>>>(u, y, v, r, batch);
    return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
  }
  size_t g = (batch + di->sms - 1) / (size_t)di->sms;  // warps per CTA: spread small batches over the SMs
  if (g < 1) g = 1;
  if (g > stage1_g<P>()) g = stage1_g<P>();
  const long gmax = env_long("HQC_S1_G", 0);  // experiments: fewer warps per CTA
  if (gmax > 0 && g > (size_t)gmax) g = (size_t)gmax;
  size_t grid = (batch + g - 1) / g;
  if (grid > (size_t)di->sms) grid = di->sms;
  k_stage1<P><<<(unsigned)grid, 32 * (unsigned)g, S1kSmem<P>::bytes((uint32_t)g), st>>>(u, y, v, r, batch);
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
  return launch_stage3_on<P>(di, sym, m, ok, batch, st);
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

// Which encrypt kernel: 2 = warp pair with per-key cached E (k_encrypt2, default), 1 = one warp per
// ciphertext (k_encrypt). HQC_ENC_KERNEL overrides (tests, experiments; read on every call).
static int enc_kernel() { return env_long("HQC_ENC_KERNEL", 2) == 1 ? 1 : 2; }

// Launch the encrypt kernel (CMP: the KEM re-encryption check writing two flags per ciphertext to eq2).
template <class P, bool CMP>
static int launch_encrypt_any(const uint64_t *h, const uint64_t *s, const uint32_t *key, const uint8_t *m,
                              const uint32_t *r1, const uint32_t *r2, const uint32_t *e, uint64_t *u, uint64_t *v,
                              size_t batch, const uint64_t *uc, const uint64_t *vc, uint8_t *eq2, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (enc_kernel() == 1) {
    const uint32_t smem = EncSmem<P>::BYTES;
    if (cudaFuncSetAttribute(k_encrypt<P, CMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return HQC_ERR_CUDA;
    size_t grid = batch;
    const size_t cap = (size_t)sms * 16;
    if (grid > cap) grid = cap;
    k_encrypt<P, CMP><<<(unsigned)grid, 32, smem, st>>>(h, s, key, m, r1, r2, e, u, v, batch, uc, vc, eq2);
    return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
  }
  // one CTA of Q u-warps + Q v-warps per SM, each CTA a contiguous range shared out job by job (encrypt.cuh)
  size_t q = (batch + sms - 1) / (size_t)sms;
  if (q < 1) q = 1;
  if (q > Enc2Smem<P>::MAX_Q) q = Enc2Smem<P>::MAX_Q;
  const uint32_t smem = Enc2Smem<P>::bytes((uint32_t)q);
  if (cudaFuncSetAttribute(k_encrypt2<P, CMP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           Enc2Smem<P>::bytes(Enc2Smem<P>::MAX_Q)) != cudaSuccess)
    return HQC_ERR_CUDA;
  size_t ctas = (batch + q - 1) / q;
  if (ctas > (size_t)sms) ctas = sms;
  const size_t per = (batch + ctas - 1) / ctas;
  const size_t grid = (batch + per - 1) / per;
  k_encrypt2<P, CMP><<<(unsigned)grid, 64 * (unsigned)q, smem, st>>>(h, s, key, m, r1, r2, e, u, v, batch, per, uc,
                                                                   vc, eq2);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P>
static int launch_encrypt(const uint64_t *h, const uint64_t *s, const uint32_t *key, const uint8_t *m,
                          const uint32_t *r1, const uint32_t *r2, const uint32_t *e, uint64_t *u, uint64_t *v,
                          size_t batch, cudaStream_t st) {
  return launch_encrypt_any<P, false>(h, s, key, m, r1, r2, e, u, v, batch, nullptr, nullptr, nullptr, st);
}

// Which fused kernel hqc_decrypt_batch launches for `batch` on the current device (1..5 as dec_kernel).
template <class P> static int kind_impl(size_t batch) {
  DevInfo *di;
  const int dev = cur_device(&di);
  if (dev < 0 || prepare<P>(dev, *di) != cudaSuccess) return HQC_ERR_CUDA;
  return dec_kernel_for<P>(di->sms, batch);
}

// How many kernel launches hqc_decrypt_batch makes for `batch` (the large-batch split, dec_split; K4x is two
// launches per part).
template <class P> static long long nlaunch_impl(size_t batch) {
  if (batch == 0) return 0;
  DevInfo *di;
  const int dev = cur_device(&di);
  if (dev < 0 || prepare<P>(dev, *di) != cudaSuccess) return HQC_ERR_CUDA;
  const size_t step = dec_part(batch, dec_split<P>(di->sms));
  long long n = 0;
  for (size_t off = 0; off < batch; off += step) {
    const size_t c = batch - off < step ? batch - off : step;
    n += (dec_kernel_for<P>(di->sms, c) == 10 || dec_kernel_for<P>(di->sms, c) == 11) ? 2 : 1;
  }
  return n;
}

template <class P> static int shape_impl(size_t batch, int *grid, int *wpc) {
  DevInfo *di;
  const int dev = cur_device(&di);
  if (dev < 0 || prepare<P>(dev, *di) != cudaSuccess) return HQC_ERR_CUDA;
  size_t per;
  decrypt_shape<P>(*di, batch, grid, &per);
  const int kind = dec_kernel_for<P>(di->sms, batch);
  *wpc = kind == 1 ? 1 : kind == 2 ? DEC_THREADS / 32 : kind == 4 ? TmDec<P>::WARPS
        : (kind == 5 || kind == 6 || kind == 8 || kind == 9 || kind == 10 || kind == 11 || kind == 12) ? (int)per
        : kind == 7 ? 2 * (int)per : 4;
  return HQC_OK;
}

}  // namespace hqc
