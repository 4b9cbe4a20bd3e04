// Stage 1 — the sparse x dense cyclic product of Eq. 1 (§III.B), XORed into v and
// truncated to n1*n2 bits (Alg. 2; R#1-R#3). One warp per ciphertext; everything in shared
// memory. DESIGN.md §6.1 gives the mapping and its roofline.
//
//   r[t] = v[t] XOR  XOR_{j<w} u[(t - y_j) mod n]          t < n12
//
// With d_j = n - y_j in [1, n] and the "doubled" u, E[b] = u[b mod n] for b < n + n12 + 32, output
// word W (bits 32W..32W+31) receives, for each j, bits [32W + d_j, 32W + d_j + 32) of E — one funnel
// shift of two adjacent E words: SHF(E[o + W], E[o + W + 1], s) with o = d_j >> 5, s = d_j & 31
// ("a coarse word rotation and a fine intra-word bit rotation ... adjacent words share carry
// bits"). The loop count is w for every ciphertext and every index (no data-dependent branches).
//
// The rows of u, y and v arrive in a per-warp staging buffer by TMA bulk copies (async_copy.cuh),
// prefetched one ciphertext ahead by the kernels in hqc_gpu.cu.
#pragma once
#include <cstdint>

#include "levels.cuh"
#include "seg_plans.cuh"

namespace hqc {

// The segmented lane layout of the product (s1_seg_product, below) in the default kernels; 0 restores the
// round-2 R-word lanes with s1_tail_words (an experiment switch, A/B in profiles/r02/ab_seg.log).
#ifndef HQC_S1_SEG
#define HQC_S1_SEG 1
#endif

// index-pair loop unroll per level, from scripts/exp_unroll.py (2: -0.5% HQC-1/3; 3: -2.4% HQC-5)
template <class P> constexpr int s1_unroll() {
#ifdef HQC_S1_UNROLL
  return HQC_S1_UNROLL;
#elif defined(HQC_S1_UNROLL_ENC)
  return P::level == 3 ? HQC_S1_UNROLL_ENC : (P::level == 5 ? 3 : 2);
#else
  return P::level == 5 ? 3 : 2;
#endif
}

// Index-pair unroll of the segmented product (s1_seg_product), per kernel family, measured against the
// R-word values above after the layout change (profiles/r02/ab_unroll*.log): the fused decrypt kernels
// want 2 at every level (HQC-5 K4c 8.61 vs 9.21 ms with 3: the 3-pair body of 57-word windows thrashed
// the instruction cache, 12.5% no_instruction stalls), the standalone product 3 (HQC-1 / 3 / 5 -0.8 /
// -1.0 / -1.1%).
template <class P> constexpr int s1_unroll_dec() {
#ifdef HQC_S1_UNROLL_DEC
  return HQC_S1_UNROLL_DEC;
#else
  return 2;
#endif
}
template <class P> constexpr int s1_unroll_s1() {
#ifdef HQC_S1_UNROLL_S1
  return HQC_S1_UNROLL_S1;
#else
  return 3;
#endif
}

// Encrypt / KeyGen products: HQC-3 prefers 3 (1.99 vs 2.06 ms per 65,536 encryptions), HQC-5 2 (4.33 vs
// 4.36), HQC-1 either (profiles/r02/ab_unroll_enc.log).
template <class P> constexpr int s1_unroll_enc() {
#ifdef HQC_S1_UNROLL_ENC2
  return HQC_S1_UNROLL_ENC2;
#else
  return P::level == 3 ? 3 : 2;
#endif
}

// Build E (S::E_WORDS words) from the staged dense row su (shared memory):
//   E[q] = u32[q]                                   q < Q0
//   E[Q0] = (last C bits of u) | u32[0] << C        the wrap of X^n = 1
//   E[q] = funnel(u32[x], u32[x + 1], 32 - C)       q = Q0 + 1 + x, x <= Q0, with u32[Q0] masked to its C
//                                                   valid bits and u32[Q0 + 1] = 0 (bits >= n ignored, R#13)
//   E[q] = 0                                        beyond (read only by lanes whose outputs are dropped)
// One warp (NT = 32): su[Q0] and su[Q0 + 1] are first rewritten in place (su is a consumed staging row),
// then each lane funnels a run of CH consecutive words (CH odd: conflict-free), loading every source
// word once and carrying the neighbour in a register (no per-word selects). The warp pair (NT = 64)
// cannot afford the in-place fix-up (two more CTA barriers: +1.6% at HQC-3), so its runs stop before
// the partial word Q0 and thread 0 adds the three words that involve it (no fix-up, no barrier: -0.5%
// for the HQC-3 fused kernel, -0.2% for the HQC-5 standalone pair, against the strided form with
// per-word selects; the one-warp kernels measured +0.4..0.5% with it and keep the in-place form).
#ifndef HQC_EBUILD_RUN2
#define HQC_EBUILD_RUN2 1
#endif
template <class P, class S, int NT = 32>
__device__ __forceinline__ void s1_build_E(uint32_t *su, uint32_t *E, int lane) {
  constexpr uint32_t NV = P::Q0 / 4;
  constexpr uint32_t MASK_C = (1u << P::C) - 1u;
  static_assert(P::Q0 + 1 < 2 * P::U_STRIDE, "the staged row has a padding word after word Q0");
  static_assert(S::E_WORDS >= 2 * P::Q0 + 2, "E holds the doubled u: every path below writes E[2 Q0 + 1]");
  const uint32_t eq0 = su[P::Q0] & MASK_C;
  for (uint32_t c = lane; c < NV; c += NT)
    reinterpret_cast<uint4 *>(E)[c] = reinterpret_cast<const uint4 *>(su)[c];
  for (uint32_t q = 4 * NV + lane; q < P::Q0; q += NT) E[q] = su[q];
  if constexpr (NT == 64 && HQC_EBUILD_RUN2) {
    // Runs over x in [0, Q0 - 2], whose two source words are both below the partial word Q0 (no
    // masking, no in-place fix-up, no barrier); thread 0 adds the three words that involve word Q0.
    constexpr uint32_t NF = P::Q0 - 1;
    constexpr uint32_t CH = ((NF + NT - 1) / NT) | 1u;  // per-thread run, odd: conflict-free
    const uint32_t x0 = (uint32_t)lane * CH;
    uint32_t lo = x0 < NF ? su[x0] : 0u;
#pragma unroll 4
    for (uint32_t t = 0; t < CH; t++) {
      const uint32_t x = x0 + t;
      if (x < NF) {
        const uint32_t hi = su[x + 1];
        E[P::Q0 + 1 + x] = __funnelshift_r(lo, hi, 32 - P::C);
        lo = hi;
      }
    }
    if (lane == 0) {
      E[P::Q0] = eq0 | (su[0] << P::C);
      E[2 * P::Q0] = __funnelshift_r(su[P::Q0 - 1], eq0, 32 - P::C);  // x = Q0 - 1
      E[2 * P::Q0 + 1] = __funnelshift_r(eq0, 0u, 32 - P::C);         // x = Q0 (u32[Q0 + 1] = 0)
    }
    for (uint32_t q = 2 * P::Q0 + 2 + lane; q < S::E_WORDS; q += NT) E[q] = 0u;
  } else if constexpr (NT == 32) {
    constexpr uint32_t NF = P::Q0 + 1;                // funnel words x = 0..Q0
    constexpr uint32_t CH = ((NF + NT - 1) / NT) | 1u;  // per-lane run, odd
    const uint32_t s0 = su[0];
    __syncwarp();  // every lane has read su[0], su[Q0] before they are rewritten
    if (lane == 0) {
      E[P::Q0] = eq0 | (s0 << P::C);
      su[P::Q0] = eq0;
      su[P::Q0 + 1] = 0u;
    }
    __syncwarp();
    const uint32_t x0 = (uint32_t)lane * CH;
    uint32_t lo = x0 < NF ? su[x0] : 0u;
#pragma unroll 4
    for (uint32_t t = 0; t < CH; t++) {
      const uint32_t x = x0 + t;
      if (x < NF) {
        const uint32_t hi = su[x + 1];
        E[P::Q0 + 1 + x] = __funnelshift_r(lo, hi, 32 - P::C);
        lo = hi;
      }
    }
    for (uint32_t q = 2 * P::Q0 + 2 + lane; q < S::E_WORDS; q += NT) E[q] = 0u;
  } else {
    if (lane == 0) E[P::Q0] = eq0 | (su[0] << P::C);
#pragma unroll 4
    for (uint32_t q = P::Q0 + 1 + lane; q < S::E_WORDS; q += NT) {
      const uint32_t x = q - P::Q0 - 1;
      const uint32_t lo = x < P::Q0 ? su[x] : (x == P::Q0 ? eq0 : 0u);
      const uint32_t hi = x + 1 < P::Q0 ? su[x + 1] : (x + 1 == P::Q0 ? eq0 : 0u);
      E[q] = __funnelshift_r(lo, hi, 32 - P::C);
    }
  }
}

// Unroll of the run loop of s1_build_E_upper (its loads are independent; the runs are 19 / 35 / 57 words):
// 19 against 4 (profiles/r02/ab_eb.log): 1,024 decryptions HQC-1 / 3 / 5 +0.4 / +2.1 / +2.8%, large
// batches within ±0.1%, HQC-1 at 148 -1%.
#ifndef HQC_EBUILD_UNROLL
#define HQC_EBUILD_UNROLL 19
#endif
// E from the u row that TMA put in E's LOWER half (E[q] = u32[q] for q <= Q0; k_stage1, k_decrypt_sb /
// _sp / _wl): only the shifted upper copy is built — E[Q0 + 1 + x] = funnel(u32[x], u32[x + 1], 32 - C),
// u32[Q0] masked to its C valid bits, u32[Q0 + 1] = 0 — then word Q0 itself (the wrap of X^n = 1) and the
// zero tail up to S::E_WORDS. One warp; the lanes' runs read only below word Q0 and write above it, and
// lane 0 reads word Q0 before it rewrites it, so the build is in place with no hazard.
template <class P, class S>
__device__ __forceinline__ void s1_build_E_upper(uint32_t *E, int lane) {
  constexpr uint32_t MASK_C = (1u << P::C) - 1u;
  constexpr uint32_t NF = P::Q0 - 1;              // x = 0 .. Q0 - 2: both sources below word Q0
  constexpr uint32_t CH = ((NF + 31) / 32) | 1u;  // per-lane run, odd: conflict-free
  static_assert(S::E_WORDS >= 2 * P::Q0 + 2, "E holds the doubled u");
  uint32_t eq0 = 0, s0 = 0, sl = 0;
  if (lane == 0) {
    eq0 = E[P::Q0] & MASK_C;
    s0 = E[0];
    sl = E[P::Q0 - 1];
  }
  const uint32_t x0 = (uint32_t)lane * CH;
  uint32_t lo = x0 < NF ? E[x0] : 0u;
  constexpr int kEU = HQC_EBUILD_UNROLL;
#pragma unroll kEU
  for (uint32_t t = 0; t < CH; t++) {
    const uint32_t x = x0 + t;
    if (x < NF) {
      const uint32_t hi = E[x + 1];
      E[P::Q0 + 1 + x] = __funnelshift_r(lo, hi, 32 - P::C);
      lo = hi;
    }
  }
  if (lane == 0) {
    E[2 * P::Q0] = __funnelshift_r(sl, eq0, 32 - P::C);      // x = Q0 - 1
    E[2 * P::Q0 + 1] = __funnelshift_r(eq0, 0u, 32 - P::C);  // x = Q0 (u32[Q0 + 1] = 0)
    E[P::Q0] = eq0 | (s0 << P::C);
  }
  for (uint32_t q = 2 * P::Q0 + 2 + lane; q < S::E_WORDS; q += 32) E[q] = 0u;
}

// A rotation amount d = 32 o + s is kept as (o << 7) | s: its low 5 bits are the funnel-shift amount
// (SHF.R.W wraps the amount mod 32) and >> 5 is the window's byte offset 4 o, one shift instead of a
// shift and a mask per index.
// Packed at every level since the segmented layout: the one-warp kernels (HQC-1 -1%, HQC-5 -0.5%,
// standalone product -0.3..-0.8%) and now HQC-3's K4l too (65,536: 1.069 -> 1.054 ms; 1,024 -3%;
// profiles/r02/ab_pack.log); only round 1's HQC-3 warp pair had preferred the plain form (+1.3%).
#ifndef HQC_PACK_D
#define HQC_PACK_D 1
#endif
template <class P> __device__ __forceinline__ uint32_t s1_pack_d(uint32_t d) {
  return HQC_PACK_D ? ((d >> 5) << 7) | (d & 31u) : d;
}
template <class P, class T> __device__ __forceinline__ const T *s1_window(const T *Eb, uint32_t dp) {
  if (HQC_PACK_D)
    return reinterpret_cast<const T *>(reinterpret_cast<const char *>(Eb) + (dp >> 5));
  return Eb + (dp >> 5);
}

// The WT rotation amounts d_j = n - y_j from the staged support row (an entry >= n is treated as 0).
template <class P, class S, int NT = 32>
__device__ __forceinline__ void s1_stage_d(const uint32_t *sy, uint32_t *dsm, int lane) {
  for (uint32_t j = lane; j < S::WPAD; j += NT) {
    const uint32_t y = sy[j];
    const uint32_t d = (j < S::WT && y < P::N) ? P::N - y : P::N;
    dsm[j] = s1_pack_d<P>(d);
  }
}

// The rotate-and-XOR over support indices [j0, j1) (j0 even; the loop count is fixed by the level,
// not by the data). acc[k] accumulates output word lane*R + k.
template <class P, class S>
__device__ __forceinline__ void s1_product_range(const uint32_t *E, const uint32_t *dsm, uint32_t (&acc)[S::R],
                                                 int lane, uint32_t j0, uint32_t j1, bool init = true) {
  constexpr int R = S::R;
  if (init) {
#pragma unroll
    for (int k = 0; k < R; k++) acc[k] = 0;
  }
  const uint32_t *Eb = E + lane * R;
  uint32_t j = j0;
  constexpr int kUnroll = s1_unroll<P>();
#pragma unroll kUnroll
  for (; j + 1 < j1; j += 2) {  // two indices per pass: one 3-input XOR per word
    const uint2 dd = *reinterpret_cast<const uint2 *>(dsm + j);
    const uint32_t *p0 = s1_window<P>(Eb, dd.x);
    const uint32_t *p1 = s1_window<P>(Eb, dd.y);
    uint32_t a0 = p0[0], b0 = p1[0];
#pragma unroll
    for (int k = 0; k < R; k++) {
      const uint32_t a1 = p0[k + 1], b1 = p1[k + 1];
      acc[k] ^= __funnelshift_r(a0, a1, dd.x) ^ __funnelshift_r(b0, b1, dd.y);
      a0 = a1;
      b0 = b1;
    }
  }
  if (j < j1) {
    const uint32_t d = dsm[j];
    const uint32_t *p0 = s1_window<P>(Eb, d);
    uint32_t a0 = p0[0];
#pragma unroll
    for (int k = 0; k < R; k++) {
      const uint32_t a1 = p0[k + 1];
      acc[k] ^= __funnelshift_r(a0, a1, d);
      a0 = a1;
    }
  }
}

// The same product with SHIFTED lane windows (ShShape, levels.cuh): lane L loads only the R words
// E[o + L R + k], k < R, and takes the word before them, E[o + L R - 1] — the last word its left neighbour
// loaded — with one SHFL.UP instead of an (R+1)-th shared-memory load: R loads per (index, lane) instead of
// R + 1, i.e. 1/R fewer shared-memory wavefronts in the loop that binds every kernel.
// acc[k] accumulates output word L R - 1 + k; lane 0's acc[0] (word -1) is garbage and never stored.
template <class P, class S>
__device__ __forceinline__ void s1_product_range_sh(const uint32_t *E, const uint32_t *dsm, uint32_t (&acc)[S::R],
                                                    int lane, uint32_t j0, uint32_t j1) {
  constexpr int R = S::R;
#pragma unroll
  for (int k = 0; k < R; k++) acc[k] = 0;
  const uint32_t *Eb = E + lane * R;
  uint32_t j = j0;
  constexpr int kUnroll = s1_unroll<P>();
#pragma unroll kUnroll
  for (; j + 1 < j1; j += 2) {
    const uint2 dd = *reinterpret_cast<const uint2 *>(dsm + j);
    const uint32_t *p0 = s1_window<P>(Eb, dd.x);
    const uint32_t *p1 = s1_window<P>(Eb, dd.y);
    const uint32_t l0 = p0[R - 1], l1 = p1[R - 1];  // the last words first: the right neighbour needs them
    uint32_t a0 = __shfl_up_sync(0xffffffffu, l0, 1), b0 = __shfl_up_sync(0xffffffffu, l1, 1);
#pragma unroll
    for (int k = 0; k < R; k++) {
      const uint32_t a1 = k + 1 < R ? p0[k] : l0, b1 = k + 1 < R ? p1[k] : l1;
      acc[k] ^= __funnelshift_r(a0, a1, dd.x) ^ __funnelshift_r(b0, b1, dd.y);
      a0 = a1;
      b0 = b1;
    }
  }
  if (j < j1) {
    const uint32_t d = dsm[j];
    const uint32_t *p0 = s1_window<P>(Eb, d);
    const uint32_t l0 = p0[R - 1];
    uint32_t a0 = __shfl_up_sync(0xffffffffu, l0, 1);
#pragma unroll
    for (int k = 0; k < R; k++) {
      const uint32_t a1 = k + 1 < R ? p0[k] : l0;
      acc[k] ^= __funnelshift_r(a0, a1, d);
      a0 = a1;
    }
  }
}

// Stores of the shifted accumulators: word L R - 1 + k (skipping lane 0's word -1), < S::NOUT.
template <class S>
__device__ __forceinline__ void s1_store_r_sh(const uint32_t (&acc)[S::R], uint32_t *rsm, int lane) {
#pragma unroll
  for (int k = 0; k < (int)S::R; k++) {
    const int w = lane * (int)S::R - 1 + k;
    if (w >= 0 && w < (int)S::NOUT) rsm[w] = acc[k];
  }
}
template <class S>
__device__ __forceinline__ void s1_store_r_xor_sh(const uint32_t (&acc)[S::R], uint32_t *rsm, const uint32_t *sv,
                                                  int lane) {
#pragma unroll
  for (int k = 0; k < (int)S::R; k++) {
    const int w = lane * (int)S::R - 1 + k;
    if (w >= 0 && w < (int)S::NOUT) rsm[w] = acc[k] ^ sv[w];
  }
}

// All S::WT indices (from 0, so dsm is 16-byte aligned at every group of four): the rotation amounts of
// four indices come in one broadcast 16-byte load (one shared-memory wavefront instead of two).
// Measured against the same build without it (profiles/r02/ab_dd4_clean.log): no difference within
// ±0.4% (the 25-50 wavefronts it saves per decryption are not what limits), so off; an experiment switch.
#ifndef HQC_S1_DD4
#define HQC_S1_DD4 0
#endif
template <class P, class S>
__device__ __forceinline__ void s1_product(const uint32_t *E, const uint32_t *dsm, uint32_t (&acc)[S::R],
                                           int lane) {
  if constexpr (!HQC_S1_DD4) {
    s1_product_range<P, S>(E, dsm, acc, lane, 0, S::WT);
  } else {
    constexpr int R = S::R;
#pragma unroll
    for (int k = 0; k < R; k++) acc[k] = 0;
    const uint32_t *Eb = E + lane * R;
    auto pair = [&](uint32_t dx, uint32_t dy) {
      const uint32_t *p0 = s1_window<P>(Eb, dx);
      const uint32_t *p1 = s1_window<P>(Eb, dy);
      uint32_t a0 = p0[0], b0 = p1[0];
#pragma unroll
      for (int k = 0; k < R; k++) {
        const uint32_t a1 = p0[k + 1], b1 = p1[k + 1];
        acc[k] ^= __funnelshift_r(a0, a1, dx) ^ __funnelshift_r(b0, b1, dy);
        a0 = a1;
        b0 = b1;
      }
    };
    uint32_t j = 0;
#pragma unroll 1
    for (; j + 3 < S::WT; j += 4) {
      const uint4 d4 = *reinterpret_cast<const uint4 *>(dsm + j);
      pair(d4.x, d4.y);
      pair(d4.z, d4.w);
    }
    if constexpr (S::WT % 4 >= 2) {
      const uint2 dd = *reinterpret_cast<const uint2 *>(dsm + j);
      pair(dd.x, dd.y);
      j += 2;
    }
    if constexpr (S::WT % 2) {
      const uint32_t d = dsm[j];
      const uint32_t *p0 = s1_window<P>(Eb, d);
      uint32_t a0 = p0[0];
#pragma unroll
      for (int k = 0; k < R; k++) {
        const uint32_t a1 = p0[k + 1];
        acc[k] ^= __funnelshift_r(a0, a1, d);
        a0 = a1;
      }
    }
  }
}

// Words [Q, Q + TW) of the product by the whole warp (the ragged top above the lanes' R-word blocks): lane
// L takes support indices L, L + 32, ... (a fixed count per level), funnels TW + 1 consecutive words of
// each window, and the warp XOR-reduces each word (REDUX). Reads E: call before r overwrites it.
template <class P, class S, uint32_t Q, uint32_t TW>
__device__ __forceinline__ void s1_tail_words(const uint32_t *E, const uint32_t *dsm, int lane, uint32_t (&t)[TW]) {
  uint32_t x[TW];
#pragma unroll
  for (uint32_t i = 0; i < TW; i++) x[i] = 0;
  for (uint32_t j = lane; j < S::WT; j += 32) {
    const uint32_t d = dsm[j];
    const uint32_t *p = s1_window<P>(E + Q, d);
    uint32_t a = p[0];
#pragma unroll
    for (uint32_t i = 0; i < TW; i++) {
      const uint32_t b = p[i + 1];
      x[i] ^= __funnelshift_r(a, b, d);
      a = b;
    }
  }
#pragma unroll
  for (uint32_t i = 0; i < TW; i++) t[i] = __reduce_xor_sync(0xffffffffu, x[i]);
}

// Store the accumulators (S::NOUT words, aliasing E). The caller synchronises the warp first.
template <class S>
__device__ __forceinline__ void s1_store_r(const uint32_t (&acc)[S::R], uint32_t *rsm, int lane) {
#pragma unroll
  for (int k = 0; k < (int)S::R; k++)
    if (lane * S::R + k < S::NOUT) rsm[lane * S::R + k] = acc[k];
}

// Store acc XOR v (v staged in shared memory): lane L reads v words L*R + k — R odd, conflict-free.
template <class S>
__device__ __forceinline__ void s1_store_r_xor(const uint32_t (&acc)[S::R], uint32_t *rsm, const uint32_t *sv,
                                               int lane) {
#pragma unroll
  for (int k = 0; k < (int)S::R; k++)
    if (lane * S::R + k < S::NOUT) rsm[lane * S::R + k] = acc[k] ^ sv[lane * S::R + k];
}

// Store acc XOR x XOR v, where x is another warp's accumulator image (same word layout).
template <class S>
__device__ __forceinline__ void s1_store_r_xor2(const uint32_t (&acc)[S::R], uint32_t *rsm, const uint32_t *xs,
                                                const uint32_t *sv, int lane) {
#pragma unroll
  for (int k = 0; k < (int)S::R; k++)
    if (lane * S::R + k < S::NOUT) rsm[lane * S::R + k] = acc[k] ^ xs[lane * S::R + k] ^ sv[lane * S::R + k];
}

// In-place XOR of the accumulators into a buffer (rsm[lane*R + k] ^= acc[k]); R odd: conflict-free.
template <class S>
__device__ __forceinline__ void s1_xor_into(const uint32_t (&acc)[S::R], uint32_t *rsm, int lane) {
#pragma unroll
  for (int k = 0; k < (int)S::R; k++)
    if (lane * S::R + k < S::NOUT) rsm[lane * S::R + k] ^= acc[k];
}

// r ^= v with v staged in shared memory (16-byte chunks).
template <uint32_t NWORDS>
__device__ __forceinline__ void s1_xor_v(uint32_t *rsm, const uint32_t *sv, int lane) {
  for (uint32_t c = lane; c < NWORDS / 4; c += 32) {
    const uint4 vv = reinterpret_cast<const uint4 *>(sv)[c];
    uint4 rr = reinterpret_cast<uint4 *>(rsm)[c];
    rr.x ^= vv.x; rr.y ^= vv.y; rr.z ^= vv.z; rr.w ^= vv.w;
    reinterpret_cast<uint4 *>(rsm)[c] = rr;
  }
}

// ------------------------------------------------------------------------------------------------
// The SEGMENTED lane layout (round 2). The R-word lanes above load R + 1 window words per
// (index, lane) for R outputs — the (R+1)-th only for the high part of the lane's last funnel — and R is
// odd (conflict-free strides), so a warp issues R + 1 = ceil(NOUT/32) + 1..2 loads per index plus, where
// 32 R < NOUT, a ragged top (s1_tail_words: lane-per-index loads with random banks). Here:
//  * lane L owns the output words [st_L, st_L + len_L), contiguous in lane order, len_L in [LMIN, LMAX]
//    (LMAX = ceil(NB/32)), the starts st_L DISTINCT mod 32 (seg_plans.cuh, generated by
//    scripts/gen_segments.py), so the lanes' loads E[o + st_L + k] of every slot k hit 32 distinct banks;
//  * a funnel splits into two shifts that do not overlap: SHF(lo, hi, s) = SHF(lo, 0, s) ^ SHF(0, hi, s).
//    A LONG lane (len_L = LMAX) loads only its own LMAX words; the high part of its last funnel comes from
//    its right neighbour, which accumulates SHF(0, first word, s) over the indices in one register (`pre`)
//    and passes it on with ONE shuffle per product (round 2's per-index SHFL variant lost: it shares the
//    shared-memory data path). A SHORT lane loads its len_L + 1 words itself, in slots the long lanes use;
//  * the top neighbour word(s) of a long last lane, E[o + NB .. o + NOUT], come from a lane-per-index pass
//    (TP words per index, one REDUX per word) — HQC-3 (1,120 = 32 x 35 words) and HQC-5.
// So a warp issues LMAX loads per index (HQC-1 18, HQC-3 35, HQC-5 57; round 2: 18 + a 9-word tail, 36, 58)
// for 1.5 (LMAX + 1) ALU ops per index (the extra shift pair of `pre`). The loop count is the level's w for
// every ciphertext; the slot predicates depend on the lane only.
template <class P, uint32_t NOUT_, uint32_t WT_> struct SegShape {
  using PL = SegPlan<NOUT_>;
  static constexpr uint32_t NOUT = NOUT_, WT = WT_, WPAD = round_up(WT_, 4);
  static constexpr uint32_t NB = PL::NB, LMAX = PL::LMAX, TP = PL::TP;
  static constexpr uint32_t lmin() {
    uint32_t m = LMAX;
    for (int i = 0; i < 32; i++) m = PL::LEN[i] < m ? PL::LEN[i] : m;
    return m;
  }
  static constexpr uint32_t LMIN = lmin();
  static constexpr uint32_t def_mask(int bit) {
    uint32_t m = 0;
    for (int i = 0; i < 32; i++) m |= (((LMAX - PL::LEN[i]) >> bit) & 1u) << i;
    return m;
  }
  static constexpr uint32_t D1 = def_mask(0), D2 = def_mask(1);  // bits of LMAX - len_L
  static constexpr bool valid() {
    uint32_t st = 0, seen = 0;
    for (int i = 0; i < 32; i++) {
      if (PL::LEN[i] > LMAX || LMAX - PL::LEN[i] > 3) return false;
      if ((seen >> (st & 31)) & 1u) return false;  // two starts in one bank
      seen |= 1u << (st & 31);
      st += PL::LEN[i];
    }
    if (st != NB) return false;
    if (TP == 0) return NB == NOUT && PL::LEN[31] < LMAX;  // the last lane loads its own neighbour word
    return NB + TP - 1 == NOUT && PL::LEN[31] == LMAX && TP <= 2;
  }
  static_assert(valid(), "seg_plans.cuh: lengths, distinct starts mod 32, top handling");
  // E must hold the window words up to o + NOUT, o <= Q0 (every d <= n)
  static constexpr uint32_t E_NEED = P::Q0 + NOUT + 1;
  __device__ __forceinline__ static uint32_t len(int lane) {
    return LMAX - ((D1 >> lane) & 1u) - 2u * ((D2 >> lane) & 1u);
  }
  __device__ __forceinline__ static uint32_t start(int lane) {
    const uint32_t lt = (1u << lane) - 1u;
    return (uint32_t)lane * LMAX - __popc(D1 & lt) - 2u * __popc(D2 & lt);
  }
};
template <class P> using DecSeg = SegShape<P, P::NW, P::W>;        // u*y truncated (decrypt r)
template <class P> using FullSeg = SegShape<P, P::Q0 + 1, P::WR>;  // h*r2, all n bits (Encrypt u)
template <class P> using KeySeg = SegShape<P, P::Q0 + 1, P::W>;    // h*y (KeyGen s)
template <class P> using EncVSeg = SegShape<P, P::NW, P::WR>;      // s*r2 truncated (Encrypt v)

// The product over support indices [j0, j1) (j0 even) in the segmented layout: acc[k] = output word
// st_L + k for k < len_L (complete, the neighbour's part included); `top` = word NB + lane for lane < TP - 1.
template <class P, class G, int UNROLL = s1_unroll<P>()>
__device__ __forceinline__ void s1_seg_product(const uint32_t *E, const uint32_t *dsm, uint32_t (&acc)[G::LMAX],
                                               uint32_t &top, int lane, uint32_t j0 = 0, uint32_t j1 = G::WT) {
  constexpr int L = (int)G::LMAX, LMIN = (int)G::LMIN;
  constexpr int NPS = L - 1 - LMIN > 0 ? L - 1 - LMIN : 1;  // predicated slots k + 1 in (LMIN, L - 1]
  const uint32_t len = G::len(lane);
  const uint32_t *Eb = E + G::start(lane);
#pragma unroll
  for (int k = 0; k < L; k++) acc[k] = 0;
  uint32_t pre = 0;
  // Slots above LMIN are loaded only by lanes whose segment reaches them; the others keep a stale value
  // (loop-carried registers, no zeroing): it reaches only accumulators above their segment, never stored.
  uint32_t ja[NPS], jb[NPS];
#pragma unroll
  for (int i = 0; i < NPS; i++) ja[i] = jb[i] = 0;
  uint32_t j = j0;
  constexpr int kUnroll = UNROLL;
#pragma unroll kUnroll
  for (; j + 1 < j1; j += 2) {
    const uint2 dd = *reinterpret_cast<const uint2 *>(dsm + j);
    const uint32_t *p0 = s1_window<P>(Eb, dd.x);
    const uint32_t *p1 = s1_window<P>(Eb, dd.y);
    uint32_t a0 = p0[0], b0 = p1[0];
    pre ^= __funnelshift_r(0u, a0, dd.x) ^ __funnelshift_r(0u, b0, dd.y);
#pragma unroll
    for (int k = 0; k < L; k++) {
      uint32_t a1, b1;
      if (k + 1 == L) {
        a1 = 0u;
        b1 = 0u;
      } else if (k + 1 <= LMIN) {
        a1 = p0[k + 1];
        b1 = p1[k + 1];
      } else {
        const int i = k - LMIN;
        if ((uint32_t)(k + 1) <= len) {
          ja[i] = p0[k + 1];
          jb[i] = p1[k + 1];
        }
        a1 = ja[i];
        b1 = jb[i];
      }
      acc[k] ^= __funnelshift_r(a0, a1, dd.x) ^ __funnelshift_r(b0, b1, dd.y);
      a0 = a1;
      b0 = b1;
    }
  }
  if (j < j1) {
    const uint32_t d = dsm[j];
    const uint32_t *p0 = s1_window<P>(Eb, d);
    uint32_t a0 = p0[0];
    pre ^= __funnelshift_r(0u, a0, d);
#pragma unroll
    for (int k = 0; k < L; k++) {
      uint32_t a1;
      if (k + 1 == L) {
        a1 = 0u;
      } else if (k + 1 <= LMIN) {
        a1 = p0[k + 1];
      } else {
        const int i = k - LMIN;
        if ((uint32_t)(k + 1) <= len) ja[i] = p0[k + 1];
        a1 = ja[i];
      }
      acc[k] ^= __funnelshift_r(a0, a1, d);
      a0 = a1;
    }
  }
  uint32_t x[G::TP > 0 ? G::TP : 1];
#pragma unroll
  for (uint32_t i = 0; i < (G::TP > 0 ? G::TP : 1); i++) x[i] = 0;
  if constexpr (G::TP > 0) {
    // E[o + NB + i], i < TP, lane per index (ceil((j1 - j0) / 32) rounds, fixed by the level)
    for (uint32_t jj = j0 + lane; jj < j1; jj += 32) {
      const uint32_t d = dsm[jj];
      const uint32_t *p = s1_window<P>(E + G::NB, d);
      uint32_t w0 = p[0];
      x[0] ^= __funnelshift_r(0u, w0, d);
#pragma unroll
      for (uint32_t i = 1; i < G::TP; i++) {
        const uint32_t w1 = p[i];
        x[i] ^= __funnelshift_r(w0, w1, d);
        w0 = w1;
      }
    }
#pragma unroll
    for (uint32_t i = 0; i < G::TP; i++) x[i] = __reduce_xor_sync(0xffffffffu, x[i]);
  }
  uint32_t nxt = __shfl_down_sync(0xffffffffu, pre, 1);
  if constexpr (G::TP > 0) nxt = lane == 31 ? x[0] : nxt;
  if (len == (uint32_t)L) acc[L - 1] ^= nxt;
  top = 0;
#pragma unroll
  for (uint32_t i = 1; i < G::TP; i++) top = (uint32_t)lane == i - 1 ? x[i] : top;
}

// Stores of the segmented accumulators (the caller synchronises the warp first when rsm aliases E):
// rsm[w] = acc (^ sv[w]) (^ xs[w]) for the lane's words w; starts distinct mod 32: conflict-free.
template <class G, int MODE>
__device__ __forceinline__ void s1_seg_store_impl(const uint32_t (&acc)[G::LMAX], uint32_t top, uint32_t *rsm,
                                                  const uint32_t *xs, const uint32_t *sv, int lane) {
  const uint32_t len = G::len(lane), st = G::start(lane);
#pragma unroll
  for (int k = 0; k < (int)G::LMAX; k++) {
    if (k < (int)G::LMIN || (uint32_t)k < len) {
      uint32_t x = acc[k];
      if (MODE >= 1) x ^= sv[st + k];
      if (MODE >= 2) x ^= xs[st + k];
      rsm[st + k] = x;
    }
  }
  if constexpr (G::TP > 1) {
    if ((uint32_t)lane < G::TP - 1) {
      uint32_t x = top;
      if (MODE >= 1) x ^= sv[G::NB + lane];
      if (MODE >= 2) x ^= xs[G::NB + lane];
      rsm[G::NB + lane] = x;
    }
  }
}
template <class G>
__device__ __forceinline__ void s1_seg_store(const uint32_t (&acc)[G::LMAX], uint32_t top, uint32_t *rsm, int lane) {
  s1_seg_store_impl<G, 0>(acc, top, rsm, nullptr, nullptr, lane);
}
template <class G>
__device__ __forceinline__ void s1_seg_store_xor(const uint32_t (&acc)[G::LMAX], uint32_t top, uint32_t *rsm,
                                                 const uint32_t *sv, int lane) {
  s1_seg_store_impl<G, 1>(acc, top, rsm, nullptr, sv, lane);
}
template <class G>
__device__ __forceinline__ void s1_seg_store_xor2(const uint32_t (&acc)[G::LMAX], uint32_t top, uint32_t *rsm,
                                                  const uint32_t *xs, const uint32_t *sv, int lane) {
  s1_seg_store_impl<G, 2>(acc, top, rsm, xs, sv, lane);
}

}  // namespace hqc
