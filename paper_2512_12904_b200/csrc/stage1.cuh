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
#pragma once
#include <cstdint>

#include "levels.cuh"

namespace hqc {

__device__ __forceinline__ uint4 ld_stream_u4(const void *p) {
  uint4 r;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const void *p) {
  uint32_t r;
  asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

// Build E (P::E_WORDS words) in shared memory from one u row (global, 16-byte aligned).
template <class P>
__device__ __forceinline__ void s1_build_E(const uint64_t *__restrict__ u_row, uint32_t *E, int lane) {
  const uint32_t *u32 = reinterpret_cast<const uint32_t *>(u_row);
  constexpr uint32_t NV = P::Q0 / 4;
  constexpr uint32_t MASK_C = (1u << P::C) - 1u;
  // words below Q0: u itself (coalesced 16-byte loads)
  for (uint32_t c = lane; c < NV; c += 32) {
    uint4 x = ld_stream_u4(u32 + 4 * c);
    *reinterpret_cast<uint4 *>(E + 4 * c) = x;
  }
  for (uint32_t q = 4 * NV + lane; q < P::Q0; q += 32) E[q] = ld_stream_u32(u32 + q);
  // word Q0: the last C bits of u, then u continues from bit 0 (the wrap of X^n = 1)
  if (lane == 0) E[P::Q0] = (ld_stream_u32(u32 + P::Q0) & MASK_C) | (ld_stream_u32(u32) << P::C);
  __syncwarp();
  const uint32_t eq0 = E[P::Q0] & MASK_C;  // u32[Q0] with the bits >= n cleared
  // words above Q0: E word q holds u bits [32q - n, 32q - n + 32) = funnel(u32[x], u32[x+1], 32 - C)
  // with x = q - Q0 - 1. Words that no valid output reads are filled with zeros.
#pragma unroll 4
  for (uint32_t q = P::Q0 + 1 + lane; q < P::E_WORDS; q += 32) {
    const uint32_t x = q - P::Q0 - 1;
    const uint32_t lo = x < P::Q0 ? E[x] : (x == P::Q0 ? eq0 : 0u);
    const uint32_t hi = x + 1 < P::Q0 ? E[x + 1] : (x + 1 == P::Q0 ? eq0 : 0u);
    E[q] = __funnelshift_r(lo, hi, 32 - P::C);
  }
}

// Stage the w rotation amounts d_j = n - y_j (an entry >= n is treated as y = 0).
template <class P>
__device__ __forceinline__ void s1_stage_d(const uint32_t *__restrict__ y_row, uint32_t *dsm, int lane) {
  for (uint32_t j = lane; j < P::WPAD; j += 32) {
    uint32_t d = P::N;
    if (j < P::W) {
      const uint32_t y = __ldg(y_row + j);
      d = y < P::N ? P::N - y : P::N;
    }
    dsm[j] = d;
  }
}

// The w-iteration rotate-and-XOR. acc[k] accumulates output word lane*R + k.
template <class P>
__device__ __forceinline__ void s1_product(const uint32_t *E, const uint32_t *dsm, uint32_t (&acc)[P::R],
                                           int lane) {
  constexpr int R = P::R;
#pragma unroll
  for (int k = 0; k < R; k++) acc[k] = 0;
  const uint32_t *Eb = E + lane * R;
#pragma unroll 1
  for (uint32_t j = 0; j + 1 < P::W; j += 2) {  // two indices per pass: one 3-input XOR per word
    const uint2 dd = *reinterpret_cast<const uint2 *>(dsm + j);
    const uint32_t *p0 = Eb + (dd.x >> 5);
    const uint32_t *p1 = Eb + (dd.y >> 5);
    uint32_t a0 = p0[0], b0 = p1[0];
#pragma unroll
    for (int k = 0; k < R; k++) {
      const uint32_t a1 = p0[k + 1], b1 = p1[k + 1];
      acc[k] ^= __funnelshift_r(a0, a1, dd.x) ^ __funnelshift_r(b0, b1, dd.y);
      a0 = a1;
      b0 = b1;
    }
  }
  if (P::W & 1) {
    const uint32_t d = dsm[P::W - 1];
    const uint32_t *p0 = Eb + (d >> 5);
    uint32_t a0 = p0[0];
#pragma unroll
    for (int k = 0; k < R; k++) {
      const uint32_t a1 = p0[k + 1];
      acc[k] ^= __funnelshift_r(a0, a1, d);
      a0 = a1;
    }
  }
}

// Full stage 1 for one ciphertext: leaves r (P::NW words) at rsm (which aliases E).
// v_row may be null (product only).
template <class P>
__device__ __forceinline__ void s1_run(const uint64_t *__restrict__ u_row, const uint32_t *__restrict__ y_row,
                                       const uint64_t *__restrict__ v_row, uint32_t *E, uint32_t *dsm, int lane) {
  s1_stage_d<P>(y_row, dsm, lane);
  s1_build_E<P>(u_row, E, lane);
  __syncwarp();
  uint32_t acc[P::R];
  s1_product<P>(E, dsm, acc, lane);
  __syncwarp();  // every lane is done reading E: r overwrites it
  uint32_t *rsm = E;
#pragma unroll
  for (int k = 0; k < (int)P::R; k++)
    if (lane * P::R + k < P::NW) rsm[lane * P::R + k] = acc[k];
  __syncwarp();
  if (v_row != nullptr) {
    const uint32_t *v32 = reinterpret_cast<const uint32_t *>(v_row);
    for (uint32_t c = lane; c < P::NW / 4; c += 32) {
      const uint4 vv = ld_stream_u4(v32 + 4 * c);
      uint4 *rp = reinterpret_cast<uint4 *>(rsm + 4 * c);
      uint4 rr = *rp;
      rr.x ^= vv.x; rr.y ^= vv.y; rr.z ^= vv.z; rr.w ^= vv.w;
      *rp = rr;
    }
    __syncwarp();
  }
}

}  // namespace hqc
