// Stage 2 — duplicated RM(1,7) decoding of one n2-bit block by one thread (Table I P:113-117,
// "byte-parallel Reed–Muller decoder" P:33; readings R#9-R#12 in DESIGN.md). DESIGN.md §6.2.
//
// The oracle defines F(a) = sum_p s_p (-1)^{a.p} with s_p = mult - 2*cnt_p (cnt_p = number of copies
// with bit p set) and picks the smallest a with maximal |F(a)|, sign -> bit 7. Here:
//   1. bit-sliced copy counting: cnt_p in 2 (mult 3) or 3 (mult 5) bit planes, 32 positions per op;
//   2. soft values -2*cnt as exact fp16 in half2 registers: register i = 16q + l holds positions
//      (32q+l, 32q+l+16); the count's bit planes are placed side by side in the mantissa and one HFMA2
//      turns 1024 + 2^l' cnt into -2 cnt;
//   3. the 128-point fast Walsh–Hadamard transform: 6 butterfly stages across registers (HADD2 on
//      the FMA pipe) and one in-register stage (HFMA2 with a (1,-1) multiplier). Every value is an
//      integer of magnitude <= 640 < 2048, so fp16 arithmetic is exact;
//   4. F = FWHT(-2 cnt) + 128*mult*[a = 0]: exactly the oracle's F;
//   5. M = max |F| (HMNMX2 tree), then 128-bit masks of {|F| = M} and {F = -M} in natural a order;
//      a* = lowest set bit (smallest a, R#11), bit 7 = [F(a*) = -M].
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

namespace hqc {

__device__ __forceinline__ __half2 u2h(uint32_t x) { return *reinterpret_cast<__half2 *>(&x); }

// (a & m) | c as ONE lop3 (keeps the compiler from re-deriving a per use); m and c in registers
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t m, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(m), "r"(c));
  return d;
}


// Argmax by a tournament that carries the signed winner and its register index (3 ops per node: one
// HSET2 on |right| > |left|, two selects), instead of a max tree and then two 128-bit equality masks
// (~5 ops per register).
#ifndef HQC_RM_TOURNAMENT
#define HQC_RM_TOURNAMENT 1
#endif

__device__ __forceinline__ uint32_t h2u(__half2 x) { return *reinterpret_cast<uint32_t *>(&x); }
__device__ __forceinline__ uint32_t sel_bits(uint32_t m, uint32_t a, uint32_t b) {  // m ? a : b, bitwise
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(d) : "r"(m), "r"(a), "r"(b));
  return d;
}

// F = FWHT(-2 cnt) in h (register i = 16q + l holds a = 32q + l, 32q + l + 16): add the constant part,
// take M = max |F|, and return the smallest a with |F(a)| = M (R#11) with bit 7 = [F(a) = -M].
template <int MULT>
__device__ __forceinline__ uint32_t rm_argmax(__half2 (&h)[64]) {
  // a = 0: F(0) += 128 * mult (the constant part of the soft values)
  h[0] = __hadd2(h[0], __halves2half2(__float2half(128.0f * MULT), __float2half(0.0f)));
#if HQC_RM_TOURNAMENT
  // Per half (a's bit 4), a = 32 (i >> 4) + (i & 15) [+ 16] grows with the register index i, so a node
  // A node joins two ADJACENT register ranges [i, i+s) and [i+s, i+2s) and keeps the left winner unless
  // |right| > |left|: ties go to the smaller a (R#11). The leaves' index words are constants (i in both
  // halves); after 6 levels each half holds its winner.
  uint32_t v[32], ix[32];
#pragma unroll
  for (int k = 0; k < 32; k++) {
    const uint32_t gt = __hgt2_mask(__habs2(h[2 * k + 1]), __habs2(h[2 * k]));
    v[k] = sel_bits(gt, h2u(h[2 * k + 1]), h2u(h[2 * k]));
    ix[k] = sel_bits(gt, (uint32_t)(2 * k + 1) * 0x10001u, (uint32_t)(2 * k) * 0x10001u);
  }
#pragma unroll
  for (int n = 16; n >= 1; n >>= 1)  // v[k] covers registers [k 64/2n, (k+1) 64/2n)
#pragma unroll
    for (int k = 0; k < n; k++) {
      const uint32_t gt = __hgt2_mask(__habs2(u2h(v[2 * k + 1])), __habs2(u2h(v[2 * k])));
      v[k] = sel_bits(gt, v[2 * k + 1], v[2 * k]);
      ix[k] = sel_bits(gt, ix[2 * k + 1], ix[2 * k]);
    }
  // the two halves: a_lo = 32 (i_lo >> 4) + (i_lo & 15), a_hi = the same for i_hi, + 16
  const uint32_t ilo = ix[0] & 0xFFFFu, ihi = ix[0] >> 16;
  const uint32_t alo = ((ilo >> 4) << 5) | (ilo & 15u), ahi = ((ihi >> 4) << 5) | (ihi & 15u) | 16u;
  const float flo = __low2float(u2h(v[0])), fhi = __high2float(u2h(v[0]));
  const float mlo = fabsf(flo), mhi = fabsf(fhi);
  const bool hi = mhi > mlo || (mhi == mlo && ahi < alo);
  const uint32_t a = hi ? ahi : alo;
  const uint32_t neg = (hi ? fhi : flo) < 0.0f ? 1u : 0u;
  return a | (neg << 7);
#else

  // M = max |F| (balanced tree for ILP)
  __half2 m[32];
#pragma unroll
  for (int i = 0; i < 32; i++) m[i] = __hmax2(__habs2(h[i]), __habs2(h[i + 32]));
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1)
#pragma unroll
    for (int i = 0; i < s; i++) m[i] = __hmax2(m[i], m[i + s]);
  const __half Mh = __hmax(__low2half(m[0]), __high2half(m[0]));
  const __half2 M2 = __half2half2(Mh);
  const __half2 nM2 = __hneg2(M2);

  // masks in natural order: word q = i >> 4 holds a in [32q, 32q+32); bit (i&15) + 16*half
  uint32_t absw[4] = {0u, 0u, 0u, 0u}, posw[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 0; i < 64; i++) {
    const uint32_t bit = 0x00010001u << (i & 15);
    absw[i >> 4] |= __heq2_mask(__habs2(h[i]), M2) & bit;
    posw[i >> 4] |= __heq2_mask(h[i], nM2) & bit;  // F(a) = -M: the codeword's bit 7 is set
  }
  // smallest a with |G(a)| = M (lowest set bit, lowest word first)
  uint32_t a = 0, pw = 0;
  bool found = false;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const bool take = !found && absw[q] != 0;
    const uint32_t bitpos = __ffs(absw[q]) - 1;
    a = take ? (32u * q + bitpos) : a;
    pw = take ? (posw[q] >> bitpos) & 1u : pw;
    found = found || take;
  }
  return a | (pw << 7);
#endif
}

// X[c*4 + q] = 32-bit word q of copy c of the block.
template <int MULT>
__device__ __forceinline__ uint32_t rm_decode_block(const uint32_t (&X)[MULT * 4]) {
  static_assert(MULT == 3 || MULT == 5, "duplicated RM(1,7) with 3 or 5 copies");
  constexpr int NPL = (MULT == 3) ? 2 : 3;
  uint32_t pl[NPL][4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t a = X[q], b = X[4 + q], c = X[8 + q];
    const uint32_t s1 = a ^ b ^ c, c1 = (a & b) | (c & (a ^ b));  // full adder
    if constexpr (MULT == 3) {
      pl[0][q] = s1;
      pl[1][q] = c1;
    } else {
      const uint32_t d = X[12 + q], e = X[16 + q];
      const uint32_t s2 = s1 ^ d ^ e, c2 = (s1 & d) | (e & (s1 ^ d));  // full adder
      pl[0][q] = s2;
      pl[1][q] = c1 ^ c2;  // half adder of the two carries (weight 2)
      pl[2][q] = c1 & c2;  // weight 4
    }
  }

  // soft values v_p = -2*cnt_p (the constant mult of s_p = mult - 2 cnt_p is added to F(0) below) as
  // exact fp16 in one HFMA2 per register: the count's bit planes are placed side by side in the mantissa,
  //   x = 0x6400 | plane0 bit at 2^l' | plane1 bit at 2^(l'+1) | plane2 bit at 2^(l'+2)  (per half)
  //     = 1024 + 2^l' cnt  (<= 1024 + 128*7 < 2048: every value exact),
  //   v = fma(x, -2^(1-l'), 2^(11-l')) = -2 cnt,
  // with l' = l for positions l <= 7 (planes pre-shifted left by 0/1/2) and l' = l - 8 for l >= 8 (planes
  // pre-shifted right by 8/7/6), so the three bits never leave their half. 3 LOP3 + 1 HFMA2 per register
  // (mult 3: 2 LOP3 + 1 HFMA2).
  __half2 h[64];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uint32_t lo[NPL], hi[NPL];
#pragma unroll
    for (int k = 0; k < NPL; k++) {
      lo[k] = pl[k][q] << k;
      hi[k] = pl[k][q] >> (8 - k);
    }
#pragma unroll
    for (int l = 0; l < 16; l++) {
      const int lp = l & 7;
      const uint32_t m0 = 0x00010001u << lp;
      uint32_t x = and_or(l < 8 ? lo[0] : hi[0], m0, 0x64006400u);
#pragma unroll
      for (int k = 1; k < NPL; k++) x = and_or(l < 8 ? lo[k] : hi[k], m0 << k, x);
      h[16 * q + l] = __hfma2(u2h(x), __float2half2_rn(-ldexpf(1.0f, 1 - lp)), __float2half2_rn(ldexpf(1.0f, 11 - lp)));
    }
  }

  // FWHT over register-index bits 0..5 (position bits 0-3, 5, 6)
#pragma unroll
  for (int b = 0; b < 6; b++) {
#pragma unroll
    for (int i = 0; i < 64; i++) {
      if (i & (1 << b)) continue;
      const __half2 x = h[i], y = h[i | (1 << b)];
      h[i] = __hadd2(x, y);
      h[i | (1 << b)] = __hsub2(x, y);
    }
  }
  // in-register stage over position bit 4: (lo, hi) -> (lo + hi, lo - hi)
  const __half2 pm = __halves2half2(__float2half(1.0f), __float2half(-1.0f));
#pragma unroll
  for (int i = 0; i < 64; i++) h[i] = __hfma2(__high2half2(h[i]), pm, __low2half2(h[i]));
  return rm_argmax<MULT>(h);
}

}  // namespace hqc
