// Compile-time parameter sets for the kernels (Table I; derived per DESIGN.md §3/§6).
// Independent of oracle/ (tests cross-check hqc_get_params against the oracle's own table).
#pragma once
#include <cstdint>

namespace hqc {

template <int LEVEL> struct Table1;
template <> struct Table1<1> { static constexpr uint32_t N = 17669, N1 = 46, N2 = 384, K = 16, D = 31, W = 66, WR = 75; };
template <> struct Table1<3> { static constexpr uint32_t N = 35851, N1 = 56, N2 = 640, K = 24, D = 33, W = 100, WR = 114; };
template <> struct Table1<5> { static constexpr uint32_t N = 57637, N1 = 90, N2 = 640, K = 32, D = 59, W = 131, WR = 149; };

constexpr uint32_t round_up(uint32_t x, uint32_t m) { return (x + m - 1) / m * m; }
constexpr uint32_t make_odd_up(uint32_t x) { return x | 1u; }

template <int LEVEL> struct Lv : Table1<LEVEL> {
  using T = Table1<LEVEL>;
  static constexpr int level = LEVEL;
  static constexpr uint32_t N = T::N, N1 = T::N1, N2 = T::N2, K = T::K, W = T::W, WR = T::WR;
  static constexpr uint32_t MULT = N2 / 128;           // copies of RM(1,7)
  static constexpr uint32_t DELTA = (T::D - 1) / 2;    // RS capacity (R#15)
  static constexpr uint32_t TWO_DELTA = 2 * DELTA;     // = N1 - K syndromes / parity bytes
  static constexpr uint32_t N12 = N1 * N2;             // truncation length (R#3)
  static constexpr uint32_t NW = N12 / 32;             // 32-bit words of r (exact)
  static constexpr uint32_t U_WORDS = (N + 63) / 64;
  static constexpr uint32_t U_STRIDE = round_up(U_WORDS, 2);
  static constexpr uint32_t V_WORDS = N12 / 64;
  static constexpr uint32_t Y_STRIDE = round_up(W, 4);
  static constexpr uint32_t E_STRIDE = round_up(WR, 4);
  static constexpr uint32_t Q0 = N / 32;               // word holding bit n-1
  static constexpr uint32_t C = N % 32;                // bits of u in word Q0 (nonzero: n is prime)
  static_assert(C != 0, "n must not be a multiple of 32");
  // bits of word Q0 inside the ceil(n/8) serialized u bytes: the KEM's byte-wise compare
  static constexpr uint32_t CB = round_up(C, 8);
  static constexpr uint32_t CB_MASK = CB >= 32 ? 0xFFFFFFFFu : (1u << CB) - 1u;
  static_assert(N12 % 128 == 0, "r is processed in 16-byte chunks");
  static_assert(N2 % 128 == 0 && (N2 / 32) % 4 == 0, "RM blocks are whole 16-byte chunks");
  static_assert(N1 - K == TWO_DELTA, "shortened RS: n1 - k = 2 delta");
  static_assert(K <= 32, "Forney root flags for message positions fit one 32-bit mask");
};

// Shape of one warp-level sparse x dense product (stage1.cuh): NOUT 32-bit output words, a sparse
// operand of weight WT. A warp owns one product; lane L owns R consecutive output words
// [L*R, L*R+R). R is odd so that the 32 lanes' shared-memory reads E[o + L*R + k] fall in 32
// distinct banks for every (o, k). E[b] = u[b mod n] for b < 32*E_WORDS: the "doubled" dense
// operand, so every rotation is a plain funnel shift.
template <class P, uint32_t NOUT_, uint32_t WT_> struct ProdShape {
  static constexpr uint32_t NOUT = NOUT_, WT = WT_;
  static constexpr uint32_t R = make_odd_up((NOUT + 31) / 32);
  // at least the doubled u (2 Q0 + 2 words, which s1_build_E always writes) for the narrow-R shapes
  static constexpr uint32_t E_WORDS = round_up(P::Q0 + 32 * R + 2 > 2 * P::Q0 + 2 ? P::Q0 + 32 * R + 2
                                                                                  : 2 * P::Q0 + 2, 4);
  static constexpr uint32_t WPAD = round_up(WT, 4);
};
template <class P> using DecShape = ProdShape<P, P::NW, P::W>;          // u*y truncated to n1*n2 bits
// The one-warp decrypt product without the ragged top: the largest odd R with 32 R <= NW words per warp,
// the remaining TW = NW - 32 R words (HQC-1: 552 = 32 * 17 + 8) added by the whole warp (s1_tail_words);
// TW = 0 where NW is already 32 x odd (HQC-3) or the rest would be too wide (HQC-5: 40 words).
#ifndef HQC_S1_TAILW
#define HQC_S1_TAILW 1
#endif
template <class P> constexpr uint32_t dec_tail_words() {
  constexpr uint32_t r = ((P::NW / 32) & 1u) ? P::NW / 32 : P::NW / 32 - 1;  // largest odd, 32 r <= NW
  return (HQC_S1_TAILW && P::NW - 32 * r > 0 && P::NW - 32 * r <= 8) ? P::NW - 32 * r : 0u;
}
template <class P> using DecShapeT = ProdShape<P, P::NW - dec_tail_words<P>(), P::W>;
// The "shifted" lane windows of s1_product_range_sh (stage1.cuh): lane L owns the R output words
// [L R - 1, L R + R - 1) (lane 0 one fewer), 32 R - 1 per warp; R odd. R is the largest odd value whose
// 32 R - 1 words leave a ragged top of at most 9 words for s1_tail_words, else the smallest odd R that
// covers all NW words.
template <class P, uint32_t NW_, uint32_t WT_> struct ShShape {
  static constexpr uint32_t NW = NW_, WT = WT_;
  static constexpr uint32_t RLO = (((NW + 1) / 32) & 1u) ? (NW + 1) / 32 : (NW + 1) / 32 - 1;
  static constexpr uint32_t RHI = make_odd_up((NW + 1 + 31) / 32);
  static constexpr bool TAILED = (32 * RLO - 1 <= NW) && (NW - (32 * RLO - 1) <= 9);
  static constexpr uint32_t R = TAILED ? RLO : RHI;
  static constexpr uint32_t NOUT = TAILED ? 32 * R - 1 : NW;  // words the lanes produce (< 32 R)
  static constexpr uint32_t TW = TAILED ? NW - NOUT : 0u;     // the ragged top (s1_tail_words)
  static constexpr uint32_t E_WORDS = round_up(P::Q0 + 32 * R + 2 > 2 * P::Q0 + 2 ? P::Q0 + 32 * R + 2
                                                                                  : 2 * P::Q0 + 2, 4);
  static constexpr uint32_t WPAD = round_up(WT, 4);
};
template <class P> using DecShapeSh = ShShape<P, P::NW, P::W>;

template <class P> using FullShape = ProdShape<P, P::Q0 + 1, P::WR>;    // h*r2: all n bits
template <class P> using KeyShape = ProdShape<P, P::Q0 + 1, P::W>;      // h*y: all n bits
template <class P> using EncVShape = ProdShape<P, P::NW, P::WR>;        // s*r2 truncated

}  // namespace hqc
