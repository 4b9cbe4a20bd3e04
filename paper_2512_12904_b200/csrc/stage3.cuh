// Stage 3 — shortened RS decoding over GF(2^8) by one thread per ciphertext ("error vector
// recovery", P:227 syndromes; readings R#4-R#7 in DESIGN.md). DESIGN.md §6.3.
//
//   syndromes  S_i = r(alpha^i), i = 1..2delta              (2delta * n1 table products)
//   Berlekamp–Massey, 2delta iterations, Lambda and x^m*B stored with delta+1 coefficients (exact
//     whenever L <= delta, DESIGN.md §3 R#7; when L > delta the decode fails regardless)
//   Chien search over j in [0, n1): root_j = [Lambda(alpha^-j) = 0]; the odd part Lambda_odd(alpha^-j)
//     is kept for j < k because x*Lambda'(x) = Lambda_odd(x) in characteristic 2
//   ok = L <= delta and deg Lambda = L and #roots = L
//   Forney (b = 1) on the k message positions: e_j = Omega(alpha^-j) / (alpha^j * Lambda_odd(alpha^-j)),
//     Omega = S(x) Lambda(x) mod x^{2 delta}
//   m_j = sym_j XOR (ok and root_j ? e_j : 0), j < k    (message-first layout, R#6)
// Every loop count is fixed by the level (2delta, delta+1, n1, k): the instruction stream does not
// depend on the data (branches are selects). Field products use the log/antilog tables of
// gf256.cuh in shared memory, with the LOG(0) = 511 sentinel making zero factors free.
#pragma once
#include <cstdint>

#include "gf256.cuh"
#include "exp_timing.cuh"
#include "levels.cuh"

namespace hqc {

__device__ __forceinline__ uint32_t mod255_sub(uint32_t e, uint32_t s) {  // (e - s) mod 255, e < 255, s < 255
  return e >= s ? e - s : e + 255u - s;
}
__device__ __forceinline__ uint32_t mod255_add(uint32_t e, uint32_t s) {  // (e + s) mod 255, e, s < 255
  const uint32_t t = e + s;
  return t >= 255u ? t - 255u : t;
}

// scratch layout per warp (uint16, [row][32 lanes]):
//   rows [0, delta+1)              : sentinel GF_LOG0 (log S_i for i <= 0)
//   rows [delta+1, delta+1+2delta) : log S_{i+1}; overwritten in place by log Omega_i
//   rows [.., +k)                  : Lambda_t (linear Chien input, t <= delta < k), then log Lambda_odd(alpha^-j)
// How many coefficients of Omega = S Lambda mod x^{2 delta} the decoders form: deg Omega < L <= delta for
// every word whose correction is applied (see rs_decode_lane), so delta; HQC_RS_OMEGA_FULL=1 forms all 2 delta
// (the A/B switch of profiles/r02/ab_omega.log).
#ifndef HQC_RS_OMEGA_FULL
#define HQC_RS_OMEGA_FULL 0
#endif
template <class P> constexpr int RS_OMEGA_TERMS = HQC_RS_OMEGA_FULL ? (int)P::TWO_DELTA : (int)P::DELTA;

template <class P> struct S3Scratch {
  static constexpr uint32_t PAD = P::DELTA + 1;
  static constexpr uint32_t ROWS = PAD + 2 * P::DELTA + P::K;
  static constexpr uint32_t BYTES = ROWS * 32 * 2;
  static_assert(P::K >= P::DELTA + 1, "Lambda rows alias the Lambda_odd rows");
};

// ---- GF(2)-linear maps as constant tables -------------------------------------------------------
// The syndromes are a GF(2)-linear function of the received bits: S = XOR over (j, b) with bit b of
// sym_j set of SYN[j][b], where SYN[j][b] packs alpha^{(i+1) j} * 2^b for i < 2delta (4 per word).
// Likewise the Chien values Lambda(alpha^-j), j < n1, and Lambda_odd(alpha^-j), j < k, are linear in
// the bits of Lambda: XOR over (t, b) with bit b of Lambda_t set of CHN[t][b] (bytes j < n1: the
// contribution 2^b alpha^{-jt}; bytes n1 + j, j < k: the same for odd t, else 0). Every lane of a warp
// reads the same table word at the same time, so the tables live in the constant bank (uniform
// LDCU loads, no shared-memory traffic and no bank conflicts) — one table set per level per
// translation unit (hqc_lN.cu). A table set larger than the bank budget falls back to log/antilog.
template <class P> struct RsLinear {
  static constexpr uint32_t SW = (P::TWO_DELTA + 3) / 4;        // syndrome words
  static constexpr uint32_t CW = (P::N1 + P::K + 3) / 4;        // Chien-vector words
  static constexpr uint32_t SYN_BYTES = P::N1 * 8 * SW * 4;
  static constexpr uint32_t CHN_BYTES = (P::DELTA + 1) * 8 * CW * 4;
  static constexpr bool LINEAR_CHIEN = SYN_BYTES + CHN_BYTES + sizeof(GfTables) <= 60 * 1024;
  static constexpr uint32_t CHN_T = LINEAR_CHIEN ? P::DELTA + 1 : 1;
  struct Tables {
    uint32_t syn[P::N1][8][SW];
    uint32_t chn[CHN_T][8][CW];
  };
  static constexpr Tables make() {
    uint32_t ex[255] = {};
    uint32_t x = 1;
    for (int e = 0; e < 255; e++) {
      ex[e] = x;
      x = gf_mul_c(x, 2);
    }
    Tables T{};
    for (uint32_t j = 0; j < P::N1; j++)
      for (uint32_t b = 0; b < 8; b++)
        for (uint32_t i = 0; i < P::TWO_DELTA; i++)
          T.syn[j][b][i / 4] |= gf_mul_c(1u << b, ex[((i + 1) * j) % 255]) << (8 * (i % 4));
    if (LINEAR_CHIEN)
      for (uint32_t t = 0; t < CHN_T; t++)
        for (uint32_t b = 0; b < 8; b++)
          for (uint32_t j = 0; j < P::N1; j++) {
            const uint32_t v = gf_mul_c(1u << b, ex[(255 - (j * t) % 255) % 255]);
            T.chn[t][b][j / 4] |= v << (8 * (j % 4));
            if (j < P::K && (t & 1)) T.chn[t][b][(P::N1 + j) / 4] |= v << (8 * ((P::N1 + j) % 4));
          }
    return T;
  }
};

#ifdef HQC_THIS_LEVEL
__device__ __constant__ RsLinear<Lv<HQC_THIS_LEVEL>>::Tables c_rs_lin = RsLinear<Lv<HQC_THIS_LEVEL>>::make();
#endif

// sym_at(j) returns the j-th received symbol of this lane's ciphertext.
// Writes K message bytes to out[0..K) (out may be null for inactive lanes). Returns ok.
// REPL (experiment, HQC_S3_REPL in k_stage3): antilog lookups from a lane-replicated copy of EXPT[0..512)
// (`rexp`, 16 KB: word row e/4, column = lane, so lane l only ever touches bank l — no bank conflicts); indices
// above 511 (a zero factor) clamp to entry 511 = 0.
template <class P, class SymAt, bool REPL = false>
__device__ __forceinline__ uint32_t rs_decode_lane(SymAt sym_at, const GfTables *gf, uint16_t *scr, int lane,
                                                   uint8_t *out, const uint8_t *rexp = nullptr) {
  constexpr int TD = P::TWO_DELTA, DL = P::DELTA, N1 = P::N1, K = P::K;
  const uint8_t *EXPT = gf->exp;
  const uint8_t *rexp_lane = rexp + 4 * lane;
  auto EX = [&](uint32_t i) -> uint32_t {
    if constexpr (REPL) {
      const uint32_t c = i < 511u ? i : 511u;
      return rexp_lane[((c & ~3u) << 5) + (c & 3u)];
    } else {
      return EXPT[i];
    }
  };
  const uint16_t *LOGT = gf->log;
  constexpr int PAD = S3Scratch<P>::PAD;
#pragma unroll
  for (int k = 0; k < PAD; k++) scr[k * 32 + lane] = GF_LOG0;
  uint16_t *lS = scr + PAD * 32;  // lS[i*32 + lane] = log S_{i+1}; rows -PAD..-1 hold the sentinel
  uint16_t *lOm = lS;  // Omega overwrites the syndromes in place (computed from the top down)
  uint16_t *lOdd = lS + TD * 32;
  uint16_t *sLam = lOdd;  // read completely before lOdd is written
  using LIN = RsLinear<P>;
  PHASE_T0();

  // ---- syndromes S_i = sum_j sym_j alpha^{ij} (i = 1..2delta) as the GF(2)-linear map SYN
  {
    uint32_t Sw[LIN::SW];
#pragma unroll
    for (int w = 0; w < (int)LIN::SW; w++) Sw[w] = 0;
#pragma unroll 1
    for (int j = 0; j < N1; j++) {
      const uint32_t x = sym_at(j);
#pragma unroll
      for (int b = 0; b < 8; b++) {
        const uint32_t m = 0u - ((x >> b) & 1u);
#pragma unroll
        for (int w = 0; w < (int)LIN::SW; w++) Sw[w] ^= c_rs_lin.syn[j][b][w] & m;
      }
    }
#pragma unroll
    for (int i = 0; i < TD; i++) lS[i * 32 + lane] = LOGT[(Sw[i / 4] >> (8 * (i % 4))) & 0xFFu];
  }
  PHASE(9);

  // ---- Berlekamp–Massey (Massey 1969) with Bx = x^m * B, logs of Bx kept
  uint32_t Lam[DL + 1], lBx[DL + 1], lLam[DL + 1];
#pragma unroll
  for (int k = 0; k <= DL; k++) {
    Lam[k] = (k == 0);
    lBx[k] = (k == 1) ? 0u : GF_LOG0;  // Bx = x * 1
  }
  uint32_t L = 0, lb = 0;
#pragma unroll 1
  for (int r = 0; r < TD; r++) {
    const uint16_t *wr = lS + r * 32 + lane;  // wr[-32k] = log S_{r+1-k} (sentinel for r < k)
    uint32_t d = 0;
#pragma unroll
    for (int k = 0; k <= DL; k++) {
      lLam[k] = LOGT[Lam[k]];
      d ^= EX(lLam[k] + wr[-32 * k]);
    }
    const uint32_t ld = LOGT[d];
    const uint32_t lc = d ? mod255_sub(ld, lb) : GF_LOG0;  // log(d / b)
    const bool grow = (d != 0) && (2 * L <= (uint32_t)r);
#pragma unroll
    for (int k = 0; k <= DL; k++) Lam[k] ^= EX(lc + lBx[k]);
#pragma unroll
    for (int k = DL; k >= 1; k--) lBx[k] = grow ? lLam[k - 1] : lBx[k - 1];
    lBx[0] = GF_LOG0;
    L = grow ? (uint32_t)r + 1 - L : L;
    lb = grow ? ld : lb;
  }
  PHASE(10);
  uint32_t deg = 0;
#pragma unroll
  for (int k = 0; k <= DL; k++) {
    deg = Lam[k] ? (uint32_t)k : deg;
    lLam[k] = LOGT[Lam[k]];
  }

  // ---- Chien search over the n1 positions (+ Lambda_odd for the k message positions)
  uint32_t nroots = 0, rootmask = 0;
  if constexpr (LIN::LINEAR_CHIEN) {
#pragma unroll
    for (int t = 0; t <= DL; t++) sLam[t * 32 + lane] = (uint16_t)Lam[t];
    uint32_t Cw[LIN::CW];
#pragma unroll
    for (int w = 0; w < (int)LIN::CW; w++) Cw[w] = 0;
#pragma unroll 1
    for (int t = 0; t <= DL; t++) {
      const uint32_t x = sLam[t * 32 + lane];
#pragma unroll
      for (int b = 0; b < 8; b++) {
        const uint32_t m = 0u - ((x >> b) & 1u);
#pragma unroll
        for (int w = 0; w < (int)LIN::CW; w++) Cw[w] ^= c_rs_lin.chn[t][b][w] & m;
      }
    }
#pragma unroll
    for (int w = 0; w < (int)((N1 + 3) / 4); w++) {
      // bit 7 of each byte of nz is set iff that byte of Cw[w] is nonzero (no carries between bytes)
      const uint32_t nz = (((Cw[w] & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | Cw[w]) & 0x80808080u;
      uint32_t zero = ~nz & 0x80808080u;
      if (4 * w + 4 > N1) zero &= 0x80808080u >> (8 * (4 * w + 4 - N1));  // only positions j < n1
      nroots += __popc(zero);
#pragma unroll
      for (int c = 0; c < 4; c++)
        if (4 * w + c < K) rootmask |= ((zero >> (8 * c + 7)) & 1u) << (4 * w + c);
    }
#pragma unroll
    for (int j = 0; j < K; j++) lOdd[j * 32 + lane] = LOGT[(Cw[(N1 + j) / 4] >> (8 * ((N1 + j) % 4))) & 0xFFu];
  } else {
    // ek = log Lambda_k - j*k (mod 255), or GF_LOG0 (never updated) for a zero coefficient
    uint32_t ek[DL + 1];
#pragma unroll
    for (int k = 0; k <= DL; k++) ek[k] = lLam[k];
#pragma unroll 1
    for (int j = 0; j < N1; j++) {
      uint32_t ev = 0, od = 0;
#pragma unroll
      for (int k = 0; k <= DL; k++) {
        const uint32_t t = EX(ek[k]);
        if (k & 1) od ^= t; else ev ^= t;
        ek[k] = ek[k] == GF_LOG0 ? GF_LOG0 : mod255_sub(ek[k], (uint32_t)k % 255u);
      }
      const uint32_t root = (ev == od) ? 1u : 0u;
      nroots += root;
      if (j < K) {
        rootmask |= root << j;
        lOdd[j * 32 + lane] = LOGT[od];
      }
    }
  }
  const bool ok = (L <= (uint32_t)DL) && (deg == L) && (nroots == L);
  PHASE(11);

  // ---- Omega_i = sum_{t <= min(i, delta)} Lambda_t S_{i-t+1}, from i = OM_N-1 down:
  //      Omega_i reads log S_{i'+1} for i' <= i only, so it may overwrite row i in place.
  //      Only i < delta is formed (RS_OMEGA_TERMS): for i >= L, Omega_i is BM's discrepancy of the FINAL
  //      Lambda at step i, sum_{t <= L} Lambda_t S_{i+1-t}, and the final Lambda generates S_{L+1..2delta}, so
  //      those coefficients are zero whenever L <= delta — and when L > delta, ok is false and no fix is applied.
  constexpr int OM_N = RS_OMEGA_TERMS<P>;
#pragma unroll 1
  for (int i = OM_N - 1; i >= 0; i--) {
    const uint16_t *wi = lS + i * 32 + lane;
    uint32_t om = 0;
#pragma unroll
    for (int t = 0; t <= DL; t++) om ^= EX(lLam[t] + wi[-32 * t]);
    lOm[i * 32 + lane] = LOGT[om];
  }

  PHASE(12);
  // ---- Forney on the message positions, then the output bytes. Omega(alpha^-j) = sum_i Omega_i alpha^{-ij}
  //      for all k message positions at once: each log Omega_i is read once, and the exponents -ij mod 255
  //      are compile-time constants (immediate offsets into EXPT; no modular arithmetic at run time).
  uint32_t om_j[K];
#pragma unroll
  for (int j = 0; j < K; j++) om_j[j] = 0;
#pragma unroll
  for (int i = 0; i < OM_N; i++) {
    const uint32_t lo = lOm[i * 32 + lane];
#pragma unroll
    for (int j = 0; j < K; j++) om_j[j] ^= EX(lo + (uint32_t)((255 - (i * j) % 255) % 255));
  }
  uint32_t outw[K / 4];
#pragma unroll
  for (int q = 0; q < K / 4; q++) outw[q] = 0;
#pragma unroll
  for (int j = 0; j < K; j++) {
    const uint32_t lodd = lOdd[j * 32 + lane];
    // log e_j = log Omega(alpha^-j) - j - log Lambda_odd(alpha^-j)   (zero Omega -> e_j = 0)
    const uint32_t lnum = LOGT[om_j[j]];
    const uint32_t le = mod255_sub(mod255_sub(lnum == GF_LOG0 ? 0u : lnum, (uint32_t)j % 255u),
                                   lodd == GF_LOG0 ? 0u : lodd);
    const uint32_t ej = (lnum == GF_LOG0 || lodd == GF_LOG0) ? 0u : EX(le);
    const uint32_t fix = (ok && ((rootmask >> j) & 1u)) ? ej : 0u;
    outw[j / 4] |= ((sym_at(j) ^ fix) & 0xFFu) << (8 * (j % 4));
  }
  PHASE(13);
  if (out != nullptr) {
    if constexpr (K % 16 == 0) {
#pragma unroll
      for (int q = 0; q < K / 16; q++)
        reinterpret_cast<uint4 *>(out)[q] = make_uint4(outw[4 * q], outw[4 * q + 1], outw[4 * q + 2], outw[4 * q + 3]);
    } else {
#pragma unroll
      for (int q = 0; q < K / 8; q++) reinterpret_cast<uint2 *>(out)[q] = make_uint2(outw[2 * q], outw[2 * q + 1]);
    }
  }
  return ok ? 1u : 0u;
}

}  // namespace hqc
