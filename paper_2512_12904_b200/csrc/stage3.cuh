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
//   rows [0, delta+1)                 : sentinel GF_LOG0 (log S_i for i <= 0)
//   rows [delta+1, delta+1+2delta)    : log S_{i+1}
//   rows [.., +2delta)                : log Omega_i
//   rows [.., +k)                     : log Lambda_odd(alpha^-j), j < k
template <class P> struct S3Scratch {
  static constexpr uint32_t PAD = P::DELTA + 1;
  static constexpr uint32_t ROWS = PAD + 4 * P::DELTA + P::K;
  static constexpr uint32_t BYTES = ROWS * 32 * 2;
};

// sym_at(j) returns the j-th received symbol of this lane's ciphertext.
// Writes K message bytes to out[0..K) (out may be null for inactive lanes). Returns ok.
template <class P, class SymAt>
__device__ __forceinline__ uint32_t rs_decode_lane(SymAt sym_at, const GfTables *gf, uint16_t *scr, int lane,
                                                   uint8_t *out) {
  constexpr int TD = P::TWO_DELTA, DL = P::DELTA, N1 = P::N1, K = P::K;
  const uint8_t *EXPT = gf->exp;
  const uint16_t *LOGT = gf->log;
  constexpr int PAD = S3Scratch<P>::PAD;
#pragma unroll
  for (int k = 0; k < PAD; k++) scr[k * 32 + lane] = GF_LOG0;
  uint16_t *lS = scr + PAD * 32;  // lS[i*32 + lane] = log S_{i+1}; rows -PAD..-1 hold the sentinel
  uint16_t *lOm = lS + TD * 32;
  uint16_t *lOdd = lOm + TD * 32;

  // ---- syndromes: S_i = sum_j sym_j alpha^{ij}, in halves of at most 32 registers
  constexpr int HALF = TD > 32 ? (TD + 1) / 2 : TD;
#pragma unroll
  for (int i0 = 0; i0 < TD; i0 += HALF) {
    uint32_t S[HALF];
#pragma unroll
    for (int i = 0; i < HALF; i++) S[i] = 0;
#pragma unroll 1
    for (int j = 0; j < N1; j++) {
      const uint32_t x = sym_at(j);
      const uint32_t zm = x ? 0xFFu : 0u;
      const uint32_t jj = (uint32_t)j % 255u;
      // e = log x + (i0 + 1 + i) * j (mod 255)
      uint32_t e = x ? LOGT[x] : 0u;
      e = (e + (uint32_t)i0 * jj) % 255u;
#pragma unroll
      for (int i = 0; i < HALF; i++) {
        e = mod255_add(e, jj);
        if (i0 + i < TD) S[i] ^= EXPT[e] & zm;
      }
    }
#pragma unroll
    for (int i = 0; i < HALF; i++)
      if (i0 + i < TD) lS[(i0 + i) * 32 + lane] = LOGT[S[i]];
  }

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
      d ^= EXPT[lLam[k] + wr[-32 * k]];
    }
    const uint32_t ld = LOGT[d];
    const uint32_t lc = d ? mod255_sub(ld, lb) : GF_LOG0;  // log(d / b)
    const bool grow = (d != 0) && (2 * L <= (uint32_t)r);
#pragma unroll
    for (int k = 0; k <= DL; k++) Lam[k] ^= EXPT[lc + lBx[k]];
#pragma unroll
    for (int k = DL; k >= 1; k--) lBx[k] = grow ? lLam[k - 1] : lBx[k - 1];
    lBx[0] = GF_LOG0;
    L = grow ? (uint32_t)r + 1 - L : L;
    lb = grow ? ld : lb;
  }
  uint32_t deg = 0;
#pragma unroll
  for (int k = 0; k <= DL; k++) {
    deg = Lam[k] ? (uint32_t)k : deg;
    lLam[k] = LOGT[Lam[k]];
  }

  // ---- Chien search over the n1 positions (+ Lambda_odd for the k message positions)
  // ek = log Lambda_k - j*k (mod 255), or GF_LOG0 (never updated) for a zero coefficient
  uint32_t ek[DL + 1];
#pragma unroll
  for (int k = 0; k <= DL; k++) ek[k] = lLam[k];
  uint32_t nroots = 0, rootmask = 0;
#pragma unroll 1
  for (int j = 0; j < N1; j++) {
    uint32_t ev = 0, od = 0;
#pragma unroll
    for (int k = 0; k <= DL; k++) {
      const uint32_t t = EXPT[ek[k]];
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
  const bool ok = (L <= (uint32_t)DL) && (deg == L) && (nroots == L);

  // ---- Omega_i = sum_{t <= min(i, delta)} Lambda_t S_{i-t+1}, i < 2delta
#pragma unroll 1
  for (int i = 0; i < TD; i++) {
    const uint16_t *wi = lS + i * 32 + lane;
    uint32_t om = 0;
#pragma unroll
    for (int t = 0; t <= DL; t++) om ^= EXPT[lLam[t] + wi[-32 * t]];
    lOm[i * 32 + lane] = LOGT[om];
  }

  // ---- Forney on the message positions, then the output bytes
  uint32_t outw[K / 4];
#pragma unroll
  for (int q = 0; q < K / 4; q++) outw[q] = 0;
#pragma unroll
  for (int j = 0; j < K; j++) {
    uint32_t acc = 0, e = 0;  // Omega(alpha^-j) = sum_i Omega_i alpha^{-ij}
#pragma unroll 4
    for (int i = 0; i < TD; i++) {
      const uint32_t lo = lOm[i * 32 + lane];
      acc ^= EXPT[lo + e];
      e = mod255_sub(e, (uint32_t)j % 255u);
    }
    const uint32_t lodd = lOdd[j * 32 + lane];
    // log e_j = log Omega(alpha^-j) - j - log Lambda_odd(alpha^-j)   (zero Omega -> e_j = 0)
    const uint32_t lnum = LOGT[acc];
    const uint32_t le = mod255_sub(mod255_sub(lnum == GF_LOG0 ? 0u : lnum, (uint32_t)j % 255u),
                                   lodd == GF_LOG0 ? 0u : lodd);
    const uint32_t ej = (lnum == GF_LOG0 || lodd == GF_LOG0) ? 0u : EXPT[le];
    const uint32_t fix = (ok && ((rootmask >> j) & 1u)) ? ej : 0u;
    outw[j / 4] |= ((sym_at(j) ^ fix) & 0xFFu) << (8 * (j % 4));
  }
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
