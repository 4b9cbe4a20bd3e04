// Stage 3 — shortened RS decoding of ONE received word by a whole warp. Same algorithm
// and the same decisions as the lane-per-word decoder of stage3.cuh (readings R#4-R#7: syndromes
// S_i = r(alpha^i), i = 1..2delta; Berlekamp–Massey with Lambda and x^m B truncated to delta+1
// coefficients; Chien search over j < n1; ok = L <= delta and deg Lambda = L and #roots = L; Forney with
// b = 1 on the k message positions; output sym[0..k) corrected iff ok), with the work spread over the
// lanes instead of over 32 words:
//   syndromes   lane i (and i + 32) accumulates S_{i+1} = XOR_j EXP[log sym_j + (i+1) j mod 255]
//   BM          lane t holds coefficient t of Lambda and of x^m B (t <= delta < 32); the discrepancy is a
//               warp XOR-reduction (REDUX), the shift by x a shuffle; L, log b, d are warp-uniform
//   Chien       lane j (and j + 32, j + 64) evaluates Lambda(alpha^-j) and its odd part
//   Omega       lane i (and i + 32) forms Omega_i = sum_t Lambda_t S_{i-t+1}
//   Forney      lane j < k corrects message byte j
// It exists for SMALL batches (k_decrypt_sb): a lane-per-word decoder runs ~15k dependent instructions on
// one lane and reads its GF(2)-linear tables from the constant bank, cold in a short launch (profiles/r02/
// sb_phases.log: 90k cycles for HQC-1); this one is a few hundred instructions per lane on the log/antilog
// tables in shared memory. Every loop count is fixed by the level; the data selects, never branches.
#pragma once
#include <cstdint>

#include "exp_timing.cuh"
#include "gf256.cuh"
#include "levels.cuh"
#include "stage3.cuh"

namespace hqc {

// Berlekamp–Massey with the discrepancy formed one iteration ahead (a shorter dependent chain, more
// instructions): BM 6.4k -> 5.4k cycles per HQC-1 word; configs[0] (HQC-1, 1,024) 18.1 -> 17.7 us, but
// HQC-3 at 65,536 (where k_decrypt_sb runs throughput-bound) 1.175 -> 1.198 ms (profiles/r02/ab_bm.log).
// So per level: on where K4s serves only small, latency-bound batches (HQC-1, HQC-5), off for HQC-3.
#ifndef HQC_BM_LOOKAHEAD
#define HQC_BM_LOOKAHEAD (P::level != 3)
#endif
// riBM (below) instead of either form of the plain recurrence: no warp reduction on the dependent chain.
#ifndef HQC_BM_RIBM
#define HQC_BM_RIBM 1
#endif

// Per-warp scratch (uint16 logs): log sym_j (n1), a sentinel pad of delta+1 rows then log S_{i+1} (2delta),
// log Lambda_t (delta+1), log Omega_i (2delta).
template <class P> struct RsWarpScratch {
  static constexpr uint32_t PAD = P::DELTA + 1;
  static constexpr uint32_t LSYM = 0, LS = P::N1 + PAD, LLAM = LS + P::TWO_DELTA, LOM = LLAM + P::DELTA + 1;
  static constexpr uint32_t HALFS = LOM + P::TWO_DELTA;
  static constexpr uint32_t BYTES = round_up(HALFS * 2, 16);
  static_assert(P::DELTA < 32 && P::K <= 32, "one lane per Lambda coefficient and per message byte");
};

// Symbols per pass of the syndrome loop: its loads are independent of each other, so a deeper unroll
// keeps more of them in flight (the loop was 2.2k of the decoder's 10.7k cycles with 2).
#ifndef HQC_WRS_SYN_UNROLL
#define HQC_WRS_SYN_UNROLL 8
#endif
// Forney's sum over the 2delta log Omega_i: unrolled by 32 (configs[0] 17.15 -> 16.89 us per launch; 4 before);
// Berlekamp–Massey stays rolled (an unroll of 2 lost 1-3%: profiles/r02/ab_wrs.log).
// Syndromes by symbol-owning lanes and one warp XOR-reduction per syndrome (instead of a syndrome per lane
// looping over all n1 symbols).
#ifndef HQC_WRS_SYN_REDUX
#define HQC_WRS_SYN_REDUX 0
#endif
#ifndef HQC_WRS_FORNEY_UNROLL
#define HQC_WRS_FORNEY_UNROLL 32
#endif
#ifndef HQC_WRS_BM_UNROLL
#define HQC_WRS_BM_UNROLL 1
#endif
// sym: the word's n1 received symbols (shared memory); scr: RsWarpScratch<P>::BYTES of shared memory;
// out: k message bytes (global), or null. Returns ok (warp-uniform).
template <class P>
__device__ __forceinline__ uint32_t rs_decode_warp(const uint8_t *sym, const GfTables *gf, uint16_t *scr, int lane,
                                                   uint8_t *out) {
  using W = RsWarpScratch<P>;
  constexpr int TD = P::TWO_DELTA, DL = P::DELTA, N1 = P::N1, K = P::K;
  constexpr int NI = (TD + 31) / 32, NJ = (N1 + 31) / 32;  // rounds of the lane-parallel loops
  const uint8_t *EXPT = gf->exp;
  const uint16_t *LOGT = gf->log;
  uint16_t *lsym = scr + W::LSYM, *lS = scr + W::LS, *lLam = scr + W::LLAM, *lOm = scr + W::LOM;
  PHASE_T0();
  if constexpr (!HQC_WRS_SYN_REDUX)
    for (int j = lane; j < N1; j += 32) lsym[j] = LOGT[sym[j]];
  for (int t = lane; t < (int)W::PAD; t += 32) lS[t - (int)W::PAD] = GF_LOG0;  // log S_i for i <= 0
  __syncwarp();

  // ---- syndromes: S_{i+1} = sum_j sym_j alpha^{(i+1) j}
  if constexpr (HQC_WRS_SYN_REDUX) {
    // lane l owns symbols j = l + 32 q; per syndrome one product per owned symbol (independent loads) and a
    // warp XOR-reduction (independent across syndromes); the exponent (i+1) j advances by j per syndrome
    uint32_t ls[NJ], e[NJ], jm[NJ], mine[NI];
#pragma unroll
    for (int q = 0; q < NJ; q++) {
      const int j = lane + 32 * q;
      ls[q] = j < N1 ? (uint32_t)LOGT[sym[j]] : GF_LOG0;
      jm[q] = (uint32_t)j % 255u;
      e[q] = jm[q];
    }
#pragma unroll
    for (int q = 0; q < NI; q++) mine[q] = 0;
#pragma unroll
    for (int i = 0; i < TD; i++) {
      uint32_t part = 0;
#pragma unroll
      for (int q = 0; q < NJ; q++) {
        part ^= EXPT[ls[q] + e[q]];
        e[q] = mod255_add(e[q], jm[q]);
      }
      const uint32_t Si = __reduce_xor_sync(0xffffffffu, part);
      mine[i / 32] = lane == i % 32 ? Si : mine[i / 32];
    }
#pragma unroll
    for (int q = 0; q < NI; q++)
      if (lane + 32 * q < TD) lS[lane + 32 * q] = LOGT[mine[q]];
  } else {
    // lane i (and i + 32) accumulates S_{i+1}; the exponent advances by i+1 per symbol
    uint32_t s[NI], e[NI];
#pragma unroll
    for (int q = 0; q < NI; q++) s[q] = 0, e[q] = 0;
    constexpr int kSynUnroll = HQC_WRS_SYN_UNROLL;
#pragma unroll kSynUnroll
    for (int j = 0; j < N1; j++) {
      const uint32_t ls = lsym[j];
#pragma unroll
      for (int q = 0; q < NI; q++) {
        s[q] ^= EXPT[ls + e[q]];
        const uint32_t i1 = (uint32_t)(lane + 32 * q + 1) % 255u;
        e[q] = mod255_add(e[q], i1);
      }
    }
#pragma unroll
    for (int q = 0; q < NI; q++)
      if (lane + 32 * q < TD) lS[lane + 32 * q] = LOGT[s[q]];
  }
  __syncwarp();
  PHASE(9);

  // ---- Berlekamp–Massey: lane t <= delta holds Lambda_t and log (x^m B)_t
  const bool coef = lane <= DL;
  uint32_t lam = lane == 0 ? 1u : 0u;
  uint32_t lbx = lane == 1 ? 0u : GF_LOG0;  // Bx = x * 1
  uint32_t L = 0, lb = 0;
  uint32_t nzmask = 0;  // bit t: Lambda_t != 0
  if constexpr (HQC_BM_RIBM) {
  // Reformulated inversionless BM (Sarwate & Shanbhag, riBM): 3delta+1 registers delta_i, theta_i (element
  // i on lane i mod 32, slot i / 32, kept as logs), delta_i = S_{i+1} (i < 2delta), delta_3delta = 1; per
  // iteration, with gamma (initially 1) and the discrepancy delta_0:
  //   delta_i <- gamma delta_{i+1} + delta_0 theta_i
  //   grow (delta_0 != 0 and 2L <= r):  theta_i <- delta_{i+1}, gamma <- delta_0, L <- r + 1 - L
  // After 2delta iterations Lambda_t = delta_{delta+t} (t <= delta) is c * (the BM connection polynomial),
  // c != 0, and delta_0 at iteration r is c_r * (BM's d_r): same L, degree, roots and Forney ratios
  // Omega / Lambda_odd as the plain recurrence. Lambda and x^m B of degree <= r fit the registers, so
  // nothing is truncated; the plain BM's truncation at delta+1 coefficients (R#7) only ever drops terms
  // once L > delta, when both decoders report failure. No warp reduction in the loop: the dependent chain
  // is one broadcast, one product and one log per iteration.
  constexpr int NE = 3 * DL + 1, NS = (NE + 31) / 32;
  uint32_t ldl[NS], lth[NS];
#pragma unroll
  for (int s = 0; s < NS; s++) {
    const int i = lane + 32 * s;
    ldl[s] = i < TD ? (uint32_t)lS[i] : (i == 3 * DL ? 0u : GF_LOG0);
    lth[s] = ldl[s];
  }
  uint32_t lg = 0;  // log gamma
#pragma unroll 1
  for (int r = 0; r < TD; r++) {
    const uint32_t ld0 = __shfl_sync(0xffffffffu, ldl[0], 0);
    uint32_t y[NS];
#pragma unroll
    for (int s = 0; s < NS; s++) y[s] = __shfl_sync(0xffffffffu, ldl[s], (lane + 1) & 31);
    const bool grow = (ld0 != GF_LOG0) && (2 * L <= (uint32_t)r);
#pragma unroll
    for (int s = 0; s < NS; s++) {
      const uint32_t nb = lane == 31 ? (s + 1 < NS ? y[s + 1 < NS ? s + 1 : s] : GF_LOG0) : y[s];  // delta_{i+1}
      const uint32_t val = EXPT[lg + nb] ^ EXPT[ld0 + lth[s]];
      lth[s] = grow ? nb : lth[s];
      ldl[s] = LOGT[val];
    }
    lg = grow ? ld0 : lg;
    L = grow ? (uint32_t)r + 1 - L : L;
  }
  uint32_t bits = 0;
#pragma unroll
  for (int s = 0; s < NS; s++) {
    const int t = lane + 32 * s - DL;
    if (t >= 0 && t <= DL) {
      lLam[t] = (uint16_t)ldl[s];
      bits |= ldl[s] != GF_LOG0 ? 1u << t : 0u;
    }
  }
  nzmask = __reduce_or_sync(0xffffffffu, bits);
  } else if constexpr (HQC_BM_LOOKAHEAD) {
  // The discrepancy of iteration r+1 is formed from iteration r's quantities, so that its dependent chain
  // is lc -> one product -> REDUX -> log, not lc -> update Lambda -> log Lambda -> product -> REDUX -> log:
  //   d_{r+1} = sum_t Lambda'_t S_{r+2-t},  Lambda' = Lambda + c x^m B   (c = d_r / b, log c = lc)
  //           = XOR_t [ Lambda_t S_{r+2-t} ]  XOR  [ c (x^m B)_t S_{r+2-t} ]
  // The first part only needs log Lambda_t of iteration r (known before lc); the update of Lambda and its
  // log run beside the chain. Same values as the plain recurrence (GF arithmetic is exact).
  uint32_t llam = LOGT[lam];
  uint32_t d = __reduce_xor_sync(0xffffffffu, coef ? EXPT[llam + lS[-lane]] : 0u);  // d_0 = S_1
  uint32_t ld = LOGT[d];
  constexpr int kBmUnroll = HQC_WRS_BM_UNROLL;
#pragma unroll kBmUnroll
  for (int r = 0; r < TD; r++) {
    // log S_{r+2-t}; at r = 2delta-1 lane 0 reads the row past the syndromes (not yet written): its d is
    // never used, and the clamp keeps every table index below 1024
    const uint32_t lsn = min((uint32_t)lS[r + 1 - lane], GF_LOG0);
    const uint32_t partA = coef ? EXPT[llam + lsn] : 0u;    // Lambda_t S_{r+2-t}
    const uint32_t lc = d ? mod255_sub(ld, lb) : GF_LOG0;  // log(d / b)
    const bool grow = (d != 0) && (2 * L <= (uint32_t)r);
    const bool zc = lc == GF_LOG0 || lbx == GF_LOG0;
    const uint32_t lcb = mod255_add(zc ? 0u : lc, zc ? 0u : lbx);  // log (c (x^m B)_t)
    const uint32_t partB = (coef && !zc) ? EXPT[lcb + lsn] : 0u;
    lam ^= (coef && !zc) ? EXPT[lcb] : 0u;
    const uint32_t up = __shfl_up_sync(0xffffffffu, grow ? llam : lbx, 1);
    lbx = (lane == 0 || !coef) ? GF_LOG0 : up;
    L = grow ? (uint32_t)r + 1 - L : L;
    lb = grow ? ld : lb;
    d = __reduce_xor_sync(0xffffffffu, partA ^ partB);  // d_{r+1} (the last one is not used)
    ld = LOGT[d];
    llam = LOGT[lam];
  }
  } else {
#pragma unroll 1
  for (int r = 0; r < TD; r++) {
    const uint32_t llam = LOGT[lam];
    const uint32_t term = coef ? EXPT[llam + lS[r - lane]] : 0u;  // Lambda_t S_{r+1-t} (sentinel for r < t)
    const uint32_t d = __reduce_xor_sync(0xffffffffu, term);
    const uint32_t ld = LOGT[d];
    const uint32_t lc = d ? mod255_sub(ld, lb) : GF_LOG0;  // log(d / b)
    const bool grow = (d != 0) && (2 * L <= (uint32_t)r);
    lam ^= coef ? EXPT[lc + lbx] : 0u;
    const uint32_t up = __shfl_up_sync(0xffffffffu, grow ? llam : lbx, 1);
    lbx = (lane == 0 || !coef) ? GF_LOG0 : up;
    L = grow ? (uint32_t)r + 1 - L : L;
    lb = grow ? ld : lb;
  }
  }
  if constexpr (!HQC_BM_RIBM) {
    nzmask = __ballot_sync(0xffffffffu, coef && lam != 0);
    if (coef) lLam[lane] = LOGT[lam];
  }
  const uint32_t deg = 31u - __clz(nzmask);  // Lambda_0 != 0 always
  __syncwarp();
  PHASE(10);

  // ---- Chien search over j < n1 (lane j + 32 q); the odd part of Lambda(alpha^-j) kept for j < k
  uint32_t nroots = 0, root_mine = 0, lodd_mine = GF_LOG0;
#pragma unroll
  for (int q = 0; q < NJ; q++) {
    const int j = lane + 32 * q;
    uint32_t ev = 0, od = 0, e = 0;  // e = (-j t) mod 255
    const uint32_t jm = (uint32_t)j % 255u;
#pragma unroll
    for (int t = 0; t <= DL; t++) {
      const uint32_t x = EXPT[lLam[t] + e];
      if (t & 1) od ^= x; else ev ^= x;
      e = mod255_sub(e, jm);
    }
    const bool root = (j < N1) && (ev == od);
    nroots += __popc(__ballot_sync(0xffffffffu, root));
    if (q == 0) {
      root_mine = root ? 1u : 0u;
      lodd_mine = LOGT[od];
    }
  }
  const bool ok = (L <= (uint32_t)DL) && (deg == L) && (nroots == L);
  PHASE(11);

  // ---- Omega_i = sum_{t <= min(i, delta)} Lambda_t S_{i-t+1}, i < delta (RS_OMEGA_TERMS: the coefficients
  //      i >= L are discrepancies of the final Lambda, zero whenever the correction is applied; riBM's
  //      Lambda is a nonzero multiple of BM's, so the same holds)
  constexpr int OM_N = RS_OMEGA_TERMS<P>;
#pragma unroll
  for (int q = 0; q < (OM_N + 31) / 32; q++) {
    const int i = lane + 32 * q;
    uint32_t om = 0;
#pragma unroll
    for (int t = 0; t <= DL; t++) om ^= EXPT[lLam[t] + lS[i - t]];
    if (i < OM_N) lOm[i] = LOGT[om];
  }
  __syncwarp();
  PHASE(12);

  // ---- Forney on message position j = lane < k: e_j = Omega(alpha^-j) / (alpha^j Lambda_odd(alpha^-j))
  if (lane < K) {
    const uint32_t jm = (uint32_t)lane % 255u;
    uint32_t acc = 0, e = 0;  // e = (-i j) mod 255
    constexpr int kFUnroll = HQC_WRS_FORNEY_UNROLL;
#pragma unroll kFUnroll
    for (int i = 0; i < OM_N; i++) {
      acc ^= EXPT[lOm[i] + e];
      e = mod255_sub(e, jm);
    }
    const uint32_t lnum = LOGT[acc];
    const uint32_t le = mod255_sub(mod255_sub(lnum == GF_LOG0 ? 0u : lnum, jm), lodd_mine == GF_LOG0 ? 0u : lodd_mine);
    const uint32_t ej = (lnum == GF_LOG0 || lodd_mine == GF_LOG0) ? 0u : EXPT[le];
    const uint32_t fix = (ok && root_mine) ? ej : 0u;
    if (out != nullptr) out[lane] = (uint8_t)(sym[lane] ^ fix);
  }
  PHASE(13);
  return ok ? 1u : 0u;
}

}  // namespace hqc
