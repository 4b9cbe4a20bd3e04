// batched HQC.PKE.Encrypt (Alg. 1) and the KeyGen product
// (Alg. 3) on the GPU, reusing the stage-1 sparse x dense machinery with full-width
// outputs. Used by bench.py to make valid ciphertexts on the device; parity-tested against the
// oracle's encrypt/keygen in tests/test_gpu_encrypt.py.
//
//   keygen:  s = x + h*y                       (n bits, pad bits zero)
//   encrypt: u = r1 + h*r2                     (n bits, pad bits zero)
//            v = trunc_{n1 n2}(mG + s*r2 + e)  mG = RM(1,7)^mult o RS(message-first)   (R#3, R#6, R#9)
// The RS encoder is the paper's table-driven LFSR (§III.D, Fig. "rs_lookup_table"): a
// constant table T[f][t] = g*_t * f (2delta x 256 bytes, "approximately 8 KB" for HQC-1) turns every
// per-byte GF multiply into a lookup; g* is the reciprocal generator (message-first layout, R#6).
#pragma once
#include <cstdint>

#include "async_copy.cuh"
#include "exp_timing.cuh"
#include "gf256.cuh"
#include "levels.cuh"
#include "stage1.cuh"

namespace hqc {

// ---- compile-time RS generator tables (gf_mul_c / gf_exp_c from gf256.cuh)
template <uint32_t TD> struct RsEncTable {
  uint8_t t[256][TD];  // t[f][j] = g*_j * f
};
// g*(x) = prod_{i=1}^{2delta} (x + alpha^{-i}) = prod (x + alpha^{255-i}); coefficients g*_0..g*_{2delta-1}
template <uint32_t TD> constexpr RsEncTable<TD> make_rs_enc_table() {
  uint32_t g[TD + 1] = {};
  g[0] = 1;
  for (uint32_t i = 1; i <= TD; i++) {
    const uint32_t root = gf_exp_c(255 - i);
    for (uint32_t t = i; t > 0; t--) g[t] = g[t - 1] ^ gf_mul_c(g[t], root);
    g[0] = gf_mul_c(g[0], root);
  }
  RsEncTable<TD> T{};
  for (uint32_t f = 0; f < 256; f++)
    for (uint32_t j = 0; j < TD; j++) T.t[f][j] = static_cast<uint8_t>(gf_mul_c(g[j], f));
  return T;
}
__device__ const RsEncTable<30> c_rs_enc30 = make_rs_enc_table<30>();
__device__ const RsEncTable<32> c_rs_enc32 = make_rs_enc_table<32>();
__device__ const RsEncTable<58> c_rs_enc58 = make_rs_enc_table<58>();
template <uint32_t TD> __device__ __forceinline__ const uint8_t (*rs_table())[TD];
template <> __device__ __forceinline__ const uint8_t (*rs_table<30>())[30] { return c_rs_enc30.t; }
template <> __device__ __forceinline__ const uint8_t (*rs_table<32>())[32] { return c_rs_enc32.t; }
template <> __device__ __forceinline__ const uint8_t (*rs_table<58>())[58] { return c_rs_enc58.t; }

// Warp-cooperative systematic RS encode of k message bytes (smem msg) into cw[0..n1) (smem).
// Lane t holds LFSR cells t and t+32. c_j = m_j (j < k); c_{n1-1-e} = remainder coefficient e.
template <class P>
__device__ __forceinline__ void rs_encode_warp(const uint8_t *msg, uint8_t *cw, int lane) {
  constexpr uint32_t TD = P::TWO_DELTA;
  const uint8_t(*T)[TD] = rs_table<TD>();
  uint32_t A = 0, B = 0;  // cells lane and lane + 32
  for (uint32_t j = 0; j < P::K; j++) {
    const uint32_t top = (TD - 1 < 32) ? __shfl_sync(0xffffffffu, A, TD - 1) : __shfl_sync(0xffffffffu, B, TD - 1 - 32);
    const uint32_t fb = msg[j] ^ top;
    const uint32_t upA = __shfl_up_sync(0xffffffffu, A, 1);
    const uint32_t upB = __shfl_up_sync(0xffffffffu, B, 1);
    const uint32_t a31 = __shfl_sync(0xffffffffu, A, 31);
    const uint32_t nA = (lane == 0 ? 0u : upA) ^ ((uint32_t)lane < TD ? T[fb][lane] : 0u);
    const uint32_t nB = (lane == 0 ? a31 : upB) ^ ((uint32_t)lane + 32 < TD ? T[fb][lane + 32] : 0u);
    A = nA;
    B = (uint32_t)lane + 32 < TD ? nB : 0u;
  }
  for (uint32_t j = lane; j < P::K; j += 32) cw[j] = msg[j];
  if ((uint32_t)lane < TD) cw[P::N1 - 1 - lane] = (uint8_t)A;
  if ((uint32_t)lane + 32 < TD) cw[P::N1 - 1 - (lane + 32)] = (uint8_t)B;
}

// The same encoder on byte-wide log/antilog tables in SHARED memory (k_encrypt2): the product g*_t * fb
// becomes EXP8[log fb + log g*_t], log g*_t a per-lane constant. The product table above lives in global
// memory (8-15 KB, too large for the shared-memory budget of k_encrypt2) and each of the k dependent steps
// waited on an L1/L2 load: 7% of k_encrypt2's stall samples at HQC-3 (profiles/r02/ncu_encrypt.md).
struct Gf8Tables {
  uint8_t log[256];  // log_alpha(x), 255 for x = 0
  uint8_t exp[512];  // alpha^(e mod 255) for e < 510; 0 for 510, 511
};
constexpr Gf8Tables make_gf8_tables() {
  Gf8Tables t{};
  uint32_t x = 1;
  for (uint32_t e = 0; e < 255; e++) {
    t.exp[e] = t.exp[e + 255] = static_cast<uint8_t>(x);
    t.log[x] = static_cast<uint8_t>(e);
    x = gf_mul_c(x, 2);
  }
  t.log[0] = 255;
  return t;
}
__device__ __align__(16) const Gf8Tables g_gf8 = make_gf8_tables();
static_assert(sizeof(Gf8Tables) % 16 == 0, "copied in 16-byte pieces");

template <uint32_t TD> struct RsGenLog {
  uint8_t lg[64];  // log g*_t for t < TD (255 for a zero coefficient), 255 beyond
};
template <uint32_t TD> constexpr RsGenLog<TD> make_rs_gen_log() {
  RsGenLog<TD> L{};
  const RsEncTable<TD> T = make_rs_enc_table<TD>();  // T[1][t] = g*_t
  const Gf8Tables g = make_gf8_tables();
  for (uint32_t t = 0; t < 64; t++) L.lg[t] = t < TD ? g.log[T.t[1][t]] : 255;
  return L;
}
__device__ const RsGenLog<30> g_rs_lg30 = make_rs_gen_log<30>();
__device__ const RsGenLog<32> g_rs_lg32 = make_rs_gen_log<32>();
__device__ const RsGenLog<58> g_rs_lg58 = make_rs_gen_log<58>();
template <uint32_t TD> __device__ __forceinline__ const uint8_t *rs_gen_log();
template <> __device__ __forceinline__ const uint8_t *rs_gen_log<30>() { return g_rs_lg30.lg; }
template <> __device__ __forceinline__ const uint8_t *rs_gen_log<32>() { return g_rs_lg32.lg; }
template <> __device__ __forceinline__ const uint8_t *rs_gen_log<58>() { return g_rs_lg58.lg; }

__device__ __forceinline__ uint32_t gf8_mul_log(const Gf8Tables *t, uint32_t la, uint32_t lb) {
  return (la == 255u || lb == 255u) ? 0u : t->exp[la + lb];
}

template <class P>
__device__ __forceinline__ void rs_encode_warp_log(const uint8_t *msg, uint8_t *cw, const Gf8Tables *g, int lane) {
  constexpr uint32_t TD = P::TWO_DELTA;
  const uint8_t *LG = rs_gen_log<TD>();
  const uint32_t lgA = __ldg(LG + lane), lgB = __ldg(LG + 32 + lane);  // 255 beyond TD
  uint32_t A = 0, B = 0;  // cells lane and lane + 32
  for (uint32_t j = 0; j < P::K; j++) {
    const uint32_t top = (TD - 1 < 32) ? __shfl_sync(0xffffffffu, A, TD - 1) : __shfl_sync(0xffffffffu, B, TD - 1 - 32);
    const uint32_t lf = g->log[msg[j] ^ top];  // one address for the whole warp: a broadcast
    const uint32_t upA = __shfl_up_sync(0xffffffffu, A, 1);
    const uint32_t upB = __shfl_up_sync(0xffffffffu, B, 1);
    const uint32_t a31 = __shfl_sync(0xffffffffu, A, 31);
    A = (lane == 0 ? 0u : upA) ^ gf8_mul_log(g, lf, lgA);
    B = (uint32_t)lane + 32 < TD ? ((lane == 0 ? a31 : upB) ^ gf8_mul_log(g, lf, lgB)) : 0u;
  }
  for (uint32_t j = lane; j < P::K; j += 32) cw[j] = msg[j];
  if ((uint32_t)lane < TD) cw[P::N1 - 1 - lane] = (uint8_t)A;
  if ((uint32_t)lane + 32 < TD) cw[P::N1 - 1 - (lane + 32)] = (uint8_t)B;
}

// The 128-bit RM(1,7) codeword of byte b (R#9): bit p = b7 ^ parity(b & 0x7F & p), word q = p >> 5.
__device__ __forceinline__ void rm_encode_byte(uint32_t b, uint32_t (&w)[4]) {
  const uint32_t rows[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};
  uint32_t base = (b & 0x80u) ? 0xFFFFFFFFu : 0u;
#pragma unroll
  for (int t = 0; t < 5; t++) base ^= ((b >> t) & 1u) ? rows[t] : 0u;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t flip = (((b >> 5) & 1u) & (q & 1)) ^ (((b >> 6) & 1u) & (q >> 1));
    w[q] = base ^ (flip ? 0xFFFFFFFFu : 0u);
  }
}

// Coalesced copy of nwords (multiple of 4) 32-bit words global -> shared.
__device__ __forceinline__ void copy_g2s(uint32_t *dst, const void *src, uint32_t nwords, int lane) {
  const uint4 *s = reinterpret_cast<const uint4 *>(src);
  for (uint32_t c = lane; c < nwords / 4; c += 32) reinterpret_cast<uint4 *>(dst)[c] = __ldg(s + c);
}
__device__ __forceinline__ void copy_s2g(void *dst, const uint32_t *src, uint32_t nwords, int lane) {
  uint4 *d = reinterpret_cast<uint4 *>(dst);
  for (uint32_t c = lane; c < nwords / 4; c += 32) d[c] = reinterpret_cast<const uint4 *>(src)[c];
}

#ifndef HQC_ENC_TAIL
#define HQC_ENC_TAIL 1
#endif
// A product over NTOT words whose odd per-lane word count R = odd ceil(NTOT / 32) wastes slots (HQC-1: 552
// / 553 words -> R = 19; HQC-3's u: 1,121 words -> R = 37) runs with the largest odd R such that 32 R <=
// NTOT, and the warp adds the TW <= 9 words above 32 R cooperatively (s1_tail_words: lane-strided support
// indices, one REDUX.XOR per word). HQC-5's tops (40+ words) keep the plain shape.
template <uint32_t NTOT> constexpr uint32_t enc_tail_words() {
  constexpr uint32_t r = ((NTOT / 32) & 1u) ? NTOT / 32 : NTOT / 32 - 1;
  return (HQC_ENC_TAIL && NTOT - 32 * r > 0 && NTOT - 32 * r <= 9) ? NTOT - 32 * r : 0u;
}
template <class P> constexpr uint32_t enc_tail() { return enc_tail_words<P::Q0 + 1>(); }       // u, s
template <class P> constexpr uint32_t enc_tail_v() { return enc_tail_words<P::NW>(); }         // v
template <class P> using FullShapeT = ProdShape<P, P::Q0 + 1 - enc_tail<P>(), P::WR>;
template <class P> using KeyShapeT = ProdShape<P, P::Q0 + 1 - enc_tail<P>(), P::W>;
template <class P> using EncVShapeT = ProdShape<P, P::NW - enc_tail_v<P>(), P::WR>;

// Store words [S::NOUT, S::NOUT + TW) of the tail (t: every lane holds all TW values) into out.
template <class S, uint32_t TW>
__device__ __forceinline__ void store_tail(const uint32_t (&t)[TW], uint32_t *out, int lane) {
  uint32_t mine = 0;
#pragma unroll
  for (uint32_t i = 0; i < TW; i++) mine = (uint32_t)lane == i ? t[i] : mine;
  if ((uint32_t)lane < TW) out[S::NOUT + lane] = mine;
}

// One warp: out (NOUT + TW words in smem, aliasing E) = dense (staged in su) * support (staged in ssup);
// the TW top words are computed by the whole warp before r overwrites E.
template <class P, class S, uint32_t TW = 0>
__device__ __forceinline__ void warp_product(uint32_t *su, const uint32_t *ssup, uint32_t *E, uint32_t *dsm,
                                             int lane) {
  s1_stage_d<P, S>(ssup, dsm, lane);
  s1_build_E<P, S>(su, E, lane);
  __syncwarp();
  uint32_t acc[S::R];
  s1_product<P, S>(E, dsm, acc, lane);
  uint32_t t[TW > 0 ? TW : 1];
  if constexpr (TW > 0) s1_tail_words<P, S, S::NOUT, TW>(E, dsm, lane, t);
  __syncwarp();
  s1_store_r<S>(acc, E, lane);
  if constexpr (TW > 0) store_tail<S, TW>(t, E, lane);
  __syncwarp();
}

// The same with the segmented layout (stage1.cuh: s1_seg_product); S sizes E, G is the product's SegShape.
template <class P, class S, class G>
__device__ __forceinline__ void warp_product_seg(uint32_t *su, const uint32_t *ssup, uint32_t *E, uint32_t *dsm,
                                                 int lane) {
  static_assert(S::E_WORDS >= G::E_NEED, "the segmented windows stay inside E");
  s1_stage_d<P, S>(ssup, dsm, lane);
  s1_build_E<P, S>(su, E, lane);
  __syncwarp();
  uint32_t acc[G::LMAX], top;
  s1_seg_product<P, G, s1_unroll_enc<P>()>(E, dsm, acc, top, lane);
  __syncwarp();
  s1_seg_store<G>(acc, top, E, lane);
  __syncwarp();
}

// XOR the bits of a support (first wt entries, positions < limit) into a bit vector in smem.
__device__ __forceinline__ void xor_support_bits(uint32_t *vec, const uint32_t *supp, uint32_t wt, uint32_t limit,
                                                 int lane) {
  for (uint32_t j = lane; j < wt; j += 32) {
    const uint32_t p = supp[j];
    if (p < limit) atomicXor(vec + (p >> 5), 1u << (p & 31));
  }
}

template <class P> struct EncSmem {
  static constexpr uint32_t EW = FullShape<P>::E_WORDS > EncVShape<P>::E_WORDS ? FullShape<P>::E_WORDS
                                                                               : EncVShape<P>::E_WORDS;
  static constexpr uint32_t E_BYTES = round_up(EW * 4, 16);
  static constexpr uint32_t STG_BYTES = round_up(P::U_STRIDE * 8, 16);
  static constexpr uint32_t SUP_BYTES = round_up(P::E_STRIDE * 4, 16) * 3;  // r1/x, r2/y, e
  static constexpr uint32_t D_BYTES = round_up(round_up(P::WR, 4) * 4, 16);
  static constexpr uint32_t MISC_BYTES = round_up(P::N1 + P::K + 16, 16);
  static constexpr uint32_t BYTES = E_BYTES + STG_BYTES + SUP_BYTES + D_BYTES + MISC_BYTES;
};

// keygen: s[k] = x[k] + h[k]*y[k]. One warp per key.
template <class P>
__global__ void __launch_bounds__(32) k_keygen(const uint64_t *__restrict__ h, const uint32_t *__restrict__ x,
                                               const uint32_t *__restrict__ y, uint64_t *__restrict__ s, size_t nkeys) {
  extern __shared__ __align__(16) uint8_t smem[];
  using M = EncSmem<P>;
  using S = KeyShapeT<P>;
  const int lane = threadIdx.x;
  uint32_t *E = reinterpret_cast<uint32_t *>(smem);
  uint32_t *stg = reinterpret_cast<uint32_t *>(smem + M::E_BYTES);
  uint32_t *sx = reinterpret_cast<uint32_t *>(smem + M::E_BYTES + M::STG_BYTES);
  uint32_t *sy = sx + M::SUP_BYTES / 12;
  uint32_t *dsm = reinterpret_cast<uint32_t *>(smem + M::E_BYTES + M::STG_BYTES + M::SUP_BYTES);
  for (size_t kk = blockIdx.x; kk < nkeys; kk += gridDim.x) {
    copy_g2s(stg, h + kk * P::U_STRIDE, 2 * P::U_STRIDE, lane);
    copy_g2s(sx, x + kk * P::Y_STRIDE, P::Y_STRIDE, lane);
    copy_g2s(sy, y + kk * P::Y_STRIDE, P::Y_STRIDE, lane);
    __syncwarp();
#if HQC_S1_SEG
    warp_product_seg<P, KeyShape<P>, KeySeg<P>>(stg, sy, E, dsm, lane);
#else
    warp_product<P, S, enc_tail<P>()>(stg, sy, E, dsm, lane);
#endif
    xor_support_bits(E, sx, P::W, P::N, lane);
    __syncwarp();
    if (lane == 0) E[P::Q0] &= (1u << P::C) - 1u;  // bits >= n are zero
    for (uint32_t q = P::Q0 + 1 + lane; q < 2 * P::U_STRIDE; q += 32) E[q] = 0;
    __syncwarp();
    copy_s2g(s + kk * P::U_STRIDE, E, 2 * P::U_STRIDE, lane);
    __syncwarp();
  }
}

// encrypt: one warp per ciphertext (the first GPU encrypt; HQC_ENC_KERNEL=1 selects it, k_encrypt2 below
// is the default). CMP = false writes (u, v) to u_out / v_out. CMP = true is the KEM's re-encryption
// check (kem.cuh): the re-encrypted (u', v') never leaves shared memory; it is compared with the
// received (u_cmp, v_cmp) word by word (bits >= n of u_cmp ignored, as in oracle/kem.c) with no early
// exit, and eq_out[2 ct] = eq_out[2 ct + 1] = 1 iff every word matched.
template <class P, bool CMP = false>
__global__ void __launch_bounds__(32) k_encrypt(const uint64_t *__restrict__ h, const uint64_t *__restrict__ s,
                                                const uint32_t *__restrict__ key_index, const uint8_t *__restrict__ m,
                                                const uint32_t *__restrict__ r1, const uint32_t *__restrict__ r2,
                                                const uint32_t *__restrict__ e, uint64_t *__restrict__ u_out,
                                                uint64_t *__restrict__ v_out, size_t batch,
                                                const uint64_t *__restrict__ u_cmp = nullptr,
                                                const uint64_t *__restrict__ v_cmp = nullptr,
                                                uint8_t *__restrict__ eq_out = nullptr) {
  extern __shared__ __align__(16) uint8_t smem[];
  using M = EncSmem<P>;
  const int lane = threadIdx.x;
  uint32_t *E = reinterpret_cast<uint32_t *>(smem);
  uint32_t *stg = reinterpret_cast<uint32_t *>(smem + M::E_BYTES);
  uint32_t *s_r1 = reinterpret_cast<uint32_t *>(smem + M::E_BYTES + M::STG_BYTES);
  uint32_t *s_r2 = s_r1 + M::SUP_BYTES / 12;
  uint32_t *s_e = s_r2 + M::SUP_BYTES / 12;
  uint32_t *dsm = reinterpret_cast<uint32_t *>(smem + M::E_BYTES + M::STG_BYTES + M::SUP_BYTES);
  uint8_t *cw = smem + M::E_BYTES + M::STG_BYTES + M::SUP_BYTES + M::D_BYTES;
  uint8_t *msg = cw + P::N1;
  for (size_t ct = blockIdx.x; ct < batch; ct += gridDim.x) {
    const size_t key = key_index ? key_index[ct] : ct;
    copy_g2s(s_r1, r1 + ct * P::E_STRIDE, P::E_STRIDE, lane);
    copy_g2s(s_r2, r2 + ct * P::E_STRIDE, P::E_STRIDE, lane);
    copy_g2s(s_e, e + ct * P::E_STRIDE, P::E_STRIDE, lane);
    copy_g2s(stg, h + key * P::U_STRIDE, 2 * P::U_STRIDE, lane);
    for (uint32_t j = lane; j < P::K; j += 32) msg[j] = m[ct * P::K + j];
    __syncwarp();
    // u = r1 + h * r2 (all n bits)
#if HQC_S1_SEG
    warp_product_seg<P, FullShape<P>, FullSeg<P>>(stg, s_r2, E, dsm, lane);
#else
    warp_product<P, FullShape<P>>(stg, s_r2, E, dsm, lane);
#endif
    xor_support_bits(E, s_r1, P::WR, P::N, lane);
    __syncwarp();
    if (lane == 0) E[P::Q0] &= (1u << P::C) - 1u;
    for (uint32_t q = P::Q0 + 1 + lane; q < 2 * P::U_STRIDE; q += 32) E[q] = 0;
    __syncwarp();
    uint32_t diff = 0;
    if constexpr (CMP) {
      const uint32_t *uc = reinterpret_cast<const uint32_t *>(u_cmp + ct * P::U_STRIDE);
      for (uint32_t q = lane; q < 2 * P::U_WORDS; q += 32) {
        const uint32_t x = q < P::Q0 ? uc[q] : (q == P::Q0 ? uc[q] & P::CB_MASK : 0u);
        diff |= x ^ E[q];
      }
    } else {
      copy_s2g(u_out + ct * P::U_STRIDE, E, 2 * P::U_STRIDE, lane);
    }
    __syncwarp();
    // v = trunc(mG + s * r2 + e)
    copy_g2s(stg, s + key * P::U_STRIDE, 2 * P::U_STRIDE, lane);
    rs_encode_warp<P>(msg, cw, lane);
    __syncwarp();
#if HQC_S1_SEG
    warp_product_seg<P, EncVShape<P>, EncVSeg<P>>(stg, s_r2, E, dsm, lane);
#else
    warp_product<P, EncVShape<P>>(stg, s_r2, E, dsm, lane);
#endif
    for (uint32_t j = lane; j < P::N1; j += 32) {  // RM-encode symbol j into block j, every copy
      uint32_t w[4];
      rm_encode_byte(cw[j], w);
      uint32_t *blk = E + j * (P::N2 / 32);
#pragma unroll
      for (uint32_t c = 0; c < P::MULT; c++)
#pragma unroll
        for (int q = 0; q < 4; q++) blk[4 * c + q] ^= w[q];
    }
    __syncwarp();
    xor_support_bits(E, s_e, P::WR, P::N12, lane);
    __syncwarp();
    if constexpr (CMP) {
      const uint4 *vc = reinterpret_cast<const uint4 *>(v_cmp + ct * P::V_WORDS);
      for (uint32_t c = lane; c < P::NW / 4; c += 32) {
        const uint4 x = __ldg(vc + c);
        const uint4 y = reinterpret_cast<const uint4 *>(E)[c];
        diff |= (x.x ^ y.x) | (x.y ^ y.y) | (x.z ^ y.z) | (x.w ^ y.w);
      }
      diff = __reduce_or_sync(0xffffffffu, diff);
      if (lane == 0) eq_out[2 * ct] = eq_out[2 * ct + 1] = diff == 0;  // the two-flag layout of k_encrypt2
    } else {
      copy_s2g(v_out + ct * P::V_WORDS, E, P::NW, lane);
    }
    __syncwarp();
  }
}

// encrypt, WARP PAIR per CTA: warp 0 computes u = r1 + h*r2, warp 1 computes v = trunc(mG + s*r2 + e),
// concurrently and without exchanging data. Each CTA owns a contiguous range of ciphertexts, and each
// warp keeps the doubled dense operand (E_h, E_s) of the current key in shared memory, rebuilding it only
// when key_index changes (one key per 256 ciphertexts in the BASELINE recipe): per ciphertext only the
// product, the encoders and the support XORs remain. CMP = true (KEM re-encryption check): each warp
// compares its half of c' with the received c and writes its own flag, eq2_out[2 ct + warp]; the KDF
// accepts iff both are set.
template <class P> struct Enc2Smem {
  using SU = FullShapeT<P>;
  using SV = EncVShapeT<P>;
  static constexpr uint32_t EU_BYTES = round_up(SU::E_WORDS * 4, 16);
  static constexpr uint32_t EV_BYTES = round_up(SV::E_WORDS * 4, 16);
  // staging of a key row (2 u_stride words), then the warp's product output
  static constexpr uint32_t OUT_WORDS = 2 * P::U_STRIDE > P::NW ? 2 * P::U_STRIDE : P::NW;
  static constexpr uint32_t OUT_BYTES = round_up(OUT_WORDS * 4, 16);
  static constexpr uint32_t SUP_BYTES = round_up(P::E_STRIDE * 4, 16);
  static_assert((P::E_STRIDE * 4) % 16 == 0, "support rows are TMA bulk copies");
  static constexpr uint32_t D_BYTES = round_up(round_up(P::WR, 4) * 4, 16);
  static constexpr uint32_t MISC_BYTES = round_up(P::N1 + P::K + 16, 16);
  // two buffers of (r2 row, r1 or e row), prefetched by TMA one ciphertext ahead; two mbarriers. The
  // rotation amounts of r2 are written over the r2 row (elementwise, in place): no separate array.
  static_assert(D_BYTES <= SUP_BYTES, "the rotation amounts fit the r2 row");
  static constexpr uint32_t SUPS_BYTES = 4 * SUP_BYTES + 16;
  static constexpr uint32_t GF8_BYTES = sizeof(Gf8Tables);  // the encoder's log/antilog (warp 1), per CTA
  static constexpr uint32_t W0_BYTES = EU_BYTES + OUT_BYTES + SUPS_BYTES;
  static constexpr uint32_t W1_BYTES = EV_BYTES + OUT_BYTES + SUPS_BYTES + MISC_BYTES;
  static constexpr uint32_t WARP_BYTES = W0_BYTES > W1_BYTES ? W0_BYTES : W1_BYTES;
  static constexpr uint32_t CTR_BYTES = 16;  // the CTA's two work counters (u jobs, v jobs)
  // a CTA of Q u-warps and Q v-warps: Q <= 8 (512 threads, <= 128 registers) — 12 for HQC-1, whose warps
  // need 80 registers (768 threads, <= 85) — and fewer where shared memory ends (HQC-3: 7, HQC-5: 4)
  static constexpr uint32_t bytes(uint32_t q) { return GF8_BYTES + CTR_BYTES + 2 * q * WARP_BYTES; }
  static constexpr uint32_t fit(uint32_t q) { return q > 1 && bytes(q) > 227u * 1024u ? fit(q - 1) : q; }
  static constexpr uint32_t MAX_Q = fit(P::level == 1 ? 12 : 8);
  static constexpr uint32_t BYTES = bytes(1);
};

#ifndef HQC_ENC2_MINB
#define HQC_ENC2_MINB 1
#endif
template <class P, bool CMP = false>
__global__ void __launch_bounds__(64 * Enc2Smem<P>::MAX_Q, HQC_ENC2_MINB) k_encrypt2(const uint64_t *__restrict__ h, const uint64_t *__restrict__ s,
                                                 const uint32_t *__restrict__ key_index, const uint8_t *__restrict__ m,
                                                 const uint32_t *__restrict__ r1, const uint32_t *__restrict__ r2,
                                                 const uint32_t *__restrict__ e, uint64_t *__restrict__ u_out,
                                                 uint64_t *__restrict__ v_out, size_t batch, size_t per,
                                                 const uint64_t *__restrict__ u_cmp = nullptr,
                                                 const uint64_t *__restrict__ v_cmp = nullptr,
                                                 uint8_t *__restrict__ eq2_out = nullptr) {
  extern __shared__ __align__(16) uint8_t smem[];
  using M = Enc2Smem<P>;
  const int lane = threadIdx.x & 31;
  // Q u-warps (role 0: u = r1 + h r2) and Q v-warps (role 1: v = mG + s r2 + e); each warp caches the
  // doubled operand of its current key and takes jobs of its role from the CTA's contiguous range through a
  // shared-memory counter (claimed one ahead for the TMA prefetch). With one warp pair per CTA and fixed
  // ranges, the CTAs sharing an SM ended up to 50% apart (profiles/r02/enc_span.log): the SM ran its tail
  // with few warps.
  const uint32_t Q = blockDim.x >> 6;
  const uint32_t w_all = threadIdx.x >> 5;
  const int wid = w_all >= Q ? 1 : 0;      // role
  const uint32_t widx = w_all - wid * Q;  // index among the warps of this role
  Gf8Tables *gf8 = reinterpret_cast<Gf8Tables *>(smem);
  unsigned int *ctr = reinterpret_cast<unsigned int *>(smem + M::GF8_BYTES);
  uint8_t *base = smem + M::GF8_BYTES + M::CTR_BYTES + (size_t)w_all * M::WARP_BYTES;
  uint32_t *E = reinterpret_cast<uint32_t *>(base);
  uint32_t *out = reinterpret_cast<uint32_t *>(base + (wid ? M::EV_BYTES : M::EU_BYTES));
  uint32_t *sups = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(out) + M::OUT_BYTES);
  uint64_t *bar = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(sups) + 4 * M::SUP_BYTES);
  uint8_t *cw = reinterpret_cast<uint8_t *>(sups) + M::SUPS_BYTES;  // warp 1 only
  uint8_t *msg = cw + P::N1;
  const size_t lo = (size_t)blockIdx.x * per;
  const size_t hi = lo + per < batch ? lo + per : batch;
  const uint32_t *xsrc = wid ? e : r1;  // r1 (u-warps) or e (v-warps)
  constexpr uint32_t SB = P::E_STRIDE * 4;
  // buffer b: r2 row at sups + 2 b SUP, the r1 / e row at sups + (2 b + 1) SUP; mbarrier bar[b]
  auto sup_r2 = [&](int b) { return sups + (2 * b) * (M::SUP_BYTES / 4); };
  auto sup_x = [&](int b) { return sups + (2 * b + 1) * (M::SUP_BYTES / 4); };
  auto prefetch = [&](size_t c, int b) {  // the supports of ciphertext c, one ciphertext ahead
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar + b, 2 * SB);
      tma_load_1d(sup_r2(b), r2 + c * P::E_STRIDE, SB, bar + b);
      tma_load_1d(sup_x(b), xsrc + c * P::E_STRIDE, SB, bar + b);
    }
  };
  // the previous ciphertext's output store (TMA, async) must have read `out` before it is rewritten
  auto out_free = [&]() {
    if (!CMP && lane == 0) tma_store_wait_read();
    __syncwarp();
  };
  WARP_SPAN(0, (size_t)blockIdx.x * 2 * Q + w_all);
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  if (threadIdx.x == 0) ctr[0] = ctr[1] = Q;  // the first Q jobs of each role are taken statically
  for (uint32_t i = threadIdx.x; i < sizeof(Gf8Tables) / 16; i += blockDim.x)
    reinterpret_cast<uint4 *>(gf8)[i] = __ldg(reinterpret_cast<const uint4 *>(&g_gf8) + i);
  __syncthreads();
  uint32_t ph0 = 0, ph1 = 0;
  size_t ct = lo + widx;
  uint32_t mnext = (wid && ct < hi && (uint32_t)lane < P::K) ? m[ct * P::K + lane] : 0u;
  if (ct < hi) prefetch(ct, 0);
  size_t cached = ~(size_t)0;
  for (int b = 0; ct < hi; b ^= 1) {
    uint32_t nx = 0;
    if (lane == 0) nx = atomicAdd(ctr + wid, 1u);
    const size_t nct = lo + __shfl_sync(0xffffffffu, nx, 0);
    const bool more = nct < hi;
    const size_t key = key_index ? key_index[ct] : ct;
    if (key != cached) {  // a public index: the only data-dependent branch, on public data
      out_free();
      copy_g2s(out, (wid ? s : h) + key * P::U_STRIDE, 2 * P::U_STRIDE, lane);
      __syncwarp();
      if (wid) s1_build_E<P, typename M::SV>(out, E, lane);
      else s1_build_E<P, typename M::SU>(out, E, lane);
      cached = key;
    }
    if (wid) {  // this ciphertext's message (loaded one job ahead), then the next one's
      if ((uint32_t)lane < P::K) msg[lane] = (uint8_t)mnext;
      mnext = (more && (uint32_t)lane < P::K) ? m[nct * P::K + lane] : 0u;
    }
    mbar_wait(bar + b, b ? ph1 : ph0);
    if (b) ph1 ^= 1u; else ph0 ^= 1u;
    __syncwarp();  // every lane has seen the rows land (and is done with buffer b ^ 1 of the previous job)
    if (more) prefetch(nct, b ^ 1);
    uint32_t *s_r2 = sup_r2(b);
    uint32_t *s_x = sup_x(b);
    uint32_t *dsm = s_r2;  // the rotation amounts replace the r2 row entry by entry
    __syncwarp();
    uint32_t diff = 0;
    if (wid == 0) {  // u = r1 + h * r2 (all n bits)   (wid: the warp's role)
      using S = typename M::SU;
      s1_stage_d<P, S>(s_r2, dsm, lane);
      __syncwarp();
#if HQC_S1_SEG
      using G = FullSeg<P>;
      static_assert(S::E_WORDS >= G::E_NEED, "the segmented windows stay inside E");
      uint32_t acc[G::LMAX], top;
      s1_seg_product<P, G, s1_unroll_enc<P>()>(E, dsm, acc, top, lane);
      out_free();
      s1_seg_store<G>(acc, top, out, lane);
#else
      uint32_t acc[S::R];
      s1_product<P, S>(E, dsm, acc, lane);
      out_free();
      s1_store_r<S>(acc, out, lane);
      if constexpr (enc_tail<P>() != 0) {
        uint32_t t[enc_tail<P>()];
        s1_tail_words<P, S, S::NOUT, enc_tail<P>()>(E, dsm, lane, t);
        store_tail<S, enc_tail<P>()>(t, out, lane);
      }
#endif
      __syncwarp();
      xor_support_bits(out, s_x, P::WR, P::N, lane);
      __syncwarp();
      if (lane == 0) out[P::Q0] &= (1u << P::C) - 1u;
      for (uint32_t q = P::Q0 + 1 + lane; q < 2 * P::U_STRIDE; q += 32) out[q] = 0;
      __syncwarp();
      if constexpr (CMP) {
        const uint32_t *uc = reinterpret_cast<const uint32_t *>(u_cmp + ct * P::U_STRIDE);
        for (uint32_t q = lane; q < 2 * P::U_WORDS; q += 32) {
          const uint32_t x = q < P::Q0 ? uc[q] : (q == P::Q0 ? uc[q] & P::CB_MASK : 0u);
          diff |= x ^ out[q];
        }
      } else {  // u row to HBM by a TMA bulk store; `out` is rewritten only after out_free()
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tma_store_1d(u_out + ct * P::U_STRIDE, out, P::U_STRIDE * 8);
      }
    } else {  // v = trunc(mG + s * r2 + e)
      using S = typename M::SV;
      rs_encode_warp_log<P>(msg, cw, gf8, lane);
      s1_stage_d<P, S>(s_r2, dsm, lane);
      __syncwarp();
#if HQC_S1_SEG
      using G = EncVSeg<P>;
      static_assert(S::E_WORDS >= G::E_NEED, "the segmented windows stay inside E");
      uint32_t acc[G::LMAX], top;
      s1_seg_product<P, G, s1_unroll_enc<P>()>(E, dsm, acc, top, lane);
      out_free();
      s1_seg_store<G>(acc, top, out, lane);
#else
      uint32_t acc[S::R];
      s1_product<P, S>(E, dsm, acc, lane);
      out_free();
      s1_store_r<S>(acc, out, lane);
      if constexpr (enc_tail_v<P>() != 0) {
        uint32_t t[enc_tail_v<P>()];
        s1_tail_words<P, S, S::NOUT, enc_tail_v<P>()>(E, dsm, lane, t);
        store_tail<S, enc_tail_v<P>()>(t, out, lane);
      }
#endif
      __syncwarp();
      for (uint32_t j = lane; j < P::N1; j += 32) {  // RM-encode symbol j into block j, every copy
        uint32_t w[4];
        rm_encode_byte(cw[j], w);
        uint32_t *blk = out + j * (P::N2 / 32);
#pragma unroll
        for (uint32_t c = 0; c < P::MULT; c++)
#pragma unroll
          for (int q = 0; q < 4; q++) blk[4 * c + q] ^= w[q];
      }
      __syncwarp();
      xor_support_bits(out, s_x, P::WR, P::N12, lane);
      __syncwarp();
      if constexpr (CMP) {
        const uint4 *vc = reinterpret_cast<const uint4 *>(v_cmp + ct * P::V_WORDS);
        for (uint32_t c = lane; c < P::NW / 4; c += 32) {
          const uint4 x = __ldg(vc + c);
          const uint4 y = reinterpret_cast<const uint4 *>(out)[c];
          diff |= (x.x ^ y.x) | (x.y ^ y.y) | (x.z ^ y.z) | (x.w ^ y.w);
        }
      } else {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tma_store_1d(v_out + ct * P::V_WORDS, out, P::V_WORDS * 8);
      }
    }
    if constexpr (CMP) {
      diff = __reduce_or_sync(0xffffffffu, diff);
      if (lane == 0) eq2_out[2 * ct + wid] = diff == 0;
    }
    __syncwarp();
    ct = nct;
  }
  WARP_SPAN(1, (size_t)blockIdx.x * 2 * Q + w_all);
  if (!CMP && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete before exit
}

}  // namespace hqc
