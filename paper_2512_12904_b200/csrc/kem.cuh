// batched HQC.KEM.Encaps / Decaps with the HHK transform and implicit
// rejection ("In Decap, the receiver decrypts the ciphertext (calling Decrypt), and then
// re-encrypts to verify correctness, and securely rejects invalid ciphertexts"). The hash inputs
// follow DESIGN.md readings R#20-R#23 (the same readings oracle/kem.c states; the two share no code):
//   H_pk  = SHAKE256(h bytes || s bytes || 0x02, 32)                         R#20, R#21
//   theta = SHAKE256(H_pk || m || 0x01, 32)                                  R#20
//   coins = SHAKE256(theta || 0x04, 12 wr) -> 3 wr LE u32 -> r1, r2, e        R#22 (sampler below)
//   K     = SHAKE256((c' == c ? m' : sigma) || u bytes || v bytes || 0x03, 64) R#23
// Decaps = the fused decrypt kernel (m') -> k_kem_coins (lane per ciphertext: theta, the coin
// squeeze and the fixed-weight sampler) -> k_encrypt2<P, true> (warp pair per ciphertext: re-encryption
// compared with c inside shared memory, one flag per half) -> k_kem_kdf (lane per ciphertext: K). No branch on the
// comparison result anywhere: the KDF input is selected with masks.
#pragma once
#include <cstdint>

#include "keccak.cuh"
#include "kernels.cuh"  // launch_decrypt, k_encrypt, EncSmem

namespace hqc {

template <class P> struct KemShape {
  static constexpr uint32_t UB = (P::N + 7) / 8;  // serialised u (and h, s) bytes
  static constexpr uint32_t VB = P::N12 / 8;      // serialised v bytes
  static constexpr uint32_t KW = P::K / 8;        // message words
  static constexpr uint32_t T3 = 3 * P::WR;       // coin words (u32)
  // sampler buffer: per lane, 3 support segments of SEG u16 each (SEG = 4 * odd >= wr: the 32 lanes'
  // 64-bit reads of one group index fall in 16 distinct bank pairs per half-warp); entries >= wr = 0xFFFF
  static constexpr uint32_t SEG = ((P::WR + 3) / 4 | 1u) * 4;
  static constexpr uint32_t PB_BYTES = round_up(32 * 3 * SEG * 2, 16);
  static_assert(P::K % 8 == 0, "messages are whole 64-bit words");
  static_assert(P::N < 65536, "sampled positions fit 16 bits");
};

// Message stream "F words (registers) || AB bytes of row a || BB bytes of row b || tag" as
// 64-bit little-endian words, for shake256_absorb. Rows a and b are 8-byte aligned.
template <uint32_t FW, uint32_t AB, uint32_t BB, uint32_t TAG> struct CatReader {
  static constexpr uint32_t LEN = 8 * FW + AB + BB + 1;
  static constexpr uint32_t QA = AB / 8, RA = AB % 8, QB = BB / 8, RB = BB % 8;
  uint64_t f[FW > 0 ? FW : 1];
  const uint64_t *a, *b;
  __device__ __forceinline__ uint64_t bw(uint32_t i) const {  // word i of (b bytes || tag || 0...)
    if (i < QB) return b[i];
    if (i == QB) {
      uint64_t x = (uint64_t)TAG << (8 * RB);
      if constexpr (RB != 0) x |= b[QB] & ((1ull << (8 * RB)) - 1ull);
      return x;
    }
    return 0;
  }
  __device__ __forceinline__ uint64_t operator()(uint32_t wi) const {
    if (wi < FW) {
      uint64_t x = 0;
#pragma unroll
      for (uint32_t t = 0; t < FW; t++) x = wi == t ? f[t] : x;
      return x;
    }
    const uint32_t j = wi - FW;
    if constexpr (RA == 0) {
      return j < QA ? a[j] : bw(j - QA);
    } else {
      if (j < QA) return a[j];
      if (j == QA) return (a[QA] & ((1ull << (8 * RA)) - 1ull)) | (bw(0) << (8 * RA));
      return (bw(j - QA - 1) >> (64 - 8 * RA)) | (bw(j - QA) << (8 * RA));
    }
  }
};

// ---- H_pk per key (lane per key)
template <class P>
__global__ void __launch_bounds__(128) k_kem_hpk(const uint64_t *__restrict__ h, const uint64_t *__restrict__ s,
                                                 uint8_t *__restrict__ hpk, size_t nkeys) {
  using KS = KemShape<P>;
  const size_t key = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (key >= nkeys) return;
  CatReader<0, KS::UB, KS::UB, 0x02> rd;
  rd.a = h + key * P::U_STRIDE;
  rd.b = s + key * P::U_STRIDE;
  uint64_t A[25];
  shake256_absorb<decltype(rd)::LEN>(A, rd);
  uint64_t *o = reinterpret_cast<uint64_t *>(hpk + key * 32);
#pragma unroll
  for (int i = 0; i < 4; i++) o[i] = A[i];
}

// ---- theta, coins and the fixed-weight sampler (lane per ciphertext; R#22):
//   p_i = i + floor(rand_i (n - i) / 2^32), then for i = w-1 down to 0: p_i = i if p_i equals a later
//   (already final) entry. The loop counts depend only on the level.
// Sampled positions of the warp's 32 ciphertexts sit in shared memory as u16, per lane three contiguous
// segments (one per support), read four at a time by the duplicate scan and row by row by the
// transposed, coalesced write-out.
template <class P, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_kem_coins(const uint8_t *__restrict__ hpk,
                                                          const uint32_t *__restrict__ key_index,
                                                          const uint8_t *__restrict__ m, uint32_t *__restrict__ r1,
                                                          uint32_t *__restrict__ r2, uint32_t *__restrict__ e,
                                                          size_t batch) {
  using KS = KemShape<P>;
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint16_t *pb = reinterpret_cast<uint16_t *>(smem + warp * KS::PB_BYTES);
  const size_t base = ((size_t)blockIdx.x * WARPS + warp) * 32;
  if (base >= batch) return;
  const size_t ct = base + lane < batch ? base + lane : batch - 1;  // tail lanes redo the last row
  const size_t key = key_index ? key_index[ct] : ct;
  uint64_t A[25];
  {  // theta = SHAKE256(H_pk || m || G)
    CatReader<4, P::K, 0, 0x01> rd;
    const uint64_t *hp = reinterpret_cast<const uint64_t *>(hpk + key * 32);
#pragma unroll
    for (int i = 0; i < 4; i++) rd.f[i] = hp[i];
    rd.a = reinterpret_cast<const uint64_t *>(m + ct * P::K);
    rd.b = nullptr;
    shake256_absorb<decltype(rd)::LEN>(A, rd);
  }
  {  // coins = SHAKE256(theta || PRNG, 12 wr)
    CatReader<4, 0, 0, 0x04> rd;
#pragma unroll
    for (int i = 0; i < 4; i++) rd.f[i] = A[i];
    rd.a = rd.b = nullptr;
    shake256_absorb<decltype(rd)::LEN>(A, rd);
  }
  uint16_t *own = pb + lane * 3 * KS::SEG;  // this lane's three segments
  for (uint32_t t = 0; t < 3; t++)
#pragma unroll
    for (uint32_t q = P::WR; q < KS::SEG; q++) own[t * KS::SEG + q] = 0xFFFFu;  // never a position (n < 65535)
  constexpr uint32_t NBLK = (KS::T3 + 2 * SHAKE256_RATE_W - 1) / (2 * SHAKE256_RATE_W);
#pragma unroll 1
  for (uint32_t blk = 0; blk < NBLK; blk++) {
    if (blk) keccak_f1600(A);
#pragma unroll
    for (uint32_t i = 0; i < 2 * SHAKE256_RATE_W; i++) {
      const uint32_t t = blk * 2 * SHAKE256_RATE_W + i;
      if (t < KS::T3) {
        const uint32_t x = (i & 1) ? (uint32_t)(A[i >> 1] >> 32) : (uint32_t)A[i >> 1];
        const uint32_t sidx = t / P::WR, idx = t % P::WR;
        own[sidx * KS::SEG + idx] = (uint16_t)(idx + __umulhi(x, P::N - idx));
      }
    }
  }
  // R#22 deduplication, 4 entries per 64-bit read: for i = wr-1 down to 0, p_i <- i if p_i equals a later
  // (final) entry. Equality of four u16 at once: x = v ^ (p_i x4) has a zero halfword iff some entry
  // matches ((x - 0x0001..) & ~x & 0x8000.. is nonzero then; a borrow can only add false positives above
  // a true zero, so "any match" is exact). Entries <= i of the first group are forced nonzero. The loop
  // counts depend on i only.
#pragma unroll 1
  for (uint32_t sidx = 0; sidx < 3; sidx++) {
    uint16_t *seg = own + sidx * KS::SEG;
    const uint2 *seg2 = reinterpret_cast<const uint2 *>(seg);
#pragma unroll 1
    for (int i = (int)P::WR - 1; i >= 0; i--) {
      const uint32_t pi = seg[i];
      const uint32_t pp = pi * 0x00010001u;
      const uint32_t g0 = (uint32_t)(i + 1) >> 2, nlo = (uint32_t)(i + 1) & 3u;  // entries g0*4 .. i are not later
      const uint32_t f0 = nlo >= 1 ? 1u : 0u, f1 = nlo >= 2 ? 1u : 0u, f2 = nlo >= 3 ? 1u : 0u;
      const uint32_t force_lo = f0 | (f1 << 16), force_hi = f2;
      uint32_t hit = 0;
      for (uint32_t g = g0; g < (P::WR + 3) / 4; g++) {
        const uint2 v = seg2[g];
        uint32_t xl = v.x ^ pp, xh = v.y ^ pp;
        if (g == g0) {
          xl |= force_lo;
          xh |= force_hi;
        }
        hit |= ((xl - 0x00010001u) & ~xl & 0x80008000u) | ((xh - 0x00010001u) & ~xh & 0x80008000u);
      }
      seg[i] = hit ? (uint16_t)i : (uint16_t)pi;
    }
  }
  __syncwarp();
  // transposed write-out: row ct of r1 / r2 / e, entries >= wr zero
  const uint32_t nl = batch - base < 32 ? (uint32_t)(batch - base) : 32u;
#pragma unroll 1
  for (uint32_t l = 0; l < nl; l++) {
    const size_t c = base + l;
    const uint16_t *src = pb + l * 3 * KS::SEG;
    for (uint32_t t = lane; t < 3 * P::E_STRIDE; t += 32) {
      const uint32_t sidx = t / P::E_STRIDE, idx = t - sidx * P::E_STRIDE;
      const uint32_t val = idx < P::WR ? src[sidx * KS::SEG + idx] : 0u;
      uint32_t *dst = sidx == 0 ? r1 : (sidx == 1 ? r2 : e);
      dst[c * P::E_STRIDE + idx] = val;
    }
  }
}

// ---- K = SHAKE256(select(eq, m, sigma) || u bytes || v bytes || 0x03, 64) (lane per ciphertext, R#23).
// eq == nullptr (Encaps): the first field is m. acc_out (nullable) receives eq.
template <class P>
__global__ void __launch_bounds__(128) k_kem_kdf(const uint8_t *__restrict__ m, const uint8_t *__restrict__ sigma,
                                                 const uint32_t *__restrict__ key_index,
                                                 const uint8_t *__restrict__ eq, const uint64_t *__restrict__ u,
                                                 const uint64_t *__restrict__ v, uint8_t *__restrict__ K_out,
                                                 uint8_t *__restrict__ acc_out, size_t batch) {
  using KS = KemShape<P>;
  const size_t ct = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ct >= batch) return;
  CatReader<KS::KW, KS::UB, KS::VB, 0x03> rd;
  const uint64_t *mp = reinterpret_cast<const uint64_t *>(m + ct * P::K);
  if (eq) {
    const size_t key = key_index ? key_index[ct] : ct;
    const uint64_t *sp = reinterpret_cast<const uint64_t *>(sigma + key * P::K);
    const uint8_t ok = eq[2 * ct] & eq[2 * ct + 1];  // both halves of c' matched (k_encrypt2 flags)
    const uint64_t sel = 0ull - (uint64_t)(ok & 1u);  // all ones when accepted
#pragma unroll
    for (uint32_t i = 0; i < KS::KW; i++) rd.f[i] = (mp[i] & sel) | (sp[i] & ~sel);
    if (acc_out) acc_out[ct] = ok;
  } else {
#pragma unroll
    for (uint32_t i = 0; i < KS::KW; i++) rd.f[i] = mp[i];
  }
  rd.a = u + ct * P::U_STRIDE;
  rd.b = v + ct * P::V_WORDS;
  uint64_t A[25];
  shake256_absorb<decltype(rd)::LEN>(A, rd);
  uint4 *o = reinterpret_cast<uint4 *>(K_out + ct * 64);
#pragma unroll
  for (int i = 0; i < 4; i++)
    o[i] = make_uint4((uint32_t)A[2 * i], (uint32_t)(A[2 * i] >> 32), (uint32_t)A[2 * i + 1],
                      (uint32_t)(A[2 * i + 1] >> 32));
}

// ---- KeyGen from a 32-byte seed (lane per key; R#24, Alg. 3):
//   (seed_sk || seed_pk) = SHAKE256(seed || PRNG, 64)
//   h = SHAKE256(seed_pk || PRNG, ceil(n/8)), bits >= n cleared          ("sample_dense")
//   SHAKE256(seed_sk || PRNG, 8w + k) -> x = sample(u32 words 0..w), y = sample(words w..2w),
//                                        sigma = bytes [8w, 8w + k)
// The product s = x + h*y is the keygen kernel's (k_keygen) and runs afterwards on the same stream.
// The sampler's duplicate scan runs in the lane's own output row (L1-resident; keys are few).
template <class P>
__global__ void __launch_bounds__(128) k_kem_keygen_seed(const uint8_t *__restrict__ seeds, uint64_t *__restrict__ h,
                                                         uint32_t *__restrict__ x, uint32_t *__restrict__ y,
                                                         uint8_t *__restrict__ sigma, size_t nkeys) {
  using KS = KemShape<P>;
  const size_t key = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (key >= nkeys) return;
  uint64_t A[25], sd[8];
  {
    CatReader<4, 0, 0, 0x04> rd;
    const uint64_t *sp = reinterpret_cast<const uint64_t *>(seeds + key * 32);
#pragma unroll
    for (int i = 0; i < 4; i++) rd.f[i] = sp[i];
    rd.a = rd.b = nullptr;
    shake256_absorb<decltype(rd)::LEN>(A, rd);
#pragma unroll
    for (int i = 0; i < 8; i++) sd[i] = A[i];
  }
  {  // h from seed_pk: ceil(n/8) bytes = words [0, U_WORDS), the last one masked to bit n
    CatReader<4, 0, 0, 0x04> rd;
#pragma unroll
    for (int i = 0; i < 4; i++) rd.f[i] = sd[4 + i];
    rd.a = rd.b = nullptr;
    shake256_absorb<decltype(rd)::LEN>(A, rd);
    uint64_t *hr = h + key * P::U_STRIDE;
    constexpr uint32_t NBLK = (P::U_WORDS + SHAKE256_RATE_W - 1) / SHAKE256_RATE_W;
    constexpr uint64_t LAST = (P::N % 64) ? (~0ull >> (64 - P::N % 64)) : ~0ull;
#pragma unroll 1
    for (uint32_t blk = 0; blk < NBLK; blk++) {
      if (blk) keccak_f1600(A);
#pragma unroll
      for (uint32_t i = 0; i < SHAKE256_RATE_W; i++) {
        const uint32_t t = blk * SHAKE256_RATE_W + i;
        if (t < P::U_WORDS) hr[t] = t == P::U_WORDS - 1 ? (A[i] & LAST) : A[i];
      }
    }
#pragma unroll
    for (uint32_t t = P::U_WORDS; t < P::U_STRIDE; t++) hr[t] = 0;
  }
  uint32_t *xr = x + key * P::Y_STRIDE, *yr = y + key * P::Y_STRIDE;
  {  // x, y positions (before deduplication) and sigma from seed_sk
    CatReader<4, 0, 0, 0x04> rd;
#pragma unroll
    for (int i = 0; i < 4; i++) rd.f[i] = sd[i];
    rd.a = rd.b = nullptr;
    shake256_absorb<decltype(rd)::LEN>(A, rd);
    constexpr uint32_t NW = P::W + KS::KW;  // 64-bit output words: 2w u32 sampler words, then sigma
    constexpr uint32_t NBLK = (NW + SHAKE256_RATE_W - 1) / SHAKE256_RATE_W;
    uint64_t *sg = reinterpret_cast<uint64_t *>(sigma + key * P::K);
#pragma unroll 1
    for (uint32_t blk = 0; blk < NBLK; blk++) {
      if (blk) keccak_f1600(A);
#pragma unroll
      for (uint32_t i = 0; i < SHAKE256_RATE_W; i++) {
        const uint32_t g = blk * SHAKE256_RATE_W + i;
        if (g < P::W) {
#pragma unroll
          for (uint32_t hf = 0; hf < 2; hf++) {
            const uint32_t t = 2 * g + hf, idx = t % P::W;
            const uint32_t rnd = (uint32_t)(A[i] >> (32 * hf));
            (t < P::W ? xr : yr)[idx] = idx + __umulhi(rnd, P::N - idx);
          }
        } else if (g < NW) {
          sg[g - P::W] = A[i];
        }
      }
    }
  }
#pragma unroll 1
  for (uint32_t which = 0; which < 2; which++) {  // R#22 deduplication, fixed w(w-1)/2 compares
    uint32_t *row = which ? yr : xr;
#pragma unroll 1
    for (int i = (int)P::W - 1; i >= 0; i--) {
      const uint32_t pi = row[i];
      uint32_t dup = 0;
#pragma unroll 4
      for (uint32_t j = i + 1; j < P::W; j++) dup |= (uint32_t)(row[j] == pi);
      row[i] = dup ? (uint32_t)i : pi;
    }
#pragma unroll
    for (uint32_t t = P::W; t < P::Y_STRIDE; t++) row[t] = 0;
  }
}

// rows dst[b] = src[key_index[b]] (16-byte chunks)
static __global__ void __launch_bounds__(256) k_gather_rows(const uint4 *__restrict__ src, const uint32_t *__restrict__ key_index,
                                                     uint4 *__restrict__ dst, uint32_t row_chunks, size_t batch) {
  const size_t total = batch * row_chunks;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / row_chunks, c = i - b * row_chunks;
    dst[i] = src[(size_t)key_index[b] * row_chunks + c];
  }
}

// ---- host side
constexpr int KEM_COIN_WARPS = 2;

template <class P> struct KemWs {  // decaps/encaps workspace carve-up (256-byte aligned regions)
  size_t y, m, r1, r2, e, eq, total;
  explicit KemWs(size_t batch) {
    auto r = [](size_t x) { return (x + 255) / 256 * 256; };
    y = 0;
    m = y + r(batch * P::Y_STRIDE * 4);
    r1 = m + r(batch * P::K);
    r2 = r1 + r(batch * P::E_STRIDE * 4);
    e = r2 + r(batch * P::E_STRIDE * 4);
    eq = e + r(batch * P::E_STRIDE * 4);
    total = eq + r(2 * batch);
  }
};

template <class P> static size_t kem_ws_bytes(size_t batch) { return KemWs<P>(batch).total; }

template <class P> static int launch_kem_hpk(const uint64_t *h, const uint64_t *s, uint8_t *hpk, size_t nkeys,
                                             cudaStream_t st) {
  k_kem_hpk<P><<<(unsigned)((nkeys + 127) / 128), 128, 0, st>>>(h, s, hpk, nkeys);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P>
static int launch_kem_coins(const uint8_t *hpk, const uint32_t *key, const uint8_t *m, uint32_t *r1, uint32_t *r2,
                            uint32_t *e, size_t batch, cudaStream_t st) {
  constexpr uint32_t smem = KEM_COIN_WARPS * KemShape<P>::PB_BYTES;
  if (cudaFuncSetAttribute(k_kem_coins<P, KEM_COIN_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess)
    return HQC_ERR_CUDA;
  const size_t per = 32 * KEM_COIN_WARPS;
  k_kem_coins<P, KEM_COIN_WARPS><<<(unsigned)((batch + per - 1) / per), 32 * KEM_COIN_WARPS, smem, st>>>(
      hpk, key, m, r1, r2, e, batch);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P>
static int launch_kem_keygen(const uint8_t *seeds, uint64_t *h, uint32_t *x, uint32_t *y, uint64_t *s, uint8_t *sigma,
                             uint8_t *hpk, size_t nkeys, cudaStream_t st) {
  k_kem_keygen_seed<P><<<(unsigned)((nkeys + 127) / 128), 128, 0, st>>>(seeds, h, x, y, sigma, nkeys);
  if (cudaGetLastError() != cudaSuccess) return HQC_ERR_CUDA;
  int rc = launch_keygen<P>(h, x, y, s, nkeys, st);
  if (rc || !hpk) return rc;
  return launch_kem_hpk<P>(h, s, hpk, nkeys, st);
}

template <class P>
static int launch_kem_encaps(const uint64_t *h, const uint64_t *s, const uint8_t *hpk, const uint32_t *key,
                             const uint8_t *m, uint64_t *u, uint64_t *v, uint8_t *K_out, size_t batch, void *ws,
                             cudaStream_t st) {
  const KemWs<P> W(batch);
  uint8_t *b = static_cast<uint8_t *>(ws);
  uint32_t *r1 = reinterpret_cast<uint32_t *>(b + W.r1), *r2 = reinterpret_cast<uint32_t *>(b + W.r2),
           *e = reinterpret_cast<uint32_t *>(b + W.e);
  int rc = launch_kem_coins<P>(hpk, key, m, r1, r2, e, batch, st);
  if (rc) return rc;
  rc = launch_encrypt_any<P, false>(h, s, key, m, r1, r2, e, u, v, batch, nullptr, nullptr, nullptr, st);
  if (rc) return rc;
  k_kem_kdf<P><<<(unsigned)((batch + 127) / 128), 128, 0, st>>>(m, nullptr, key, nullptr, u, v, K_out, nullptr, batch);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P>
static int launch_kem_decaps(const uint64_t *h, const uint64_t *s, const uint8_t *hpk, const uint8_t *sigma,
                             const uint32_t *key, const uint32_t *y, const uint64_t *u, const uint64_t *v,
                             uint8_t *K_out, uint8_t *acc_out, size_t batch, void *ws, cudaStream_t st) {
  const KemWs<P> W(batch);
  uint8_t *b = static_cast<uint8_t *>(ws);
  const uint32_t *yr = y;
  if (key) {  // the fused decrypt reads one support row per ciphertext
    uint32_t *yg = reinterpret_cast<uint32_t *>(b + W.y);
    const uint32_t chunks = P::Y_STRIDE / 4;
    size_t grid = (batch * chunks + 255) / 256;
    if (grid > 4096) grid = 4096;
    k_gather_rows<<<(unsigned)grid, 256, 0, st>>>(reinterpret_cast<const uint4 *>(y), key,
                                                  reinterpret_cast<uint4 *>(yg), chunks, batch);
    if (cudaGetLastError() != cudaSuccess) return HQC_ERR_CUDA;
    yr = yg;
  }
  uint8_t *mp = b + W.m;
  uint32_t *r1 = reinterpret_cast<uint32_t *>(b + W.r1), *r2 = reinterpret_cast<uint32_t *>(b + W.r2),
           *e = reinterpret_cast<uint32_t *>(b + W.e);
  uint8_t *eq = b + W.eq;
  int rc = launch_decrypt<P>(u, v, yr, mp, batch, st);
  if (rc) return rc;
  rc = launch_kem_coins<P>(hpk, key, mp, r1, r2, e, batch, st);
  if (rc) return rc;
  rc = launch_encrypt_any<P, true>(h, s, key, mp, r1, r2, e, nullptr, nullptr, batch, u, v, eq, st);
  if (rc) return rc;
  k_kem_kdf<P><<<(unsigned)((batch + 127) / 128), 128, 0, st>>>(mp, sigma, key, eq, u, v, K_out, acc_out, batch);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

}  // namespace hqc
