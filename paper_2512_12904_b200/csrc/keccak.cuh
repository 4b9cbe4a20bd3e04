// SHAKE256 (FIPS 202) on the GPU, one thread per message: the paper's "multi-buffer parallelism"
// for the hash calls of the KEM (§III.C) taken to its B200 form, 32 independent sponges
// per warp. The 1600-bit state is 25 64-bit lanes in registers; the round
// body is fully unrolled so the rho/pi permutation and every rotation amount are compile-time
// constants and chi becomes one 3-input LOP3 per 32-bit half. Parity: tests/test_gpu_kem.py
// (against hashlib and the oracle).
#pragma once
#include <cstdint>

namespace hqc {

// 64-bit rotation as two 32-bit funnel shifts of the register halves (r is a compile-time constant in
// every use, so the branches fold). Written as (x << r) | (x >> (64 - r)), nvcc emitted up to four shifts
// plus an OR for many of the rotation amounts.
__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) {
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  uint32_t nl, nh;
  if (r == 0) return x;
  if (r < 32) {
    nh = __funnelshift_l(lo, hi, r);
    nl = __funnelshift_l(hi, lo, r);
  } else if (r == 32) {
    nh = lo;
    nl = hi;
  } else {
    nh = __funnelshift_l(hi, lo, r - 32);
    nl = __funnelshift_l(lo, hi, r - 32);
  }
  return ((uint64_t)nh << 32) | nl;
}

__constant__ uint64_t c_keccak_rc[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808Aull, 0x8000000080008000ull,
    0x000000000000808Bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull,
    0x000000000000008Aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000Aull,
    0x000000008000808Bull, 0x800000000000008Bull, 0x8000000000008089ull, 0x8000000000008003ull,
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800Aull, 0x800000008000000Aull,
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};

// Keccak-f[1600]: 24 rounds of theta, rho, pi, chi, iota on lanes A[x + 5y].
#ifndef HQC_KECCAK_UNROLL  // round-loop unroll; measured (scripts/time_kem_lib.py): 2 and 4 are 1-2% slower,
#define HQC_KECCAK_UNROLL 1  // 24 (straight line) 15-17% slower (instruction-cache misses)
#endif
constexpr int kKeccakUnroll = HQC_KECCAK_UNROLL;
__device__ __forceinline__ void keccak_f1600(uint64_t (&A)[25]) {
  constexpr int RHO[25] = {0, 1, 62, 28, 27, 36, 44, 6, 55, 20, 3, 10, 43, 25, 39, 41, 45, 15, 21, 8, 18, 2, 61, 56, 14};
#pragma unroll kKeccakUnroll
  for (int round = 0; round < 24; round++) {
    uint64_t C[5], D[5], B[25];
#pragma unroll
    for (int x = 0; x < 5; x++) C[x] = A[x] ^ A[x + 5] ^ A[x + 10] ^ A[x + 15] ^ A[x + 20];
#pragma unroll
    for (int x = 0; x < 5; x++) D[x] = C[(x + 4) % 5] ^ rotl64(C[(x + 1) % 5], 1);
    // rho then pi: lane (x, y) moves to (y, 2x + 3y)
#pragma unroll
    for (int x = 0; x < 5; x++)
#pragma unroll
      for (int y = 0; y < 5; y++) B[y + 5 * ((2 * x + 3 * y) % 5)] = rotl64(A[x + 5 * y] ^ D[x], RHO[x + 5 * y]);
#pragma unroll
    for (int x = 0; x < 5; x++)
#pragma unroll
      for (int y = 0; y < 5; y++) A[x + 5 * y] = B[x + 5 * y] ^ (~B[(x + 1) % 5 + 5 * y] & B[(x + 2) % 5 + 5 * y]);
    A[0] ^= c_keccak_rc[round];
  }
}

constexpr uint32_t SHAKE256_RATE_W = 17;  // 136-byte rate = 17 lanes

#ifndef HQC_SHAKE_PREFETCH  // 1: load the next absorb block during the current permutation (KEM -1.5%)
#define HQC_SHAKE_PREFETCH 1
#endif

// Absorb a LEN-byte message into a fresh SHAKE256 state and apply the final permutation; A[0..17)
// then holds the first 136 output bytes (call keccak_f1600 for each further block). mw(i) returns
// message bytes [8i, 8i + 8) as a little-endian word and is called once per word, in increasing i
// (bytes past LEN may be anything: they are masked). SHAKE padding: 0x1F after the message, 0x80
// in the last byte of the rate (FIPS 202 pad10*1 with the 1111 XOF suffix).
template <uint32_t LEN, class MsgWord>
__device__ __forceinline__ void shake256_absorb(uint64_t (&A)[25], MsgWord &mw) {
  constexpr uint32_t NB = LEN / 136 + 1;  // the last block holds the padding
  constexpr uint32_t LASTW = LEN / 8, NBYTE = LEN % 8;
#pragma unroll
  for (int i = 0; i < 25; i++) A[i] = 0;
  auto word = [&](uint32_t b, uint32_t i) -> uint64_t {  // rate word i of padded block b
    const uint32_t wi = b * SHAKE256_RATE_W + i;
    uint64_t x = 0;
    if (wi < LASTW) {
      x = mw(wi);
    } else if (wi == LASTW) {
      if constexpr (NBYTE != 0) x = mw(wi) & ((1ull << (8 * NBYTE)) - 1ull);
      x |= 0x1Full << (8 * NBYTE);
    }
    if (i == SHAKE256_RATE_W - 1 && b == NB - 1) x ^= 0x80ull << 56;
    return x;
  };
  if constexpr (NB == 1) {
#pragma unroll
    for (uint32_t i = 0; i < SHAKE256_RATE_W; i++) A[i] ^= word(0, i);
    keccak_f1600(A);
  } else {
#if HQC_SHAKE_PREFETCH == 1
    // the next block's message words are loaded before the current permutation, so their (global
    // memory) latency overlaps the 24 rounds instead of stalling the absorb
    uint64_t nxt[SHAKE256_RATE_W];
#pragma unroll
    for (uint32_t i = 0; i < SHAKE256_RATE_W; i++) nxt[i] = word(0, i);
#pragma unroll 1
    for (uint32_t b = 0; b < NB; b++) {
#pragma unroll
      for (uint32_t i = 0; i < SHAKE256_RATE_W; i++) A[i] ^= nxt[i];
      if (b + 1 < NB) {
#pragma unroll
        for (uint32_t i = 0; i < SHAKE256_RATE_W; i++) nxt[i] = word(b + 1, i);
      }
      keccak_f1600(A);
    }
#else
#pragma unroll 1
    for (uint32_t b = 0; b < NB; b++) {
#pragma unroll
      for (uint32_t i = 0; i < SHAKE256_RATE_W; i++) A[i] ^= word(b, i);
      keccak_f1600(A);
    }
#endif
  }
}

}  // namespace hqc
