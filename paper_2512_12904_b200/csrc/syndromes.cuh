// SURVEY §8(a) row a6 on its own, in three ways: the RS syndromes
//   S_i = sum_{j < n1} sym_j alpha^{i j},  i = 1..2delta     (R#5: byte j <-> X^j, 0x11D, alpha = 0x02)
// of a batch of received words, one lane per word (a warp holds 32 words, symbols staged [j][lane]).
//   SYN_LINEAR (0): the GF(2)-linear map of the fused kernel (stage3.cuh, RsLinear): for every set bit b
//       of sym_j XOR the packed vector alpha^{(i+1)j} 2^b; tables in the constant bank, uniform LDCU
//       loads, ALU-only arithmetic (8 * ceil(2delta/4) LOP3 per symbol).
//   SYN_NIBBLE (1): the paper's nibble-sliced tables ("two nibble-sliced lookup tables ... the
//       contributions of alpha^{i(j-1)} for all high and low nibbles ... each byte multiplication resolved
//       through a pair of XOR lookups (hi XOR lo)"), widened to 4 syndromes per 32-bit entry:
//       T[q][j][h][x] = pack_{t<4} alpha^{(4q+t+1) j} * (h ? x << 4 : x). Tables in shared memory, x
//       fastest (16 consecutive words: the 32 lanes' lookups of one (q, j, h) hit 16 distinct banks).
//   SYN_LOGEXP (2): log/antilog tables in shared memory: S_i ^= EXP[LOG[sym_j] + (i j mod 255)] with the
//       LOG(0) sentinel of gf256.cuh; one byte lookup per (i, j), the exponent offset an immediate.
// All three give the same bytes (GF arithmetic is exact); tests/test_gpu_parity.py checks each
// against oracle/rs.c: orc_rs_syndromes.
#pragma once
#include <cstdint>

#include "gf256.cuh"
#include "levels.cuh"
#include "stage3.cuh"

namespace hqc {

enum { SYN_LINEAR = 0, SYN_NIBBLE = 1, SYN_LOGEXP = 2 };

template <class P> struct NibbleSyn {
  static constexpr uint32_t SW = (P::TWO_DELTA + 3) / 4;  // packed syndrome words
  static constexpr uint32_t WORDS = SW * P::N1 * 2 * 16;
  static constexpr uint32_t BYTES = WORDS * 4;
  struct Tables {
    uint32_t t[SW][P::N1][2][16];
  };
  static constexpr Tables make() {
    Tables T{};
    uint32_t ex[255] = {};
    uint32_t e = 1;
    for (uint32_t k = 0; k < 255; k++) {
      ex[k] = e;
      e = gf_mul_c(e, 2);
    }
    for (uint32_t q = 0; q < SW; q++)
      for (uint32_t j = 0; j < P::N1; j++)
        for (uint32_t t = 0; t < 4; t++) {
          const uint32_t i = 4 * q + t;  // syndrome S_{i+1}
          if (i >= P::TWO_DELTA) continue;
          uint32_t cb[8] = {};  // alpha^{(i+1) j} * 2^b
          cb[0] = ex[((i + 1) * j) % 255];
          for (int b = 1; b < 8; b++) cb[b] = (cb[b - 1] << 1) ^ ((cb[b - 1] & 0x80u) ? 0x11Du : 0u);
          for (uint32_t x = 0; x < 16; x++) {
            uint32_t lo = 0, hi = 0;
            for (int b = 0; b < 4; b++)
              if ((x >> b) & 1) {
                lo ^= cb[b];
                hi ^= cb[b + 4];
              }
            T.t[q][j][0][x] |= lo << (8 * t);
            T.t[q][j][1][x] |= hi << (8 * t);
          }
        }
    return T;
  }
};

#ifdef HQC_THIS_LEVEL
__device__ const NibbleSyn<Lv<HQC_THIS_LEVEL>>::Tables g_nib_syn = NibbleSyn<Lv<HQC_THIS_LEVEL>>::make();
#endif

template <class P> constexpr uint32_t syn_smem_bytes(int method) {
  return method == SYN_NIBBLE ? NibbleSyn<P>::BYTES : (method == SYN_LOGEXP ? (uint32_t)sizeof(GfTables) : 0u);
}

// One lane's syndromes, packed 4 per word (byte t of Sw[q] = S_{4q+t+1}).
template <class P, int METHOD, class SymAt>
__device__ __forceinline__ void syndromes_lane(SymAt sym_at, const uint8_t *tab, uint32_t (&Sw)[(P::TWO_DELTA + 3) / 4]) {
  constexpr uint32_t SW = (P::TWO_DELTA + 3) / 4;
#pragma unroll
  for (uint32_t q = 0; q < SW; q++) Sw[q] = 0;
  if constexpr (METHOD == SYN_LINEAR) {
#pragma unroll 1
    for (uint32_t j = 0; j < P::N1; j++) {
      const uint32_t x = sym_at(j);
#pragma unroll
      for (int b = 0; b < 8; b++) {
        const uint32_t m = 0u - ((x >> b) & 1u);
#pragma unroll
        for (uint32_t q = 0; q < SW; q++) Sw[q] ^= c_rs_lin.syn[j][b][q] & m;
      }
    }
  } else if constexpr (METHOD == SYN_NIBBLE) {
    const uint32_t *T = reinterpret_cast<const uint32_t *>(tab);
#pragma unroll 2
    for (uint32_t j = 0; j < P::N1; j++) {
      const uint32_t x = sym_at(j);
      const uint32_t *lo = T + j * 32 + (x & 15u);
      const uint32_t *hi = T + j * 32 + 16 + (x >> 4);
#pragma unroll
      for (uint32_t q = 0; q < SW; q++) Sw[q] ^= lo[q * P::N1 * 32] ^ hi[q * P::N1 * 32];
    }
  } else {
    const GfTables *gf = reinterpret_cast<const GfTables *>(tab);
#pragma unroll
    for (uint32_t j = 0; j < P::N1; j++) {
      const uint8_t *e = gf->exp + gf->log[sym_at(j)];
#pragma unroll
      for (uint32_t i = 0; i < P::TWO_DELTA; i++) Sw[i / 4] ^= (uint32_t)e[((i + 1) * j) % 255] << (8 * (i % 4));
    }
  }
}

// Stage a6 alone: syn_out[b][i-1] = S_i of received word sym[b], i = 1..2delta. Persistent grid,
// warp per 32 words; the CTA first stages the method's tables into shared memory.
template <class P, int METHOD>
__global__ void __launch_bounds__(128) k_syndromes(const uint8_t *__restrict__ sym, uint8_t *__restrict__ syn_out,
                                                   size_t batch) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr uint32_t TB = round_up(syn_smem_bytes<P>(METHOD), 16);
  if constexpr (METHOD == SYN_NIBBLE) {
    const uint4 *src = reinterpret_cast<const uint4 *>(&g_nib_syn);
    uint4 *d = reinterpret_cast<uint4 *>(smem);
    for (uint32_t i = threadIdx.x; i < NibbleSyn<P>::BYTES / 16; i += blockDim.x) d[i] = src[i];
  } else if constexpr (METHOD == SYN_LOGEXP) {
    gf_tables_to_smem(reinterpret_cast<GfTables *>(smem));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t *sb = smem + TB + (size_t)wib * round_up(P::N1 * 32, 16);
  const size_t nwarps = (size_t)gridDim.x * (blockDim.x >> 5);
  constexpr uint32_t SW = (P::TWO_DELTA + 3) / 4;
  for (size_t base = ((size_t)blockIdx.x * (blockDim.x >> 5) + wib) * 32; base < batch; base += nwarps * 32) {
    const size_t rows = batch - base < 32 ? batch - base : 32;
    for (uint32_t e = lane; e < 32 * P::N1; e += 32) {  // e = row*N1 + j (coalesced read)
      const uint32_t row = e / P::N1, j = e % P::N1;
      sb[j * 32 + row] = row < rows ? sym[(base + row) * P::N1 + j] : 0;
    }
    __syncwarp();
    auto sym_at = [&](uint32_t j) -> uint32_t { return sb[j * 32 + lane]; };
    uint32_t Sw[SW];
    syndromes_lane<P, METHOD>(sym_at, smem, Sw);
    if ((size_t)lane < rows) {
      uint8_t *o = syn_out + (base + lane) * P::TWO_DELTA;
#pragma unroll
      for (uint32_t i = 0; i < P::TWO_DELTA; i++) o[i] = (uint8_t)(Sw[i / 4] >> (8 * (i % 4)));
    }
    __syncwarp();
  }
}

template <class P, int METHOD> static int launch_syndromes_m(const uint8_t *sym, uint8_t *syn, size_t batch,
                                                             cudaStream_t st) {
  constexpr uint32_t smem = round_up(syn_smem_bytes<P>(METHOD), 16) + 4 * round_up(P::N1 * 32, 16);
  if (cudaFuncSetAttribute(k_syndromes<P, METHOD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return HQC_ERR_CUDA;
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_syndromes<P, METHOD>, 128, smem) != cudaSuccess ||
      per_sm < 1)
    return HQC_ERR_CUDA;
  size_t grid = (batch + 127) / 128;
  const size_t cap = (size_t)sms * per_sm;
  if (grid > cap) grid = cap;
  k_syndromes<P, METHOD><<<(unsigned)grid, 128, smem, st>>>(sym, syn, batch);
  return cudaGetLastError() == cudaSuccess ? HQC_OK : HQC_ERR_CUDA;
}

template <class P> static int launch_syndromes(const uint8_t *sym, uint8_t *syn, size_t batch, int method,
                                               cudaStream_t st) {
  switch (method) {
    case SYN_LINEAR: return launch_syndromes_m<P, SYN_LINEAR>(sym, syn, batch, st);
    case SYN_NIBBLE: return launch_syndromes_m<P, SYN_NIBBLE>(sym, syn, batch, st);
    case SYN_LOGEXP: return launch_syndromes_m<P, SYN_LOGEXP>(sym, syn, batch, st);
    default: return HQC_ERR_SIZE;
  }
}

}  // namespace hqc
