// GF(2^8) log/antilog tables for the RS stage (R#4: field polynomial x^8+x^4+x^3+x^2+1 = 0x11D,
// alpha = 0x02). Generated at compile time, copied to shared memory once per CTA.
//   EXPT[e] = alpha^(e mod 255) for e < 510, and 0 for 510 <= e < 1024;
//   LOGT[x] = log_alpha(x) for x != 0, and LOGT[0] = GF_LOG0 = 511.
// With the sentinel, a product of logs la + lb (each < 255, or 511 for a zero factor) indexes EXPT
// directly: EXPT[la + lb] = a*b including the zero cases, with no branch and no mask.
#pragma once
#include <cstdint>

namespace hqc {

constexpr uint32_t GF_LOG0 = 511;
constexpr uint32_t GF_EXP_SIZE = 1024;

struct GfTables {
  uint8_t exp[GF_EXP_SIZE];
  uint16_t log[256];
};

constexpr GfTables make_gf_tables() {
  GfTables t{};
  uint32_t x = 1;
  for (uint32_t e = 0; e < 255; e++) {
    t.exp[e] = static_cast<uint8_t>(x);
    t.exp[e + 255] = static_cast<uint8_t>(x);
    t.log[x] = static_cast<uint16_t>(e);
    x <<= 1;                    // multiply by alpha = x
    if (x & 0x100) x ^= 0x11D;  // reduce
  }
  for (uint32_t e = 510; e < GF_EXP_SIZE; e++) t.exp[e] = 0;
  t.log[0] = GF_LOG0;
  return t;
}

// in global memory, not the constant bank: every thread of the copy below reads a different word, which
// the constant cache would serialise (a ~3.7k-cycle prologue per CTA; profiles/r02/sb_phases.log)
__device__ __align__(16) const GfTables g_gf = make_gf_tables();
static_assert(sizeof(GfTables) % 16 == 0, "copied in 16-byte pieces");

// compile-time GF(2^8) arithmetic for building the constant tables below and in encrypt.cuh
constexpr uint32_t gf_mul_c(uint32_t a, uint32_t b) {  // carry-less product mod 0x11D
  uint32_t r = 0;
  for (int i = 0; i < 8; i++)
    if ((b >> i) & 1) r ^= a << i;
  for (int d = 14; d >= 8; d--)
    if ((r >> d) & 1) r ^= 0x11Du << (d - 8);
  return r;
}
constexpr uint32_t gf_exp_c(uint32_t e) {  // alpha^e, alpha = 0x02
  uint32_t r = 1;
  for (uint32_t i = 0; i < e % 255; i++) r = gf_mul_c(r, 2);
  return r;
}

// Copy the tables into a CTA's shared memory (all threads of the CTA participate).
__device__ __forceinline__ void gf_tables_to_smem(GfTables *dst) {
  const uint4 *src = reinterpret_cast<const uint4 *>(&g_gf);
  uint4 *d = reinterpret_cast<uint4 *>(dst);
  for (uint32_t i = threadIdx.x; i < sizeof(GfTables) / 16; i += blockDim.x) d[i] = __ldg(src + i);
}

}  // namespace hqc
