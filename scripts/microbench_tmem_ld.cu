// Load bandwidth of tensor memory against shared memory, per SM (question for the stage-1 product:
// could a skewed copy of E in TMEM, read with tcgen05.ld at a warp-uniform column, add load bandwidth
// to the shared-memory-bound funnel-shift loop? profiles/r01b/NOTES.md item 18).
//   mode 0: every warp reads TMEM (tcgen05.ld.sync.aligned.32x32b.x{W}, warp w -> lane quarter w%4)
//   mode 1: every warp reads shared memory (W LDS.32 per lane, conflict-free, lane-consecutive)
//   mode 2: even warps TMEM, odd warps shared memory (do the two paths add up?)
// Consumption: the loaded words are folded into W/2 accumulators with 3-input XORs (LOP3), so the
// ALU work per word is half an instruction.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mbtm scripts/microbench_tmem_ld.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int W> struct Ld;
template <> struct Ld<32> {
  static __device__ __forceinline__ void tm(uint32_t (&r)[32], uint32_t ta) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(ta));
  }
};

template <int MODE, int NWARPS, int COLS>
__global__ void __launch_bounds__(NWARPS * 32, 1) k_bw(uint32_t *out, int iters) {
  __shared__ __align__(16) uint32_t sm[10 * 1024];  // 40 KB
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 10 * 1024; i += blockDim.x) sm[i] = i * 2654435761u;
  if (MODE != 1 && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = MODE != 1 ? tmem_base : 0;
  const uint32_t ta0 = tb + ((uint32_t)((warp & 3) * 32) << 16);
  if (MODE != 1) {  // fill this warp's lane quarter (values are irrelevant, keep them defined)
    for (int c = 0; c < COLS; c++)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta0 + c), "r"(c * 977u + lane));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  __syncthreads();
  const bool use_tm = MODE == 0 || (MODE == 2 && (warp & 1) == 0);
  uint32_t acc[16];
#pragma unroll
  for (int k = 0; k < 16; k++) acc[k] = 0;
  uint32_t col = (uint32_t)warp * 7u;
  if (use_tm) {
#pragma unroll 1
    for (int it = 0; it < iters; it++) {
      uint32_t r[32];
      Ld<32>::tm(r, ta0 + col);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 16; k++) acc[k] ^= r[k] ^ r[k + 16];
      col += 37u;
      if (col >= COLS - 32) col -= COLS - 32;
    }
  } else {
    const uint32_t *b = sm + lane;  // word lane + 32*k: 32 banks, one wavefront per LDS
#pragma unroll 1
    for (int it = 0; it < iters; it++) {
      const uint32_t *p = b + (col & 255u) * 32;
      uint32_t r[32];
#pragma unroll
      for (int k = 0; k < 32; k++) r[k] = p[k * 32];
#pragma unroll
      for (int k = 0; k < 16; k++) acc[k] ^= r[k] ^ r[k + 16];
      col += 37u;
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < 16; k++) x ^= acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (MODE != 1 && warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(COLS));
}

template <int MODE, int NWARPS, int COLS> void run(int sms, uint32_t *out, int clk_khz) {
  const int iters = 20000;
  auto k = k_bw<MODE, NWARPS, COLS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NWARPS * 32, 0);
  const int grid = sms;  // one CTA per SM (launch bounds min 1; occupancy printed below is not used)
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<grid, NWARPS * 32>>>(out, 100);
  cudaEventRecord(a);
  k<<<grid, NWARPS * 32>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)grid * NWARPS * iters * 32 * 32 * 4;
  const double per_clk = bytes / (ms * 1e-3) / sms / (clk_khz * 1e3);
  printf("mode %d (%s) warps/CTA %2d cols %3d: %.3f ms  %.1f B/clk/SM  (%s)\n", MODE,
         MODE == 0 ? "tmem" : MODE == 1 ? "smem" : "half+half", NWARPS, COLS, ms, per_clk,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  uint32_t *out;
  cudaMalloc(&out, 148 * 1024 * 4 * 4);
  printf("SMs %d, clock %d kHz (B/clk/SM computed at this clock)\n", sms, clk);
  run<1, 4, 512>(sms, out, clk);
  run<1, 8, 512>(sms, out, clk);
  run<1, 16, 512>(sms, out, clk);
  run<0, 4, 512>(sms, out, clk);
  run<0, 8, 512>(sms, out, clk);
  run<0, 16, 512>(sms, out, clk);
  run<2, 8, 512>(sms, out, clk);
  run<2, 16, 512>(sms, out, clk);
  cudaFree(out);
  return 0;
}
