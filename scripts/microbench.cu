// K7: measured ceilings on this B200 for the operations the decrypt path is made of.
//   lds   : conflict-free LDS.32 with the stage-1 address pattern (lane L reads base + L*R + k, R odd)
//   alu   : SHF.R.W + LOP3 (3-input XOR) throughput, many independent chains
//   s1    : the stage-1 inner loop itself (R words per lane, 2 indices per pass) on a synthetic E
// Each kernel runs with `warps` warps per SM (1-warp CTAs, grid = 148 * warps) for a fixed amount of
// work per warp; we report per-SM rates using the CUDA-event time and the SM clock from clock64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int R = 35;
constexpr int EW = 2400;

__global__ void k_lds(uint32_t *out, int iters, long long *clk) {
  __shared__ uint32_t E[EW + 64];
  const int lane = threadIdx.x;
  for (int i = lane; i < EW + 64; i += 32) E[i] = i * 2654435761u;
  __syncwarp();
  long long t0 = clock64();
  uint32_t acc[8] = {0};
  uint32_t o = (blockIdx.x * 97u) % 1100u;
  const uint32_t *p = E + lane * R;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < 32; k++) acc[k & 7] ^= p[o + k];
    o = (o + 37u) % 1100u;
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) x ^= acc[k];
  out[blockIdx.x * 32 + lane] = x;
  if (lane == 0) clk[blockIdx.x] = clock64() - t0;
}

__global__ void k_alu(uint32_t *out, int iters, long long *clk, uint32_t s) {
  const int lane = threadIdx.x;
  uint32_t a[16];
#pragma unroll
  for (int k = 0; k < 16; k++) a[k] = lane * 7919u + k;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      a[k] = __funnelshift_r(a[k], a[(k + 1) & 15], s + k);
      a[k] ^= a[(k + 3) & 15] ^ a[(k + 5) & 15];
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < 16; k++) x ^= a[k];
  out[blockIdx.x * 32 + lane] = x;
  if (lane == 0) clk[blockIdx.x] = clock64() - t0;
}

__global__ void k_s1(uint32_t *out, int iters, long long *clk) {
  __shared__ __align__(16) uint32_t E[EW + 64];
  __shared__ uint32_t dsm[128];
  const int lane = threadIdx.x;
  for (int i = lane; i < EW + 64; i += 32) E[i] = i * 2654435761u + blockIdx.x;
  for (int i = lane; i < 128; i += 32) dsm[i] = (i * 7919u + blockIdx.x * 131u) % 35851u + 1;
  __syncwarp();
  long long t0 = clock64();
  uint32_t acc[R];
#pragma unroll
  for (int k = 0; k < R; k++) acc[k] = 0;
  const uint32_t *Eb = E + lane * R;
  for (int it = 0; it < iters; it++) {
#pragma unroll 1
    for (int j = 0; j < 100; j += 2) {
      const uint2 dd = *reinterpret_cast<const uint2 *>(dsm + j);
      const uint32_t *p0 = Eb + (dd.x >> 5);
      const uint32_t *p1 = Eb + (dd.y >> 5);
      uint32_t a0 = p0[0], b0 = p1[0];
#pragma unroll
      for (int k = 0; k < R; k++) {
        const uint32_t a1 = p0[k + 1], b1 = p1[k + 1];
        acc[k] ^= __funnelshift_r(a0, a1, dd.x) ^ __funnelshift_r(b0, b1, dd.y);
        a0 = a1;
        b0 = b1;
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < R; k++) x ^= acc[k];
  out[blockIdx.x * 32 + lane] = x;
  if (lane == 0) clk[blockIdx.x] = clock64() - t0;
}

// stage-1 loop where a fraction of the words use the FMA pipe: funnel(lo, hi, s) = hi*m + umulhi(lo, m),
// m = 2^(32-s), s in [1, 32] (word offset adjusted by one when the bit offset is 0)
template <int MODE>
__global__ void k_s1mix(uint32_t *out, int iters, long long *clk) {
  __shared__ __align__(16) uint32_t E[EW + 64];
  __shared__ uint32_t dsm[128];
  const int lane = threadIdx.x;
  for (int i = lane; i < EW + 64; i += 32) E[i] = i * 2654435761u + blockIdx.x;
  for (int i = lane; i < 128; i += 32) dsm[i] = (i * 7919u + blockIdx.x * 131u) % 35851u + 1;
  __syncwarp();
  long long t0 = clock64();
  uint32_t acc[R];
#pragma unroll
  for (int k = 0; k < R; k++) acc[k] = 0;
  const uint32_t *Eb = E + lane * R;
  for (int it = 0; it < iters; it++) {
#pragma unroll 1
    for (int j = 0; j < 100; j += 2) {
      const uint2 dd = *reinterpret_cast<const uint2 *>(dsm + j);
      const uint32_t s0 = ((dd.x - 1) & 31) + 1, s1 = ((dd.y - 1) & 31) + 1;
      const uint32_t m0 = 1u << (32 - s0), m1 = 1u << (32 - s1);
      const uint32_t *p0 = Eb + ((dd.x - s0) >> 5);
      const uint32_t *p1 = Eb + ((dd.y - s1) >> 5);
      uint32_t a0 = p0[0], b0 = p1[0];
#pragma unroll
      for (int k = 0; k < R; k++) {
        const uint32_t a1 = p0[k + 1], b1 = p1[k + 1];
        const bool fma = MODE == 1 ? (k % 2 == 1) : MODE == 2 ? (k % 8 < 3) : false;
        if (fma) {
          const uint32_t fa = a1 * m0 + __umulhi(a0, m0);
          const uint32_t fb = b1 * m1 + __umulhi(b0, m1);
          acc[k] ^= fa ^ fb;
        } else {
          acc[k] ^= __funnelshift_r(a0, a1, s0) ^ __funnelshift_r(b0, b1, s1);
        }
        a0 = a1;
        b0 = b1;
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < R; k++) x ^= acc[k];
  out[blockIdx.x * 32 + lane] = x;
  if (lane == 0) clk[blockIdx.x] = clock64() - t0;
}

__global__ void k_imadhi(uint32_t *out, int iters, long long *clk, uint32_t m) {
  const int lane = threadIdx.x;
  uint32_t a[16];
#pragma unroll
  for (int k = 0; k < 16; k++) a[k] = lane * 7919u + k;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < 16; k++) a[k] = __umulhi(a[k], m + k) + a[(k + 1) & 15];
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < 16; k++) x ^= a[k];
  out[blockIdx.x * 32 + lane] = x;
  if (lane == 0) clk[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint32_t *out;
  long long *clk;
  CK(cudaMalloc(&out, 148 * 64 * 32 * 4));
  CK(cudaMalloc(&clk, 148 * 64 * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  long long hc[148 * 64];
  for (int kind = 0; kind < 7; kind++) {
    for (int warps : {8, 12, 16}) {
      const int grid = sms * warps;
      const int iters = kind == 0 ? 4000 : (kind == 1 || kind == 3) ? 20000 : 40;
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        if (kind == 0) k_lds<<<grid, 32>>>(out, iters, clk);
        else if (kind == 1) k_alu<<<grid, 32>>>(out, iters, clk, 3);
        else if (kind == 2) k_s1<<<grid, 32>>>(out, iters, clk);
        else if (kind == 3) k_imadhi<<<grid, 32>>>(out, iters, clk, 0x9E3779B9u);
        else if (kind == 4) k_s1mix<0><<<grid, 32>>>(out, iters, clk);
        else if (kind == 5) k_s1mix<1><<<grid, 32>>>(out, iters, clk);
        else k_s1mix<2><<<grid, 32>>>(out, iters, clk);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
      }
      CK(cudaGetLastError());
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(hc, clk, grid * 8, cudaMemcpyDeviceToHost));
      double mx = 0;
      for (int i = 0; i < grid; i++) mx = hc[i] > mx ? hc[i] : mx;
      const double clk_hz = mx / (ms * 1e-3);
      if (kind == 0) {
        const double lds = (double)grid * iters * 32;  // warp-level LDS instructions
        printf("lds  warps/SM %2d: %.3f LDS.32 warp-instr/clk/SM  (%.0f MHz)\n", warps, lds / sms / (ms * 1e-3) / clk_hz, clk_hz / 1e6);
      } else if (kind == 1) {
        const double ops = (double)grid * iters * 16 * 2 * 32;  // SHF + LOP3 lane-ops
        printf("alu  warps/SM %2d: %.1f lane-ops/clk/SM (SHF+LOP3)  (%.0f MHz)\n", warps, ops / sms / (ms * 1e-3) / clk_hz, clk_hz / 1e6);
      } else if (kind == 3) {
        const double ops = (double)grid * iters * 16 * 32;
        printf("imadhi warps/SM %2d: %.1f lane-ops/clk/SM (IMAD.HI + dependent add)  (%.0f MHz)\n", warps, ops / sms / (ms * 1e-3) / clk_hz, clk_hz / 1e6);
      } else {
        const double pairs = (double)grid * iters * 100 * R * 32;  // (index, word) pairs
        printf("s1[kind %d] warps/SM %2d: %.2f pairs/clk/SM  (LDS wavefront bound 32/1.029=%.1f)  (%.0f MHz)\n", warps,
               kind, pairs / sms / (ms * 1e-3) / clk_hz, 32.0 / (36.0 / 35.0), clk_hz / 1e6);
      }
    }
  }
  return 0;
}
