// Stage-1 inner-loop variants (HQC-3 shape, R = 35): per-warp latency tolerance vs resident warps.
//   v0: as in stage1.cuh (offset pair loaded at the top of each pass)
//   v1: the next pass's offsets prefetched one pass ahead (register double buffer)
//   v2: v1 + the first window word of the next pass loaded before this pass's tail
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbs1 scripts/microbench_s1.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int R = 35;
constexpr int EW = 2400;
constexpr int NIDX = 100;

template <int V>
__global__ void __launch_bounds__(32) k_s1(uint32_t *out, int iters, long long *clk) {
  __shared__ __align__(16) uint32_t E[EW + 64];
  __shared__ __align__(16) uint32_t dsm[NIDX + 4];
  const int lane = threadIdx.x;
  for (int i = lane; i < EW + 64; i += 32) E[i] = i * 2654435761u + blockIdx.x;
  for (int i = lane; i < NIDX + 4; i += 32) dsm[i] = (i * 7919u + blockIdx.x * 131u) % 35851u + 1;
  __syncwarp();
  long long t0 = clock64();
  uint32_t acc[R];
#pragma unroll
  for (int k = 0; k < R; k++) acc[k] = 0;
  const uint32_t *Eb = E + lane * R;
  for (int it = 0; it < iters; it++) {
    if (V == 0) {
#pragma unroll 2
      for (int j = 0; j < NIDX; j += 2) {
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
    } else {
      uint2 dd = *reinterpret_cast<const uint2 *>(dsm);
#pragma unroll 1
      for (int j = 0; j < NIDX; j += 2) {
        const uint2 dn = *reinterpret_cast<const uint2 *>(dsm + j + 2);  // next pass (padding row at the end)
        const uint32_t *p0 = Eb + (dd.x >> 5);
        const uint32_t *p1 = Eb + (dd.y >> 5);
        uint32_t a0 = p0[0], b0 = p1[0];
        if (V == 2) {
#pragma unroll
          for (int k = 0; k < R; k++) {
            const uint32_t a1 = p0[k + 1];
            acc[k] ^= __funnelshift_r(a0, a1, dd.x);
            a0 = a1;
          }
#pragma unroll
          for (int k = 0; k < R; k++) {
            const uint32_t b1 = p1[k + 1];
            acc[k] ^= __funnelshift_r(b0, b1, dd.y);
            b0 = b1;
          }
        } else {
#pragma unroll
          for (int k = 0; k < R; k++) {
            const uint32_t a1 = p0[k + 1], b1 = p1[k + 1];
            acc[k] ^= __funnelshift_r(a0, a1, dd.x) ^ __funnelshift_r(b0, b1, dd.y);
            a0 = a1;
            b0 = b1;
          }
        }
        dd = dn;
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < R; k++) x ^= acc[k];
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
  static long long hc[148 * 64];
  for (int v = 0; v < 3; v++) {
    for (int warps : {2, 4, 6, 8, 10, 12, 16}) {
      const int grid = sms * warps;
      const int iters = 60;
      float ms = 0;
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        if (v == 0) k_s1<0><<<grid, 32>>>(out, iters, clk);
        else if (v == 1) k_s1<1><<<grid, 32>>>(out, iters, clk);
        else k_s1<2><<<grid, 32>>>(out, iters, clk);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
      }
      CK(cudaGetLastError());
      CK(cudaMemcpy(hc, clk, grid * 8, cudaMemcpyDeviceToHost));
      double mx = 0;
      for (int i = 0; i < grid; i++) mx = hc[i] > mx ? hc[i] : mx;
      const double clk_hz = mx / (ms * 1e-3);
      const double pairs = (double)grid * iters * NIDX * R * 32;
      printf("v%d warps/SM %2d: %.2f pairs/clk/SM (bound %.1f)  %.3f ms  (%.0f MHz est)\n", v, warps,
             pairs / sms / (ms * 1e-3) / clk_hz, 32.0 * 35.0 / 36.0, ms, clk_hz / 1e6);
    }
  }
  return 0;
}
