// Why does the in-kernel stage-1 loop run below the pure loop? Variants of the HQC-3 product loop
// (R = 35, 100 indices = one ciphertext per "iteration"):
//   a: pure loop, compiler's register choice                      (as microbench_s1 v0)
//   b: pure loop, capped at 64 registers (k_stage1's allocation)
//   c: a + per-ciphertext E rebuild from a staging row (funnel shifts) + syncwarp, as k_stage1
//   d: c capped at 64 registers
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mbs1b scripts/microbench_s1b.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int R = 35;
constexpr int Q0 = 1120, C = 11;
constexpr int EW = 2244;
constexpr int NIDX = 100;

template <bool REBUILD>
__device__ __forceinline__ void body(uint32_t *out, int iters, long long *clk) {
  __shared__ __align__(16) uint32_t E[EW + 64];
  __shared__ __align__(16) uint32_t su[Q0 + 8];
  __shared__ __align__(16) uint32_t dsm[NIDX + 4];
  const int lane = threadIdx.x;
  for (int i = lane; i < EW + 64; i += 32) E[i] = i * 2654435761u + blockIdx.x;
  for (int i = lane; i < Q0 + 8; i += 32) su[i] = i * 0x9E3779B9u + blockIdx.x;
  for (int i = lane; i < NIDX + 4; i += 32) dsm[i] = (i * 7919u + blockIdx.x * 131u) % 35851u + 1;
  __syncwarp();
  long long t0 = clock64();
  uint32_t acc[R];
#pragma unroll
  for (int k = 0; k < R; k++) acc[k] = 0;
  const uint32_t *Eb = E + lane * R;
  for (int it = 0; it < iters; it++) {
    if (REBUILD) {
      for (uint32_t c = lane; c < Q0 / 4; c += 32) reinterpret_cast<uint4 *>(E)[c] = reinterpret_cast<const uint4 *>(su)[c];
#pragma unroll 4
      for (uint32_t q = Q0 + 1 + lane; q < EW; q += 32) {
        const uint32_t x = q - Q0 - 1;
        const uint32_t lo = x < Q0 ? su[x] : 0u;
        const uint32_t hi = x + 1 < Q0 ? su[x + 1] : 0u;
        E[q] = __funnelshift_r(lo, hi, 32 - C);
      }
      __syncwarp();
    }
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
    if (REBUILD) {
      __syncwarp();
#pragma unroll
      for (int k = 0; k < R; k++) E[lane * R + k] = acc[k];  // r overwrites E, as in S1Pipe::run
      __syncwarp();
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < R; k++) x ^= acc[k];
  out[blockIdx.x * 32 + lane] = x;
  if (lane == 0) clk[blockIdx.x] = clock64() - t0;
}

__global__ void __launch_bounds__(32) k_a(uint32_t *o, int it, long long *c) { body<false>(o, it, c); }
__global__ void __launch_bounds__(32, 32) k_b(uint32_t *o, int it, long long *c) { body<false>(o, it, c); }
__global__ void __launch_bounds__(32) k_c(uint32_t *o, int it, long long *c) { body<true>(o, it, c); }
__global__ void __launch_bounds__(32, 32) k_d(uint32_t *o, int it, long long *c) { body<true>(o, it, c); }

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
  const char *names = "abcd";
  for (int v = 0; v < 4; v++) {
    for (int warps : {4, 8, 12, 16}) {
      const int grid = sms * warps;
      const int iters = 60;
      float ms = 0;
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        if (v == 0) k_a<<<grid, 32>>>(out, iters, clk);
        else if (v == 1) k_b<<<grid, 32>>>(out, iters, clk);
        else if (v == 2) k_c<<<grid, 32>>>(out, iters, clk);
        else k_d<<<grid, 32>>>(out, iters, clk);
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
      printf("%c warps/SM %2d: %.2f pairs/clk/SM (bound %.1f)  %.3f ms  (%.0f MHz est)\n", names[v], warps,
             pairs / sms / (ms * 1e-3) / clk_hz, 32.0 * 35.0 / 36.0, ms, clk_hz / 1e6);
    }
  }
  return 0;
}
