// The north star's conditional option, measured: the RM(1,7) Hadamard step as a batched tcgen05 GEMM
// (F = S · H over 128-position blocks, fp16 x fp16 -> fp32 in TMEM) against the register butterfly of
// stage2.cuh (rm_decode_block), on the same random HQC-3-shaped blocks (5 copies of 128 bits each).
// Both produce the decoded byte of every block (smallest a with maximal |F(a)|, bit 7 = sign); the
// program checks they agree and prints blocks/s for each.
//   TC path, CTA = 4 warps, one tile = 128 blocks: every thread builds its block's soft values
//   s_p = 5 - 2 cnt_p as fp16 and stores them as row `tid` of the A tile (K-major, no swizzle: 8x8
//   core matrices, LBO = 128 B along K, SBO = 2048 B along M); one thread issues 8 tcgen05.mma
//   (M = N = 128, K = 16 each) against the constant Hadamard B tile and commits to an mbarrier; every
//   thread then reads its row of F (128 fp32 accumulators) back with tcgen05.ld and takes the argmax.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mbtc scripts/microbench_tc_fht.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstdlib>

#include "../paper_2512_12904_b200/csrc/stage2.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int MULT = 5;
constexpr int WORDS = MULT * 4;  // 32-bit words per block

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---- the butterfly path: one thread per block
__global__ void __launch_bounds__(128) k_fwht(const uint32_t *__restrict__ bits, uint8_t *__restrict__ out, int nblk) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nblk; b += gridDim.x * blockDim.x) {
    uint32_t X[WORDS];
    const uint4 *src = reinterpret_cast<const uint4 *>(bits + (size_t)b * WORDS);
#pragma unroll
    for (int c = 0; c < MULT; c++) {
      const uint4 x = src[c];
      X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
    }
    out[b] = (uint8_t)hqc::rm_decode_block<MULT>(X);
  }
}

// ---- the tensor-core path
constexpr int TILE = 128;
constexpr uint32_t A_BYTES = TILE * 128 * 2, B_BYTES = 128 * 128 * 2;
constexpr uint32_t LBO = 128, SBO = 2048;

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((LBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((SBO >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100); base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
  return d;
}
// byte offset of element (row r, k) in the K-major interleaved layout
__device__ __forceinline__ uint32_t kmaj_off(int r, int k) {
  return (r >> 3) * SBO + (k >> 3) * LBO + (r & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
  return ok != 0;
}

__global__ void __launch_bounds__(128, 3) k_tc(const uint32_t *__restrict__ bits, uint8_t *__restrict__ out, int nblk,
                                               int *__restrict__ err) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *A = smem, *Bt = smem + A_BYTES;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B = H: row n = output index a, column k = position p: (-1)^popcount(a & p)
  for (int e = tid; e < 128 * 128; e += 128) {
    const int n = e >> 7, k = e & 127;
    const int i = k >> 1, hh = k & 1, pos = 32 * (i >> 4) + (i & 15) + 16 * hh;
    const int j = n >> 1, jh = n & 1, a = 32 * (j >> 4) + (j & 15) + 16 * jh;  // output order = h[] layout
    *reinterpret_cast<__half *>(Bt + kmaj_off(n, k)) = __float2half((__popc(a & pos) & 1) ? -1.0f : 1.0f);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  // instruction descriptor: D f32, A/B f16, both K-major, N = 128, M = 128
#ifdef TC_F32
  const uint32_t idesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
#else
  const uint32_t idesc = (0u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);  // f16 accumulators (exact: |F| <= 1280)
#endif
  const uint32_t a0 = smem_u32(A), b0 = smem_u32(Bt);
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile * TILE < nblk; tile += gridDim.x) {
    const int b = tile * TILE + tid;
    // soft values -2 cnt_p as fp16 in the butterfly's register layout: half2 register i = 16q + l holds
    // positions (32q + l, 32q + l + 16); the K index of the GEMM follows that order (k = 2i, 2i + 1),
    // and the Hadamard tile B is built in the same order, so the registers go to A as they are
    {
      uint32_t X[WORDS];
      const uint4 *src = reinterpret_cast<const uint4 *>(bits + (size_t)(b < nblk ? b : nblk - 1) * WORDS);
#pragma unroll
      for (int c = 0; c < MULT; c++) {
        const uint4 x = src[c];
        X[4 * c] = x.x; X[4 * c + 1] = x.y; X[4 * c + 2] = x.z; X[4 * c + 3] = x.w;
      }
      uint32_t pl[3][4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const uint32_t a = X[q], bb = X[4 + q], c = X[8 + q], d = X[12 + q], e = X[16 + q];
        const uint32_t s1 = a ^ bb ^ c, c1 = (a & bb) | (c & (a ^ bb));
        const uint32_t s2 = s1 ^ d ^ e, c2 = (s1 & d) | (e & (s1 ^ d));
        pl[0][q] = s2; pl[1][q] = c1 ^ c2; pl[2][q] = c1 & c2;
      }
#pragma unroll
      for (int q = 0; q < 4; q++) {
        uint32_t lo[3], hi[3];
#pragma unroll
        for (int k = 0; k < 3; k++) { lo[k] = pl[k][q] << k; hi[k] = pl[k][q] >> (8 - k); }
#pragma unroll
        for (int g = 0; g < 4; g++) {  // 4 registers l = 4g .. 4g+3 -> one 16-byte chunk
          uint32_t w[4];
#pragma unroll
          for (int t = 0; t < 4; t++) {
            const int l = 4 * g + t, lp = l & 7;
            const uint32_t m0 = 0x00010001u << lp;
            uint32_t x = hqc::and_or(l < 8 ? lo[0] : hi[0], m0, 0x64006400u);
            x = hqc::and_or(l < 8 ? lo[1] : hi[1], m0 << 1, x);
            x = hqc::and_or(l < 8 ? lo[2] : hi[2], m0 << 2, x);
            const __half2 v = __hfma2(hqc::u2h(x), __float2half2_rn(-ldexpf(1.0f, 1 - lp)),
                                      __float2half2_rn(ldexpf(1.0f, 11 - lp)));
            w[t] = *reinterpret_cast<const uint32_t *>(&v);
          }
          const int i = 16 * q + 4 * g;  // half2 register index -> k = 2i
          *reinterpret_cast<uint4 *>(A + kmaj_off(tid, 2 * i)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int s = 0; s < 8; s++) {  // K = 16 per MMA: two 8-element core matrices along K
        const uint64_t ad = umma_desc(a0 + s * 2 * LBO), bd = umma_desc(b0 + s * 2 * LBO);
        const uint32_t acc = s > 0;
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                     ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(smem_u32(&mbar)) : "memory");
    }
    // bounded wait (a lost arrival reports an error instead of hanging the GPU)
    bool done = false;
    for (long it = 0; it < (1L << 24) && !done; it++) done = mbar_try(smem_u32(&mbar), phase);
    if (!done) {
      atomicExch(err, 1);
      break;
    }
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;");
    // row tid of F: TMEM lane tid (warp w reads lanes 32w..32w+31); f16 accumulators, two adjacent
    // columns packed per register -> exactly the butterfly's h[64] layout, then its argmax
    __half2 hF[64];
#pragma unroll
    for (int q = 0; q < 2; q++) {
      uint32_t r[32];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + 64 * q;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; i++) hF[32 * q + i] = hqc::u2h(r[i]);
    }
    const uint32_t sym = hqc::rm_argmax<MULT>(hF);
    if (b < nblk) out[b] = (uint8_t)sym;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // A may be overwritten; TMEM may be overwritten by the next MMAs
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  const int nblk = 56 * 65536;  // HQC-3: 56 blocks per ciphertext, 65,536 ciphertexts
  std::vector<uint32_t> h((size_t)nblk * WORDS);
  uint64_t x = 0x9E3779B97F4A7C15ull;
  for (auto &w : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    w = (uint32_t)x;
  }
  uint32_t *d_bits;
  uint8_t *d1, *d2;
  int *d_err;
  CK(cudaMalloc(&d_bits, h.size() * 4));
  CK(cudaMalloc(&d1, nblk));
  CK(cudaMalloc(&d2, nblk));
  CK(cudaMalloc(&d_err, 4));
  CK(cudaMemset(d_err, 0, 4));
  CK(cudaMemcpy(d_bits, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t smem = A_BYTES + B_BYTES;
  CK(cudaFuncSetAttribute(k_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_tc, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tc, 128, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k_tc));
  printf("k_tc: regs %d static smem %zu max dyn %d occupancy %d\n", fa.numRegs, fa.sharedSizeBytes,
         fa.maxDynamicSharedSizeBytes, per_sm);
  if (getenv("TC_CTAS")) per_sm = atoi(getenv("TC_CTAS"));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms_f = 0, ms_t = 0;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    k_fwht<<<sms * 16, 128>>>(d_bits, d1, nblk);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms_f, e0, e1);
    cudaEventRecord(e0);
    k_tc<<<sms * per_sm, 128, smem>>>(d_bits, d2, nblk, d_err);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms_t, e0, e1);
  }
  CK(cudaGetLastError());
  int err = 0;
  CK(cudaMemcpy(&err, d_err, 4, cudaMemcpyDeviceToHost));
  std::vector<uint8_t> o1(nblk), o2(nblk);
  CK(cudaMemcpy(o1.data(), d1, nblk, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(o2.data(), d2, nblk, cudaMemcpyDeviceToHost));
  long mism = 0;
  for (int i = 0; i < nblk; i++) mism += o1[i] != o2[i];
  printf("blocks %d  butterfly %.3f ms (%.2f Gblk/s)  tcgen05 %.3f ms (%.2f Gblk/s, %d CTAs/SM)  mismatches %ld  mbar_timeout %d\n",
         nblk, ms_f, nblk / ms_f / 1e6, ms_t, nblk / ms_t / 1e6, per_sm, mism, err);
  return mism == 0 && err == 0 ? 0 : 2;
}
