// Stage 1 (the sparse x dense product of Eq. 1, §III.B) with its windows read from TENSOR
// MEMORY instead of shared memory: K1t, an opt-in kernel of hqc_sparse_dense_mul_batch (HQC_S1_KERNEL=3),
// and the product of the fused variant K4t (HQC_DEC_KERNEL=4). Same arithmetic as stage1.cuh
// (r[W] ^= SHF(E[o + W], E[o + W + 1], s) for each support index, o = d >> 5, s = d & 31), different
// load path.
//
// NOT CONSTANT-FLOW: the support is bucketed by offset range, so the trip count of each range's loop
// (and whether a range ends with a single-index pass) depends on the secret y. The total arithmetic is
// fixed, but the control flow is not (R#8, P:171 ask for execution independent of secret data), which
// is why the library's defaults are the shared-memory kernels and these are opt-in.
//
// Why: the shared-memory kernels read one 32-bit word per (index, output word) pair and run at ~90% of
// the 128 B/clk/SM shared-memory bound (profiles/r01b/NOTES.md, item 1); tcgen05.ld reads tensor memory
// at ~300-400 B/clk/SM with 8-16 warps (scripts/microbench_tmem_ld.cu, NOTES item 18).
//
// Layout. tcgen05.ld.32x32b gives lane l of a warp the columns [c, c + x) of TMEM row (32 q + l) at a
// WARP-UNIFORM column c. Lane l owns output words [l R, l R + R) and needs, for an index with word
// offset o, the window E[o + l R .. o + l R + R]. So row l holds a SKEWED copy of E:
//     row l, column c  =  E[l R + t G + c]        c < COLS,  range t: o in [t G, t G + G),  G = COLS - R
// and the index reads columns (o - t G) .. (o - t G) + R, all < COLS. The support indices are bucketed
// by range (ballot compaction), and for each range the warp refills its columns from E in shared memory
// (16-byte loads, see TmShape) with tcgen05.st, then runs that range's indices.
// Shared-memory traffic per ciphertext drops from w * NW words (the windows) to NR * 32 * COLS (the
// refills), HQC-3: 112,000 -> 49,152 words; the windows come from TMEM.
//
// CTA = 16 warps (HQC-1/3; 4 per TMEM lane quarter, COLS = 128 columns each) or 8 warps (HQC-5, whose
// buffers are larger; COLS = 256); one CTA per SM (the dynamic shared memory request is padded so that a
// second CTA never waits in tcgen05.alloc). Measured choices: profiles/r01b/NOTES.md item 18.
#pragma once
#include <cstdint>

#include "async_copy.cuh"
#include "levels.cuh"
#include "stage1.cuh"

namespace hqc {

// ---- tcgen05 tensor-memory access (PTX ISA 8.7, sm_100a) -----------------------------------------
template <int N> struct TmLd;
#define HQC_TM_R8(o) "=r"(r[o]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]), "=r"(r[o + 5]), "=r"(r[o + 6]), "=r"(r[o + 7])
#define HQC_TM_W8(o) "r"(r[o]), "r"(r[o + 1]), "r"(r[o + 2]), "r"(r[o + 3]), "r"(r[o + 4]), "r"(r[o + 5]), "r"(r[o + 6]), "r"(r[o + 7])
template <> struct TmLd<32> {
  static __device__ __forceinline__ void ld(uint32_t *r, uint32_t ta) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : HQC_TM_R8(0), HQC_TM_R8(8), HQC_TM_R8(16), HQC_TM_R8(24)
        : "r"(ta));
  }
  static __device__ __forceinline__ void st(const uint32_t *r, uint32_t ta) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        HQC_TM_W8(0), HQC_TM_W8(8), HQC_TM_W8(16), HQC_TM_W8(24)
        : "memory");
  }
};
template <> struct TmLd<16> {
  static __device__ __forceinline__ void ld(uint32_t *r, uint32_t ta) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : HQC_TM_R8(0), HQC_TM_R8(8)
                 : "r"(ta));
  }
};
template <> struct TmLd<8> {
  static __device__ __forceinline__ void ld(uint32_t *r, uint32_t ta) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : HQC_TM_R8(0) : "r"(ta));
  }
};
template <> struct TmLd<4> {
  static __device__ __forceinline__ void ld(uint32_t *r, uint32_t ta) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(ta));
  }
};
template <> struct TmLd<2> {
  static __device__ __forceinline__ void ld(uint32_t *r, uint32_t ta) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(ta));
  }
};
template <> struct TmLd<1> {
  static __device__ __forceinline__ void ld(uint32_t *r, uint32_t ta) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(ta));
  }
};
#undef HQC_TM_R8
#undef HQC_TM_W8

// N consecutive columns from ta into r[0..N) as power-of-two pieces (largest first).
template <int N> __device__ __forceinline__ void tm_ld_n(uint32_t *r, uint32_t ta) {
  if constexpr (N >= 32) {
    TmLd<32>::ld(r, ta);
    tm_ld_n<N - 32>(r + 32, ta + 32);
  } else if constexpr (N >= 16) {
    TmLd<16>::ld(r, ta);
    tm_ld_n<N - 16>(r + 16, ta + 16);
  } else if constexpr (N >= 8) {
    TmLd<8>::ld(r, ta);
    tm_ld_n<N - 8>(r + 8, ta + 8);
  } else if constexpr (N >= 4) {
    TmLd<4>::ld(r, ta);
    tm_ld_n<N - 4>(r + 4, ta + 4);
  } else if constexpr (N >= 2) {
    TmLd<2>::ld(r, ta);
    tm_ld_n<N - 2>(r + 2, ta + 2);
  } else if constexpr (N == 1) {
    TmLd<1>::ld(r, ta);
  }
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ---- K1t -----------------------------------------------------------------------------------------
// Output words per lane: R = ceil(NW / 32) rounded up so that the refills (lane l reads E from word
// l R on) use V-word loads that are aligned and conflict-free: V = 4, R = 4 x odd (16-byte loads; the 8
// lanes of a wavefront hit 8 distinct 4-bank groups: (R/4) l mod 8 is a permutation for R/4 odd);
// V = 2, R = 2 x odd (8-byte loads, 16 lanes per wavefront); V = 1, R odd (the shared-memory kernels'
// choice). A larger R wastes up to 3 words per lane in the product (HQC-3: 36 x 32 = 1152 >= 1120).
#ifndef HQC_S1T_V
#define HQC_S1T_V 4
#endif
template <class P, uint32_t V> constexpr uint32_t s1t_r() {
  constexpr uint32_t r = (P::NW + 31) / 32;
  if constexpr (V == 1) return make_odd_up(r);
  else if constexpr (V == 2) return (r % 4 == 2) ? r : (r % 4 == 3 ? r + 3 : r + (2 - r % 4));
  else return round_up(r, 4);
}
template <class P, uint32_t V> struct TmShape {
  static constexpr uint32_t NOUT = P::NW, WT = P::W;
  static constexpr uint32_t R = s1t_r<P, V>();
  static constexpr uint32_t E_WORDS = round_up(P::Q0 + 32 * R + 2, 4);
  static constexpr uint32_t WPAD = round_up(WT, 4);
};

#ifndef HQC_S1T_WARPS
#define HQC_S1T_WARPS (P::level == 5 ? 8 : 16)
#endif
#ifndef HQC_S1T_COLS
#define HQC_S1T_COLS (P::level == 5 ? 256 : 128)
#endif
#ifndef HQC_S1T_FU
#define HQC_S1T_FU 2
#endif

// Per-warp shared-memory layout of the tensor-memory product (after a per-CTA prefix of PRE bytes):
// E | staging row (u, then v) | bucketed rotation amounts + range starts | mbarrier | EXTRA bytes (the
// fused kernel's symbol chunk). E is at least E_MIN bytes (the fused kernel's RS scratch aliases it).
template <class P, int WARPS_, uint32_t COLS_, uint32_t PRE_ = 16, uint32_t EXTRA_ = 0, uint32_t E_MIN_ = 0>
struct TmS1 {
  static constexpr uint32_t V = HQC_S1T_V;
  using S = TmShape<P, V>;
  static constexpr int WARPS = WARPS_;                // WARPS / 4 per lane quarter
  static constexpr uint32_t COLS = COLS_;             // TMEM columns per warp
  static constexpr uint32_t WIN = S::R + 1;           // window words per index
  static constexpr int FU = HQC_S1T_FU;               // refill pieces in flight
  static constexpr uint32_t G = COLS - S::R;          // word offsets per range
  static constexpr uint32_t NR = P::Q0 / G + 1;       // ranges (o = d >> 5 <= n >> 5 = Q0)
  static constexpr uint32_t JPL = (P::W + 31) / 32;   // support slots per lane (registers, one ahead)
  // E is read by the refills up to word 31 R + (NR - 1) G + round_up(COLS, 32 FU) - 1 (columns past a
  // range's last window hold words no index reads; the buffer only has to be addressable there)
  static constexpr uint32_t EW_FILL = 31 * S::R + (NR - 1) * G + round_up(COLS, 32 * FU);
  static constexpr uint32_t EW = EW_FILL > S::E_WORDS ? EW_FILL : S::E_WORDS;
  static constexpr uint32_t E_BYTES = round_up(EW * 4 > E_MIN_ ? EW * 4 : E_MIN_, 16);
  static constexpr uint32_t UB = P::U_STRIDE * 8, VB = P::V_WORDS * 8;
  static constexpr uint32_t STG_BYTES = round_up(UB > VB ? UB : VB, 16);
  static constexpr uint32_t L_BYTES = round_up((S::WPAD + NR + 1) * 4, 16);  // bucketed d, then range starts
  static constexpr uint32_t EXTRA_OFF = E_BYTES + STG_BYTES + L_BYTES + 16;
  static constexpr uint32_t WARP_BYTES = round_up(EXTRA_OFF + EXTRA_, 16);
  static constexpr uint32_t PRE = PRE_;               // per-CTA prefix; its last 16 bytes hold the TMEM address
  // one CTA per SM: more than half of the 228 KB so that no second CTA is co-resident
  static constexpr uint32_t SMEM_BYTES = PRE + WARPS * WARP_BYTES > 120 * 1024 ? PRE + WARPS * WARP_BYTES : 120 * 1024;
  static_assert(PRE + WARPS * WARP_BYTES <= 227 * 1024, "per-warp buffers fit in one CTA");
  static_assert(WARPS % 4 == 0 && COLS * (WARPS / 4) <= 512 && COLS % 32 == 0, "TMEM columns");
  static_assert(G >= 32, "ranges wider than a fill piece");
  static_assert(S::R % V == 0 && G % V == 0 && (V == 1 || (V == 2 && S::R % 4 == 2) || (V == 4 && S::R % 4 == 0)),
                "V-word aligned, conflict-free refill loads");
};

// CTA start: warp 0 allocates all 512 TMEM columns (one CTA per SM), every lane learns its warp's base.
template <class M> __device__ __forceinline__ uint32_t tm_cta_alloc(uint8_t *smem, int wib) {
  uint32_t *slot = reinterpret_cast<uint32_t *>(smem + M::PRE - 16);
  if (wib == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  // this warp's TMEM: lanes 32 (w % 4) .. + 31, columns (w / 4) * COLS .. + COLS - 1
  return *slot + ((uint32_t)(32 * (wib & 3)) << 16) + (uint32_t)(wib >> 2) * M::COLS;
}
template <class M> __device__ __forceinline__ void tm_cta_free(uint8_t *smem, int wib) {
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (wib == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(
        *reinterpret_cast<uint32_t *>(smem + M::PRE - 16)));
}

// One warp's product pipeline: u of the current ciphertext staged by TMA, its support in registers
// (loaded one ciphertext ahead), the windows from this warp's TMEM columns.
template <class P, class M> struct TmPipe {
  using S = typename M::S;
  static constexpr int R = S::R;
  uint32_t *E, *stg, *list, *starts;
  uint64_t *bar;
  uint8_t *extra;
  uint32_t phase, ta;
  uint32_t yn[M::JPL];
  const uint64_t *u, *v;
  const uint32_t *y;

  __device__ __forceinline__ TmPipe(uint8_t *ws, uint32_t ta_, const uint64_t *u_, const uint64_t *v_,
                                    const uint32_t *y_, int lane)
      : ta(ta_), u(u_), v(v_), y(y_) {
    E = reinterpret_cast<uint32_t *>(ws);
    stg = reinterpret_cast<uint32_t *>(ws + M::E_BYTES);
    list = reinterpret_cast<uint32_t *>(ws + M::E_BYTES + M::STG_BYTES);
    starts = list + S::WPAD;
    bar = reinterpret_cast<uint64_t *>(ws + M::E_BYTES + M::STG_BYTES + M::L_BYTES);
    extra = ws + M::EXTRA_OFF;
    phase = 0;
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
  }
  __device__ __forceinline__ void wait() {
    mbar_wait(bar, phase);
    phase ^= 1u;
  }
  __device__ __forceinline__ void tma_row(const void *src, uint32_t bytes, int lane) {
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(bar, bytes);
      tma_load_1d(stg, src, bytes, bar);
    }
  }
  // request ciphertext ct's u (TMA) and its support row (registers)
  __device__ __forceinline__ void fetch(size_t ct, int lane) {
    tma_row(u + ct * P::U_STRIDE, M::UB, lane);
#pragma unroll
    for (uint32_t s = 0; s < M::JPL; s++) {
      const uint32_t j = lane + 32 * s;
      yn[s] = j < P::W ? __ldg(y + ct * P::Y_STRIDE + j) : 0u;
    }
  }

  // Stage 1 of ciphertext ct (fetched): leaves r = v XOR trunc(u * y) (or the product alone when v is
  // NULL) in E[0 .. NW); requests `next` when has_next (v: after r is stored, else during the product).
  __device__ __forceinline__ void run(size_t ct, bool has_next, size_t next, int lane) {
    wait();
    // rotation amounts d_j = n - y_j (an entry >= n counts as y = 0, R#13) and their ranges
    uint32_t dj[M::JPL], tj[M::JPL];
#pragma unroll
    for (uint32_t s = 0; s < M::JPL; s++) {
      const uint32_t j = lane + 32 * s;
      dj[s] = yn[s] < P::N ? P::N - yn[s] : P::N;
      tj[s] = j < P::W ? (dj[s] >> 5) / M::G : M::NR;
    }
    s1_build_E<P, S>(stg, E, lane);
    __syncwarp();
    if (v) tma_row(v + ct * P::V_WORDS, M::VB, lane);  // v lands in the consumed staging row
    else if (has_next) tma_row(u + next * P::U_STRIDE, M::UB, lane);
    if (has_next) {
#pragma unroll
      for (uint32_t s = 0; s < M::JPL; s++) {  // in flight during this product
        const uint32_t j = lane + 32 * s;
        yn[s] = j < P::W ? __ldg(y + next * P::Y_STRIDE + j) : 0u;
      }
    }
    {  // bucket by range: ballot compaction, range by range (w entries in total, whatever the split)
      uint32_t pos = 0;
      const uint32_t lt = (1u << lane) - 1u;
#pragma unroll 1
      for (uint32_t t = 0; t < M::NR; t++) {
        if (lane == 0) starts[t] = pos;
#pragma unroll
        for (uint32_t s = 0; s < M::JPL; s++) {
          const uint32_t m = __ballot_sync(0xffffffffu, tj[s] == t);
          if (tj[s] == t) list[pos + __popc(m & lt)] = dj[s];
          pos += __popc(m);
        }
      }
      if (lane == 0) starts[M::NR] = pos;
    }
    __syncwarp();
    uint32_t acc[R];
#pragma unroll
    for (int k = 0; k < R; k++) acc[k] = 0;
    const uint32_t *Erow = E + lane * R;
#pragma unroll 1
    for (uint32_t t = 0; t < M::NR; t++) {
      // refill: row l, column c <- E[l R + t G + c], the columns this range's windows reach:
      // (min(t G + G - 1, Q0) - t G) + WIN (the last range is short); FU pieces of 32 in flight
      const uint32_t omax = (t + 1) * M::G - 1 < P::Q0 ? (t + 1) * M::G - 1 : P::Q0;
      const uint32_t nc = omax - t * M::G + M::WIN;
      const uint32_t *src = Erow + t * M::G;  // V-word aligned: R, G and c are multiples of V
#pragma unroll 1
      for (uint32_t c = 0; c < nc; c += 32 * M::FU) {
        uint32_t f[M::FU][32];
#pragma unroll
        for (int q = 0; q < M::FU; q++)
#pragma unroll
          for (int k = 0; k < 32; k += M::V) {
            if constexpr (M::V == 4) {
              const uint4 x = *reinterpret_cast<const uint4 *>(src + c + 32 * q + k);
              f[q][k] = x.x; f[q][k + 1] = x.y; f[q][k + 2] = x.z; f[q][k + 3] = x.w;
            } else if constexpr (M::V == 2) {
              const uint2 x = *reinterpret_cast<const uint2 *>(src + c + 32 * q + k);
              f[q][k] = x.x; f[q][k + 1] = x.y;
            } else {
              f[q][k] = src[c + 32 * q + k];
            }
          }
#pragma unroll
        for (int q = 0; q < M::FU; q++)
          if (q == 0 || c + 32 * q < nc) TmLd<32>::st(f[q], ta + c + 32 * q);
      }
      tm_wait_st();
      const uint32_t j1 = starts[t + 1], tg = t * M::G;
      uint32_t j = starts[t];
#pragma unroll 1
      for (; j + 1 < j1; j += 2) {  // two indices per pass: one 3-input XOR per word
        const uint32_t d0 = list[j], d1 = list[j + 1];
        uint32_t a[M::WIN], b[M::WIN];
        tm_ld_n<M::WIN>(a, ta + (d0 >> 5) - tg);
        tm_ld_n<M::WIN>(b, ta + (d1 >> 5) - tg);
        tm_wait_ld();
#pragma unroll
        for (int k = 0; k < R; k++) acc[k] ^= __funnelshift_r(a[k], a[k + 1], d0) ^ __funnelshift_r(b[k], b[k + 1], d1);
      }
      if (j < j1) {
        const uint32_t d0 = list[j];
        uint32_t a[M::WIN];
        tm_ld_n<M::WIN>(a, ta + (d0 >> 5) - tg);
        tm_wait_ld();
#pragma unroll
        for (int k = 0; k < R; k++) acc[k] ^= __funnelshift_r(a[k], a[k + 1], d0);
      }
    }
    __syncwarp();  // every lane's refills have read E: r overwrites it
    if (v) {
      wait();
      s1_store_r_xor<S>(acc, E, stg, lane);
    } else {
      s1_store_r<S>(acc, E, lane);
    }
    __syncwarp();
    if (v && has_next) tma_row(u + next * P::U_STRIDE, M::UB, lane);  // staging row free again
  }
};

template <class P> using TmS1Std = TmS1<P, HQC_S1T_WARPS, HQC_S1T_COLS>;

#ifndef HQC_S1T_MINB
#define HQC_S1T_MINB 1
#endif
// K1t: stage 1 alone, one warp per ciphertext (grid-stride over the CTA's warps), one CTA per SM.
template <class P>
__global__ void __launch_bounds__(32 * TmS1Std<P>::WARPS, HQC_S1T_MINB)
    k_stage1t(const uint64_t *__restrict__ u, const uint32_t *__restrict__ y, const uint64_t *__restrict__ v,
              uint64_t *__restrict__ r_out, size_t batch) {
  using M = TmS1Std<P>;
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t ta = tm_cta_alloc<M>(smem, wib);
  TmPipe<P, M> pipe(smem + M::PRE + (size_t)wib * M::WARP_BYTES, ta, u, v, y, lane);
  const size_t nwarps = (size_t)gridDim.x * M::WARPS;
  size_t ct = (size_t)blockIdx.x * M::WARPS + wib;
  if (ct < batch) pipe.fetch(ct, lane);
  for (; ct < batch; ct += nwarps) {
    pipe.run(ct, ct + nwarps < batch, ct + nwarps, lane);
    uint4 *dst = reinterpret_cast<uint4 *>(r_out + ct * P::V_WORDS);
    const uint4 *src = reinterpret_cast<const uint4 *>(pipe.E);
    for (uint32_t c = lane; c < P::NW / 4; c += 32) dst[c] = src[c];
    __syncwarp();
  }
  tm_cta_free<M>(smem, wib);
}

}  // namespace hqc
