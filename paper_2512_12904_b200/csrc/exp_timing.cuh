// Experiments only (scripts/exp_variants.py, scripts/exp_sb_phases.py): with -DHQC_EXP_TIMING, PHASE(i)
// adds the clock64() cycles since the previous mark to g_phase_cycles[i] (lane 0 of each warp); read and
// cleared by hqc_exp_phases_lN (kernels.cuh). Without it both macros are empty: product builds carry none.
#pragma once

#ifdef HQC_EXP_TIMING
__device__ unsigned long long g_phase_cycles[16];
#define PHASE_T0() long long _t = clock64()
#define PHASE(i)                                                                                   \
  do {                                                                                             \
    long long _n = clock64();                                                                      \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase_cycles[i], (unsigned long long)(_n - _t));     \
    _t = _n;                                                                                       \
  } while (0)
// per-warp start / end times (%globaltimer, ns) of k_decrypt_sb, indexed by global warp id
__device__ unsigned long long g_warp_span[8192][2];
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define WARP_SPAN(i, w)                                                      \
  do {                                                                       \
    if ((threadIdx.x & 31) == 0 && (w) < 8192) g_warp_span[(w)][(i)] = gtimer_ns(); \
  } while (0)
#else
#define PHASE_T0()
#define PHASE(i)
#define WARP_SPAN(i, w)
#endif
