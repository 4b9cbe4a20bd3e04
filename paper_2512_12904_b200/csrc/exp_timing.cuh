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
#else
#define PHASE_T0()
#define PHASE(i)
#endif
