/* ORACLE (test infrastructure only) — parameter sets.
 * Table I "HQC parameter sets", P:107-122:
 *   HQC-1  N=17,669  w=66   w_e=w_r=75   RS [46,16,31]  RM [384,8,192]
 *   HQC-3  N=35,851  w=100  w_e=w_r=114  RS [56,24,33]  RM [640,8,320]
 *   HQC-5  N=57,637  w=131  w_e=w_r=149  RS [90,32,59]  RM [640,8,320]
 * Derived: delta = (d-1)/2 (R#15), mult = n2/128, n12 = n1*n2 (R#3).
 * This table is the oracle's own copy; tests cross-check it against the CUDA library's
 * hqc_get_params and against tests/golden/table1_params.txt (retyped from P:115-117). */
#include "oracle.h"

int orc_get_params(int level, orc_params *out) {
  uint32_t n, w, wr, n1, k, d, n2, dp;
  switch (level) {
    case 1: n = 17669; w = 66;  wr = 75;  n1 = 46; k = 16; d = 31; n2 = 384; dp = 192; break;
    case 3: n = 35851; w = 100; wr = 114; n1 = 56; k = 24; d = 33; n2 = 640; dp = 320; break;
    case 5: n = 57637; w = 131; wr = 149; n1 = 90; k = 32; d = 59; n2 = 640; dp = 320; break;
    default: return -1;
  }
  out->level = level;
  out->n = n; out->w = w; out->wr = wr;
  out->n1 = n1; out->k = k; out->d = d; out->delta = (d - 1) / 2;
  out->n2 = n2; out->mult = n2 / 128; out->dprime = dp;
  out->n12 = n1 * n2;
  out->words = (n + 63) / 64;
  out->vwords = (out->n12 + 63) / 64;
  return 0;
}
