/* ORACLE (test infrastructure only) — SHAKE256 (FIPS 202) for the KEM row of SURVEY §8(f).
 *
 * The paper uses SHAKE256 as HQC's PRNG and for the domain-separated G, H, K (§II.A, §III.C
 * P:183-192) but gives no construction; this is the textbook sponge: Keccak-f[1600] (24 rounds of
 * theta, rho, pi, chi, iota, written from the standard's step definitions), rate 136 bytes,
 * domain padding 0x1F ... 0x80. Pins (tests/test_oracle_kem.py): the SPEC S:102 vector
 * SHAKE256("", 32) and Python's hashlib.shake_256 on many lengths (a library implementation). */
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

static uint64_t rotl(uint64_t x, unsigned r) { return r ? (x << r) | (x >> (64 - r)) : x; }

/* round constants from the LFSR rc(t) of FIPS 202 §3.2.5 */
static int rc_bit(unsigned t) {
  if (t % 255 == 0) return 1;
  unsigned R = 1;  /* 8-bit LFSR state, R = 10000000 in the standard's bit order (bit 0 first) */
  for (unsigned i = 1; i <= t % 255; i++) {
    unsigned r0 = 0;
    /* R = 0 || R; R[0] ^= R[8]; R[4] ^= R[8]; R[5] ^= R[8]; R[6] ^= R[8]; R = Trunc8(R) */
    R <<= 1;
    unsigned r8 = (R >> 8) & 1;
    R ^= r8 | (r8 << 4) | (r8 << 5) | (r8 << 6);
    R &= 0xFF;
    (void)r0;
  }
  return (int)(R & 1);
}

void orc_keccak_f1600(uint64_t A[25]) {
  /* A[x + 5y] is lane (x, y) */
  for (unsigned ir = 0; ir < 24; ir++) {
    uint64_t C[5], D[5], B[25];
    for (int x = 0; x < 5; x++) C[x] = A[x] ^ A[x + 5] ^ A[x + 10] ^ A[x + 15] ^ A[x + 20];  /* theta */
    for (int x = 0; x < 5; x++) D[x] = C[(x + 4) % 5] ^ rotl(C[(x + 1) % 5], 1);
    for (int i = 0; i < 25; i++) A[i] ^= D[i % 5];
    /* rho: offsets (t+1)(t+2)/2 along the walk (x, y) -> (y, 2x + 3y), starting at (1, 0) */
    uint64_t R[25];
    memcpy(R, A, sizeof R);
    {
      int x = 1, y = 0;
      for (int t = 0; t < 24; t++) {
        R[x + 5 * y] = rotl(A[x + 5 * y], (unsigned)(((t + 1) * (t + 2) / 2) % 64));
        int nx = y, ny = (2 * x + 3 * y) % 5;
        x = nx;
        y = ny;
      }
    }
    /* pi: A'[x, y] = A[(x + 3y) mod 5, x] */
    for (int x = 0; x < 5; x++)
      for (int y = 0; y < 5; y++) B[x + 5 * y] = R[((x + 3 * y) % 5) + 5 * x];
    /* chi */
    for (int x = 0; x < 5; x++)
      for (int y = 0; y < 5; y++)
        A[x + 5 * y] = B[x + 5 * y] ^ ((~B[(x + 1) % 5 + 5 * y]) & B[(x + 2) % 5 + 5 * y]);
    /* iota: RC[j] bit at position 2^j - 1 is rc(j + 7 ir) */
    uint64_t RC = 0;
    for (unsigned j = 0; j <= 6; j++)
      if (rc_bit(j + 7 * ir)) RC |= 1ull << ((1u << j) - 1);
    A[0] ^= RC;
  }
}

/* SHAKE256(msg, outlen): rate 136 bytes, suffix 0x1F, final bit 0x80 */
void orc_shake256(const uint8_t *msg, size_t len, uint8_t *out, size_t outlen) {
  const size_t rate = 136;
  uint64_t A[25];
  memset(A, 0, sizeof A);
  uint8_t block[136];
  size_t off = 0;
  for (;;) {
    size_t take = len - off < rate ? len - off : rate;
    memset(block, 0, rate);
    memcpy(block, msg + off, take);
    off += take;
    int last = take < rate;
    if (last) {
      block[take] ^= 0x1F;
      block[rate - 1] ^= 0x80;
    }
    for (size_t i = 0; i < rate / 8; i++) {
      uint64_t w = 0;
      for (int b = 0; b < 8; b++) w |= (uint64_t)block[8 * i + b] << (8 * b);
      A[i] ^= w;
    }
    orc_keccak_f1600(A);
    if (last) break;
  }
  size_t got = 0;
  for (;;) {
    for (size_t i = 0; i < rate && got < outlen; i++, got++) out[got] = (uint8_t)(A[i / 8] >> (8 * (i % 8)));
    if (got >= outlen) break;
    orc_keccak_f1600(A);
  }
}
