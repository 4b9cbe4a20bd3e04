/*
 * hqc_gpu.h — C ABI of libhqcgpu.so: batched HQC.PKE.Decrypt on NVIDIA B200 (sm_100a).
 *
 * What it computes (PAPER.md = arxiv 2512.12904 "OptHQC"; P:n = line n; R#k = DESIGN.md §3 reading k):
 *   HQC.PKE.Decrypt (Alg. 2): m' = C.Decode(v - u*y) over many independent ciphertexts,
 *   in three stages:
 *     (1) the sparse x dense cyclic product of Eq. 1 (§III.B) in GF(2)[X]/(X^n - 1),
 *         XORed into v and truncated to n1*n2 bits (R#1-R#3);
 *     (2) duplicated RM(1,7) decoding of each n2-bit block (Table I; R#9-R#12);
 *     (3) shortened RS decoding over GF(2^8) (R#4-R#7): syndromes, Berlekamp–Massey,
 *         Chien root search over the n1 positions, Forney error values, message-first output.
 *   The results are bit-identical to the CPU oracle in oracle/ (tests/test_gpu_*.py).
 *   Also here: step a6 alone in three GF-product methods, batched Encrypt and the KeyGen
 *   product, KeyGen from seeds, and the HHK KEM (Encaps / Decaps with implicit rejection, SHAKE256),
 *   plus two host-buffer end-to-end calls (ABI rows, or serialized ciphertexts with resident keys).
 *
 * Conventions for every entry point
 *   - All functions are host functions and reentrant. Global state: per-device launch attributes and
 *     the two internal streams of the host-buffer calls (created once, guarded by a mutex).
 *   - Array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) unless the name says
 *     _host; they are allocated and owned by the caller and must be 16-byte aligned. The library
 *     allocates no device memory. Outputs must not alias inputs.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream). Every call only
 *     enqueues work on it and returns; asynchronous faults surface at the caller's next sync.
 *   - batch == 0 returns HQC_OK and launches nothing. Argument checks run on the host before any
 *     launch: unknown level (HQC_ERR_LEVEL), NULL pointer with batch > 0 (HQC_ERR_NULL), pointer not
 *     16-byte aligned (HQC_ERR_ALIGN), batch > HQC_MAX_BATCH (HQC_ERR_SIZE). A failed launch returns
 *     HQC_ERR_CUDA: every entry point clears a launch error left pending by earlier, unrelated work
 *     before it launches, so the status reflects this call (a sticky error — a dead context — still
 *     shows). RS decoding failure is a RESULT (uncorrected bytes), never an error.
 *   - Bit order: bit t of a ring element is bit t%64 of uint64 word t/64 (little endian).
 *   - Unchecked preconditions (checking costs a pass): y_support[b][0..w) are distinct and < n
 *     (S:263); use hqc_validate_support in debug builds. A support entry >= n is treated as 0 (no
 *     fault, unspecified output). Bits >= n of u and the padding words/entries of every row are
 *     ignored.
 */
#ifndef HQC_GPU_H
#define HQC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HQC_OK = 0,
  HQC_ERR_LEVEL = -1,
  HQC_ERR_NULL = -2,
  HQC_ERR_ALIGN = -3,
  HQC_ERR_SIZE = -4,
  HQC_ERR_CUDA = -5
} hqc_status;

#define HQC_MAX_BATCH ((size_t)1 << 31)

/* Table I plus the derived row layout of this library. Filled by hqc_get_params;
   treat as read-only. */
typedef struct {
  int32_t level;     /* 1, 3, 5 */
  uint32_t n;        /* ring length N: 17669 / 35851 / 57637 */
  uint32_t n1;       /* RS length: 46 / 56 / 90 */
  uint32_t n2;       /* duplicated RM length: 384 / 640 / 640 */
  uint32_t mult;     /* n2 / 128: 3 / 5 / 5 */
  uint32_t k;        /* message bytes: 16 / 24 / 32 */
  uint32_t delta;    /* RS correction capacity (d-1)/2: 15 / 16 / 29 */
  uint32_t w;        /* omega, weight of y: 66 / 100 / 131 */
  uint32_t wr;       /* omega_r = omega_e: 75 / 114 / 149 */
  uint32_t n12;      /* n1*n2: 17664 / 35840 / 57600 */
  uint32_t u_words;  /* ceil(n/64): 277 / 561 / 901 */
  uint32_t u_stride; /* uint64 per u row = u_words rounded up to even (16-byte rows) */
  uint32_t v_words;  /* uint64 per v / r row = n12/64: 276 / 560 / 900 */
  uint32_t y_stride; /* uint32 per support row = w rounded up to a multiple of 4 */
  uint32_t e_stride; /* uint32 per r1/r2/e support row = wr rounded up to a multiple of 4 */
} hqc_params;

/* Fills *out for level 1, 3 or 5. Returns HQC_OK or HQC_ERR_LEVEL / HQC_ERR_NULL. */
int hqc_get_params(int level, hqc_params *out);

/* Static string for a status code (never NULL). */
const char *hqc_status_str(int status);

/* ---------------------------------------------------------------------------------------------
 * Fused decrypt (Alg. 2):  m_out[b] = C.Decode(v[b] XOR trunc_{n12}(u[b] * y[b]))
 *   u         [batch][u_stride] uint64   ciphertext part u (bits >= n ignored)
 *   v         [batch][v_words]  uint64   ciphertext part v (n1*n2 bits)
 *   y_support [batch][y_stride] uint32   the secret y's support, first w entries used (R#1)
 *   m_out     [batch][k]        uint8    decrypted messages (RS failure -> uncorrected bytes)
 * The launch policy picks the kernel by level and batch (hqc_decrypt_launch_kernel
 * reports it): one fused kernel — stage 1 in shared memory, stage 2 lane-per-RM-block, stage 3 by a
 * warp per word (small batches) or a lane per word (large ones), no intermediate leaving the SM — except
 * HQC-5 above ~16,000 (kernel 11; kernel 10 is its round-2 predecessor), which runs stages 1+2 in
 * one launch, writes the n1 received symbols of each ciphertext to a scratch buffer and decodes them
 * in a second launch. That scratch
 * (batch x n1 bytes, at most 1,048,576 rows per launch) comes from a memory pool the library creates
 * per device on first use; it is stream-ordered (allocated and freed on `stream`, so concurrent calls
 * on different streams are safe and the call can be captured in a CUDA graph) and the pool keeps freed
 * memory for later calls (up to ~94 MB). A large batch may run as consecutive launches
 * (hqc_decrypt_launch_count). All default kernels are constant-flow (R#8). HQC_DEC_KERNEL=1..11
 * forces a kernel (same results; 4 is the tensor-memory product, whose loop counts depend on y,
 * DESIGN.md §6.1b); the variable is read once per process.
 * ------------------------------------------------------------------------------------------- */
int hqc_decrypt_batch(const hqc_params *p, const uint64_t *u, const uint64_t *v,
                      const uint32_t *y_support, uint8_t *m_out, size_t batch, void *stream);

/* Stage 1 alone (Eq. 1; truncation R#3):
 *   r_out[b] = v[b] XOR trunc_{n12}(u[b] * y[b]), [batch][v_words] uint64.
 *   v may be NULL: r_out is then the truncated product alone (the standalone sparse x dense
 *   product of BASELINE configs[4]). Constant-flow (fixed loop counts, R#8); the environment
 *   variable HQC_S1_KERNEL=3 selects a faster tensor-memory kernel whose loop counts depend on
 *   y. */
int hqc_sparse_dense_mul_batch(const hqc_params *p, const uint64_t *u, const uint32_t *y_support,
                               const uint64_t *v, uint64_t *r_out, size_t batch, void *stream);

/* Stage 2 alone: sym_out[b][j] = RM-decode(bits [j*n2, (j+1)*n2) of r[b]), j < n1 (R#9-R#11).
 *   r [batch][v_words] uint64 -> sym_out [batch][n1] uint8. */
int hqc_rm_decode_batch(const hqc_params *p, const uint64_t *r, uint8_t *sym_out, size_t batch,
                        void *stream);

/* Stage 3 alone: m_out[b] = RS-decode(sym[b]) (bounded-distance decoding, R#7).
 *   sym [batch][n1] uint8 -> m_out [batch][k] uint8; ok_out [batch] (nullable) = 1 if a codeword
 *   within distance delta was found (and corrected), else 0 (m_out = sym[b][0..k)). */
int hqc_rs_decode_batch(const hqc_params *p, const uint8_t *sym, uint8_t *m_out, size_t batch,
                        void *stream);
int hqc_rs_decode_batch_ex(const hqc_params *p, const uint8_t *sym, uint8_t *m_out,
                           uint8_t *ok_out, size_t batch, void *stream);

/* Step a6 alone (§8(f) row 4): syn_out[b][i-1] = S_i = sum_{j<n1} sym[b][j] alpha^{i j},
 * i = 1..2delta (readings R#4, R#5). sym [batch][n1] uint8 -> syn_out [batch][2 delta] uint8.
 * method selects how the GF(2^8) products are formed; all give the same bytes:
 *   0 = GF(2)-linear map with constant-bank tables (the fused kernel's method),
 *   1 = the paper's nibble-sliced tables (two 16-entry lookups per byte, "hi XOR lo") in shared
 *       memory, 4 syndromes per 32-bit entry,
 *   2 = log/antilog tables in shared memory.
 * An unknown method returns HQC_ERR_SIZE. */
int hqc_rs_syndromes_batch(const hqc_params *p, const uint8_t *sym, uint8_t *syn_out, size_t batch, int method,
                           void *stream);

/* Helpers for tests and the bench.
 * hqc_count_mismatch: *d_count += #{b : m_out[b] != m_ref[b]} (d_count: one device uint64, the
 *   caller zeroes it). hqc_validate_support: *d_bad += #{rows with an entry >= n or a repeated
 *   entry among the first w}. Same pointer rules as every entry point (non-NULL, 16-byte aligned). */
int hqc_count_mismatch(const hqc_params *p, const uint8_t *m_out, const uint8_t *m_ref,
                       size_t batch, unsigned long long *d_count, void *stream);
int hqc_validate_support(const hqc_params *p, const uint32_t *y_support, size_t batch,
                         unsigned long long *d_bad, void *stream);

/* ---------------------------------------------------------------------------------------------
 * the KeyGen product and batched Encrypt on the GPU (used by bench.py to
 * build valid ciphertexts on the device; parity-tested against the oracle).
 * hqc_keygen_batch (Alg. 3):  s[i] = x[i] + h[i]*y[i]
 *   h [nkeys][u_stride] uint64 (bits >= n ignored), x, y [nkeys][y_stride] uint32 (first w used),
 *   s_out [nkeys][u_stride] uint64 (bits >= n and padding words written as zero).
 * hqc_encrypt_batch (Alg. 1):  u = r1 + h*r2,  v = trunc_{n1 n2}(mG + s*r2 + e)
 *   h, s [nkeys][u_stride] (the public key of each ciphertext, rows selected by key_index[b], or row b
 *   when key_index is NULL; PRECONDITION key_index[b] < nkeys (or batch <= nkeys without key_index),
 *   unchecked: the ABI carries no key count and the indices are device data — the Python binding checks
 *   them), m [batch][k], r1, r2, e [batch][e_stride] uint32 (first wr used, distinct,
 *   < n), u_out [batch][u_stride], v_out [batch][v_words]. mG is the concatenated RS/RM encoding of m
 *   (message-first RS by the table-driven LFSR of §III.D, duplicated RM(1,7) per R#9/R#12).
 * ------------------------------------------------------------------------------------------- */
int hqc_keygen_batch(const hqc_params *p, const uint64_t *h, const uint32_t *x, const uint32_t *y,
                     uint64_t *s_out, size_t nkeys, void *stream);
int hqc_encrypt_batch(const hqc_params *p, const uint64_t *h, const uint64_t *s,
                      const uint32_t *key_index, const uint8_t *m, const uint32_t *r1,
                      const uint32_t *r2, const uint32_t *e, uint64_t *u_out, uint64_t *v_out,
                      size_t batch, void *stream);

/* ---------------------------------------------------------------------------------------------
 * batched HQC.KEM with the HHK transform and implicit rejection (Decap
 * "decrypts the ciphertext (calling Decrypt), and then re-encrypts to verify correctness, and
 * securely rejects invalid ciphertexts"). The paper gives no byte-level hash inputs; this library
 * follows DESIGN.md readings R#20-R#23 (SHAKE256 = FIPS 202 XOF; tags G=0x01, H=0x02, K=0x03,
 * PRNG=0x04 appended to the hashed bytes):
 *   H_pk  = SHAKE256(h bytes || s bytes || 0x02, 32)     h, s serialised as ceil(n/8) LE bytes
 *   theta = SHAKE256(H_pk || m || 0x01, 32)
 *   (r1, r2, e) = fixed-weight sampling of SHAKE256(theta || 0x04, 12 wr) (3 wr LE uint32 words)
 *   c     = u bytes (ceil(n/8)) || v bytes (n1 n2 / 8)
 *   Encaps:  (u, v) = Encrypt(pk, m; r1, r2, e),  K = SHAKE256(m || c || 0x03, 64)
 *   Decaps:  m' = Decrypt(y, c); c' = Encrypt(pk, m'; coins(m')); K = SHAKE256((c' == c ? m' : sigma)
 *            || c || 0x03, 64). c' == c byte-wise over the serialized length: bits [n, 8 ceil(n/8))
 *            of a received u are part of c (a ciphertext with any of them set is rejected); the row's
 *            words beyond the ceil(n/8) u bytes are not part of c and are ignored.
 * Layouts: h, s [nkeys][u_stride] uint64 (rows as written by hqc_keygen_batch), hpk [nkeys][32],
 * sigma [nkeys][k], y_support [nkeys][y_stride] (per KEY), key_index [batch] uint32 (NULL = row b
 * uses key b; the precondition key_index[b] < nkeys of hqc_encrypt_batch applies), m [batch][k], u [batch][u_stride], v [batch][v_words], K_out [batch][64],
 * accepted_out [batch] uint8 (nullable; 1 = c' == c). d_work: caller-owned device scratch of at
 * least hqc_kem_workspace_bytes(p, batch) bytes (else HQC_ERR_SIZE); it holds m', the sampled
 * supports and the comparison flags and may be reused once the stream has passed the call.
 * Encaps takes m from the caller (the message draw is the caller's randomness).
 * ------------------------------------------------------------------------------------------- */
/* KeyGen from seeds (Alg. 3; reading R#24), one key per seed:
 *   (seed_sk || seed_pk) = SHAKE256(seed || 0x04, 64)
 *   h     = SHAKE256(seed_pk || 0x04, ceil(n/8)) as LE bits, bits >= n cleared
 *   SHAKE256(seed_sk || 0x04, 8w + k) -> x = sample(u32 words 0..w), y = sample(words w..2w) with the
 *           fixed-weight sampler of R#22, sigma = bytes [8w, 8w + k)
 *   s     = x + h*y (the product of hqc_keygen_batch); hpk = H_pk (as hqc_kem_hpk_batch) if hpk_out != NULL
 * seeds [nkeys][32] uint8; h_out, s_out [nkeys][u_stride] uint64 (padding words zero); x_out, y_out
 * [nkeys][y_stride] uint32 (entries >= w zero; positions distinct, in [0, n), unsorted); sigma_out
 * [nkeys][k]; hpk_out [nkeys][32] (nullable). All device pointers, 16-byte aligned; nkeys = 0 is a no-op. */
int hqc_kem_keygen_batch(const hqc_params *p, const uint8_t *seeds, uint64_t *h_out, uint32_t *x_out,
                         uint32_t *y_out, uint64_t *s_out, uint8_t *sigma_out, uint8_t *hpk_out, size_t nkeys,
                         void *stream);
size_t hqc_kem_workspace_bytes(const hqc_params *p, size_t batch);
int hqc_kem_hpk_batch(const hqc_params *p, const uint64_t *h, const uint64_t *s, uint8_t *hpk_out,
                      size_t nkeys, void *stream);
int hqc_kem_encaps_batch(const hqc_params *p, const uint64_t *h, const uint64_t *s, const uint8_t *hpk,
                         const uint32_t *key_index, const uint8_t *m, uint64_t *u_out, uint64_t *v_out,
                         uint8_t *K_out, size_t batch, void *d_work, size_t work_bytes, void *stream);
int hqc_kem_decaps_batch(const hqc_params *p, const uint64_t *h, const uint64_t *s, const uint8_t *hpk,
                         const uint8_t *sigma, const uint32_t *key_index, const uint32_t *y_support,
                         const uint64_t *u, const uint64_t *v, uint8_t *K_out, uint8_t *accepted_out,
                         size_t batch, void *d_work, size_t work_bytes, void *stream);

/* ---------------------------------------------------------------------------------------------
 * Host-buffer decrypt (the end-to-end call): u_h, v_h, y_h, m_h are HOST arrays in the layouts of
 * hqc_decrypt_batch (page-locked memory recommended; pageable memory works but copies synchronously).
 * The batch is processed in chunks of `chunk` ciphertexts (0 = 8192) on two internal streams so that
 * the H2D copy of chunk i+1, the fused kernel on chunk i and the D2H copy of chunk i-1 overlap.
 * d_work: caller-owned DEVICE workspace of at least hqc_decrypt_host_workspace_bytes(p, chunk)
 * bytes (else HQC_ERR_SIZE). Asynchronous with respect to the host: the work is ordered after prior
 * work on `stream` and later work on `stream` waits for it; m_h is valid after synchronising `stream`.
 * ------------------------------------------------------------------------------------------- */
size_t hqc_decrypt_host_workspace_bytes(const hqc_params *p, size_t chunk);
int hqc_decrypt_batch_host(const hqc_params *p, const uint64_t *u_h, const uint64_t *v_h,
                           const uint32_t *y_h, uint8_t *m_h, size_t batch, void *d_work,
                           size_t work_bytes, size_t chunk, void *stream);

/* ---------------------------------------------------------------------------------------------
 * Serialized-ciphertext host call (the server-side end-to-end path): ct_h is a HOST array of batch
 * ciphertexts in the serialized layout c = u bytes (ceil(n/8), LE bits) || v bytes (n1 n2 / 8), i.e.
 * hqc_ct_bytes(p) bytes each (4,417 for HQC-1), back to back with no padding; key_h (HOST,
 * [batch] uint32, nullable only when nkeys == 1) selects each ciphertext's key; y_keys is a DEVICE
 * table [nkeys][y_stride] uint32 of the keys' supports (provisioned once; it stays resident); m_h is
 * the HOST output [batch][k]. Per chunk of `chunk` ciphertexts (0 = 8192) the library copies the
 * bytes and key indices in, unpacks them into the rows of hqc_decrypt_batch on the device
 * (k_unpack_ct), runs the fused kernel and copies m out, pipelined over two internal streams.
 * Key indices are host data here and are checked before anything is enqueued: an index >= nkeys
 * returns HQC_ERR_SIZE. d_work: DEVICE
 * workspace of at least hqc_decrypt_ct_host_workspace_bytes(p, chunk) bytes. Stream semantics as
 * hqc_decrypt_batch_host.
 * ------------------------------------------------------------------------------------------- */
size_t hqc_ct_bytes(const hqc_params *p);
size_t hqc_decrypt_ct_host_workspace_bytes(const hqc_params *p, size_t chunk);
int hqc_decrypt_ct_batch_host(const hqc_params *p, const uint8_t *ct_h, const uint32_t *key_h,
                              const uint32_t *y_keys, size_t nkeys, uint8_t *m_h, size_t batch, void *d_work,
                              size_t work_bytes, size_t chunk, void *stream);

/* Number of persistent CTAs / warps the fused kernel launches for `batch` on the current device
 * (introspection for the bench's launch accounting). Returns HQC_OK. */
int hqc_decrypt_launch_shape(const hqc_params *p, size_t batch, int *grid, int *warps_per_cta);
/* Which fused kernel hqc_decrypt_batch runs for `batch`: 1 = k_decrypt_w1 (one warp
 * per ciphertext range, lane-per-word RS), 2 = k_decrypt (warp pair), 3 = k_decrypt_ws (warp-specialised),
 * 4 = k_decrypt_t (tensor-memory product, opt-in), 5 = k_decrypt_sb (one warp per ciphertext, warp-parallel
 * RS), 6 = k_decrypt_wd (k_decrypt_w1 with CTA-shared work), 7 = k_decrypt_sp (a warp pair per ciphertext,
 * small batches), 8 = k_decrypt_wl (compact warps, CTA-shared work, lane-per-word RS), 9 = k_decrypt_wl with
 * static ranges, 10 = k_decrypt_s12 + k_stage3 (stages 1+2, then stage 3 lane-per-word: two launches);
 * negative hqc_status on error. The default depends on the level and the batch; the environment variable
 * HQC_DEC_KERNEL=1..10 forces one (tests, experiments). */
int hqc_decrypt_launch_kernel(const hqc_params *p, size_t batch);
/* How many kernel launches hqc_decrypt_batch makes for `batch` (a large batch runs as consecutive
 * launches of at most a per-level size; kernel 10 is two launches per part); negative
 * hqc_status on error. */
long long hqc_decrypt_launch_count(const hqc_params *p, size_t batch);

#ifdef __cplusplus
}
#endif
#endif /* HQC_GPU_H */
