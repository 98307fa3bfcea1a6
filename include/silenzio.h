/*
 * silenzio.h -- C ABI of the B200-native batched TFHE PBS library that runs the
 * data-parallel hot path of Silenzio (arXiv 2504.17785).
 *
 * The paper evaluates every non-linear step of its integer training circuit as
 * a TFHE programmable-bootstrapping table lookup (§II-C1 l.101 "TFHE's
 * programmable bootstrapping (PBS)"; §III-D l.257 lookupComp /
 * multivariateLookupComp) on integers of at most 8 bits, plus linear
 * add/sub/scalar-mul (l.101). The paper contains no TFHE internals (it cites
 * CGGI, l.48); the conventions used here are SURVEY.md §8(c) C1-C8 and are
 * listed as readings R1-R21 in DESIGN.md.
 *
 * Conventions for every entry point:
 *  - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *    unless the name ends in _host. The caller owns all memory; the library
 *    allocates nothing and keeps no per-call state. The only process-wide
 *    state is a read-only table of FFT twiddles, built once per device.
 *  - Torus elements are uint64_t (q = 2^64, wrapping). LWE ciphertexts are
 *    mask-then-body, row-major: [count][dim+1].
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All calls are stream-ordered and asynchronous; kernel faults surface at
 *    the caller's next synchronisation.
 *  - Return 0 (SILENZIO_OK) or a negative silenzio_status. No exceptions cross
 *    the ABI. No CPU fallback exists: if a shape is not supported by a kernel,
 *    SILENZIO_ERR_UNSUPPORTED is returned and nothing is launched.
 *  - Deterministic: same inputs give bit-identical outputs (fixed reduction
 *    order, no floating-point atomics).
 */
#ifndef SILENZIO_H
#define SILENZIO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t lwe_dim;      /* n, small-key LWE dimension            742 | 900 | 1024 */
  uint32_t glwe_dim;     /* k (only k = 1 is supported)           1 */
  uint32_t poly_size;    /* N, power of two                       2048 | 8192 | 32768 */
  uint32_t pbs_base_log; /* log2 B_pbs                            23 | 15 | 15 */
  uint32_t pbs_level;    /* l                                     1 | 2 | 2 */
  uint32_t ks_base_log;  /* log2 B_ks                             3 | 4 | 4 */
  uint32_t ks_level;     /* l_ks                                  5 | 4 | 5 */
  uint32_t ks_in_dim;    /* KS input dimension (k*N of the producing set) */
  uint32_t fft_limbs;    /* P in {1,2,3}: signed limbs per Fourier BSK coefficient */
  uint32_t limb_bits;    /* width of the low limbs; the top limb takes 64-(P-1)*limb_bits */
} silenzio_params;

typedef enum {
  SILENZIO_OK = 0,
  SILENZIO_ERR_INVALID_PARAM = -1, /* inconsistent or out-of-range parameter */
  SILENZIO_ERR_UNSUPPORTED = -2,   /* valid TFHE parameters no kernel implements */
  SILENZIO_ERR_NULL_POINTER = -3,
  SILENZIO_ERR_MISALIGNED = -4,    /* pointer not aligned: 16 B for the Fourier BSK and workspaces
                                      (vector / bulk-copy access), the element size (8 B u64, 4 B u32)
                                      for ciphertext, LUT, KSK and id arrays (rows of k*N+1 words
                                      cannot all be 16-byte aligned) */
  SILENZIO_ERR_COUNT = -5,         /* count = 0 where not allowed, or overflow */
  SILENZIO_ERR_WINDOW = -6,        /* gadget driver: value window larger than a PBS can evaluate */
  SILENZIO_ERR_CUDA = -7,          /* a CUDA launch / runtime call failed */
  SILENZIO_ERR_WORKSPACE = -8      /* workspace missing or too small */
} silenzio_status;

const char *silenzio_status_string(int status);
/* Library version string (build id). */
const char *silenzio_version(void);

/* ---------------------------------------------------------------- sizing */
/* Bytes of the Fourier-domain bootstrapping key: n*(k+1)l*(k+1)*P*(N/2)*16. */
size_t silenzio_fourier_bsk_bytes(const silenzio_params *params);
/* Bytes of workspace silenzio_pbs_batch needs for `count` ciphertexts
 * (the keyswitched small-key LWEs, count*(n+1)*8, rounded up, plus the
 * blind-rotation workspace). */
size_t silenzio_pbs_workspace_bytes(const silenzio_params *params, size_t count);

/* Number of kernel launches silenzio_pbs_batch makes for `count` ciphertexts:
 * the keyswitch (tensor-core path: KSK byte-plane preparation + digit matrix
 * and GEMM per 65535 x 128 ciphertexts; CUDA-core path: one) plus the blind
 * rotation (N = 2048, level 1: one persistent launch; otherwise one launch per
 * resident wave, all CTAs of a wave sweeping the Fourier BSK together).
 * -1 if the parameters are unsupported. */
long silenzio_pbs_launch_count(const silenzio_params *params, size_t count);

/* ------------------------------------------------------- hot-path calls */
/* BSK -> Fourier (offline, once per key).
 *  bsk          [n][(k+1)l][k+1][N] u64, standard domain (GGSW of s_i, C6).
 *  fourier_bsk  opaque, silenzio_fourier_bsk_bytes() bytes: each coefficient is
 *               lifted to a signed integer, split into P signed limbs, folded
 *               with the negacyclic twist and transformed with the same f64 FFT
 *               the blind rotation uses, pre-scaled by 2/N. Layout is tiled to
 *               the blind-rotation thread mapping (not user-visible). */
int silenzio_bsk_to_fourier(const uint64_t *bsk, void *fourier_bsk,
                            const silenzio_params *params, void *stream);

/* Device bytes of the keyswitch workspace for `count` ciphertexts: the KSK
 * split into byte planes and the int8 digit matrix, both in the tensor-core
 * operand layout (63 MB + count x 10 KiB at set A); 0 when the parameters do
 * not admit the tensor-core path (digits must fit int8: ks_base_log <= 7, and
 * ks_in_dim * l_ks * 2^(ks_base_log-1) * 255 < 2^31). */
size_t silenzio_keyswitch_workspace_bytes(const silenzio_params *params, size_t count);

/* LWE keyswitch big key -> small key.
 *  lwe_in  [count][ks_in_dim+1], ksk [ks_in_dim][l_ks][n+1], lwe_out [count][n+1].
 *  out = (0,...,0,b) - sum_j sum_t Dec_t(a_j) * KSK[j][t], exact mod 2^64.
 *  workspace: >= silenzio_keyswitch_workspace_bytes(params, count) device
 *  bytes, 16-byte aligned, or NULL. With a workspace the product runs on the tensor cores
 *  (tcgen05 int8 MMA over the KSK byte planes, re-derived from ksk on every
 *  call); without one (or when the byte count is 0) on the CUDA cores. Both
 *  are exact, so the result is identical. */
int silenzio_keyswitch_batch(const uint64_t *lwe_in, const uint64_t *ksk, uint64_t *lwe_out,
                             size_t count, const silenzio_params *params, void *workspace,
                             void *stream);

/* Programmable bootstrapping, atomic pattern KS -> MS -> BR -> SE
 * (R1).
 *  lwe_in      [count][kN+1] big-key LWE ciphertexts
 *  lut_ids     [count] u32 index into luts (ids >= num_luts are clamped to 0);
 *              may be NULL (all ciphertexts use luts[0])
 *  luts        [num_luts][N] test polynomials (silenzio_build_testpoly)
 *  fourier_bsk from silenzio_bsk_to_fourier; ksk as in silenzio_keyswitch_batch
 *  lwe_out     [count][kN+1] big-key LWE ciphertexts of LUT(message)
 *  workspace   >= silenzio_pbs_workspace_bytes(params, count) device bytes.
 * lwe_in and lwe_out must not alias. */
int silenzio_pbs_batch(const uint64_t *lwe_in, const uint32_t *lut_ids, const uint64_t *luts,
                       uint32_t num_luts, const void *fourier_bsk, const uint64_t *ksk,
                       uint64_t *lwe_out, size_t count, const silenzio_params *params,
                       void *workspace, void *stream);

/* KSK byte planes, a once-per-key conversion like silenzio_bsk_to_fourier
 * (SURVEY.md §8(a) a1): the keyswitching key split into its 8 byte planes in
 * the tensor-core operand layout, silenzio_ksk_planes_bytes()
 * device bytes (63 MB at set A; 0 when the parameters do not admit the
 * tensor-core keyswitch, in which case silenzio_ksk_to_planes returns
 * SILENZIO_ERR_UNSUPPORTED). planes: 16-byte aligned. */
size_t silenzio_ksk_planes_bytes(const silenzio_params *params);
int silenzio_ksk_to_planes(const uint64_t *ksk, void *planes, const silenzio_params *params,
                           void *stream);

/* PBS of linear combinations, the gadgets' "linear op, then lookup" step as
 * one call (SURVEY.md §8(a) a0 fused into a1):
 *   x_i   = sum_{t<terms} coef[i][t] * in[idx[i][t]] + (0,...,0,cst[i])   mod 2^64
 *   out_i = PBS(x_i; luts[lut_ids[i]])
 * The combination is formed inside the keyswitch's digit-decomposition kernel
 * and never written to memory; the keyswitch uses the prepared byte planes
 * (silenzio_ksk_to_planes). Bit-identical to silenzio_lwe_linear_batch followed
 * by silenzio_pbs_batch.
 *  in        [*][kN+1] big-key LWE; idx [count][terms] u32 rows of `in`,
 *            coef [count][terms] i64, cst [count] u64 or NULL. idx = NULL (then
 *            coef and cst must be NULL too): x_i = in[i], a plain PBS.
 *  lut_ids, luts, num_luts, fourier_bsk, lwe_out as in silenzio_pbs_batch;
 *            lwe_out may alias `in` (every input is consumed by the keyswitch
 *            before the blind rotation writes).
 *  workspace >= silenzio_pbs_linear_workspace_bytes(params, count), 16-byte aligned.
 * SILENZIO_ERR_UNSUPPORTED when the parameters have no tensor-core keyswitch. */
size_t silenzio_pbs_linear_workspace_bytes(const silenzio_params *params, size_t count);
int silenzio_pbs_linear_batch(const uint64_t *in, const uint32_t *idx, const int64_t *coef,
                              const uint64_t *cst, uint32_t terms, const uint32_t *lut_ids,
                              const uint64_t *luts, uint32_t num_luts, const void *fourier_bsk,
                              const void *ksk_planes, uint64_t *lwe_out, size_t count,
                              const silenzio_params *params, void *workspace, void *stream);

/* Blind rotation + sample extraction only (MS -> BR -> SE) of small-key
 * inputs [count][n+1]; output [count][kN+1]. Used to check the stages
 * separately against the oracle, for the literal MS->BR->SE->KS order and for
 * cross-parameter pipelines (set B). `workspace` must hold
 * silenzio_blind_rotate_workspace_bytes(params, count) bytes (0 for N <= 8192,
 * where it may be NULL; N = 32768 keeps each in-flight ciphertext's accumulator
 * and spectra there, 1.75 MiB per ciphertext, at most 48 in flight). */
size_t silenzio_blind_rotate_workspace_bytes(const silenzio_params *params, size_t count);
int silenzio_blind_rotate_batch(const uint64_t *lwe_small, const uint32_t *lut_ids,
                                const uint64_t *luts, uint32_t num_luts, const void *fourier_bsk,
                                uint64_t *lwe_out, size_t count, const silenzio_params *params,
                                void *workspace, void *stream);

/* Same as silenzio_pbs_batch but lwe_in / lwe_out are HOST buffers (pinned
 * memory recommended). Copies are chunked (`chunk` ciphertexts, 0 = auto) and
 * overlapped with compute on two internal streams created per call; the call
 * returns after the last output chunk has landed in host memory (synchronous).
 * workspace must hold silenzio_pbs_host_workspace_bytes(params, chunk).
 * Ordering: the internal streams wait for the work already queued on `stream`
 * (the stream that produced luts / fourier_bsk / ksk / workspace), so the
 * caller needs no synchronisation before the call. */
size_t silenzio_pbs_host_workspace_bytes(const silenzio_params *params, size_t chunk);
int silenzio_pbs_batch_host(const uint64_t *lwe_in_host, const uint32_t *lut_ids_host,
                            const uint64_t *luts, uint32_t num_luts, const void *fourier_bsk,
                            const uint64_t *ksk, uint64_t *lwe_out_host, size_t count,
                            size_t chunk, const silenzio_params *params, void *workspace,
                            void *stream);

/* Linear LWE combination (PAPER.md l.101 linear ops):
 *  out[i] = sum_{t<terms} coef[i][t] * in[idx[i][t]] + (0,...,0,cst[i])  mod 2^64.
 *  in [*][dim+1], idx [count][terms] u32, coef [count][terms] i64,
 *  cst [count] u64 (may be NULL), out [count][dim+1]; out must not alias in. */
int silenzio_lwe_linear_batch(const uint64_t *in, const uint32_t *idx, const int64_t *coef,
                              const uint64_t *cst, uint32_t terms, uint32_t dim, size_t count,
                              uint64_t *out, void *stream);

/* Test polynomial of a LUT:
 *  v' = sum_{j<N} T[floor(j/box)] X^j, box = N / 2^p;  v = X^{-box/2} * v'.
 *  tables [num][2^p] u64 torus values, polys [num][N] u64. */
int silenzio_build_testpoly(const uint64_t *tables, uint32_t num, uint32_t p, uint32_t N,
                            uint64_t *polys, void *stream);

/* ------------------------------------------------------------ gadgets */
/* Encrypted Matmul^RNS (Alg. 2, l.280-307) at
 * parameter set A (N = 2048, 4-bit messages + padding, Delta = 2^59). A thin
 * driver: it only sequences silenzio_lwe_linear_batch and silenzio_pbs_batch
 * calls (schedule: DESIGN.md §Config 3).
 *  X        [a][b] big-key LWE, each an integer in [-8, 8) encoded (x mod 32) Delta
 *  W        [b][c] likewise
 *  moduli   [k], each in {5, 7, 9, 11, 13, 16} (pairwise coprime; else
 *           SILENZIO_ERR_WINDOW: no 16-value PBS window schedule for it)
 *  out      [k][a][c] big-key LWE: residue (X W)_{ij} mod m at scale Delta for
 *           m != 16, and at scale 2^60 for m = 16 (native wrap channel)
 *  workspace >= silenzio_rns_matmul_workspace_bytes(params, a, b, c) device bytes.
 * The call synchronises `stream` internally (host-built index arrays). */
size_t silenzio_rns_matmul_workspace_bytes(const silenzio_params *params, uint32_t a, uint32_t b,
                                           uint32_t c);
int silenzio_rns_matmul(const uint64_t *X, const uint64_t *W, uint32_t a, uint32_t b, uint32_t c,
                        const uint32_t *moduli_host, uint32_t k, uint64_t *out, const void *fourier_bsk,
                        const uint64_t *ksk, const silenzio_params *params, void *workspace,
                        size_t workspace_bytes, void *stream);

/* Config-4 gadgets at parameter set A (DESIGN.md §Config 4). Each call composes
 * linear LWE ops and PBS only. Ciphertext arrays are big-key LWE [*][kN+1];
 * residues / digits / bits are encoded at Delta = 2^59; `moduli_host` must be
 * ascending with every m <= 16 (SILENZIO_ERR_WINDOW otherwise); workspace >=
 * silenzio_gadget_workspace_bytes(params, k, count). Calls synchronise `stream`.
 *  silenzio_rns2mrns        Alg. 1 RNS2MRNS: in [k][count]
 *                           residues -> out [k][count] MRNS digits (least significant first).
 *  silenzio_rns_sign_abs    Sign_(-1,1,1) via the top MRNS digit >= r_k/2 (l.309-323; r_k even)
 *                           -> sign_out [count] in {0 (>= 0), 1 (< 0)}; |x| per residue
 *                           (Alg. 4, l.414-415) -> abs_out [k][count].
 *  silenzio_mrns_bitlen_max Alg. 3 step 2 (l.344-349): bitlen_out [k][count] = bit length of
 *                           every digit; max_out [k] = tensor-wide maximum per digit position.
 *  silenzio_int_ce_grad     Alg. 5 IntCELossDeriv (l.433-450) at Gamma = 4, kappa = 0 (DESIGN
 *                           R10, R12): Yhat [a][b] signed in [-8,8), Y [a][b] one-hot bits,
 *                           b <= 13 -> out [a][b] in {-1, 0, 1}. */
size_t silenzio_gadget_workspace_bytes(const silenzio_params *params, uint32_t k, size_t count);
int silenzio_rns2mrns(const uint64_t *in, const uint32_t *moduli_host, uint32_t k, size_t count,
                      uint64_t *out, const void *fourier_bsk, const uint64_t *ksk,
                      const silenzio_params *params, void *workspace, size_t workspace_bytes,
                      void *stream);
int silenzio_rns_sign_abs(const uint64_t *in, const uint32_t *moduli_host, uint32_t k, size_t count,
                          uint64_t *sign_out, uint64_t *abs_out, const void *fourier_bsk,
                          const uint64_t *ksk, const silenzio_params *params, void *workspace,
                          size_t workspace_bytes, void *stream);
int silenzio_mrns_bitlen_max(const uint64_t *digits, uint32_t k, size_t count, uint64_t *bitlen_out,
                             uint64_t *max_out, const void *fourier_bsk, const uint64_t *ksk,
                             const silenzio_params *params, void *workspace, size_t workspace_bytes,
                             void *stream);
int silenzio_int_ce_grad(const uint64_t *Yhat, const uint64_t *Y, uint32_t a, uint32_t b, uint64_t *out,
                         const void *fourier_bsk, const uint64_t *ksk, const silenzio_params *params,
                         void *workspace, size_t workspace_bytes, void *stream);

/* g7: Shift2MSBs+- digit combine with the 8-bit stage (Alg. 3 steps 3-6, Alg. 4
 * re-sign; DESIGN.md §Config 4). Inputs at set A (pa): top_digit [count] = most
 * significant MRNS digit of x (sign: >= top_radix / 2), abs_digits [k][count] =
 * MRNS digits of |x|, maxes [k] = silenzio_mrns_bitlen_max output. One 8-bit PBS
 * at set B (pb, N = 32768) per element and digit, reached through keyswitches
 * ksk_ab (pab: set-A big key -> set-B small key) and ksk_ba (pba: set-B big key
 * -> set-A big key). Output out [count] = Shift2MSBs+-(x) in [-(2^gamma - 1),
 * 2^gamma - 1] at Delta (set A); maxbit_out [1] = encrypted maxBit at 2^55
 * (shift = maxBit - gamma). */
size_t silenzio_mrns_combine_workspace_bytes(const silenzio_params *pa, const silenzio_params *pb, uint32_t k,
                                             size_t count);
int silenzio_mrns_digit_combine(const uint64_t *top_digit, const uint64_t *abs_digits, const uint64_t *maxes,
                                uint32_t k, size_t count, uint32_t top_radix, uint32_t w, uint32_t gamma,
                                uint64_t *out, uint64_t *maxbit_out, const void *fbsk_a, const uint64_t *ksk_a,
                                const silenzio_params *pa, const void *fbsk_b, const silenzio_params *pb,
                                const uint64_t *ksk_ab, const silenzio_params *pab, const uint64_t *ksk_ba,
                                const silenzio_params *pba, void *workspace, size_t workspace_bytes, void *stream);

/* Shift2MSBs+- (Alg. 4, l.408-423, over Alg. 3 Shift2MSBs+,
 * l.337-374) in one call: residues [k][count] at Delta (set A, moduli
 * ascending, top modulus even) -> out [count] = Shift2MSBs+-(x) in
 * [-(2^gamma - 1), 2^gamma - 1] at Delta, maxbit_out [1] as in
 * silenzio_mrns_digit_combine (w = modulus bit width, gamma = Gamma - 1).
 * Composes RNS2MRNS, sign / abs, RNS2MRNS of |x|, bit lengths + block max and
 * the 8-bit digit combine (parameters and keys as silenzio_mrns_digit_combine);
 * the digits-of-x chain and the |x| chain run concurrently on two streams.
 * workspace >= silenzio_shift2msbs_workspace_bytes(pa, pb, k, count);
 * synchronises `stream`. */
size_t silenzio_shift2msbs_workspace_bytes(const silenzio_params *pa, const silenzio_params *pb, uint32_t k,
                                           size_t count);
int silenzio_shift2msbs_pm(const uint64_t *residues, const uint32_t *moduli_host, uint32_t k, size_t count,
                           uint32_t w, uint32_t gamma, uint64_t *out, uint64_t *maxbit_out, const void *fbsk_a,
                           const uint64_t *ksk_a, const silenzio_params *pa, const void *fbsk_b,
                           const silenzio_params *pb, const uint64_t *ksk_ab, const silenzio_params *pab,
                           const uint64_t *ksk_ba, const silenzio_params *pba, void *workspace,
                           size_t workspace_bytes, void *stream);

/* Training-step gadgets (Alg. 6, l.466-502; SURVEY.md §8(f) NEXT #1;
 * schedules DESIGN.md §6b'', readings R23-R26) at parameter set A. Thin
 * drivers over linear LWE ops and PBS; ciphertext arrays are big-key LWE
 * [*][kN+1] at Delta = 2^59 unless stated; workspace >=
 * silenzio_train_workspace_bytes(params, k, count) (k = 1 except sign3);
 * calls synchronise `stream`; shapes without a 16-value window schedule
 * return SILENZIO_ERR_WINDOW.
 *  silenzio_channel16     in [count]: residue r in [0,16) at 2^60 (the m = 16
 *                         channel of silenzio_rns_matmul) -> out: r at Delta (2 PBS).
 *  silenzio_rns_sign3     Sign^RNS_(-1,0,1) (l.309-323, zero test l.313): residues
 *                         [k][count] at Delta, moduli ascending with 16 last, k <= 7
 *                         -> out [count] in {-1, 0, 1}.
 *  silenzio_relu_cap      ReLU_x(x) = min(max(x, 0), cap) (l.269-274), x in [-8, 8),
 *                         0 <= cap <= 7.
 *  silenzio_relu_mask     out = e [0 < s < cap] for e in {-1, 0, 1}, s in [-8, 8)
 *                         (the ReLU_x derivative applied to an error sign, R25).
 *  silenzio_weight_update out = clip(w - g, wmin, wmax) for w in [wmin, wmax] within
 *                         [-8, 8), g in {-1, 0, 1}; fresh output (identity refresh). */
size_t silenzio_train_workspace_bytes(const silenzio_params *params, uint32_t k, size_t count);
int silenzio_channel16(const uint64_t *in, size_t count, uint64_t *out, const void *fbsk, const uint64_t *ksk,
                       const silenzio_params *params, void *workspace, size_t workspace_bytes, void *stream);
int silenzio_rns_sign3(const uint64_t *residues, const uint32_t *moduli_host, uint32_t k, size_t count,
                       uint64_t *out, const void *fbsk, const uint64_t *ksk, const silenzio_params *params,
                       void *workspace, size_t workspace_bytes, void *stream);
int silenzio_relu_cap(const uint64_t *in, size_t count, int32_t cap, uint64_t *out, const void *fbsk,
                      const uint64_t *ksk, const silenzio_params *params, void *workspace, size_t workspace_bytes,
                      void *stream);
int silenzio_relu_mask(const uint64_t *e, const uint64_t *s, size_t count, int32_t cap, uint64_t *out,
                       const void *fbsk, const uint64_t *ksk, const silenzio_params *params, void *workspace,
                       size_t workspace_bytes, void *stream);
int silenzio_weight_update(const uint64_t *w, const uint64_t *g, size_t count, int32_t wmin, int32_t wmax,
                           uint64_t *out, const void *fbsk, const uint64_t *ksk, const silenzio_params *params,
                           void *workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------- client-side key / ciphertext generation
 * All random numbers are inputs (drawn by the caller), so every key and
 * ciphertext is a deterministic function of the caller's seeded draws. */
/* out[c] = (mask[c], <mask[c], key> + noise[c] + plaintext[c])  (C2). */
int silenzio_lwe_encrypt_batch(const uint64_t *mask, const int64_t *noise,
                               const uint64_t *plaintext, const uint64_t *key, uint32_t dim,
                               size_t count, uint64_t *out, void *stream);
/* phase[c] = b - <a, key>  (C2). */
int silenzio_lwe_phase_batch(const uint64_t *ct, const uint64_t *key, uint32_t dim, size_t count,
                             uint64_t *phase, void *stream);
/* GGSW bootstrapping key (C6): mask [n][(k+1)l][k][N], noise [n][(k+1)l][N],
 * lwe_key [n] in {0,1}, glwe_key [k][N] in {0,1} -> bsk [n][(k+1)l][k+1][N].
 * N = 32768 computes the GLWE bodies with an exact limb-split FFT and needs
 * silenzio_bsk_generate_workspace_bytes() of workspace (0 otherwise; NULL ok). */
size_t silenzio_bsk_generate_workspace_bytes(const silenzio_params *params);
int silenzio_bsk_generate(const uint64_t *lwe_key, const uint64_t *glwe_key, const uint64_t *mask,
                          const int64_t *noise, uint64_t *bsk, const silenzio_params *params,
                          void *workspace, void *stream);
/* Keyswitching key (C3): KSK[j][t] = LWE_s(s_in[j] * 2^{64 - t*base_log}),
 * mask [in_dim][level][n], noise [in_dim][level] -> ksk [in_dim][level][n+1]. */
int silenzio_ksk_generate(const uint64_t *in_key, const uint64_t *lwe_key, const uint64_t *mask,
                          const int64_t *noise, uint64_t *ksk, uint32_t in_dim, uint32_t n,
                          uint32_t base_log, uint32_t level, void *stream);

/* ------------------------------------------ sampled-PBS trace (test / debug)
 * The gadget drivers evaluate their PBS internally; an oracle replay of a
 * sample of them ("Replay 1 024 sampled PBS" of configs 3 and
 * 4) needs their inputs. While a trace of `kind` is active, every `stride`-th
 * PBS element (global element counter across calls, offset `phase` < stride)
 * evaluated by that kind of call site is copied, stream-ordered, into
 * `records` (DEVICE, [max_records][in_words + out_words + lut_words + 2] u64):
 *   [input LWE][output LWE][test polynomial][global element index, lut id].
 * kind 0: set-A PBS of the gadget drivers (in/out: big-key LWE, k*N+1 words;
 *         lut: N words). kind 1: the set-B blind rotation + sample extraction
 *         of the 8-bit stage (in: set-B small-key LWE, n+1 words; out: set-B
 *         big-key LWE, k*N+1 words; lut: N words).
 * Records whose sizes do not match the call site are skipped (counted only).
 * Process-wide state (one trace per kind, mutex-guarded); off by default,
 * and the drivers' results do not depend on it. end() stops the trace and
 * returns the number of records written (or a negative status), and the
 * number of elements seen through `elements_seen` (may be NULL). */
int silenzio_pbs_trace_begin(int kind, uint64_t *records, size_t max_records, uint64_t stride, uint64_t phase,
                             size_t in_words, size_t out_words, size_t lut_words);
long silenzio_pbs_trace_end(int kind, uint64_t *elements_seen);

/* Debug builds only (-DSZ_FFT_MARGIN=1, tools/fft_margin.py): per limb p < 3,
 * over every limb value the set-A blind rotations rounded since the last call
 * (R20: exact while the FFT error < 1/2 and |x| < 2^51):
 * out[4p] = max |x - round(x)|, out[4p+1] = max |x|, out[4p+2] = number of
 * values with |x - round(x)| >= 1/4, out[4p+3] = number >= 1/2; resets them.
 * Release builds return SILENZIO_ERR_UNSUPPORTED. */
int silenzio_debug_fft_margin(double *out);
/* Debug builds only (-DSZ_PHASE_TIMING=1, tools/phase_times.py): clock64 cycles
 * accumulated per phase of the set-A CMux loop, out[warp][phase] (8 x 8, CTA 0,
 * phases: publish, digits, forward FFT, spectra exchange, stage wait, MAC,
 * inverse FFT, recombination; for batches the latency kernel takes,
 * tools/phase_times_lat.py names its phases); resets them. Release builds:
 * UNSUPPORTED. */
int silenzio_debug_phase_times(unsigned long long *out);
/* The same for the set-B (N = 32768) cluster kernel: out[12] cycles per phase
 * of CTA 0 thread 0 (forward free-wait, digits + radix-4 + sends, forward
 * full-wait, block FFT, MAC, block IFFT, inverse free-wait, sends, inverse
 * full-wait, combine + ACC update). Release builds: UNSUPPORTED. */
int silenzio_debug_phase_times_b(unsigned long long *out);

#ifdef __cplusplus
}
#endif
#endif /* SILENZIO_H */
