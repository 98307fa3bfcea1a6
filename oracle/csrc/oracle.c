/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU reference of the TFHE operations on the
 * Silenzio hot path (batched programmable bootstrapping, §II-C1 l.101
 * "TFHE's programmable bootstrapping (PBS)", and the lookups of §III-D l.257).
 * The paper gives no TFHE internals (it cites CGGI, and only
 * lists KeyGen/Enc/Eval/Dec abstractly, l.90-98), so every step below follows
 * the reading fixed in SURVEY.md §8(c) C1-C8 and listed in DESIGN.md §Readings.
 *
 * Everything is exact integer arithmetic mod 2^64 (uint64_t wraps). Polynomial
 * products are schoolbook negacyclic (N^2 multiply-adds, sign flip on wrap):
 * no FFT, no blocking, no reordering of the arithmetic. OpenMP splits
 * independent ciphertexts (or key rows) across threads; at N >= 8192 a batch
 * smaller than the thread count instead splits the N^2 terms of each external
 * product into private partial sums added afterwards (exact: integer addition mod 2^64 is
 * associative and commutative, so the result is bit-identical).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library. It shares no code with paper_2504_17785_b200/.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;
typedef int64_t i64;

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* out += a * b  in Z_{2^64}[X]/(X^N + 1), schoolbook.
 * Term a_i b_j lands on X^{i+j}; if i+j >= N it wraps to X^{i+j-N} with a
 * minus sign because X^N = -1.  (SURVEY.md §8(c) C6 "schoolbook negacyclic
 * mod 2^64: N^2 u64 MACs with sign flip on wrap".)
 * _part adds only the terms with i in [i0, i1), so that the N^2 terms of one
 * product can be split across threads (the sum mod 2^64 does not depend on
 * the order in which the terms are added). */
#if defined(__x86_64__) && defined(__GNUC__) && !defined(__clang__)
__attribute__((target_clones("arch=x86-64-v4", "arch=x86-64-v3", "default")))
#endif
void oracle_negacyclic_mac_part(u64 *out, const u64 *a, const u64 *b, int N, int i0, int i1) {
  for (int i = i0; i < i1; i++) {
    const u64 ai = a[i];
    if (ai == 0) continue; /* exact: a zero term adds nothing */
    for (int j = 0; j < N - i; j++) out[i + j] += ai * b[j];
    for (int j = N - i; j < N; j++) out[i + j - N] -= ai * b[j];
  }
}

/* The full product: the terms a_i b_j for every i (the sum above over i in [0, N)). */
void oracle_negacyclic_mac(u64 *out, const u64 *a, const u64 *b, int N) {
  oracle_negacyclic_mac_part(out, a, b, N, 0, N);
}

/* out = X^e * in, e in [0, 2N) (negacyclic rotation; X^N = -1). */
void oracle_rotate(u64 *out, const u64 *in, int N, int e) {
  const int twoN = 2 * N;
  e %= twoN;
  if (e < 0) e += twoN;
  for (int j = 0; j < N; j++) {
    int idx = j + e; /* X^j * X^e = X^{j+e} */
    if (idx >= twoN) idx -= twoN;
    if (idx < N) out[idx] = in[j];
    else out[idx - N] = (u64)0 - in[j];
  }
}

/* Signed gadget decomposition (R3/R4):
 *   r = floor((a + 2^{63-l*beta}) / 2^{64-l*beta}) mod 2^{l*beta}
 *   for t = l..1: d_t = r mod 2^beta; r >>= beta;
 *                 if d_t >= 2^{beta-1}: d_t -= 2^beta, r += 1
 *   (final carry dropped).  digits[t-1] holds d_t; d_t has weight q/B^t.
 * Edge case l*beta = 64: nothing to round, r = a. */
void oracle_decompose(u64 a, int base_log, int level, i64 *digits) {
  const int lb = base_log * level;
  u64 r;
  if (lb >= 64) r = a;
  else r = (a + ((u64)1 << (63 - lb))) >> (64 - lb);
  const u64 mask = (base_log >= 64) ? ~(u64)0 : (((u64)1 << base_log) - 1);
  const i64 half = (i64)1 << (base_log - 1);
  for (int t = level; t >= 1; t--) {
    i64 d = (i64)(r & mask);
    r = (base_log >= 64) ? 0 : (r >> base_log);
    if (d >= half) {
      d -= (i64)1 << base_log;
      r += 1;
    }
    digits[t - 1] = d;
  }
}

/* Modulus switch to 2N: round half up by
 * add-half-then-shift, wrapping mod 2N.  log2_2N = log2(N) + 1. */
u64 oracle_modswitch(u64 a, int log2_2N) {
  return (a + ((u64)1 << (63 - log2_2N))) >> (64 - log2_2N);
}

/* Fresh LWE encryption:
 *   b = <a, s> + e + plaintext  (mod 2^64); ciphertext = (a_0..a_{dim-1}, b). */
void oracle_lwe_encrypt(const u64 *mask, const i64 *noise, const u64 *plaintext,
                        const u64 *key, int dim, long count, u64 *out) {
#pragma omp parallel for schedule(static)
  for (long c = 0; c < count; c++) {
    const u64 *a = mask + (size_t)c * dim;
    u64 *o = out + (size_t)c * (dim + 1);
    u64 b = 0;
    for (int i = 0; i < dim; i++) {
      o[i] = a[i];
      b += a[i] * key[i];
    }
    o[dim] = b + (u64)noise[c] + plaintext[c];
  }
}

/* Phase b - <a, s> of `count` LWE ciphertexts. */
void oracle_lwe_phase(const u64 *ct, const u64 *key, int dim, long count, u64 *phase) {
#pragma omp parallel for schedule(static)
  for (long c = 0; c < count; c++) {
    const u64 *a = ct + (size_t)c * (dim + 1);
    u64 acc = 0;
    for (int i = 0; i < dim; i++) acc += a[i] * key[i];
    phase[c] = a[dim] - acc;
  }
}

/* Bootstrapping key = n GGSW encryptions of the small-key bits s_i under the
 * GLWE key S:
 *   row (r, j), r in [0,k], j in [1,l]: GLWE_S(0) + s_i * q/B^j added to
 *   component r (mask r for r < k, body for r = k).
 *   GLWE_S(0) = (A_0..A_{k-1}, B = sum_m A_m*S_m + E).
 * Layouts: mask [n][(k+1)l][k][N], noise [n][(k+1)l][N], out [n][(k+1)l][k+1][N]. */
void oracle_bsk_generate(const u64 *lwe_key, const u64 *glwe_key, const u64 *mask,
                         const i64 *noise, int n, int k, int N, int base_log,
                         int level, u64 *bsk) {
  const int rows = (k + 1) * level;
#pragma omp parallel for schedule(dynamic)
  for (long ir = 0; ir < (long)n * rows; ir++) {
    const int i = (int)(ir / rows), row = (int)(ir % rows);
    const int r = row / level, j = row % level + 1;
    const u64 *A = mask + (size_t)ir * k * N;
    const i64 *E = noise + (size_t)ir * N;
    u64 *G = bsk + (size_t)ir * (k + 1) * N;
    u64 *body = G + (size_t)k * N;
    for (int m = 0; m < k; m++) memcpy(G + (size_t)m * N, A + (size_t)m * N, sizeof(u64) * N);
    for (int c = 0; c < N; c++) body[c] = (u64)E[c];
    for (int m = 0; m < k; m++)
      oracle_negacyclic_mac(body, glwe_key + (size_t)m * N, A + (size_t)m * N, N);
    const int shift = 64 - j * base_log; /* q / B^j = 2^{64 - j*beta} */
    G[(size_t)r * N] += lwe_key[i] << shift;
  }
}

/* Keyswitching key:
 *   KSK[j][t] = LWE_s(s_big[j] * q/B_ks^t), t = 1..l_ks, sigma_LWE.
 * Layouts: mask [in_dim][l_ks][n], noise [in_dim][l_ks], out [in_dim][l_ks][n+1]. */
void oracle_ksk_generate(const u64 *big_key, const u64 *lwe_key, const u64 *mask,
                         const i64 *noise, int in_dim, int n, int base_log,
                         int level, u64 *ksk) {
#pragma omp parallel for schedule(static)
  for (long jt = 0; jt < (long)in_dim * level; jt++) {
    const int j = (int)(jt / level), t = (int)(jt % level) + 1;
    const u64 *a = mask + (size_t)jt * n;
    u64 *o = ksk + (size_t)jt * (n + 1);
    u64 b = 0;
    for (int i = 0; i < n; i++) {
      o[i] = a[i];
      b += a[i] * lwe_key[i];
    }
    o[n] = b + (u64)noise[jt] + (big_key[j] << (64 - t * base_log));
  }
}

/* Keyswitch big key -> small key:
 *   out = (0,...,0, b') - sum_j sum_t d_{j,t} * KSK[j][t]. */
void oracle_keyswitch(const u64 *in, const u64 *ksk, u64 *out, long count, int in_dim,
                      int n, int base_log, int level) {
#pragma omp parallel for schedule(dynamic)
  for (long c = 0; c < count; c++) {
    const u64 *a = in + (size_t)c * (in_dim + 1);
    u64 *o = out + (size_t)c * (n + 1);
    i64 d[64];
    for (int i = 0; i <= n; i++) o[i] = 0;
    o[n] = a[in_dim];
    for (int j = 0; j < in_dim; j++) {
      oracle_decompose(a[j], base_log, level, d);
      for (int t = 0; t < level; t++) {
        if (d[t] == 0) continue;
        const u64 *row = ksk + ((size_t)j * level + t) * (n + 1);
        const u64 dt = (u64)d[t];
        for (int i = 0; i <= n; i++) o[i] -= dt * row[i];
      }
    }
  }
}

/* Blind rotation of one small-key LWE (n+1 words):
 *   ACC <- (0, ..., 0, X^{-b~} * v)
 *   for i = 0..n-1: ACC <- ACC + ExtProd(BSK_i, X^{a~_i} * ACC - ACC)
 *   ExtProd(G, c) = sum_{r<=k} sum_{j=1..l} Dec_j(c_r) * G[r*l + j-1].
 * acc: (k+1) x N output. */
void oracle_blind_rotate(const u64 *lwe, const u64 *testpoly, const u64 *bsk, int n,
                         int k, int N, int base_log, int level, u64 *acc) {
  int logN = 0;
  while ((1 << logN) < N) logN++;
  const int log2_2N = logN + 1;
  const int K1 = k + 1, rows = K1 * level;
  u64 *rot = (u64 *)malloc(sizeof(u64) * N);
  u64 *diff = (u64 *)malloc(sizeof(u64) * K1 * N);
  u64 *digit_poly = (u64 *)malloc(sizeof(u64) * rows * N);
  u64 *prod = (u64 *)malloc(sizeof(u64) * K1 * N);
  i64 d[64];
  /* a large ring (N >= 8192) outside any parallel region (a few ciphertexts):
   * split each external product across the threads; otherwise stay serial */
  enum { kSplit = 4 };
  const int ntask = rows * K1 * kSplit;
  u64 *part = NULL;
#ifdef _OPENMP
  if (N >= 8192 && !omp_in_parallel() && omp_get_max_threads() > 1) part = (u64 *)malloc(sizeof(u64) * ntask * N);
#endif

  /* ACC init: X^{-b~} * v = X^{2N - b~} * v */
  const u64 bt = oracle_modswitch(lwe[n], log2_2N);
  for (int m = 0; m < k; m++) memset(acc + (size_t)m * N, 0, sizeof(u64) * N);
  oracle_rotate(acc + (size_t)k * N, testpoly, N, (int)((2 * (u64)N - bt) % (2 * (u64)N)));

  for (int i = 0; i < n; i++) {
    const int at = (int)oracle_modswitch(lwe[i], log2_2N);
    /* D_r = X^{a~_i} * ACC_r - ACC_r */
    for (int r = 0; r < K1; r++) {
      oracle_rotate(rot, acc + (size_t)r * N, N, at);
      for (int c = 0; c < N; c++) diff[(size_t)r * N + c] = rot[c] - acc[(size_t)r * N + c];
    }
    /* decompose every coefficient into l signed digits */
    for (int r = 0; r < K1; r++)
      for (int c = 0; c < N; c++) {
        oracle_decompose(diff[(size_t)r * N + c], base_log, level, d);
        for (int j = 0; j < level; j++) digit_poly[((size_t)r * level + j) * N + c] = (u64)d[j];
      }
    /* external product with the GGSW BSK_i */
    memset(prod, 0, sizeof(u64) * K1 * N);
    const u64 *G = bsk + (size_t)i * rows * K1 * N;
    if (!part) {
      for (int row = 0; row < rows; row++)
        for (int o = 0; o < K1; o++)
          oracle_negacyclic_mac(prod + (size_t)o * N, digit_poly + (size_t)row * N,
                                G + ((size_t)row * K1 + o) * N, N);
    } else {
      /* the same terms, split over (row, o, i-range) tasks into private sums
       * (one blind rotation alone, e.g. a single set-B PBS, uses every core) */
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic)
#endif
      for (int t = 0; t < ntask; t++) {
        const int row = t / (K1 * kSplit), o = (t / kSplit) % K1, s = t % kSplit;
        u64 *dst = part + (size_t)t * N;
        memset(dst, 0, sizeof(u64) * N);
        oracle_negacyclic_mac_part(dst, digit_poly + (size_t)row * N, G + ((size_t)row * K1 + o) * N, N,
                                   s * N / kSplit, (s + 1) * N / kSplit);
      }
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
      for (int c = 0; c < N; c++)
        for (int t = 0; t < ntask; t++) prod[(size_t)((t / kSplit) % K1) * N + c] += part[(size_t)t * N + c];
    }
    for (size_t c = 0; c < (size_t)K1 * N; c++) acc[c] += prod[c];
  }
  free(rot);
  free(diff);
  free(digit_poly);
  free(prod);
  free(part);
}

/* Sample extraction of coefficient 0:
 *   a'[jN] = A_j[0]; a'[jN+i] = -A_j[N-i] (i in [1,N)); b' = B[0]. */
void oracle_sample_extract(const u64 *acc, int k, int N, u64 *out) {
  for (int j = 0; j < k; j++) {
    const u64 *A = acc + (size_t)j * N;
    out[(size_t)j * N] = A[0];
    for (int i = 1; i < N; i++) out[(size_t)j * N + i] = (u64)0 - A[N - i];
  }
  out[(size_t)k * N] = acc[(size_t)k * N];
}

/* Atomic pattern PBS(ct) = SE(BR(MS(KS(ct)))) (R1):
 * input and output are big-key LWE ciphertexts [count][kN+1]. */
void oracle_pbs(const u64 *lwe_in, const uint32_t *lut_ids, const u64 *luts, int num_luts,
                const u64 *bsk, const u64 *ksk, u64 *lwe_out, long count, int n, int k,
                int N, int pbs_base_log, int pbs_level, int ks_base_log, int ks_level) {
  const int big = k * N;
#pragma omp parallel for schedule(dynamic) if (count >= oracle_num_threads() || N < 8192)
  for (long c = 0; c < count; c++) {
    u64 *small = (u64 *)malloc(sizeof(u64) * (n + 1));
    u64 *acc = (u64 *)malloc(sizeof(u64) * (k + 1) * N);
    oracle_keyswitch(lwe_in + (size_t)c * (big + 1), ksk, small, 1, big, n, ks_base_log,
                     ks_level);
    uint32_t id = lut_ids ? lut_ids[c] : 0;
    if ((int)id >= num_luts) id = 0;
    oracle_blind_rotate(small, luts + (size_t)id * N, bsk, n, k, N, pbs_base_log, pbs_level,
                        acc);
    oracle_sample_extract(acc, k, N, lwe_out + (size_t)c * (big + 1));
    free(small);
    free(acc);
  }
}

/* Blind rotation + sample extraction only (input already a small-key LWE),
 * used to replay the PBS stage on the keyswitch output the GPU consumed. */
void oracle_br_se(const u64 *lwe_small, const uint32_t *lut_ids, const u64 *luts,
                  int num_luts, const u64 *bsk, u64 *lwe_out, long count, int n, int k,
                  int N, int pbs_base_log, int pbs_level) {
  const int big = k * N;
#pragma omp parallel for schedule(dynamic) if (count >= oracle_num_threads() || N < 8192)
  for (long c = 0; c < count; c++) {
    u64 *acc = (u64 *)malloc(sizeof(u64) * (k + 1) * N);
    uint32_t id = lut_ids ? lut_ids[c] : 0;
    if ((int)id >= num_luts) id = 0;
    oracle_blind_rotate(lwe_small + (size_t)c * (n + 1), luts + (size_t)id * N, bsk, n, k, N,
                        pbs_base_log, pbs_level, acc);
    oracle_sample_extract(acc, k, N, lwe_out + (size_t)c * (big + 1));
    free(acc);
  }
}

/* Linear LWE combination ("linear operations
 * addition, subtraction, and multiplication"):
 *   out[i] = sum_t coef[i][t] * in[idx[i][t]] + (0,...,0,cst[i])   (mod 2^64). */
void oracle_lwe_linear(const u64 *in, const uint32_t *idx, const i64 *coef, const u64 *cst,
                       int terms, int dim, long count, u64 *out) {
#pragma omp parallel for schedule(static)
  for (long i = 0; i < count; i++) {
    u64 *o = out + (size_t)i * (dim + 1);
    for (int c = 0; c <= dim; c++) o[c] = 0;
    for (int t = 0; t < terms; t++) {
      const u64 *src = in + (size_t)idx[(size_t)i * terms + t] * (dim + 1);
      const u64 w = (u64)coef[(size_t)i * terms + t];
      for (int c = 0; c <= dim; c++) o[c] += w * src[c];
    }
    o[dim] += cst ? cst[i] : 0;
  }
}
