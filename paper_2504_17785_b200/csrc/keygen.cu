// keygen.cu -- client-side key and ciphertext generation, test polynomials and
// linear LWE combinations (all exact integer arithmetic mod 2^64).
// Random numbers (masks, noise) are inputs; see silenzio.h.
#include "common.cuh"

namespace sz {

// ---------------------------------------------------------------- LWE encrypt
// out[c] = (mask[c], <mask[c], key> + noise[c] + plaintext[c])   (C2)
// one warp per ciphertext, fixed reduction order (deterministic).
__global__ void lwe_encrypt_kernel(const u64 *mask, const i64 *noise, const u64 *pt, const u64 *key,
                                   int dim, long count, u64 *out) {
  const long c = (long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= count) return;
  const u64 *a = mask + (size_t)c * dim;
  u64 *o = out + (size_t)c * (dim + 1);
  u64 s = 0;
  for (int i = lane; i < dim; i += 32) {
    const u64 ai = a[i];
    o[i] = ai;
    s += ai * key[i];
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) o[dim] = s + (u64)noise[c] + pt[c];
}

// phase[c] = b - <a, key>   (C2)
__global__ void lwe_phase_kernel(const u64 *ct, const u64 *key, int dim, long count, u64 *phase) {
  const long c = (long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= count) return;
  const u64 *a = ct + (size_t)c * (dim + 1);
  u64 s = 0;
  for (int i = lane; i < dim; i += 32) s += a[i] * key[i];
#pragma unroll
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) phase[c] = a[dim] - s;
}

// ----------------------------------------------------------- BSK (GGSW) gen
// One CTA per GLWE (i, row): body = E + sum_m A_m * S_m (negacyclic, binary S),
// then s_i * q/B^j added to component r (C6).
__global__ void bsk_generate_kernel(const u64 *lwe_key, const u64 *glwe_key, const u64 *mask,
                                    const i64 *noise, u64 *bsk, int k, int N, int base_log, int level) {
  extern __shared__ __align__(16) unsigned char kg_smem[];
  u64 *A = reinterpret_cast<u64 *>(kg_smem);                // [N]
  int *nz = reinterpret_cast<int *>(kg_smem + N * sizeof(u64));  // nonzero key positions
  __shared__ int nnz;
  const long ir = blockIdx.x;
  const int rows = (k + 1) * level;
  const int i = (int)(ir / rows), row = (int)(ir % rows);
  const int r = row / level, j = row % level + 1;
  u64 *G = bsk + (size_t)ir * (k + 1) * N;
  const u64 *Am_all = mask + (size_t)ir * k * N;
  const i64 *E = noise + (size_t)ir * N;
  // body accumulators: each thread owns coefficients c = tid + blockDim*q
  for (int c = threadIdx.x; c < N; c += blockDim.x) G[(size_t)k * N + c] = (u64)E[c];
  for (int m = 0; m < k; m++) {
    __syncthreads();
    if (threadIdx.x == 0) nnz = 0;
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
      const u64 a = Am_all[(size_t)m * N + c];
      A[c] = a;
      G[(size_t)m * N + c] = a;
    }
    __syncthreads();
    // compact list of key positions with S_m[e] = 1 (order irrelevant: exact sums)
    for (int e = threadIdx.x; e < N; e += blockDim.x)
      if (glwe_key[(size_t)m * N + e] & 1) nz[atomicAdd(&nnz, 1)] = e;
    __syncthreads();
    const int cnt = nnz;
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
      u64 s = 0;
      for (int q = 0; q < cnt; q++) {
        const int e = nz[q];
        // S[e] X^e * A: coefficient c receives A[c - e] (negated on wrap)
        const int src = c - e;
        s += (src >= 0) ? A[src] : (u64)0 - A[src + N];
      }
      G[(size_t)k * N + c] += s;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) G[(size_t)r * N] += lwe_key[i] << (64 - j * base_log);
}

// BSK rows for large N: copy masks into G, then (after the GLWE body kernel)
// add s_i * q / B^j to component r.
__global__ void bsk_rows_copy_kernel(const u64 *mask, u64 *bsk, long rows_total, int N) {
  const long total = rows_total * (long)N;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long ir = e / N;
    const int c = (int)(e % N);
    bsk[(size_t)ir * 2 * N + c] = mask[(size_t)ir * N + c];
  }
}
__global__ void bsk_rows_finish_kernel(const u64 *lwe_key, u64 *bsk, long rows_total, int level, int N, int base_log) {
  const long ir = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (ir >= rows_total) return;
  const int rows = 2 * level;
  const int i = (int)(ir / rows), row = (int)(ir % rows);
  const int r = row / level, j = row % level + 1;
  bsk[((size_t)ir * 2 + r) * N] += lwe_key[i] << (64 - j * base_log);
}

// ----------------------------------------------------------------- KSK gen
// KSK[j][t] = (a, <a, s> + e + s_in[j] * 2^{64 - t beta}); one warp per row (C3).
__global__ void ksk_generate_kernel(const u64 *in_key, const u64 *lwe_key, const u64 *mask,
                                    const i64 *noise, u64 *ksk, int in_dim, int n, int base_log,
                                    int level) {
  const long jt = (long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (jt >= (long)in_dim * level) return;
  const int j = (int)(jt / level), t = (int)(jt % level) + 1;
  const u64 *a = mask + (size_t)jt * n;
  u64 *o = ksk + (size_t)jt * (n + 1);
  u64 s = 0;
  for (int i = lane; i < n; i += 32) {
    const u64 ai = a[i];
    o[i] = ai;
    s += ai * lwe_key[i];
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) o[n] = s + (u64)noise[jt] + (in_key[j] << (64 - t * base_log));
}

// --------------------------------------------------------- test polynomial
// v'[j] = T[j / box]; v = X^{-box/2} v'  =>  v[j] = v'[j + box/2], negated past N (C5).
__global__ void testpoly_kernel(const u64 *tables, int num, int p, int N, u64 *polys) {
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long)num * N) return;
  const int l = (int)(e / N), j = (int)(e % N);
  const int box = N >> p;
  const int src = j + box / 2;
  const u64 *T = tables + (size_t)l * (1 << p);
  polys[e] = (src < N) ? T[src / box] : (u64)0 - T[(src - N) / box];
}

// ------------------------------------------------------------- linear ops
// out[i] = sum_t coef[i][t] * in[idx[i][t]] + (0,...,0,cst[i])  (a0)
__global__ void lwe_linear_kernel(const u64 *in, const u32 *idx, const i64 *coef, const u64 *cst,
                                  int terms, int dim, long count, u64 *out) {
  const long i = blockIdx.x;
  if (i >= count) return;
  for (int c = threadIdx.x; c <= dim; c += blockDim.x) {
    u64 s = 0;
    for (int t = 0; t < terms; t++) {
      const u64 *src = in + (size_t)idx[(size_t)i * terms + t] * (dim + 1);
      s += (u64)coef[(size_t)i * terms + t] * src[c];
    }
    if (c == dim && cst) s += cst[i];
    out[(size_t)i * (dim + 1) + c] = s;
  }
}

// out[e] = ca A[e] + cb B[e] + cc C[e] + (0,...,0,cst)   (elementwise, exact mod 2^64)
__global__ void lwe_axpy3_kernel(u64 *out, const u64 *A, i64 ca, const u64 *B, i64 cb, const u64 *C, i64 cc,
                                 u64 cst, long count, int dim) {
  const long total = count * (long)(dim + 1);
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    u64 s = 0;
    if (A) s += (u64)ca * A[e];
    if (B) s += (u64)cb * B[e];
    if (C) s += (u64)cc * C[e];
    if (e % (dim + 1) == dim) s += cst;
    out[e] = s;
  }
}

// out[e] = ca A[e] + cb B[e] + cc C[e mod (dim+1)]: C is ONE ciphertext broadcast to all
__global__ void lwe_axpy_bcast_kernel(u64 *out, const u64 *A, i64 ca, const u64 *B, i64 cb, const u64 *C, i64 cc,
                                      long count, int dim) {
  const long total = count * (long)(dim + 1);
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    u64 s = (u64)cc * C[e % (dim + 1)];
    if (A) s += (u64)ca * A[e];
    if (B) s += (u64)cb * B[e];
    out[e] = s;
  }
}

// ------------------------------------------------------------ host launch
int launch_lwe_encrypt(const u64 *mask, const i64 *noise, const u64 *pt, const u64 *key, int dim,
                       size_t count, u64 *out, cudaStream_t st) {
  const long blocks = (long)((count + 7) / 8);
  lwe_encrypt_kernel<<<(unsigned)blocks, 256, 0, st>>>(mask, noise, pt, key, dim, (long)count, out);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

int launch_lwe_phase(const u64 *ct, const u64 *key, int dim, size_t count, u64 *phase, cudaStream_t st) {
  const long blocks = (long)((count + 7) / 8);
  lwe_phase_kernel<<<(unsigned)blocks, 256, 0, st>>>(ct, key, dim, (long)count, phase);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

int launch_glwe_body_huge(const u64 *, size_t, const u64 *, const i64 *, u64 *, size_t, long, void *, cudaStream_t);

int launch_bsk_generate_huge(const u64 *lwe_key, const u64 *glwe_key, const u64 *mask, const i64 *noise, u64 *bsk,
                             int n, int N, int base_log, int level, void *workspace, cudaStream_t st) {
  const long rows_total = (long)n * 2 * level;
  bsk_rows_copy_kernel<<<148 * 8, 256, 0, st>>>(mask, bsk, rows_total, N);
  SZ_LAUNCH_OK();
  int rc = launch_glwe_body_huge(mask, (size_t)N, glwe_key, noise, bsk + N, (size_t)2 * N, rows_total, workspace, st);
  if (rc) return rc;
  bsk_rows_finish_kernel<<<(unsigned)((rows_total + 255) / 256), 256, 0, st>>>(lwe_key, bsk, rows_total, level, N,
                                                                              base_log);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

int launch_bsk_generate(const u64 *lwe_key, const u64 *glwe_key, const u64 *mask, const i64 *noise,
                        u64 *bsk, int n, int k, int N, int base_log, int level, cudaStream_t st) {
  const size_t smem = (size_t)N * (sizeof(u64) + sizeof(int));
  if (smem > 227 * 1024) return SILENZIO_ERR_UNSUPPORTED;
  SZ_CUDA_OK(cudaFuncSetAttribute(bsk_generate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long blocks = (long)n * (k + 1) * level;
  bsk_generate_kernel<<<(unsigned)blocks, 512, smem, st>>>(lwe_key, glwe_key, mask, noise, bsk, k, N,
                                                           base_log, level);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

int launch_ksk_generate(const u64 *in_key, const u64 *lwe_key, const u64 *mask, const i64 *noise, u64 *ksk,
                        int in_dim, int n, int base_log, int level, cudaStream_t st) {
  const long rows = (long)in_dim * level;
  ksk_generate_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(in_key, lwe_key, mask, noise, ksk, in_dim, n,
                                                                 base_log, level);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

int launch_testpoly(const u64 *tables, int num, int p, int N, u64 *polys, cudaStream_t st) {
  const long total = (long)num * N;
  testpoly_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(tables, num, p, N, polys);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

int launch_lwe_axpy3(u64 *out, const u64 *A, i64 ca, const u64 *B, i64 cb, const u64 *C, i64 cc, u64 cst,
                     size_t count, int dim, cudaStream_t st) {
  if (count == 0) return SILENZIO_OK;
  const long total = (long)count * (dim + 1);
  long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  lwe_axpy3_kernel<<<(unsigned)blocks, 256, 0, st>>>(out, A, ca, B, cb, C, cc, cst, (long)count, dim);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

int launch_lwe_axpy_bcast(u64 *out, const u64 *A, i64 ca, const u64 *B, i64 cb, const u64 *C, i64 cc, size_t count,
                          int dim, cudaStream_t st) {
  if (count == 0) return SILENZIO_OK;
  const long total = (long)count * (dim + 1);
  long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  lwe_axpy_bcast_kernel<<<(unsigned)blocks, 256, 0, st>>>(out, A, ca, B, cb, C, cc, (long)count, dim);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

int launch_lwe_linear(const u64 *in, const u32 *idx, const i64 *coef, const u64 *cst, int terms, int dim,
                      size_t count, u64 *out, cudaStream_t st) {
  lwe_linear_kernel<<<(unsigned)count, 256, 0, st>>>(in, idx, coef, cst, terms, dim, (long)count, out);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

}  // namespace sz
