// keyswitch.cu -- batched LWE keyswitch big key -> small key (SURVEY.md §8(a) a1,
// §8(c) C3):  out = (0,...,0,b) - sum_j sum_t Dec_t(a_j) * KSK[j][t]  mod 2^64.
//
// GEMM-shaped over the batch: [count x in_dim*l] digits times
// [in_dim*l x (n+1)] KSK rows. A CTA owns a 32-ciphertext x 128-output tile;
// per chunk of 8 input coefficients it decomposes 32x8 coefficients once into
// shared memory and stages the matching 8*l KSK row segments (coalesced 1 KiB
// rows), then every thread accumulates a 4x4 register tile of u64 sums.
#include "common.cuh"

namespace sz {

constexpr int KS_CT = 32;    // ciphertexts per CTA
constexpr int KS_OUT = 128;  // output coefficients per CTA
constexpr int KS_J = 8;      // input coefficients per chunk
constexpr int KS_MAXL = 8;   // max l_ks supported by the smem tile

struct KSArgs {
  const u64 *in;   // [count][in_dim+1]
  const u64 *ksk;  // [in_dim][l][n+1]
  u64 *out;        // [count][n+1]
  long count;
  int in_dim, n, base_log, level;
  int kchunk;      // input coefficients per blockIdx.z (split-K); == in_dim: no split
};

__global__ void __launch_bounds__(256) keyswitch_kernel(KSArgs A) {
  extern __shared__ __align__(16) unsigned char ks_smem[];
  u64 (*ks)[KS_OUT] = reinterpret_cast<u64 (*)[KS_OUT]>(ks_smem);  // [8 l][128]
  int (*dig)[KS_CT] = reinterpret_cast<int (*)[KS_CT]>(ks_smem + (size_t)KS_J * A.level * KS_OUT * sizeof(u64));
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  const long c0 = (long)blockIdx.x * KS_CT;
  const int o0 = blockIdx.y * KS_OUT;
  const int n1 = A.n + 1, L = A.level;

  u64 acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const long c = c0 + ty + 8 * r;
      const int o = o0 + tx + 32 * q;
      acc[r][q] = (c < A.count && o == A.n && blockIdx.z == 0) ? A.in[(size_t)c * (A.in_dim + 1) + A.in_dim] : 0ull;
    }

  const int jbeg = blockIdx.z * A.kchunk;
  const int jend = (jbeg + A.kchunk < A.in_dim) ? jbeg + A.kchunk : A.in_dim;
  for (int j0 = jbeg; j0 < jend; j0 += KS_J) {
    __syncthreads();
    // decompose 32 ciphertexts x 8 coefficients (one per thread)
    {
      const int cc = tid & 31, jj = tid >> 5;
      const long c = c0 + cc;
      const int j = j0 + jj;
      u64 r = 0;
      if (c < A.count && j < jend) r = sz_decomp_round(A.in[(size_t)c * (A.in_dim + 1) + j], A.base_log, L);
      for (int t = L; t >= 1; t--) {
        const i64 d = sz_decomp_next(r, A.base_log);
        dig[jj * L + (t - 1)][cc] = (c < A.count && j < jend) ? (int)d : 0;
      }
    }
    // stage KSK rows (j0..j0+7, all t) x this CTA's 128 outputs
    const int nrows = KS_J * L;
    for (int e = tid; e < nrows * KS_OUT; e += 256) {
      const int rr = e / KS_OUT, oo = e % KS_OUT;
      const int j = j0 + rr / L, t = rr % L;
      const int o = o0 + oo;
      ks[rr][oo] = (j < jend && o < n1) ? A.ksk[((size_t)j * L + t) * n1 + o] : 0ull;
    }
    __syncthreads();
    for (int rr = 0; rr < nrows; rr++) {
      u64 kv[4];
      i64 dv[4];
#pragma unroll
      for (int q = 0; q < 4; q++) kv[q] = ks[rr][tx + 32 * q];
#pragma unroll
      for (int r = 0; r < 4; r++) dv[r] = dig[rr][ty + 8 * r];
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[r][q] -= (u64)dv[r] * kv[q];
    }
  }
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const long c = c0 + ty + 8 * r;
      const int o = o0 + tx + 32 * q;
      if (c < A.count && o < n1) {
        // split-K partial sums: exact u64 (mod 2^64) additions commute, so the
        // result is bit-identical whatever order the atomics land in
        if (gridDim.z > 1) atomicAdd(reinterpret_cast<unsigned long long *>(&A.out[(size_t)c * n1 + o]), acc[r][q]);
        else A.out[(size_t)c * n1 + o] = acc[r][q];
      }
    }
}

int launch_keyswitch(const u64 *in, const u64 *ksk, u64 *out, size_t count, int in_dim, int n,
                     int base_log, int level, cudaStream_t stream) {
  if (level > KS_MAXL) return SILENZIO_ERR_UNSUPPORTED;
  KSArgs A{in, ksk, out, (long)count, in_dim, n, base_log, level, in_dim};
  dim3 grid((unsigned)((count + KS_CT - 1) / KS_CT), (unsigned)((n + 1 + KS_OUT - 1) / KS_OUT));
  // few ciphertexts x a long input (e.g. the 32768 -> 2048 cross keyswitch of
  // the 8-bit stage): split the input dimension over blockIdx.z so that about
  // 4 CTAs per SM stream the KSK; partial sums are added atomically
  {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long tiles = (long)grid.x * grid.y;
    long split = (4L * sms + tiles - 1) / tiles;
    const long max_split = in_dim / (8 * KS_J);  // keep >= 8 chunks per split
    if (split > max_split) split = max_split;
    if (split > 1) {
      const int kc = (int)(((in_dim + split - 1) / split + KS_J - 1) / KS_J * KS_J);
      A.kchunk = kc;
      grid.z = (unsigned)((in_dim + kc - 1) / kc);
      SZ_CUDA_OK(cudaMemsetAsync(out, 0, count * (size_t)(n + 1) * sizeof(u64), stream));
    }
  }
  const size_t smem = (size_t)KS_J * level * (KS_OUT * sizeof(u64) + KS_CT * sizeof(int));
  SZ_CUDA_OK(cudaFuncSetAttribute(keyswitch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  keyswitch_kernel<<<grid, 256, smem, stream>>>(A);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

}  // namespace sz
