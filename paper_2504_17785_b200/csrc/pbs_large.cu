// pbs_large.cu -- blind rotation and BSK -> Fourier for N = 8192 (parameter
// set C, BASELINE configs[2]: 6-bit messages, PBS 2^15 x 2).
//
// Same steps and conventions as pbs.cu;
// the difference is size: M = N/2 = 4096 complex points per transform.
// One 256-thread CTA per ciphertext (one FFT "team"), 16 complex values per
// thread, four-step 16 x 16 x 16 decimation in frequency with two shared-memory
// exchanges through a 64 KiB buffer (swizzle p ^ ((p >> 4) & 7) makes all
// three access patterns bank-conflict free). ACC (2 x 8192 u64 = 128 KiB)
// stays in shared memory. The (k+1)l = 4 digit spectra of a CMux are
// thread-private (each thread's MAC reads exactly the slots its own forward
// pass produced), so they live in this thread's lane of tensor memory (4 x 64
// columns per lane quadrant, 1; the 1 = 0 build keeps
// them in per-thread local memory), with no synchronisation and no workspace.
#include <cmath>
#include <mutex>
#include <vector>

#include <cooperative_groups.h>

#include "fft.cuh"
#include "limbs.cuh"
#include "tmem.cuh"

namespace sz {

__constant__ double2 c_twistL[16];  // e^{i pi m / 32}: w^{256 m} for N = 8192 (same values as N = 2048)

constexpr int kNL = 8192;
constexpr int kML = 4096;
constexpr int kTL = 256;
constexpr int kLog2_2NL = 14;

struct TablesL {
  double2 tw1[16 * 256];  // w^{t (4k+1)}, w = e^{i pi / 8192}
  double2 tw2[16 * 16];   // W_256^{s k}
};
__device__ TablesL g_tabL;

static std::once_flag g_tabL_once[64];
static int g_tabL_status[64];

static int init_tabL(int dev) {
  TablesL h;
  const long double PI = 3.141592653589793238462643383279502884L;
  for (int k = 0; k < 16; k++)
    for (int t = 0; t < 256; t++) {
      long double ang = PI * (long double)(t * (4 * k + 1)) / 8192.0L;
      h.tw1[k * 256 + t] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
  for (int k = 0; k < 16; k++)
    for (int s = 0; s < 16; s++) {
      long double ang = 2.0L * PI * (long double)(s * k) / 256.0L;
      h.tw2[k * 16 + s] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return SILENZIO_ERR_CUDA;
  if (prev != dev && cudaSetDevice(dev) != cudaSuccess) return SILENZIO_ERR_CUDA;
  double2 tw[16];
  for (int m = 0; m < 16; m++) {
    long double ang = PI * (long double)m / 32.0L;
    tw[m] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  cudaError_t e = cudaMemcpyToSymbol(g_tabL, &h, sizeof(TablesL));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_twistL, tw, sizeof(tw));
  if (prev != dev) cudaSetDevice(prev);
  return e == cudaSuccess ? SILENZIO_OK : SILENZIO_ERR_CUDA;
}

static int ensure_tables_large() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SILENZIO_ERR_CUDA;
  std::call_once(g_tabL_once[dev], [dev] { g_tabL_status[dev] = init_tabL(dev); });
  return g_tabL_status[dev];
}

__device__ __forceinline__ int swzL(int p) { return p ^ ((p >> 4) & 7); }

// Forward: x[m] = folded value at j = t + 256 m. Out: x[r] = spectrum at
// position 16 t + bitrev4(r) (slot r).
__device__ __forceinline__ void fwd_fft_L(double2 (&x)[16], double2 *buf, int t) {
  const TablesL &T = g_tabL;
#pragma unroll
  for (int m = 0; m < 16; m++) x[m] = cmul(x[m], c_twistL[m]);
  dft<16, false>(x);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int k = bitrev4(r);
    buf[swzL(t + 256 * k)] = cmul(x[r], __ldg(&T.tw1[k * 256 + t]));
  }
  __syncthreads();
  const int b = t >> 4, s = t & 15;
  double2 y[16];
#pragma unroll
  for (int m = 0; m < 16; m++) y[m] = buf[swzL(256 * b + s + 16 * m)];
  dft<16, false>(y);
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int k = bitrev4(r);
    buf[swzL(256 * b + s + 16 * k)] = (k == 0) ? y[r] : cmul(y[r], __ldg(&T.tw2[k * 16 + s]));
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < 16; m++) x[m] = buf[swzL(16 * t + m)];
  dft<16, false>(x);
}

// Inverse (unnormalised) of fwd_fft_L; out x[m] = (c_j + i c_{j+4096}) M at j = t + 256 m.
__device__ __forceinline__ void inv_fft_L(double2 (&x)[16], double2 *buf, int t) {
  const TablesL &T = g_tabL;
  {
    double2 z[16];
#pragma unroll
    for (int k = 0; k < 16; k++) z[k] = x[bitrev4(k)];
    dft<16, true>(z);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; q++) buf[swzL(16 * t + bitrev4(q))] = z[q];
  }
  __syncthreads();
  const int b = t >> 4, s = t & 15;
  double2 y[16];
#pragma unroll
  for (int k = 0; k < 16; k++) {
    const double2 v = buf[swzL(256 * b + s + 16 * k)];
    y[k] = (k == 0) ? v : cmulc(v, __ldg(&T.tw2[k * 16 + s]));
  }
  dft<16, true>(y);
#pragma unroll
  for (int q = 0; q < 16; q++) buf[swzL(256 * b + s + 16 * bitrev4(q))] = y[q];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 16; k++) x[k] = cmulc(buf[swzL(t + 256 * k)], __ldg(&T.tw1[k * 256 + t]));
  dft<16, true>(x);
  double2 o[16];
#pragma unroll
  for (int q = 0; q < 16; q++) o[bitrev4(q)] = x[q];
#pragma unroll
  for (int m = 0; m < 16; m++) x[m] = cmulc(o[m], c_twistL[m]);
}

__device__ __forceinline__ i64 sextL(i64 x, int bits) {
  return (bits >= 64) ? x : (i64)((u64)x << (64 - bits)) >> (64 - bits);
}

__device__ __forceinline__ double limb_of(u64 g, int P, int w, int p) {
  if (P == 1) return (double)(i64)g;
  const i64 l0 = sextL((i64)g, w);
  const u64 rem = (g - (u64)l0) >> w;
  if (p == 0) return (double)l0;
  if (P == 2) return (double)sextL((i64)rem, 64 - w);
  const i64 l1 = sextL((i64)rem, w);
  if (p == 1) return (double)l1;
  const i64 rem2 = ((i64)rem - l1) >> w;
  return (double)sextL(rem2, 64 - 2 * w);
}

__device__ __forceinline__ u64 f64_to_torus_L(double x) {
  const double hi = floor(x * 0x1p-32);
  const double lo = fma(hi, -0x1p32, x);
  return ((u64)__double2ll_rn(hi) << 32) + (u64)__double2ll_rn(lo);
}

__device__ __forceinline__ u64 limb_to_torus_L(double x, int p, int P, int w) {
  // P = 3: |x| < 2^51 (R20), rounded on the FP64 pipe (1.5 * 2^52 trick)
  // instead of a 64-bit F2I conversion
  if (P == 3) return rint_small(x) << (p * w);
  if (p > 0) return (u64)__double2ll_rn(x) << (p * w);
  return f64_to_torus_L(x);
}

struct BRLArgs {
  const u64 *lwe_small;
  const u32 *lut_ids;
  const u64 *luts;
  u32 num_luts;
  const double2 *fbsk;  // [n][2][rows][P][16][256]
  u64 *lwe_out;
  long count;
  int n, base_log, w;
};

__host__ __device__ constexpr size_t brl_smem_bytes(int n) {
  return 2 * kNL * sizeof(u64) + kML * sizeof(double2) + ((size_t)n * 2 + 15) / 16 * 16;
}

// one thread asks the copy engine to pull a contiguous chunk into L2 (no
// registers, no completion tracking): the next round's BSK rows arrive while
// the current round computes, so the MAC's loads hit L2 instead of HBM
__device__ __forceinline__ void l2_prefetch_bulk(const void *ptr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

template <int L, int P>
__global__ void __launch_bounds__(256, 1) blind_rotate_large_kernel(BRLArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int rows = 2 * L;
  u64 *acc = reinterpret_cast<u64 *>(smem);                                   // [2][8192]
  double2 *buf = reinterpret_cast<double2 *>(smem + 2 * kNL * sizeof(u64));   // [4096]
  unsigned short *abar = reinterpret_cast<unsigned short *>(buf + kML);
  const int t = threadIdx.x;
  const int n = A.n, w = A.w, blog = A.base_log;
  // thread-private digit spectra: in tensor memory when they fit (rows <= 4:
  // threads t and t + 128 share a lane (warps w, w + 4), columns [0, 256) and
  // [256, 512); row r, slot sl at column 64 r + 4 sl), else in local memory
  constexpr bool kTm = rows <= 4;
  __shared__ uint32_t tmem_slot;
  const int wid = t >> 5;
  if constexpr (kTm) {
    if (wid == 0) tmem_alloc(&tmem_slot, 512);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
  }
  const uint32_t ta_spec = kTm ? tmem_slot + ((uint32_t)(32 * (wid & 3)) << 16) + 256 * (wid >> 2) : 0u;
  double2 spec[kTm ? 1 : rows][16];
  for (long c = blockIdx.x; c < A.count; c += gridDim.x) {
    const u64 *lwe = A.lwe_small + (size_t)c * (n + 1);
    for (int i = t; i < n; i += kTL) abar[i] = (unsigned short)sz_modswitch(lwe[i], kLog2_2NL);
    const int bt = (int)sz_modswitch(lwe[n], kLog2_2NL);
    u32 id = A.lut_ids ? A.lut_ids[c] : 0u;
    if (id >= A.num_luts) id = 0;
    const u64 *v = A.luts + (size_t)id * kNL;
    for (int j = t; j < kNL; j += kTL) {
      acc[j] = 0;
      const int idx = (j + bt) & (2 * kNL - 1);
      acc[kNL + j] = (idx < kNL) ? v[idx] : (u64)0 - v[idx - kNL];
    }
    __syncthreads();
    // rows of (i, o, p) for this CTA: rows chunks of kML double2, stride P kML
    auto prefetch_round = [&](int i, int o, int p) {
      if (t == 0 && i < n)
        for (int row = 0; row < rows; row++)
          l2_prefetch_bulk(A.fbsk + (((size_t)i * 2 + o) * rows + row) * P * kML + (size_t)p * kML,
                           kML * sizeof(double2));
    };
    // MAC round k of CMux i (k = o P + P - 1 - p, 2P rounds) -> prefetch k + 1
    auto prefetch_ahead = [&](int i, int k) {
      i += k / (2 * P);
      k %= 2 * P;
      prefetch_round(i, k / P, P - 1 - k % P);
    };
    prefetch_ahead(0, 0);
    for (int i = 0; i < n; i++) {
      const int a = abar[i];
      // -------- forward: every (component r, level lvl) digit polynomial
#pragma unroll 1
      for (int r = 0; r < 2; r++) {
        const u64 *accr = acc + r * kNL;
        // L = 2: the level-1 pass decomposes every coefficient once and keeps the
        // level-2 digits (|d| <= 2^{base_log-1} < 2^15) as packed int16 pairs for the
        // level-2 pass (no second read of the rotated ACC, no second decomposition)
        constexpr bool kPack = (L == 2);
        uint32_t pk[kPack ? 16 : 1];
#pragma unroll 1
        for (int lvl = 1; lvl <= L; lvl++) {
          double2 x[16];
          if (kPack && lvl == 2 && blog <= 15) {
#pragma unroll
            for (int m = 0; m < 16; m++)
              x[m] = make_double2((double)(short)(pk[kPack ? m : 0] & 0xffffu), (double)(short)(pk[kPack ? m : 0] >> 16));
          } else {
#pragma unroll
          for (int m = 0; m < 16; m++) {
            double dv[2];
            int d2[2] = {0, 0};
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int j = t + 256 * m + 4096 * h;
              const int src = (j - a) & (2 * kNL - 1);
              const u64 rv = accr[src & (kNL - 1)];
              const u64 rot = (src < kNL) ? rv : (u64)0 - rv;
              u64 rr = sz_decomp_round(rot - accr[j], blog, L);
              i64 d = 0;
#pragma unroll
              for (int tt = L; tt >= 1; tt--) {
                const i64 dd = sz_decomp_next(rr, blog);
                if (tt == lvl) d = dd;
                if (kPack && tt == 2) d2[h] = (int)dd;
              }
              dv[h] = (double)d;
            }
            x[m] = make_double2(dv[0], dv[1]);
            if (kPack) pk[m] = ((uint32_t)d2[0] & 0xffffu) | ((uint32_t)d2[1] << 16);
          }
          }
          fwd_fft_L(x, buf, t);
          const int row = r * L + (lvl - 1);
          if constexpr (kTm) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
              uint32_t r16[16];
              pack4(&x[4 * j], r16);
              tmem_st16(ta_spec + 64 * row + 16 * j, r16);
            }
          } else {
#pragma unroll
            for (int sl = 0; sl < 16; sl++) spec[row][sl] = x[sl];
          }
        }
      }
      if constexpr (kTm) tmem_wait_st();
      __syncthreads();  // all reads of ACC done before the inverse updates it
      // -------- inverse: per output component o, limbs top -> 0
#pragma unroll 1
      for (int o = 0; o < 2; o++) {
        const double2 *Gi = A.fbsk + ((size_t)i * 2 + o) * rows * P * kML + t;
        u64 *acco = acc + o * kNL;
#pragma unroll 1
        for (int p = P - 1; p >= 0; p--) {
          prefetch_ahead(i, o * P + (P - 1 - p) + 1);
          double2 y[16];
#pragma unroll
          for (int sl = 0; sl < 16; sl++) y[sl] = make_double2(0.0, 0.0);
#pragma unroll 1
          for (int row = 0; row < rows; row++) {
            const double2 *G = Gi + ((size_t)row * P + p) * kML;
            if constexpr (kTm) {
#pragma unroll
            for (int qq = 0; qq < 4; qq += 2) {
              double2 g[8];
#pragma unroll
              for (int q = 0; q < 8; q++) g[q] = __ldg(&G[(4 * qq + q) * kTL]);
              uint32_t d0[16], d1[16];
              tmem_ld16(ta_spec + 64 * row + 16 * qq, d0);
              tmem_ld16(ta_spec + 64 * row + 16 * (qq + 1), d1);
              tmem_wait_ld16x2(d0, d1);
#pragma unroll
              for (int q = 0; q < 4; q++) {
                cmac(y[4 * qq + q], unpack1(d0, q), g[q]);
                cmac(y[4 * qq + 4 + q], unpack1(d1, q), g[4 + q]);
              }
            }
            } else {
#pragma unroll
            for (int qq = 0; qq < 4; qq++) {
              double2 g[4];
#pragma unroll
              for (int q = 0; q < 4; q++) g[q] = __ldg(&G[(4 * qq + q) * kTL]);
#pragma unroll
              for (int q = 0; q < 4; q++) cmac(y[4 * qq + q], spec[kTm ? 0 : row][4 * qq + q], g[q]);
            }
            }
          }
          inv_fft_L(y, buf, t);
#pragma unroll
          for (int m = 0; m < 16; m++) {
            acco[t + 256 * m] += limb_to_torus_L(y[m].x, p, P, w);
            acco[t + 256 * m + 4096] += limb_to_torus_L(y[m].y, p, P, w);
          }
        }
      }
      __syncthreads();
    }
    u64 *out = A.lwe_out + (size_t)c * (kNL + 1);
    for (int j = t; j <= kNL; j += kTL) {
      u64 val;
      if (j == 0) val = acc[0];
      else if (j < kNL) val = (u64)0 - acc[kNL - j];
      else val = acc[kNL];
      out[j] = val;
    }
    __syncthreads();
  }
  if constexpr (kTm) {
    tmem_fence_before();
    __syncthreads();
    if (wid == 0) tmem_dealloc(tmem_slot, 512);
  }
}

struct B2FLArgs {
  const u64 *bsk;  // [n][rows][2][N]
  double2 *fbsk;   // [n][2][rows][P][16][256]
  int rows, P, w;
};

__global__ void __launch_bounds__(256) bsk_to_fourier_large_kernel(B2FLArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2 *buf = reinterpret_cast<double2 *>(smem);
  const int t = threadIdx.x;
  long blk = blockIdx.x;
  const int p = blk % A.P; blk /= A.P;
  const int o = blk % 2; blk /= 2;
  const int row = blk % A.rows; blk /= A.rows;
  const int i = (int)blk;
  const u64 *g = A.bsk + (((size_t)i * A.rows + row) * 2 + o) * kNL;
  double2 x[16];
#pragma unroll
  for (int m = 0; m < 16; m++)
    x[m] = make_double2(limb_of(g[t + 256 * m], A.P, A.w, p), limb_of(g[t + 256 * m + 4096], A.P, A.w, p));
  fwd_fft_L(x, buf, t);
  double2 *dst = A.fbsk + ((((size_t)i * 2 + o) * A.rows + row) * A.P + p) * kML;
  const double scale = 1.0 / kML;
#pragma unroll
  for (int sl = 0; sl < 16; sl++) dst[sl * kTL + t] = make_double2(x[sl].x * scale, x[sl].y * scale);
}

long blind_rotate_large_wave(const silenzio_params *P) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  (void)P;
  return sms;  // one 256-thread CTA (192 KiB smem) per SM
}

int launch_blind_rotate_large(const u64 *lwe_small, const u32 *lut_ids, const u64 *luts, u32 num_luts,
                              const void *fbsk, u64 *lwe_out, size_t count, const silenzio_params *P,
                              cudaStream_t stream) {
  int st = ensure_tables_large();
  if (st) return st;
  BRLArgs A;
  A.lwe_small = lwe_small;
  A.lut_ids = lut_ids;
  A.luts = luts;
  A.num_luts = num_luts;
  A.fbsk = reinterpret_cast<const double2 *>(fbsk);
  A.lwe_out = lwe_out;
  A.n = (int)P->lwe_dim;
  A.base_log = (int)P->pbs_base_log;
  A.w = (int)P->limb_bits;
  void (*kern)(BRLArgs) = nullptr;
  const int L = (int)P->pbs_level, PP = (int)P->fft_limbs;
#define SZ_BRL_CASE(LL, QQ) \
  if (L == LL && PP == QQ) kern = blind_rotate_large_kernel<LL, QQ>;
  SZ_BRL_CASE(1, 3) SZ_BRL_CASE(2, 3) SZ_BRL_CASE(2, 2) SZ_BRL_CASE(2, 1) SZ_BRL_CASE(3, 3) SZ_BRL_CASE(4, 3)
#undef SZ_BRL_CASE
  if (!kern) return SILENZIO_ERR_UNSUPPORTED;
  const size_t smem = brl_smem_bytes(A.n);
  if (smem > 227 * 1024) return SILENZIO_ERR_UNSUPPORTED;
  SZ_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long wave = blind_rotate_large_wave(P);
  if (wave <= 0) return SILENZIO_ERR_CUDA;
  for (long c0 = 0; c0 < (long)count; c0 += wave) {
    BRLArgs W = A;
    const long cnt = ((long)count - c0 < wave) ? (long)count - c0 : wave;
    W.lwe_small = A.lwe_small + (size_t)c0 * (A.n + 1);
    W.lut_ids = A.lut_ids ? A.lut_ids + c0 : nullptr;
    W.lwe_out = A.lwe_out + (size_t)c0 * (kNL + 1);
    W.count = cnt;
    kern<<<(unsigned)cnt, kTL, smem, stream>>>(W);
    SZ_LAUNCH_OK();
  }
  return SILENZIO_OK;
}

int launch_bsk_to_fourier_large(const u64 *bsk, void *fbsk, const silenzio_params *P, cudaStream_t stream) {
  int st = ensure_tables_large();
  if (st) return st;
  B2FLArgs A;
  A.bsk = bsk;
  A.fbsk = reinterpret_cast<double2 *>(fbsk);
  A.rows = 2 * (int)P->pbs_level;
  A.P = (int)P->fft_limbs;
  A.w = (int)P->limb_bits;
  const size_t smem = kML * sizeof(double2);
  SZ_CUDA_OK(cudaFuncSetAttribute(bsk_to_fourier_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long blocks = (long)P->lwe_dim * A.rows * 2 * A.P;
  bsk_to_fourier_large_kernel<<<(unsigned)blocks, kTL, smem, stream>>>(A);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

// =====================================================================
// N = 32768 (parameter set B, BASELINE configs[4] 8-bit stage).
// M = 16384 = 4 x 4096. Negacyclic transform of one polynomial:
//   Z[q + 4k'] = DFT_4096(y_q)[k'],  y_q[p] = W_M^{pq} sum_{m'<4} z[p + 4096 m'] W_4^{m' q},
//   z_j = (a_j + i a_{j+M}) w^j, w = e^{i pi / 32768}.
// fwd_fft_L computes DFT_4096(x_p w8^p) (w8 = e^{i pi / 8192}, the N=8192
// twist), so the input handed to it is
//   x_q[p] = F[q][p] sum_{m'} (a_{p+4096m'} + i a_{p+4096m'+M}) C[m'][q],
//   F[q][p] = e^{i pi p (4q - 3) / 32768},  C[m'][q] = e^{i pi m'/8} i^{m' q}.
// The inverse applies inv_fft_L per block then the conjugate combination.
// Per ciphertext the state lives in global memory (L2-resident by limiting
// the ciphertexts in flight): ACC [2][32768] u64, spectra [rows][4][4096]
// complex, block scratch [4][4096] complex. One 256-thread CTA per ciphertext.
constexpr int kNH = 32768;
constexpr int kMH = 16384;
constexpr int kLog2_2NH = 16;
// Ciphertexts in flight = one CTA per SM (measured on B200, tools/time_setb.py:
// 48 in flight (L2-resident state) 107 PBS/s, 96: 160, 148: 265, 296: 269 --
// the kernel is latency-bound per CTA, so every SM should hold one).
static long huge_inflight() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      sms <= 0)
    return 148;
  return sms;
}

__device__ double2 g_FH[4 * 4096];  // F[q][p]
__constant__ double2 c_CH[16];     // C[m'][q], index m' * 4 + q

static std::once_flag g_tabH_once[64];
static int g_tabH_status[64];

static int init_tabH(int dev) {
  std::vector<double2> F(4 * 4096);
  const long double PI = 3.141592653589793238462643383279502884L;
  for (int q = 0; q < 4; q++)
    for (int p = 0; p < 4096; p++) {
      long double ang = PI * (long double)p * (long double)(4 * q - 3) / 32768.0L;
      F[q * 4096 + p] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
  double2 C[16];
  for (int mp = 0; mp < 4; mp++)
    for (int q = 0; q < 4; q++) {
      long double ang = PI * (long double)mp / 8.0L + PI / 2.0L * (long double)((mp * q) % 4);
      C[mp * 4 + q] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return SILENZIO_ERR_CUDA;
  if (prev != dev && cudaSetDevice(dev) != cudaSuccess) return SILENZIO_ERR_CUDA;
  cudaError_t e = cudaMemcpyToSymbol(g_FH, F.data(), F.size() * sizeof(double2));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_CH, C, sizeof(C));
  if (prev != dev) cudaSetDevice(prev);
  return e == cudaSuccess ? SILENZIO_OK : SILENZIO_ERR_CUDA;
}

static int ensure_tables_huge() {
  int st = ensure_tables_large();
  if (st) return st;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SILENZIO_ERR_CUDA;
  std::call_once(g_tabH_once[dev], [dev] { g_tabH_status[dev] = init_tabH(dev); });
  return g_tabH_status[dev];
}

// Radix-4 step of the M = 4 x 4096 transform in butterfly form: C[m'][q] =
// e^{i pi m'/8} i^{m' q}, so sum_m' v[m'] C[m'][q] is a 4-point DFT (positive
// exponent) of the twisted inputs v[m'] e^{i pi m'/8}: 3 complex multiplications
// + 8 complex additions (28 FP64 instructions) instead of 16 general complex
// multiplications by table constants (96). The twist constants are the table's
// own C[m'][0], so the values multiplied are the ones the tables define.
__device__ __forceinline__ void radix4_fwd(const double2 (&v)[4], double2 (&S)[4]) {
  const double2 w1 = cmul(v[1], c_CH[4]), w2 = cmul(v[2], c_CH[8]), w3 = cmul(v[3], c_CH[12]);
  const double2 a = cadd(v[0], w2), b = csub(v[0], w2), c = cadd(w1, w3), d = csub(w1, w3);
  S[0] = cadd(a, c);
  S[2] = csub(a, c);
  S[1] = make_double2(b.x - d.y, b.y + d.x);  // b + i d
  S[3] = make_double2(b.x + d.y, b.y - d.x);  // b - i d
}
// conjugate step: o[m'] = conj(C[m'][0]) sum_q u[q] (-i)^{m' q}
__device__ __forceinline__ void radix4_inv(const double2 (&u)[4], double2 (&o)[4]) {
  const double2 a = cadd(u[0], u[2]), b = csub(u[0], u[2]), c = cadd(u[1], u[3]), d = csub(u[1], u[3]);
  o[0] = cadd(a, c);
  o[2] = cmulc(csub(a, c), c_CH[8]);
  o[1] = cmulc(make_double2(b.x + d.y, b.y - d.x), c_CH[4]);   // (b - i d) conj(C[1][0])
  o[3] = cmulc(make_double2(b.x - d.y, b.y + d.x), c_CH[12]);  // (b + i d) conj(C[3][0])
}

__host__ __device__ constexpr size_t brh_ws_per_ct(int rows) {
  return 2 * (size_t)kNH * sizeof(u64) + (size_t)rows * kMH * sizeof(double2) + (size_t)kMH * sizeof(double2);
}

struct BRHArgs {
  const u64 *lwe_small;
  const u32 *lut_ids;
  const u64 *luts;
  u32 num_luts;
  const double2 *fbsk;  // [n][2][rows][P][4 blocks][16][256]
  u64 *lwe_out;
  long count;
  int n, base_log, w;
  unsigned char *ws;    // gridDim.x * brh_ws_per_ct(rows)
};

// forward radix-4 step of one polynomial given by a coefficient functor:
// writes x_q[p] (input of block q's fwd_fft_L, natural order p = t + 256 m) to X[q][m][t]
template <class Coef>
__device__ __forceinline__ void huge_radix4_in(double2 *X, int t, Coef coef) {
#pragma unroll 1
  for (int m = 0; m < 16; m++) {
    const int p = t + 256 * m;
    double2 v[4];
#pragma unroll
    for (int mp = 0; mp < 4; mp++) {
      const int j = p + 4096 * mp;
      v[mp] = make_double2(coef(j), coef(j + kMH));
    }
    double2 S[4];
    radix4_fwd(v, S);
#pragma unroll
    for (int q = 0; q < 4; q++) X[((size_t)q * 16 + m) * 256 + t] = cmul(S[q], g_FH[q * 4096 + p]);
  }
}

template <int L, int P>
__global__ void __launch_bounds__(256, 1) blind_rotate_huge_kernel(BRHArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int rows = 2 * L;
  double2 *buf = reinterpret_cast<double2 *>(smem);  // [4096] exchange
  unsigned short *abar = reinterpret_cast<unsigned short *>(buf + kML);
  const int t = threadIdx.x;
  const int n = A.n, w = A.w, blog = A.base_log;
  unsigned char *ws = A.ws + (size_t)blockIdx.x * brh_ws_per_ct(rows);
  u64 *acc = reinterpret_cast<u64 *>(ws);                                     // [2][32768]
  double2 *spec = reinterpret_cast<double2 *>(ws + 2 * (size_t)kNH * 8);      // [rows][4][16][256]
  double2 *X = spec + (size_t)rows * kMH;                                     // [4][16][256]

  for (long c = blockIdx.x; c < A.count; c += gridDim.x) {
    const u64 *lwe = A.lwe_small + (size_t)c * (n + 1);
    for (int i = t; i < n; i += 256) abar[i] = (unsigned short)sz_modswitch(lwe[i], kLog2_2NH);
    const int bt = (int)sz_modswitch(lwe[n], kLog2_2NH);
    u32 id = A.lut_ids ? A.lut_ids[c] : 0u;
    if (id >= A.num_luts) id = 0;
    const u64 *v = A.luts + (size_t)id * kNH;
    for (int j = t; j < kNH; j += 256) {
      acc[j] = 0;
      const int idx = (j + bt) & (2 * kNH - 1);
      acc[kNH + j] = (idx < kNH) ? v[idx] : (u64)0 - v[idx - kNH];
    }
    __syncthreads();
    for (int i = 0; i < n; i++) {
      const int a = abar[i];
      // -------- forward: every (r, lvl) digit polynomial -> 4 block spectra
#pragma unroll 1
      for (int r = 0; r < 2; r++) {
        const u64 *accr = acc + (size_t)r * kNH;
#pragma unroll 1
        for (int lvl = 1; lvl <= L; lvl++) {
          huge_radix4_in(X, t, [&](int j) {
            const int src = (j - a) & (2 * kNH - 1);
            const u64 rv = accr[src & (kNH - 1)];
            const u64 rot = (src < kNH) ? rv : (u64)0 - rv;
            u64 rr = sz_decomp_round(rot - accr[j], blog, L);
            i64 d = 0;
#pragma unroll
            for (int tt = L; tt >= 1; tt--) {
              const i64 dd = sz_decomp_next(rr, blog);
              if (tt == lvl) d = dd;
            }
            return (double)d;
          });
          const int row = r * L + (lvl - 1);
#pragma unroll 1
          for (int q = 0; q < 4; q++) {
            double2 x[16];
#pragma unroll
            for (int m = 0; m < 16; m++) x[m] = X[((size_t)q * 16 + m) * 256 + t];
            fwd_fft_L(x, buf, t);
            double2 *dst = spec + ((size_t)row * 4 + q) * kML;
#pragma unroll
            for (int sl = 0; sl < 16; sl++) dst[sl * 256 + t] = x[sl];
          }
        }
      }
      __syncthreads();  // ACC reads done before the inverse updates it
      // -------- inverse: per output o and limb p
#pragma unroll 1
      for (int o = 0; o < 2; o++) {
        u64 *acco = acc + (size_t)o * kNH;
#pragma unroll 1
        for (int p = P - 1; p >= 0; p--) {
#pragma unroll 1
          for (int q = 0; q < 4; q++) {
            double2 y[16];
#pragma unroll
            for (int sl = 0; sl < 16; sl++) y[sl] = make_double2(0.0, 0.0);
#pragma unroll 1
            for (int row = 0; row < rows; row++) {
              const double2 *G = A.fbsk + (((((size_t)i * 2 + o) * rows + row) * P + p) * 4 + q) * kML + t;
              const double2 *D = spec + ((size_t)row * 4 + q) * kML + t;
#pragma unroll
              for (int sl = 0; sl < 16; sl++) cmac(y[sl], D[sl * 256], __ldg(&G[sl * 256]));
            }
            inv_fft_L(y, buf, t);
#pragma unroll
            for (int m = 0; m < 16; m++) X[((size_t)q * 16 + m) * 256 + t] = y[m];
          }
          // conjugate radix-4 combination, untwist folded in conj(F), conj(C); round; ACC +=
#pragma unroll 1
          for (int m = 0; m < 16; m++) {
            const int pp = t + 256 * m;
            double2 u[4];
#pragma unroll
            for (int q = 0; q < 4; q++) u[q] = cmulc(X[((size_t)q * 16 + m) * 256 + t], g_FH[q * 4096 + pp]);
            double2 so[4];
            radix4_inv(u, so);
#pragma unroll
            for (int mp = 0; mp < 4; mp++) {
              const int j = pp + 4096 * mp;
              acco[j] += limb_to_torus_L(so[mp].x, p, P, w);
              acco[j + kMH] += limb_to_torus_L(so[mp].y, p, P, w);
            }
          }
        }
      }
      __syncthreads();
    }
    u64 *out = A.lwe_out + (size_t)c * (kNH + 1);
    for (int j = t; j <= kNH; j += 256) {
      u64 val;
      if (j == 0) val = acc[0];
      else if (j < kNH) val = (u64)0 - acc[kNH - j];
      else val = acc[kNH];
      out[j] = val;
    }
    __syncthreads();
  }
}

// BSK -> Fourier at N = 32768: one CTA per (i, row, o, limb); the radix-4 inputs
// of each block are recomputed in registers (offline conversion, no scratch).
struct B2FHArgs {
  const u64 *bsk;  // [n][rows][2][N]
  double2 *fbsk;   // [n][2][rows][P][4][16][256]
  int rows, P, w;
  long total;
};

__global__ void __launch_bounds__(256) bsk_to_fourier_huge_kernel(B2FHArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2 *buf = reinterpret_cast<double2 *>(smem);
  const int t = threadIdx.x;
  for (long blk0 = blockIdx.x; blk0 < A.total; blk0 += gridDim.x) {
    long blk = blk0;
    const int p = blk % A.P; blk /= A.P;
    const int o = blk % 2; blk /= 2;
    const int row = blk % A.rows; blk /= A.rows;
    const long i = blk;
    const u64 *g = A.bsk + (((size_t)i * A.rows + row) * 2 + o) * kNH;
    double2 *dst = A.fbsk + ((((size_t)i * 2 + o) * A.rows + row) * A.P + p) * (size_t)kMH;
    const double scale = 1.0 / kMH;
#pragma unroll 1
    for (int q = 0; q < 4; q++) {
      double2 x[16];
#pragma unroll 1
      for (int m = 0; m < 16; m++) {
        const int pp = t + 256 * m;
        double2 s = make_double2(0.0, 0.0);
#pragma unroll
        for (int mp = 0; mp < 4; mp++) {
          const int j = pp + 4096 * mp;
          const double2 v = make_double2(limb_of(g[j], A.P, A.w, p), limb_of(g[j + kMH], A.P, A.w, p));
          s = cadd(s, cmul(v, c_CH[mp * 4 + q]));
        }
        x[m] = cmul(s, g_FH[q * 4096 + pp]);
      }
      fwd_fft_L(x, buf, t);
#pragma unroll
      for (int sl = 0; sl < 16; sl++)
        dst[(size_t)q * kML + sl * 256 + t] = make_double2(x[sl].x * scale, x[sl].y * scale);
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------
// N = 32768 on a thread-block cluster: the four CTAs of a cluster are the
// four radix-4 blocks q of one ciphertext (M = 4 x 4096, same transform and
// tables as blind_rotate_huge_kernel, so the arithmetic is identical), and the
// per-ciphertext state stays on chip:
//  * ACC is split by fold position: CTA s owns positions pp in [1024 s, 1024 s
//    + 1024) of every block mp and both fold halves h (coefficient j = h 16384
//    + mp 4096 + pp), [comp][h][mp][1024] u64 = 128 KiB of shared memory;
//  * block q's four digit spectra live in CTA q's tensor memory (as set C);
//  * the radix-4 steps are all-to-all exchanges through distributed shared
//    memory: forward, CTA s computes the block inputs x_q[pp] of its positions
//    from the rotated ACC (remote reads) and stores them into CTA q's FFT
//    buffer; inverse, CTA q stores its block output at pp into the owner of pp,
//    which combines the four blocks, rounds and updates its ACC slice.
// Cluster barriers order the exchanges (two per forward row and per (o, p)).
constexpr int kClQ = 4;  // CTAs per ciphertext = radix-4 blocks
__host__ __device__ constexpr size_t brc_acc_bytes() { return 2 * 2 * 4 * 1024 * sizeof(u64); }
__host__ __device__ constexpr size_t brc_smem_bytes(int n) {
  return brc_acc_bytes() + kML * sizeof(double2) + ((size_t)n * 2 + 15) / 16 * 16;
}
__device__ __forceinline__ int brc_aidx(int comp, int h, int mp, int loc) { return ((comp * 2 + h) * 4 + mp) * 1024 + loc; }

// ---- cluster exchange primitives (shared::cluster addresses are 32-bit)
__device__ __forceinline__ uint32_t cl_mapa(uint32_t saddr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
// arm this CTA's receive barrier for `bytes` of incoming st.async data (one arrival)
__device__ __forceinline__ void cl_mbar_expect(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
// relaxed arrive: ordering comes from a preceding fence.release.cluster (ptxas
// emits the full MEMBAR.GPU + ERRBAR sequence once per fence instead of once per
// release-arrive)
__device__ __forceinline__ void cl_fence_release() { asm volatile("fence.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void cl_mbar_arrive_remote_relaxed(uint32_t rmbar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rmbar) : "memory");
}
__device__ __forceinline__ void cl_mbar_wait_acq(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nSZ_CLW_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SZ_CLW_%=;\n}\n" ::"r"(mbar),
      "r"(parity)
      : "memory");
}
// 16-byte remote store that completes `16` transaction bytes on the receiver's barrier
__device__ __forceinline__ void cl_st_async(uint32_t raddr, double2 v, uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(v.x), "d"(v.y), "r"(rmbar)
               : "memory");
}

#ifndef SZ_PHASE_TIMING
#define SZ_PHASE_TIMING 0  // 1: debug build accumulating clock64 per CMux phase (CTA 0, thread 0)
#endif
#if SZ_PHASE_TIMING
__device__ unsigned long long g_phase_b[12];
#define SZB_PT_INIT long long szb_prev = clock64();
#define SZB_PT(k)                                                              \
  do {                                                                         \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                 \
      const long long now = clock64();                                         \
      g_phase_b[k] += (unsigned long long)(now - szb_prev);                    \
      szb_prev = now;                                                          \
    }                                                                          \
  } while (0)
#else
#define SZB_PT_INIT
#define SZB_PT(k) \
  do {            \
  } while (0)
#endif

template <int L, int P>
__global__ void __cluster_dims__(kClQ, 1, 1) __launch_bounds__(256, 1) blind_rotate_cluster_kernel(BRHArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  constexpr int rows = 2 * L;
  static_assert(rows <= 4, "digit spectra must fit tensor memory");
  u64 *acc = reinterpret_cast<u64 *>(smem);                          // [2][2][4][1024]
  double2 *buf = reinterpret_cast<double2 *>(smem + brc_acc_bytes()); // [4096] FFT / exchange buffer
  unsigned short *abar = reinterpret_cast<unsigned short *>(buf + kML);
  const int t = threadIdx.x, wid = t >> 5;
  const int q = (int)cl.block_rank();
  const int n = A.n, w = A.w, blog = A.base_log;
  // remote (distributed shared memory) addresses: one mapa per access
  auto racc = [&](int rank, int idx) -> const u64 & { return *cl.map_shared_rank(acc + idx, rank); };
  __shared__ uint32_t tmem_slot;
  if (wid == 0) tmem_alloc(&tmem_slot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t ta_spec = tmem_slot + ((uint32_t)(32 * (wid & 3)) << 16) + 256 * (wid >> 2);
  // exchange rounds: every round fills each CTA's buffer with
  // 4 x 16 KiB from the 4 senders. full = this CTA's receive barrier (armed
  // with 64 KiB per round); freeb = counts the 4 receivers that released their
  // buffer for the next round (this CTA sends only after all 4 did).
  __shared__ __align__(8) uint64_t xbar[2];
  const uint32_t full = smem_u32(&xbar[0]), freeb = smem_u32(&xbar[1]);
  const uint32_t buf_s = smem_u32(buf);
  uint32_t xround = 0;
  auto release_buf = [&]() {  // after a __syncthreads: this CTA is done with its buffer
    if (t == 0) {
      cl_mbar_expect(full, 4 * 1024 * sizeof(double2));
      // one release fence, then relaxed remote arrivals (a release-arrive per
      // remote barrier costs a MEMBAR + ERRBAR each: 4 % slower)
      cl_fence_release();
#pragma unroll
      for (int r = 0; r < kClQ; r++) cl_mbar_arrive_remote_relaxed(cl_mapa(freeb, r));
    }
  };
  if (t == 0) {
    cl_mbar_init(full, 1);
    cl_mbar_init(freeb, kClQ);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  const long ncl = gridDim.x / kClQ;
  for (long c = blockIdx.x / kClQ; c < A.count; c += ncl) {
    const u64 *lwe = A.lwe_small + (size_t)c * (n + 1);
    for (int i = t; i < n; i += 256) abar[i] = (unsigned short)sz_modswitch(lwe[i], kLog2_2NH);
    const int bt = (int)sz_modswitch(lwe[n], kLog2_2NH);
    u32 id = A.lut_ids ? A.lut_ids[c] : 0u;
    if (id >= A.num_luts) id = 0;
    const u64 *v = A.luts + (size_t)id * kNH;
    // ACC = (0, X^{-b~} v) on the owned positions
    for (int e = t; e < 2 * 4 * 1024; e += 256) {
      const int loc = e & 1023, mp = (e >> 10) & 3, h = e >> 12;
      const int j = h * kMH + mp * 4096 + 1024 * q + loc;
      const int idx = (j + bt) & (2 * kNH - 1);
      acc[brc_aidx(0, h, mp, loc)] = 0;
      acc[brc_aidx(1, h, mp, loc)] = (idx < kNH) ? v[idx] : (u64)0 - v[idx - kNH];
    }
    __syncthreads();
    SZB_PT_INIT
    for (int i = 0; i < n; i++) {
      const int a = abar[i];
      // -------- forward: (r, lvl) digit polynomial -> radix-4 inputs -> block FFT
#pragma unroll 1
      for (int r = 0; r < 2; r++) {
#pragma unroll 1
        for (int lvl = 1; lvl <= L; lvl++) {
          __syncthreads();  // this CTA's previous use of its buffer (FFT / combination) is over
          release_buf();
          cl_mbar_wait_acq(freeb, xround & 1);  // all 4 buffers free, all ACC slices final (release/acquire)
          SZB_PT(0);

#pragma unroll 1
          for (int mm = 0; mm < 4; mm++) {
            const int loc = t + 256 * mm, pp = 1024 * q + loc;
            double2 vv[4];
#pragma unroll
            for (int mp = 0; mp < 4; mp++) {
              double dv[2];
#pragma unroll
              for (int h = 0; h < 2; h++) {
                const int j = h * kMH + mp * 4096 + pp;
                const int src = (j - a) & (2 * kNH - 1);
                const int sj = src & (kNH - 1);
                const int spp = sj & 4095;
                const u64 rv = racc(spp >> 10, brc_aidx(r, sj >> 14, (sj >> 12) & 3, spp & 1023));
                const u64 rot = (src < kNH) ? rv : (u64)0 - rv;
                u64 rr = sz_decomp_round(rot - acc[brc_aidx(r, h, mp, loc)], blog, L);
                i64 d = 0;
#pragma unroll
                for (int tt = L; tt >= 1; tt--) {
                  const i64 dd = sz_decomp_next(rr, blog);
                  if (tt == lvl) d = dd;
                }
                dv[h] = (double)d;
              }
              vv[mp] = make_double2(dv[0], dv[1]);
            }
            double2 S4[4];
            radix4_fwd(vv, S4);
#pragma unroll
            for (int qq = 0; qq < 4; qq++) {
              const double2 xv = cmul(S4[qq], g_FH[qq * 4096 + pp]);
              cl_st_async(cl_mapa(buf_s + pp * 16, qq), xv, cl_mapa(full, qq));
            }
          }
          SZB_PT(1);
          cl_mbar_wait_acq(full, xround & 1);  // block inputs delivered
          xround++;
          SZB_PT(2);

          double2 x[16];
#pragma unroll
          for (int m = 0; m < 16; m++) x[m] = buf[t + 256 * m];
          fwd_fft_L(x, buf, t);
          const int row = r * L + (lvl - 1);
#pragma unroll
          for (int jj = 0; jj < 4; jj++) {
            uint32_t r16[16];
            pack4(&x[4 * jj], r16);
            tmem_st16(ta_spec + 64 * row + 16 * jj, r16);
          }
          SZB_PT(3);
        }
      }
      tmem_wait_st();
      // -------- inverse: per output o and limb p: MAC, block IFFT, exchange, combine
#pragma unroll 1
      for (int o = 0; o < 2; o++) {
#pragma unroll 1
        for (int p = P - 1; p >= 0; p--) {
          double2 y[16];
#pragma unroll
          for (int sl = 0; sl < 16; sl++) y[sl] = make_double2(0.0, 0.0);
#pragma unroll 1
          for (int row = 0; row < rows; row++) {
            const double2 *G = A.fbsk + (((((size_t)i * 2 + o) * rows + row) * P + p) * 4 + q) * kML + t;
#pragma unroll
            for (int qq = 0; qq < 4; qq += 2) {
              double2 g[8];
#pragma unroll
              for (int k = 0; k < 8; k++) g[k] = __ldg(&G[(4 * qq + k) * 256]);
              uint32_t d0[16], d1[16];
              tmem_ld16(ta_spec + 64 * row + 16 * qq, d0);
              tmem_ld16(ta_spec + 64 * row + 16 * (qq + 1), d1);
              tmem_wait_ld16x2(d0, d1);
#pragma unroll
              for (int k = 0; k < 4; k++) {
                cmac(y[4 * qq + k], unpack1(d0, k), g[k]);
                cmac(y[4 * qq + 4 + k], unpack1(d1, k), g[4 + k]);
              }
            }
          }
          SZB_PT(4);
          inv_fft_L(y, buf, t);
          SZB_PT(5);
          __syncthreads();  // this CTA's IFFT is done with its buffer
          release_buf();
          cl_mbar_wait_acq(freeb, xround & 1);
          SZB_PT(6);
#pragma unroll
          for (int m = 0; m < 16; m++) {
            const int pp = t + 256 * m;
            cl_st_async(cl_mapa(buf_s + (q * 1024 + (pp & 1023)) * 16, pp >> 10), y[m], cl_mapa(full, pp >> 10));
          }
          SZB_PT(7);
          cl_mbar_wait_acq(full, xround & 1);  // block outputs delivered to the owners
          xround++;
          SZB_PT(8);

#pragma unroll 1
          for (int mm = 0; mm < 4; mm++) {
            const int loc = t + 256 * mm, pp = 1024 * q + loc;
            double2 u[4];
#pragma unroll
            for (int qq = 0; qq < 4; qq++) u[qq] = cmulc(buf[qq * 1024 + loc], g_FH[qq * 4096 + pp]);
            double2 so[4];
            radix4_inv(u, so);
#pragma unroll
            for (int mp = 0; mp < 4; mp++) {
              acc[brc_aidx(o, 0, mp, loc)] += limb_to_torus_L(so[mp].x, p, P, w);
              acc[brc_aidx(o, 1, mp, loc)] += limb_to_torus_L(so[mp].y, p, P, w);
            }
          }
          SZB_PT(9);
        }
      }
    }
    __syncthreads();
    // ---- sample extraction of the owned coefficients: a'[0] = A[0], a'[i] = -A[N-i], b' = B[0]
    u64 *out = A.lwe_out + (size_t)c * (kNH + 1);
    for (int e = t; e < 2 * 4 * 1024; e += 256) {
      const int loc = e & 1023, mp = (e >> 10) & 3, h = e >> 12;
      const int j = h * kMH + mp * 4096 + 1024 * q + loc;
      const u64 a0 = acc[brc_aidx(0, h, mp, loc)];
      if (j == 0) {
        out[0] = a0;
        out[kNH] = acc[brc_aidx(1, h, mp, loc)];
      } else {
        out[kNH - j] = (u64)0 - a0;
      }
    }
    __syncthreads();
  }
  cl.sync();  // no CTA leaves while its shared memory may still be accessed
  tmem_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tmem_slot, 512);
}

static bool cluster_path(const silenzio_params *P) {
  return P->pbs_level <= 2 && P->fft_limbs == 3 && brc_smem_bytes((int)P->lwe_dim) <= 227 * 1024;
}

// max co-resident clusters for (device, kernel, dynamic smem), cached (the
// query is cheap but not free); guarded for concurrent host threads
static long cluster_grid(const silenzio_params *P, void (*kern)(BRHArgs), size_t smem) {
  struct Entry { int dev; void (*kern)(BRHArgs); size_t smem; long ncl; };
  static std::mutex m;
  static std::vector<Entry> cache;
  (void)P;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  {
    std::lock_guard<std::mutex> lk(m);
    for (const Entry &e : cache)
      if (e.dev == dev && e.kern == kern && e.smem == smem) return e.ncl;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kClQ * 64, 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = kClQ;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, (void *)kern, &cfg) != cudaSuccess || ncl <= 0) return -1;
  std::lock_guard<std::mutex> lk(m);
  cache.push_back({dev, kern, smem, (long)ncl});
  return ncl;
}

size_t blind_rotate_huge_ws_bytes(const silenzio_params *P, size_t count) {
  const long cap = huge_inflight();
  const long inflight = (long)count < cap ? (long)count : cap;
  return (size_t)inflight * brh_ws_per_ct(2 * (int)P->pbs_level);
}

long blind_rotate_huge_wave(const silenzio_params *P) {
  if (cluster_path(P)) return 1L << 40;  // one persistent launch for any count
  return huge_inflight();
}

int launch_blind_rotate_huge(const u64 *lwe_small, const u32 *lut_ids, const u64 *luts, u32 num_luts,
                             const void *fbsk, u64 *lwe_out, size_t count, const silenzio_params *P,
                             void *workspace, cudaStream_t stream) {
  int st = ensure_tables_huge();
  if (st) return st;
  BRHArgs A;
  A.lwe_small = lwe_small;
  A.lut_ids = lut_ids;
  A.luts = luts;
  A.num_luts = num_luts;
  A.fbsk = reinterpret_cast<const double2 *>(fbsk);
  A.lwe_out = lwe_out;
  A.n = (int)P->lwe_dim;
  A.base_log = (int)P->pbs_base_log;
  A.w = (int)P->limb_bits;
  A.ws = reinterpret_cast<unsigned char *>(workspace);
  A.count = (long)count;
  if (cluster_path(P)) {
    void (*ck)(BRHArgs) = P->pbs_level == 2 ? blind_rotate_cluster_kernel<2, 3> : blind_rotate_cluster_kernel<1, 3>;
    const size_t csmem = brc_smem_bytes(A.n);
    SZ_CUDA_OK(cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
    const long ncl = cluster_grid(P, ck, csmem);
    if (ncl <= 0) return SILENZIO_ERR_CUDA;
    const long grid = (long)count < ncl ? (long)count : ncl;
    ck<<<(unsigned)(grid * kClQ), 256, csmem, stream>>>(A);  // persistent: cluster g takes ciphertexts g, g + grid, ...
    SZ_LAUNCH_OK();
    return SILENZIO_OK;
  }
  if (!workspace) return SILENZIO_ERR_WORKSPACE;
  void (*kern)(BRHArgs) = nullptr;
  const int L = (int)P->pbs_level, PP = (int)P->fft_limbs;
  if (L == 2 && PP == 3) kern = blind_rotate_huge_kernel<2, 3>;
  if (L == 4 && PP == 3) kern = blind_rotate_huge_kernel<4, 3>;
  if (L == 1 && PP == 3) kern = blind_rotate_huge_kernel<1, 3>;
  if (!kern) return SILENZIO_ERR_UNSUPPORTED;
  const size_t smem = kML * sizeof(double2) + ((size_t)A.n * 2 + 15) / 16 * 16;
  SZ_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long inflight = huge_inflight();
  for (long c0 = 0; c0 < (long)count; c0 += inflight) {
    BRHArgs W = A;
    const long cnt = ((long)count - c0 < inflight) ? (long)count - c0 : inflight;
    W.lwe_small = A.lwe_small + (size_t)c0 * (A.n + 1);
    W.lut_ids = A.lut_ids ? A.lut_ids + c0 : nullptr;
    W.lwe_out = A.lwe_out + (size_t)c0 * (kNH + 1);
    W.count = cnt;
    kern<<<(unsigned)cnt, 256, smem, stream>>>(W);
    SZ_LAUNCH_OK();
  }
  return SILENZIO_OK;
}

int launch_bsk_to_fourier_huge(const u64 *bsk, void *fbsk, const silenzio_params *P, cudaStream_t stream) {
  int st = ensure_tables_huge();
  if (st) return st;
  B2FHArgs A;
  A.bsk = bsk;
  A.fbsk = reinterpret_cast<double2 *>(fbsk);
  A.rows = 2 * (int)P->pbs_level;
  A.P = (int)P->fft_limbs;
  A.w = (int)P->limb_bits;
  A.total = (long)P->lwe_dim * A.rows * 2 * A.P;
  const int grid = 296;
  const size_t smem = kML * sizeof(double2);
  SZ_CUDA_OK(cudaFuncSetAttribute(bsk_to_fourier_huge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  bsk_to_fourier_huge_kernel<<<grid, 256, smem, stream>>>(A);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

}  // namespace sz

namespace sz {

// GLWE bodies at N = 32768 for key generation: body = E + A * S (negacyclic,
// binary S), exact via three 22/22/20-bit limbs of A and the f64 transform
// above (|sum| <= 2^21 * 16384 < 2^53, rounded to the exact integer).
// One CTA per GLWE (grid-stride); scratch per CTA: X, S^ (2 x 256 KiB) + res (256 KiB).
struct GBHArgs {
  const u64 *A;      // row g: A + g * a_stride
  const u64 *key;    // [N] binary
  const i64 *E;      // row g: E + g * N
  u64 *body;         // row g: body + g * out_stride
  long count;
  size_t a_stride, out_stride;
  unsigned char *ws;
};

__host__ __device__ constexpr size_t gbh_ws_per_cta() { return 2 * (size_t)kMH * sizeof(double2) + (size_t)kNH * sizeof(u64); }

__global__ void __launch_bounds__(256) glwe_body_huge_kernel(GBHArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2 *buf = reinterpret_cast<double2 *>(smem);
  const int t = threadIdx.x;
  unsigned char *ws = A.ws + (size_t)blockIdx.x * gbh_ws_per_cta();
  double2 *X = reinterpret_cast<double2 *>(ws);
  double2 *Sh = X + kMH;
  u64 *res = reinterpret_cast<u64 *>(Sh + kMH);
  // S^ once per CTA
  huge_radix4_in(X, t, [&](int j) { return (double)(A.key[j] & 1); });
#pragma unroll 1
  for (int q = 0; q < 4; q++) {
    double2 x[16];
#pragma unroll
    for (int m = 0; m < 16; m++) x[m] = X[((size_t)q * 16 + m) * 256 + t];
    fwd_fft_L(x, buf, t);
#pragma unroll
    for (int sl = 0; sl < 16; sl++) Sh[(size_t)q * kML + sl * 256 + t] = make_double2(x[sl].x / kMH, x[sl].y / kMH);
    __syncthreads();
  }
  for (long g = blockIdx.x; g < A.count; g += gridDim.x) {
    const u64 *a = A.A + (size_t)g * A.a_stride;
    const i64 *e = A.E + (size_t)g * kNH;
    for (int j = t; j < kNH; j += 256) res[j] = (u64)e[j];
#pragma unroll 1
    for (int p = 0; p < 3; p++) {
      __syncthreads();
      huge_radix4_in(X, t, [&](int j) { return limb_of(a[j], 3, 22, p); });
#pragma unroll 1
      for (int q = 0; q < 4; q++) {
        double2 x[16];
#pragma unroll
        for (int m = 0; m < 16; m++) x[m] = X[((size_t)q * 16 + m) * 256 + t];
        fwd_fft_L(x, buf, t);
#pragma unroll
        for (int sl = 0; sl < 16; sl++) x[sl] = cmul(x[sl], Sh[(size_t)q * kML + sl * 256 + t]);
        inv_fft_L(x, buf, t);
#pragma unroll
        for (int m = 0; m < 16; m++) X[((size_t)q * 16 + m) * 256 + t] = x[m];
      }
#pragma unroll 1
      for (int m = 0; m < 16; m++) {
        const int pp = t + 256 * m;
        double2 u[4];
#pragma unroll
        for (int q = 0; q < 4; q++) u[q] = cmulc(X[((size_t)q * 16 + m) * 256 + t], g_FH[q * 4096 + pp]);
#pragma unroll
        for (int mp = 0; mp < 4; mp++) {
          double2 s = make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < 4; q++) s = cadd(s, cmulc(u[q], c_CH[mp * 4 + q]));
          const int j = pp + 4096 * mp;
          res[j] += (u64)__double2ll_rn(s.x) << (22 * p);
          res[j + kMH] += (u64)__double2ll_rn(s.y) << (22 * p);
        }
      }
    }
    __syncthreads();
    u64 *out = A.body + (size_t)g * A.out_stride;
    for (int j = t; j < kNH; j += 256) out[j] = res[j];
  }
}

size_t glwe_body_huge_ws_bytes() { return 148 * gbh_ws_per_cta(); }

int launch_glwe_body_huge(const u64 *Amask, size_t a_stride, const u64 *key, const i64 *E, u64 *body,
                          size_t out_stride, long count, void *workspace, cudaStream_t stream) {
  int st = ensure_tables_huge();
  if (st) return st;
  if (!workspace) return SILENZIO_ERR_WORKSPACE;
  GBHArgs A{Amask, key, E, body, count, a_stride, out_stride, reinterpret_cast<unsigned char *>(workspace)};
  const size_t smem = kML * sizeof(double2);
  SZ_CUDA_OK(cudaFuncSetAttribute(glwe_body_huge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long grid = count < 148 ? count : 148;
  glwe_body_huge_kernel<<<(unsigned)grid, 256, smem, stream>>>(A);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

}  // namespace sz

// SZ_PHASE_TIMING debug builds: clock64 cycles per phase of the set-B cluster
// kernel's CMux loop (CTA 0, thread 0): 0 forward release/free-wait, 1 digits +
// radix-4 + sends, 2 forward full-wait, 3 block FFT + TMEM store, 4 MAC,
// 5 block IFFT, 6 inverse release/free-wait, 7 sends, 8 inverse full-wait,
// 9 combine + rounding + ACC update; read and reset
extern "C" int silenzio_debug_phase_times_b(unsigned long long *out /* [12] */) {
#if SZ_PHASE_TIMING
  unsigned long long z[12] = {0};
  SZ_CUDA_OK(cudaMemcpyFromSymbol(out, sz::g_phase_b, sizeof(z)));
  SZ_CUDA_OK(cudaMemcpyToSymbol(sz::g_phase_b, z, sizeof(z)));
  return SILENZIO_OK;
#else
  (void)out;
  return SILENZIO_ERR_UNSUPPORTED;
#endif
}
