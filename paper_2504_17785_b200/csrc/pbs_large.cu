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
// pass produced), so they live in per-thread local memory (L1/L2), with no
// synchronisation and no workspace.
#include <cmath>
#include <mutex>

#include "fft.cuh"

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
  if (P == 3 || p > 0) return (u64)__double2ll_rn(x) << (p * w);
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

template <int L, int P>
__global__ void __launch_bounds__(256, 1) blind_rotate_large_kernel(BRLArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int rows = 2 * L;
  u64 *acc = reinterpret_cast<u64 *>(smem);                                   // [2][8192]
  double2 *buf = reinterpret_cast<double2 *>(smem + 2 * kNL * sizeof(u64));   // [4096]
  unsigned short *abar = reinterpret_cast<unsigned short *>(buf + kML);
  const int t = threadIdx.x;
  const int n = A.n, w = A.w, blog = A.base_log;
  double2 spec[rows][16];  // thread-private digit spectra (local memory)

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
    for (int i = 0; i < n; i++) {
      const int a = abar[i];
      // -------- forward: every (component r, level lvl) digit polynomial
#pragma unroll 1
      for (int r = 0; r < 2; r++) {
        const u64 *accr = acc + r * kNL;
#pragma unroll 1
        for (int lvl = 1; lvl <= L; lvl++) {
          double2 x[16];
#pragma unroll
          for (int m = 0; m < 16; m++) {
            double dv[2];
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
              }
              dv[h] = (double)d;
            }
            x[m] = make_double2(dv[0], dv[1]);
          }
          fwd_fft_L(x, buf, t);
          const int row = r * L + (lvl - 1);
#pragma unroll
          for (int sl = 0; sl < 16; sl++) spec[row][sl] = x[sl];
        }
      }
      __syncthreads();  // all reads of ACC done before the inverse updates it
      // -------- inverse: per output component o, limbs top -> 0
#pragma unroll 1
      for (int o = 0; o < 2; o++) {
        const double2 *Gi = A.fbsk + ((size_t)i * 2 + o) * rows * P * kML + t;
        u64 *acco = acc + o * kNL;
#pragma unroll 1
        for (int p = P - 1; p >= 0; p--) {
          double2 y[16];
#pragma unroll
          for (int sl = 0; sl < 16; sl++) y[sl] = make_double2(0.0, 0.0);
#pragma unroll 1
          for (int row = 0; row < rows; row++) {
            const double2 *G = Gi + ((size_t)row * P + p) * kML;
#pragma unroll
            for (int qq = 0; qq < 4; qq++) {
              double2 g[4];
#pragma unroll
              for (int q = 0; q < 4; q++) g[q] = __ldg(&G[(4 * qq + q) * kTL]);
#pragma unroll
              for (int q = 0; q < 4; q++) cmac(y[4 * qq + q], spec[row][4 * qq + q], g[q]);
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

}  // namespace sz
