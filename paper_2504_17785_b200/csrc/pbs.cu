// pbs.cu -- blind rotation (MS + ACC init + n x CMux + SE) and BSK -> Fourier
// for k = 1, N = 2048 on sm_100a.
//
// Steps (conventions §8(c) C4-C7, R3-R6):
//   MS:   a~_i = round(a_i * 2N / 2^64)                                  (a2)
//   init: ACC = (0, X^{-b~} v)                                           (a3)
//   CMux: ACC += ExtProd(BSK_i, X^{a~_i} ACC - ACC)   for i < n          (a4)
//         rotate-diff -> signed digits -> forward FFT -> pointwise MAC with
//         the Fourier BSK (P limbs) -> inverse FFT -> exact rounding and
//         limb recombination mod 2^64 -> ACC +=
//   SE:   coefficient 0 of ACC as a big-key LWE                          (a5)
//
// Design: persistent CTAs of 128 threads = two teams of
// 64; team g owns GLWE component g (mask / body). ACC (2 x 2048 u64) stays in
// shared memory for the whole CMux loop; the decomposed digits' spectra are
// staged in shared memory (one 16 KiB array per GGSW row); every transform is
// register resident (16 complex per thread) with two shared-memory exchanges.
// The BSK is streamed from L2 (it is read once per CMux per ciphertext and is
// laid out so each warp load is 512 contiguous bytes).
#include <cmath>
#include <mutex>

#include "fft.cuh"
#include "tmem.cuh"

#ifndef SZ_PAIR_LIMBS
#define SZ_PAIR_LIMBS 0  // limb pairs in the inverse: measured slower (17.3k vs 27.5k PBS/s, register pressure)
#endif

namespace sz {

__device__ Tables g_tables;
__constant__ double2 c_twist[16];

static std::once_flag g_tables_once[64];
static int g_tables_status[64];

// Build the twiddle tables on the host in long double and round once to double.
static int init_tables_for_device(int dev) {
  Tables h;
  const long double PI = 3.141592653589793238462643383279502884L;
  for (int k = 0; k < 16; k++)
    for (int t = 0; t < 64; t++) {
      long double ang = PI * (long double)(t * (4 * k + 1)) / 2048.0L;
      h.tw1[k * 64 + t] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
  for (int k = 0; k < 16; k++)
    for (int s = 0; s < 4; s++) {
      long double ang = 2.0L * PI * (long double)(s * k) / 64.0L;
      h.tw2[k * 4 + s] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
  for (int m = 0; m < 16; m++) {
    long double ang = PI * (long double)m / 32.0L;
    h.twist[m] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return SILENZIO_ERR_CUDA;
  if (prev != dev && cudaSetDevice(dev) != cudaSuccess) return SILENZIO_ERR_CUDA;
  cudaError_t e = cudaMemcpyToSymbol(g_tables, &h, sizeof(Tables));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_twist, h.twist, sizeof(h.twist));
  if (prev != dev) cudaSetDevice(prev);
  return e == cudaSuccess ? SILENZIO_OK : SILENZIO_ERR_CUDA;
}

int ensure_tables() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SILENZIO_ERR_CUDA;
  std::call_once(g_tables_once[dev], [dev] { g_tables_status[dev] = init_tables_for_device(dev); });
  return g_tables_status[dev];
}

// ------------------------------------------------------------------ team FFT
// named barrier per 64-thread team (id 1 + team index within the CTA)
__device__ __forceinline__ void team_sync(int team) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(kTeam) : "memory");
}
// named barrier `id` over `count` threads (whole warps)
__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Forward transform. In: x[m] = folded value at j = t + 64 m (natural m).
// Out: x[4u + r] = spectrum at position 4 (t + 64 u) + bitrev2(r) ("slot" order).
// `buf` (16 KiB) is the exchange buffer; on return the caller must team_sync
// before overwriting it (other threads may still be reading pass-3 data).
__device__ __forceinline__ void fwd_fft(double2 (&x)[16], double2 *buf, int t, int team) {
  const Tables &T = g_tables;
  // negacyclic twist, part 1: w^{64 m} (the w^t part is folded into tw1)
#pragma unroll
  for (int m = 0; m < 16; m++) x[m] = cmul(x[m], c_twist[m]);
  // pass 1: radix 16 over stride 64 (thread owns offset s = t)
  dft<16, false>(x);
  const int c1 = t ^ ((t >> 3) & 3);  // swz(t + 64 k) = 64 k + (c1 ^ 4 (k & 1))
  team_sync(team);
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int k = bitrev4(r);
#ifdef SZ_DIAG_TW
    const double2 w = make_double2(0.7 + k, 0.1 * t);
#else
    const double2 w = __ldg(&T.tw1[k * 64 + t]);
#endif
    buf[64 * k + (c1 ^ ((k & 1) << 2))] = cmul(x[r], w);
  }
  team_sync(team);
  // pass 2: radix 16 over stride 4 inside blocks of 64
  const int b = t >> 2, s = t & 3;
  double2 y[16];
#pragma unroll
  for (int m = 0; m < 16; m++) y[m] = buf[swz(64 * b + s + 4 * m)];
  dft<16, false>(y);
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int k = bitrev4(r);
    const double2 w = __ldg(&T.tw2[k * 4 + s]);
    buf[swz(64 * b + s + 4 * k)] = (k == 0) ? y[r] : cmul(y[r], w);
  }
  team_sync(team);
  // pass 3: radix 4 over stride 1, four groups per thread
#pragma unroll
  for (int u = 0; u < 4; u++) {
    double2 z[4];
#pragma unroll
    for (int m = 0; m < 4; m++) z[m] = buf[swz(4 * (t + 64 * u) + m)];
    dft<4, false>(z);
#pragma unroll
    for (int r = 0; r < 4; r++) x[4 * u + r] = z[r];
  }
}

// Inverse transform (unnormalised). In: slot order as produced by fwd_fft.
// Out: x[m] = value at j = t + 64 m, untwisted: (c_j + i c_{j+1024}) * M.
__device__ __forceinline__ void inv_fft(double2 (&x)[16], double2 *buf, int t, int team) {
  const Tables &T = g_tables;
  team_sync(team);  // previous users of buf are done
  // pass 3^-1
#pragma unroll
  for (int u = 0; u < 4; u++) {
    double2 z[4];
#pragma unroll
    for (int k = 0; k < 4; k++) z[k] = x[4 * u + bitrev2(k)];
    dft<4, true>(z);
#pragma unroll
    for (int q = 0; q < 4; q++) buf[swz(4 * (t + 64 * u) + bitrev2(q))] = z[q];
  }
  team_sync(team);
  // pass 2^-1
  const int b = t >> 2, s = t & 3;
  double2 y[16];
#pragma unroll
  for (int k = 0; k < 16; k++) {
    const double2 v = buf[swz(64 * b + s + 4 * k)];
    y[k] = (k == 0) ? v : cmulc(v, __ldg(&T.tw2[k * 4 + s]));
  }
  dft<16, true>(y);
#pragma unroll
  for (int q = 0; q < 16; q++) buf[swz(64 * b + s + 4 * bitrev4(q))] = y[q];
  team_sync(team);
  // pass 1^-1
  const int c1 = t ^ ((t >> 3) & 3);
#pragma unroll
  for (int k = 0; k < 16; k++) x[k] = cmulc(buf[64 * k + (c1 ^ ((k & 1) << 2))], __ldg(&T.tw1[k * 64 + t]));
  dft<16, true>(x);
  // x[q] now holds m = bitrev4(q); reorder to natural m and untwist
  double2 o[16];
#pragma unroll
  for (int q = 0; q < 16; q++) o[bitrev4(q)] = x[q];
#pragma unroll
  for (int m = 0; m < 16; m++) x[m] = cmulc(o[m], c_twist[m]);
}

// Two inverse transforms interleaved (independent data, shared twiddle loads
// and barriers): xa through buffer ba, xb through buffer bb.
__device__ __forceinline__ void inv_fft2(double2 (&xa)[16], double2 (&xb)[16], double2 *ba, double2 *bb, int t,
                                         int team) {
  const Tables &T = g_tables;
  team_sync(team);
#pragma unroll
  for (int u = 0; u < 4; u++) {
    double2 za[4], zb[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      za[k] = xa[4 * u + bitrev2(k)];
      zb[k] = xb[4 * u + bitrev2(k)];
    }
    dft<4, true>(za);
    dft<4, true>(zb);
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int pos = swz(4 * (t + 64 * u) + bitrev2(q));
      ba[pos] = za[q];
      bb[pos] = zb[q];
    }
  }
  team_sync(team);
  {
    const int b = t >> 2, s = t & 3;
    double2 ya[16], yb[16];
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const int pos = swz(64 * b + s + 4 * k);
      const double2 va = ba[pos], vb = bb[pos];
      if (k == 0) {
        ya[k] = va;
        yb[k] = vb;
      } else {
        const double2 w = __ldg(&T.tw2[k * 4 + s]);
        ya[k] = cmulc(va, w);
        yb[k] = cmulc(vb, w);
      }
    }
    dft<16, true>(ya);
    dft<16, true>(yb);
#pragma unroll
    for (int q = 0; q < 16; q++) {
      const int pos = swz(64 * b + s + 4 * bitrev4(q));
      ba[pos] = ya[q];
      bb[pos] = yb[q];
    }
  }
  team_sync(team);
  const int c1 = t ^ ((t >> 3) & 3);
#pragma unroll
  for (int k = 0; k < 16; k++) {
    const int pos = 64 * k + (c1 ^ ((k & 1) << 2));
    const double2 w = __ldg(&T.tw1[k * 64 + t]);
    xa[k] = cmulc(ba[pos], w);
    xb[k] = cmulc(bb[pos], w);
  }
  dft<16, true>(xa);
  dft<16, true>(xb);
  double2 oa[16], ob[16];
#pragma unroll
  for (int q = 0; q < 16; q++) {
    oa[bitrev4(q)] = xa[q];
    ob[bitrev4(q)] = xb[q];
  }
#pragma unroll
  for (int m = 0; m < 16; m++) {
    xa[m] = cmulc(oa[m], c_twist[m]);
    xb[m] = cmulc(ob[m], c_twist[m]);
  }
}

// ------------------------------------------------------------- limb helpers
__device__ __forceinline__ i64 sext(i64 x, int bits) {
  return (bits >= 64) ? x : (i64)((u64)x << (64 - bits)) >> (64 - bits);
}

// Split a u64 torus coefficient into P signed limbs, limb p weighted 2^{p*w};
// the top limb is reduced mod 2^{64-(P-1)w} (its weight makes higher bits vanish).
__device__ __forceinline__ void limb_split(u64 g, int P, int w, double (&l)[3]) {
  if (P == 1) {
    l[0] = (double)(i64)g;
    return;
  }
  const i64 l0 = sext((i64)g, w);
  const u64 rem = (g - (u64)l0) >> w;  // exact: g - l0 = 0 mod 2^w
  l[0] = (double)l0;
  if (P == 2) {
    l[1] = (double)sext((i64)rem, 64 - w);
    return;
  }
  const i64 l1 = sext((i64)rem, w);
  const i64 rem2 = ((i64)rem - l1) >> w;
  l[1] = (double)l1;
  l[2] = (double)sext(rem2, 64 - 2 * w);
}

// double (integer-valued up to rounding) -> round to nearest, mod 2^64
__device__ __forceinline__ u64 f64_to_torus(double x) {
  const double hi = floor(x * 0x1p-32);
  const double lo = fma(hi, -0x1p32, x);  // exact
  return ((u64)__double2ll_rn(hi) << 32) + (u64)__double2ll_rn(lo);
}

// x mod 2^bits for an integer-valued double |x| < 2^53 (exact)
__device__ __forceinline__ double fmod_pow2(double x, double two_bits, double inv_two_bits) {
  return fma(-floor(x * inv_two_bits), two_bits, x);
}

// ---------------------------------------------------------------- v3 (TMEM)
// CTA = two ciphertexts x two 64-thread teams (256 threads). Warp w:
// team g = w >> 2 (GLWE component), ciphertext slot cs = (w >> 1) & 1, half h = w & 1.
// The two teams of a ciphertext sit on warps {2cs+h} and {4+2cs+h}, i.e. in the
// same TMEM lane quadrant, so thread t of team 0 and thread t of team 1 own the
// same TMEM lane. The digit spectra D^_0, D^_1 (one per team) are exchanged
// through TMEM columns [0,64) and [64,128) instead of shared memory, and the
// pass-1 twiddles w^{t(4k+1)} live in TMEM columns [128,192), so neither uses
// the L1/shared-memory data path. Shared memory holds only the per-team
// transient buffer (ACC copy for the rotation, then every FFT exchange).
#ifndef SZ_TW_TMEM
#define SZ_TW_TMEM 0  // twiddles from TMEM: measured slower in v2 (17.2k vs 27.6k PBS/s): tcgen05.ld latency
#endif
#ifndef SZ_V3
#define SZ_V3 0  // TMEM spectrum exchange: measured slower (21.7k vs 27.6k PBS/s, TMEM load latency)
#endif
constexpr uint32_t kTmCols = 256, kColD = 0, kColTw = 128;

__device__ __forceinline__ void fwd_fft_tm(double2 (&x)[16], double2 *buf, int t, int team, uint32_t tw_ta) {
  const Tables &T = g_tables;
#pragma unroll
  for (int m = 0; m < 16; m++) x[m] = cmul(x[m], c_twist[m]);
  dft<16, false>(x);
  const int c1 = t ^ ((t >> 3) & 3);
  team_sync(team);
#if SZ_TW_TMEM
#pragma unroll
  for (int j = 0; j < 4; j += 2) {
    uint32_t ra[16], rb[16];
    tmem_ld16(tw_ta + 16 * j, ra);
    tmem_ld16(tw_ta + 16 * (j + 1), rb);
    tmem_wait_ld16x2(ra, rb);
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int r = 4 * j + q, k = bitrev4(r);
      buf[64 * k + (c1 ^ ((k & 1) << 2))] = cmul(x[r], unpack1(ra, q));
      const int r2 = 4 * (j + 1) + q, k2 = bitrev4(r2);
      buf[64 * k2 + (c1 ^ ((k2 & 1) << 2))] = cmul(x[r2], unpack1(rb, q));
    }
  }
#else
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int k = bitrev4(r);
    buf[64 * k + (c1 ^ ((k & 1) << 2))] = cmul(x[r], __ldg(&T.tw1[k * 64 + t]));
  }
#endif
  team_sync(team);
  const int b = t >> 2, s = t & 3;
  double2 y[16];
#pragma unroll
  for (int m = 0; m < 16; m++) y[m] = buf[swz(64 * b + s + 4 * m)];
  dft<16, false>(y);
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int k = bitrev4(r);
    buf[swz(64 * b + s + 4 * k)] = (k == 0) ? y[r] : cmul(y[r], __ldg(&T.tw2[k * 4 + s]));
  }
  team_sync(team);
#pragma unroll
  for (int u = 0; u < 4; u++) {
    double2 z[4];
#pragma unroll
    for (int m = 0; m < 4; m++) z[m] = buf[swz(4 * (t + 64 * u) + m)];
    dft<4, false>(z);
#pragma unroll
    for (int r = 0; r < 4; r++) x[4 * u + r] = z[r];
  }
}

__device__ __forceinline__ void inv_fft_tm(double2 (&x)[16], double2 *buf, int t, int team, uint32_t tw_ta) {
  const Tables &T = g_tables;
  team_sync(team);
#pragma unroll
  for (int u = 0; u < 4; u++) {
    double2 z[4];
#pragma unroll
    for (int k = 0; k < 4; k++) z[k] = x[4 * u + bitrev2(k)];
    dft<4, true>(z);
#pragma unroll
    for (int q = 0; q < 4; q++) buf[swz(4 * (t + 64 * u) + bitrev2(q))] = z[q];
  }
  team_sync(team);
  {
    const int b = t >> 2, s = t & 3;
    double2 y[16];
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const double2 v = buf[swz(64 * b + s + 4 * k)];
      y[k] = (k == 0) ? v : cmulc(v, __ldg(&T.tw2[k * 4 + s]));
    }
    dft<16, true>(y);
#pragma unroll
    for (int q = 0; q < 16; q++) buf[swz(64 * b + s + 4 * bitrev4(q))] = y[q];
  }
  team_sync(team);
  const int c1 = t ^ ((t >> 3) & 3);
#if SZ_TW_TMEM
#pragma unroll
  for (int j = 0; j < 4; j += 2) {
    uint32_t ra[16], rb[16];
    tmem_ld16(tw_ta + 16 * j, ra);
    tmem_ld16(tw_ta + 16 * (j + 1), rb);
    tmem_wait_ld16x2(ra, rb);
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int k = bitrev4(4 * j + q), k2 = bitrev4(4 * (j + 1) + q);
      x[k] = cmulc(buf[64 * k + (c1 ^ ((k & 1) << 2))], unpack1(ra, q));
      x[k2] = cmulc(buf[64 * k2 + (c1 ^ ((k2 & 1) << 2))], unpack1(rb, q));
    }
  }
#else
#pragma unroll
  for (int k = 0; k < 16; k++) x[k] = cmulc(buf[64 * k + (c1 ^ ((k & 1) << 2))], __ldg(&T.tw1[k * 64 + t]));
#endif
  dft<16, true>(x);
  double2 o[16];
#pragma unroll
  for (int q = 0; q < 16; q++) o[bitrev4(q)] = x[q];
#pragma unroll
  for (int m = 0; m < 16; m++) x[m] = cmulc(o[m], c_twist[m]);
}

// ------------------------------------------------------------ BR kernel
struct BRArgs {
  const u64 *lwe_small;  // [count][n+1]
  const u32 *lut_ids;    // [count] or null
  const u64 *luts;       // [num_luts][N]
  u32 num_luts;
  const double2 *fbsk;   // [n][2][rows][P][16][64]
  u64 *lwe_out;          // [count][N+1]
  long count;
  int n, level, base_log, P, w;
};

constexpr int kN = 2048;
constexpr int kLog2_2N = 12;

__host__ __device__ constexpr size_t br_smem_bytes(int rows, int n) {
  return (SZ_PAIR_LIMBS ? 4 : 2) * kM * sizeof(double2)  // transient buffers per team (ACC copy / IFFT exchanges)
         + (size_t)rows * kM * sizeof(double2)    // digit spectra (also forward exchange buffers)
         + ((size_t)n * sizeof(unsigned short) + 15) / 16 * 16;  // modswitched masks
}

// limb p of the inverse transform -> its exact contribution round(x) * 2^{p w} mod 2^64
__device__ __forceinline__ u64 limb_to_torus(double x, int p, int P, int w) {
  if (P == 3 || p > 0) return (u64)__double2ll_rn(x) << (p * w);  // |x| < 2^53: exact
  return f64_to_torus(x);                                          // P <= 2, low limb may exceed 2^53
}

// ACC lives in registers for the whole CMux loop: thread t of team g owns
// ACC_g[j] for j = t + 64 m + 1024 h (m < 16, h < 2) -- exactly the
// coefficients its inverse FFT produces, so the update never leaves registers.
// Shared memory per CTA: two 16 KiB transient buffers (the ACC copy the
// rotation reads, later the IFFT exchange) + one 16 KiB spectrum per GGSW row.
constexpr int kMaxCPB = 1;  // ciphertexts per CTA (lockstep CTAs measured slower: shared stalls)
#ifndef SZ_BR_MINBLOCKS
#define SZ_BR_MINBLOCKS 2
#endif

template <int L, int P>
__global__ void __launch_bounds__(128 * kMaxCPB, SZ_BR_MINBLOCKS) blind_rotate_kernel(BRArgs A) {
  extern __shared__ __align__(16) unsigned char smem_all[];
  constexpr int rows = 2 * L;
  const int slot = threadIdx.x >> 7;  // which ciphertext of the CTA
  unsigned char *smem = smem_all + slot * br_smem_bytes(rows, A.n);
  double2 *tbuf_all = reinterpret_cast<double2 *>(smem);  // [2 teams][2][1024]
  double2 *dsm = tbuf_all + (SZ_PAIR_LIMBS ? 4 : 2) * kM;  // [rows][16][64]
  unsigned short *abar = reinterpret_cast<unsigned short *>(dsm + (size_t)rows * kM);

  const int tid = threadIdx.x & 127;
  const int team = tid >> 6, t = tid & 63;
  const int bar_team = slot * 2 + team;
  double2 *tbuf = tbuf_all + team * (SZ_PAIR_LIMBS ? 2 : 1) * kM;
  double2 *tbuf2 = tbuf + kM;  // used only with SZ_PAIR_LIMBS
  u64 *accs = reinterpret_cast<u64 *>(tbuf);  // ACC_g copy [2048]
  const int n = A.n, w = A.w, blog = A.base_log;
#if SZ_TW_TMEM
  // pass-1 twiddles w^{t(4k+1)} of this thread's t in its own TMEM lane
  // (64 columns per CTA): they leave the L1 data path entirely.
  __shared__ uint32_t tmem_slot;
  const int wid = threadIdx.x >> 5;
  if (wid == 0) tmem_alloc(&tmem_slot, 64);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t ta_tw = tmem_slot + ((uint32_t)(32 * (wid & 3)) << 16);
#pragma unroll
  for (int j = 0; j < 4; j++) {
    double2 v[4];
#pragma unroll
    for (int q = 0; q < 4; q++) v[q] = g_tables.tw1[bitrev4(4 * j + q) * 64 + t];
    uint32_t r16[16];
    pack4(v, r16);
    tmem_st16(ta_tw + 16 * j, r16);
  }
  tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
#define SZ_FWD(x, b, tt, tm) fwd_fft_tm(x, b, tt, tm, ta_tw)
#define SZ_INV(x, b, tt, tm) inv_fft_tm(x, b, tt, tm, ta_tw)
#else
#define SZ_FWD(x, b, tt, tm) fwd_fft(x, b, tt, tm)
#define SZ_INV(x, b, tt, tm) inv_fft(x, b, tt, tm)
#endif

  // all CTA slots iterate the same number of times (idle slots keep the barriers)
  const int cpb = blockDim.x >> 7;
  const long ngroups = (A.count + cpb - 1) / cpb;
  for (long grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const long c = grp * cpb + slot;
    const bool live = c < A.count;
    const u64 *lwe = A.lwe_small + (size_t)c * (n + 1);
    // ---- modulus switch (a2)
    for (int i = tid; i < n; i += 128) abar[i] = live ? (unsigned short)sz_modswitch(lwe[i], kLog2_2N) : 0;
    const int bt = live ? (int)sz_modswitch(lwe[n], kLog2_2N) : 0;
    // ---- ACC init (a3): ACC = (0, X^{-b~} v), (X^{-b} v)[j] = v[j + b] (negacyclic)
    u32 id = (A.lut_ids && live) ? A.lut_ids[c] : 0u;
    if (id >= A.num_luts) id = 0;
    const u64 *v = A.luts + (size_t)id * kN;
    u64 accr[16][2];
#pragma unroll
    for (int m = 0; m < 16; m++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int j = t + 64 * m + 1024 * h;
        const int idx = (j + bt) & (2 * kN - 1);
        const u64 vv = (idx < kN) ? v[idx] : (u64)0 - v[idx - kN];
        accr[m][h] = team ? vv : 0ull;
      }
    __syncthreads();  // abar visible

    for (int i = 0; i < n; i++) {
      const int a = abar[i];
      // ---------------- publish ACC_g for the rotation
#pragma unroll
      for (int m = 0; m < 16; m++)
#pragma unroll
        for (int h = 0; h < 2; h++) accs[t + 64 * m + 1024 * h] = accr[m][h];
      team_sync(bar_team);
      // ---------------- forward: digits of X^a ACC_g - ACC_g, one FFT per level
#pragma unroll 1
      for (int lvl = 1; lvl <= L; lvl++) {
        double2 x[16];
#pragma unroll
        for (int m = 0; m < 16; m++) {
          double dv[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int j = t + 64 * m + 1024 * h;
            const int src = (j - a) & (2 * kN - 1);
            const u64 rv = accs[src & (kN - 1)];
            const u64 rot = (src < kN) ? rv : (u64)0 - rv;
            u64 r = sz_decomp_round(rot - accr[m][h], blog, L);
            i64 d = 0;
            // peel digits t = l, l-1, ..., lvl  (level lvl has weight q/B^lvl)
#pragma unroll
            for (int tt = L; tt >= 1; tt--) {
              const i64 dd = sz_decomp_next(r, blog);
              if (tt == lvl) d = dd;
            }
            dv[h] = (double)d;
          }
          x[m] = make_double2(dv[0], dv[1]);
        }
        double2 *drow = dsm + (size_t)(team * L + (lvl - 1)) * kM;
        SZ_FWD(x, drow, t, bar_team);  // the row's own spectrum buffer is the exchange buffer
        team_sync(bar_team);
#pragma unroll
        for (int sl = 0; sl < 16; sl++) drow[sl * 64 + t] = x[sl];
      }
      __syncthreads();  // every row's spectrum is complete
      // ---------------- inverse: output component o = team, limbs top -> 0
      const int o = team;
#ifdef SZ_DIAG_G_L1
      const double2 *Gi = A.fbsk + ((size_t)(i & 0) * 2 + o) * rows * P * kM;
#else
      const double2 *Gi = A.fbsk + ((size_t)i * 2 + o) * rows * P * kM;
#endif
#pragma unroll 1
      for (int p = P - 1; p >= 0; p -= (SZ_PAIR_LIMBS ? 2 : 1)) {
        if (SZ_PAIR_LIMBS && p >= 1) {
          // limbs p and p-1 together: one pass over the spectra, two interleaved IFFTs
          const int pa = p, pb = p - 1;
          double2 ya[16], yb[16];
#pragma unroll
          for (int sl = 0; sl < 16; sl++) {
            ya[sl] = make_double2(0.0, 0.0);
            yb[sl] = make_double2(0.0, 0.0);
          }
#pragma unroll 1
          for (int row = 0; row < rows; row++) {
            const double2 *Ga = Gi + ((size_t)row * P + pa) * kM + t;
            const double2 *Gb = Gi + ((size_t)row * P + pb) * kM + t;
            const double2 *D = dsm + (size_t)row * kM + t;
#pragma unroll
            for (int qq = 0; qq < 4; qq++) {
              double2 ga[4], gb[4], dd[4];
#pragma unroll
              for (int q = 0; q < 4; q++) {
                ga[q] = __ldg(&Ga[(4 * qq + q) * 64]);
                gb[q] = __ldg(&Gb[(4 * qq + q) * 64]);
              }
#pragma unroll
              for (int q = 0; q < 4; q++) dd[q] = D[(4 * qq + q) * 64];
#pragma unroll
              for (int q = 0; q < 4; q++) {
                cmac(ya[4 * qq + q], dd[q], ga[q]);
                cmac(yb[4 * qq + q], dd[q], gb[q]);
              }
            }
          }
          inv_fft2(ya, yb, tbuf, tbuf2, t, bar_team);
#pragma unroll
          for (int m = 0; m < 16; m++) {
            accr[m][0] += limb_to_torus(ya[m].x, pa, P, w) + limb_to_torus(yb[m].x, pb, P, w);
            accr[m][1] += limb_to_torus(ya[m].y, pa, P, w) + limb_to_torus(yb[m].y, pb, P, w);
          }
        } else {
          double2 y[16];
#pragma unroll
          for (int sl = 0; sl < 16; sl++) y[sl] = make_double2(0.0, 0.0);
#pragma unroll 1
          for (int row = 0; row < rows; row++) {
            const double2 *G = Gi + ((size_t)row * P + p) * kM + t;
            const double2 *D = dsm + (size_t)row * kM + t;
#pragma unroll
            for (int qq = 0; qq < 4; qq++) {
              double2 g[4], dd[4];
#pragma unroll
              for (int q = 0; q < 4; q++) g[q] = __ldg(&G[(4 * qq + q) * 64]);
#pragma unroll
              for (int q = 0; q < 4; q++) dd[q] = D[(4 * qq + q) * 64];
#pragma unroll
              for (int q = 0; q < 4; q++) cmac(y[4 * qq + q], dd[q], g[q]);
            }
          }
          SZ_INV(y, tbuf, t, bar_team);
#pragma unroll
          for (int m = 0; m < 16; m++) {
            accr[m][0] += limb_to_torus(y[m].x, p, P, w);
            accr[m][1] += limb_to_torus(y[m].y, p, P, w);
          }
        }
      }
      __syncthreads();  // spectra and transient buffers free for the next CMux
    }
    // ---- sample extraction (a5): a'[0] = A[0], a'[i] = -A[N-i], b' = B[0]
    u64 *out = A.lwe_out + (size_t)c * (kN + 1);
#pragma unroll
    for (int m = 0; m < 16; m++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int j = t + 64 * m + 1024 * h;
        if (!live) {
        } else if (team == 0) {
          if (j == 0) out[0] = accr[m][h];
          else out[kN - j] = (u64)0 - accr[m][h];
        } else if (j == 0) {
          out[kN] = accr[m][h];
        }
      }
    __syncthreads();  // abar reuse
  }
#if SZ_TW_TMEM
  tmem_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tmem_slot, 64);
#endif
#undef SZ_FWD
#undef SZ_INV
}


__host__ __device__ constexpr size_t br3_smem_per_ct(int n) {
  return 2 * kM * sizeof(double2) + ((size_t)n * sizeof(unsigned short) + 15) / 16 * 16;
}

template <int P>
__global__ void __launch_bounds__(256, 1) blind_rotate_tmem_kernel(BRArgs A) {
  extern __shared__ __align__(16) unsigned char smem_all[];
  __shared__ uint32_t tmem_slot;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = wid >> 2, cs = (wid >> 1) & 1, h = wid & 1;
  const int t = h * 32 + lane;             // FFT thread index within the team
  const int ti = g * 64 + t;               // index within the ciphertext's 128 threads
  const int team = cs * 2 + g;             // team_sync id 1 + team, 64 threads
  const int pair_id = 5 + cs;              // both teams of this ciphertext, 128 threads
  const int n = A.n, w = A.w, blog = A.base_log;
  unsigned char *sm = smem_all + cs * br3_smem_per_ct(n);
  double2 *tbuf = reinterpret_cast<double2 *>(sm) + g * kM;
  u64 *accs = reinterpret_cast<u64 *>(tbuf);
  unsigned short *abar = reinterpret_cast<unsigned short *>(sm + 2 * kM * sizeof(double2));

  if (wid == 0) tmem_alloc(&tmem_slot, kTmCols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tlane = tmem_slot + ((uint32_t)(32 * (wid & 3)) << 16);
  const uint32_t ta_tw = tlane + kColTw, ta_d0 = tlane + kColD, ta_d1 = tlane + kColD + 64;
  if (g == 0) {  // pass-1 twiddles of this lane's t, in register order r (k = bitrev4(r))
#pragma unroll
    for (int j = 0; j < 4; j++) {
      double2 v[4];
#pragma unroll
      for (int q = 0; q < 4; q++) v[q] = g_tables.tw1[bitrev4(4 * j + q) * 64 + t];
      uint32_t r16[16];
      pack4(v, r16);
      tmem_st16(ta_tw + 16 * j, r16);
    }
    tmem_wait_st();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();

  const long ngroups = (A.count + 1) / 2;
  for (long grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const long c = grp * 2 + cs;
    const bool live = c < A.count;
    const u64 *lwe = A.lwe_small + (size_t)(live ? c : 0) * (n + 1);
    for (int i = ti; i < n; i += 128) abar[i] = live ? (unsigned short)sz_modswitch(lwe[i], kLog2_2N) : 0;
    const int bt = live ? (int)sz_modswitch(lwe[n], kLog2_2N) : 0;
    u32 id = (A.lut_ids && live) ? A.lut_ids[c] : 0u;
    if (id >= A.num_luts) id = 0;
    const u64 *v = A.luts + (size_t)id * kN;
    u64 accr[16][2];
#pragma unroll
    for (int m = 0; m < 16; m++)
#pragma unroll
      for (int hh = 0; hh < 2; hh++) {
        const int j = t + 64 * m + 1024 * hh;
        const int idx = (j + bt) & (2 * kN - 1);
        const u64 vv = (idx < kN) ? v[idx] : (u64)0 - v[idx - kN];
        accr[m][hh] = g ? vv : 0ull;
      }
    bar_sync(pair_id, 128);  // abar visible to both teams
    for (int i = 0; i < n; i++) {
      const int a = abar[i];
#pragma unroll
      for (int m = 0; m < 16; m++)
#pragma unroll
        for (int hh = 0; hh < 2; hh++) accs[t + 64 * m + 1024 * hh] = accr[m][hh];
      team_sync(team);
      double2 x[16];
#pragma unroll
      for (int m = 0; m < 16; m++) {
        double dv[2];
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
          const int j = t + 64 * m + 1024 * hh;
          const int src = (j - a) & (2 * kN - 1);
          const u64 rv = accs[src & (kN - 1)];
          const u64 rot = (src < kN) ? rv : (u64)0 - rv;
          u64 r = sz_decomp_round(rot - accr[m][hh], blog, 1);
          dv[hh] = (double)sz_decomp_next(r, blog);
        }
        x[m] = make_double2(dv[0], dv[1]);
      }
      fwd_fft_tm(x, tbuf, t, team, ta_tw);
      {
        const uint32_t ta_dg = g ? ta_d1 : ta_d0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
          uint32_t r16[16];
          pack4(&x[4 * j], r16);
          tmem_st16(ta_dg + 16 * j, r16);
        }
        tmem_wait_st();
      }
      tmem_fence_before();
      bar_sync(pair_id, 128);
      tmem_fence_after();
      // ---------------- inverse: output component o = g, limbs top -> 0
      const double2 *Gi = A.fbsk + ((size_t)i * 2 + g) * 2 * P * kM;
#pragma unroll 1
      for (int p = P - 1; p >= 0; p--) {
        double2 y[16];
        const double2 *G0 = Gi + ((size_t)0 * P + p) * kM + t;
        const double2 *G1 = Gi + ((size_t)1 * P + p) * kM + t;
#pragma unroll
        for (int j = 0; j < 4; j++) {
          double2 g0[4], g1[4];
#pragma unroll
          for (int q = 0; q < 4; q++) {
            g0[q] = __ldg(&G0[(4 * j + q) * 64]);
            g1[q] = __ldg(&G1[(4 * j + q) * 64]);
          }
          uint32_t d0[16], d1[16];
          tmem_ld16(ta_d0 + 16 * j, d0);
          tmem_ld16(ta_d1 + 16 * j, d1);
          tmem_wait_ld16x2(d0, d1);
#pragma unroll
          for (int q = 0; q < 4; q++) {
            double2 acc = make_double2(0.0, 0.0);
            cmac(acc, unpack1(d0, q), g0[q]);
            cmac(acc, unpack1(d1, q), g1[q]);
            y[4 * j + q] = acc;
          }
        }
        inv_fft_tm(y, tbuf, t, team, ta_tw);
#pragma unroll
        for (int m = 0; m < 16; m++) {
          accr[m][0] += limb_to_torus(y[m].x, p, P, w);
          accr[m][1] += limb_to_torus(y[m].y, p, P, w);
        }
      }
      tmem_fence_before();
      bar_sync(pair_id, 128);  // both teams done reading D^ (TMEM) before the next CMux writes it
      tmem_fence_after();
    }
    if (live) {
      u64 *out = A.lwe_out + (size_t)c * (kN + 1);
#pragma unroll
      for (int m = 0; m < 16; m++)
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
          const int j = t + 64 * m + 1024 * hh;
          if (g == 0) {
            if (j == 0) out[0] = accr[m][hh];
            else out[kN - j] = (u64)0 - accr[m][hh];
          } else if (j == 0) {
            out[kN] = accr[m][hh];
          }
        }
    }
    bar_sync(pair_id, 128);  // abar reuse
  }
  tmem_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tmem_slot, kTmCols);
}

// --------------------------------------------------------- BSK -> Fourier
struct B2FArgs {
  const u64 *bsk;  // [n][rows][2][N]
  double2 *fbsk;   // [n][2][rows][P][16][64]
  int n, rows, P, w;
};

// one team (64 threads) per (i, row, o, p)
__global__ void __launch_bounds__(64) bsk_to_fourier_kernel(B2FArgs A) {
  __shared__ __align__(16) double2 buf[kM];
  const int t = threadIdx.x;
  long blk = blockIdx.x;
  const int p = blk % A.P; blk /= A.P;
  const int o = blk % 2; blk /= 2;
  const int row = blk % A.rows; blk /= A.rows;
  const int i = (int)blk;
  const u64 *g = A.bsk + (((size_t)i * A.rows + row) * 2 + o) * kN;
  double2 x[16];
#pragma unroll
  for (int m = 0; m < 16; m++) {
    double l0[3], l1[3];
    limb_split(g[t + 64 * m], A.P, A.w, l0);
    limb_split(g[t + 64 * m + 1024], A.P, A.w, l1);
    x[m] = make_double2(l0[p], l1[p]);
  }
  fwd_fft(x, buf, t, 0);
  double2 *dst = A.fbsk + ((((size_t)i * 2 + o) * A.rows + row) * A.P + p) * kM;
  const double scale = 1.0 / kM;
#pragma unroll
  for (int sl = 0; sl < 16; sl++) dst[sl * 64 + t] = make_double2(x[sl].x * scale, x[sl].y * scale);
}

// ------------------------------------------------------------ host launch
// Kernel variant, CTA shape and resident ciphertexts per wave for these params.
struct BRPlan {
  void (*kern)(BRArgs);
  int cpb;
  size_t smem;
  long wave;  // ciphertexts per launch (resident on the whole GPU)
};

static int plan_blind_rotate(const silenzio_params *P, BRPlan *plan) {
  const int level = (int)P->pbs_level, limbs = (int)P->fft_limbs, n = (int)P->lwe_dim;
  void (*kern)(BRArgs) = nullptr;
#define SZ_BR_CASE(LL, PP) \
  if (level == LL && limbs == PP) kern = blind_rotate_kernel<LL, PP>;
  SZ_BR_CASE(1, 1) SZ_BR_CASE(1, 2) SZ_BR_CASE(1, 3)
  SZ_BR_CASE(2, 1) SZ_BR_CASE(2, 2) SZ_BR_CASE(2, 3)
  SZ_BR_CASE(4, 1) SZ_BR_CASE(4, 2) SZ_BR_CASE(4, 3)
#undef SZ_BR_CASE
  if (!kern) return SILENZIO_ERR_UNSUPPORTED;
  const size_t per_ct = br_smem_bytes(2 * level, n);
  int cpb = (int)((227 * 1024) / per_ct);
  if (cpb > kMaxCPB) cpb = kMaxCPB;
  if (cpb < 1) return SILENZIO_ERR_UNSUPPORTED;
  const size_t smem = cpb * per_ct;
  SZ_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 0, per_sm = 0;
  SZ_CUDA_OK(cudaGetDevice(&dev));
  SZ_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SZ_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128 * cpb, smem));
  if (per_sm < 1) return SILENZIO_ERR_UNSUPPORTED;
  plan->kern = kern;
  plan->cpb = cpb;
  plan->smem = smem;
  plan->wave = (long)sms * per_sm * cpb;
  return SILENZIO_OK;
}

static int launch_blind_rotate_tmem(const BRArgs &A, const silenzio_params *P, size_t count, cudaStream_t stream) {
  void (*kern)(BRArgs) = nullptr;
  if (P->fft_limbs == 1) kern = blind_rotate_tmem_kernel<1>;
  if (P->fft_limbs == 2) kern = blind_rotate_tmem_kernel<2>;
  if (P->fft_limbs == 3) kern = blind_rotate_tmem_kernel<3>;
  if (!kern) return SILENZIO_ERR_UNSUPPORTED;
  const size_t smem = 2 * br3_smem_per_ct(A.n);
  if (smem > 200 * 1024) return SILENZIO_ERR_UNSUPPORTED;
  SZ_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 0;
  SZ_CUDA_OK(cudaGetDevice(&dev));
  SZ_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const long wave = 2L * sms;  // one CTA (two ciphertexts) per SM
  for (long c0 = 0; c0 < (long)count; c0 += wave) {
    BRArgs W = A;
    const long cnt = ((long)count - c0 < wave) ? (long)count - c0 : wave;
    W.lwe_small = A.lwe_small + (size_t)c0 * (A.n + 1);
    W.lut_ids = A.lut_ids ? A.lut_ids + c0 : nullptr;
    W.lwe_out = A.lwe_out + (size_t)c0 * (kN + 1);
    W.count = cnt;
    kern<<<(unsigned)((cnt + 1) / 2), 256, smem, stream>>>(W);
    SZ_LAUNCH_OK();
  }
  return SILENZIO_OK;
}

long blind_rotate_wave(const silenzio_params *P) {
#if SZ_V3
  if (P->pbs_level == 1) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return 2L * sms;
  }
#endif
  BRPlan plan;
  if (ensure_tables() != SILENZIO_OK || plan_blind_rotate(P, &plan) != SILENZIO_OK) return -1;
  return plan.wave;
}

int launch_blind_rotate(const u64 *lwe_small, const u32 *lut_ids, const u64 *luts, u32 num_luts,
                        const void *fbsk, u64 *lwe_out, size_t count, const silenzio_params *P,
                        cudaStream_t stream) {
  int st = ensure_tables();
  if (st != SILENZIO_OK) return st;
  BRArgs A;
  A.lwe_small = lwe_small;
  A.lut_ids = lut_ids;
  A.luts = luts;
  A.num_luts = num_luts;
  A.fbsk = reinterpret_cast<const double2 *>(fbsk);
  A.lwe_out = lwe_out;
  A.count = (long)count;
  A.n = (int)P->lwe_dim;
  A.level = (int)P->pbs_level;
  A.base_log = (int)P->pbs_base_log;
  A.P = (int)P->fft_limbs;
  A.w = (int)P->limb_bits;
#if SZ_V3
  if (P->pbs_level == 1) return launch_blind_rotate_tmem(A, P, count, stream);
#endif
  BRPlan plan;
  if ((st = plan_blind_rotate(P, &plan))) return st;
  void (*kern)(BRArgs) = plan.kern;
  const int cpb = plan.cpb;
  const size_t smem = plan.smem;
  // One launch per resident wave: every CTA of a wave sweeps BSK_0..BSK_{n-1}
  // at the same pace, so the streamed Fourier BSK (146 MB at set A, > L2)
  // is fetched from HBM about once per wave instead of once per drifting CTA.
  const long resident_cts = plan.wave;
  for (long c0 = 0; c0 < (long)count; c0 += resident_cts) {
    BRArgs W = A;
    const long cnt = ((long)count - c0 < resident_cts) ? (long)count - c0 : resident_cts;
    W.lwe_small = A.lwe_small + (size_t)c0 * (A.n + 1);
    W.lut_ids = A.lut_ids ? A.lut_ids + c0 : nullptr;
    W.lwe_out = A.lwe_out + (size_t)c0 * (kN + 1);
    W.count = cnt;
    const long grid = (cnt + cpb - 1) / cpb;
    kern<<<(unsigned)grid, 128 * cpb, smem, stream>>>(W);
    SZ_LAUNCH_OK();
  }
  return SILENZIO_OK;
}

int launch_bsk_to_fourier(const u64 *bsk, void *fbsk, const silenzio_params *P, cudaStream_t stream) {
  int st = ensure_tables();
  if (st != SILENZIO_OK) return st;
  B2FArgs A;
  A.bsk = bsk;
  A.fbsk = reinterpret_cast<double2 *>(fbsk);
  A.n = (int)P->lwe_dim;
  A.rows = 2 * (int)P->pbs_level;
  A.P = (int)P->fft_limbs;
  A.w = (int)P->limb_bits;
  const long blocks = (long)A.n * A.rows * 2 * A.P;
  bsk_to_fourier_kernel<<<(unsigned)blocks, 64, 0, stream>>>(A);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

}  // namespace sz
