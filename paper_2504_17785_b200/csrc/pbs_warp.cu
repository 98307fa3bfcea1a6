// pbs_warp.cu -- blind rotation for k = 1, N = 2048, level-1 gadget (parameter
// set A, the benchmark configuration) with warp-synchronous FFTs, the
// accumulator and the digit spectra in tensor memory, and the Fourier BSK
// staged into shared memory by the bulk-copy (TMA) engine.
//
// Same method and conventions as pbs.cu (SURVEY.md §8(a) a2-a5, §8(c) C4-C7,
// DESIGN.md R3-R6, R20); only the data movement differs:
//
//  * FFT: M = 1024 = 32 x 32 complex points per transform, one warp per
//    transform, 32 values per thread: pass 1 (radix 32 in registers), one
//    transposition through shared memory (XOR-swizzled, conflict free),
//    pass 2 (radix 32). Only __syncwarp between passes.
//  * CTA = 8 warps = 4 ciphertexts; ciphertext s uses warp s (GLWE mask
//    component) and warp s + 4 (body). Both warps of a ciphertext access the
//    same TMEM lane quadrant, so a thread and its partner share one lane:
//      columns [  0,128)  ACC_0 (warp s),  [128,256) ACC_1 (warp s + 4)
//      columns [256,384)  D^_0 (row 0 spectrum), [384,512) D^_1
//    The MAC reads both digit spectra from TMEM (off the L1/shared path).
//  * The four ciphertexts of a CTA run the CMux loop in lock step and share
//    the Fourier BSK: one 64 KiB bulk copy per (i, limb) into shared memory,
//    issued by one thread right after the previous limb's MAC and landing
//    during the inverse FFT (mbarrier completion).
//
// Fourier BSK layout for this kernel: [n][P][2 (o)][2 (row)][32 (r)][32 (lane)]
// where (r, lane) holds the spectrum at index lane + 32 r, times 1/M.
#include <cmath>
#include <cstring>
#include <mutex>

#include "fft.cuh"
#include "limbs.cuh"
#include "tmem.cuh"

namespace sz {
namespace w32 {

constexpr int kN = 2048;
constexpr int kLog2_2N = 12;
constexpr int kM = 1024;
constexpr int kCts = 4;       // ciphertexts per CTA
constexpr uint32_t kTmemCols = 512;

// cos(2 pi e / 32), e = 0..31 (correctly rounded doubles)
struct C32 {
  static constexpr double c[32] = {
      1.0, 0.9807852804032304, 0.9238795325112867, 0.8314696123025452, 0.7071067811865476, 0.5555702330196022,
      0.3826834323650898, 0.19509032201612828, 0.0, -0.19509032201612828, -0.3826834323650898,
      -0.5555702330196022, -0.7071067811865476, -0.8314696123025452, -0.9238795325112867, -0.9807852804032304,
      -1.0, -0.9807852804032304, -0.9238795325112867, -0.8314696123025452, -0.7071067811865476,
      -0.5555702330196022, -0.3826834323650898, -0.19509032201612828, 0.0, 0.19509032201612828,
      0.3826834323650898, 0.5555702330196022, 0.7071067811865476, 0.8314696123025452, 0.9238795325112867,
      0.9807852804032304};
};

// Radix-2 decimation-in-time butterflies.
// tan(2 pi r / 32), r = 0..4 (correctly rounded doubles)
struct T32 {
  static constexpr double t[5] = {0.0, 0.198912367379658, 0.41421356237309503, 0.6681786379192989, 1.0};
};

// DIT butterfly a' = a + W^E b, b' = a - W^E b, W = e^{+2 pi i / 32} (conjugate
// when INV), 6 FP64 instructions when nontrivial: with W^e = i^q e^{i theta},
//   e^{i theta} b = cos (b.x - tan b.y, b.y + tan b.x) = sin (cot b.x - b.y, cot b.y + b.x)
// and the cos / sin scale folds into the four output FMAs.
template <int E, bool INV>
__device__ __forceinline__ void bfly(double2 &a, double2 &b) {
  constexpr int e = INV ? ((32 - (E & 31)) & 31) : (E & 31);
  constexpr int q = e >> 3, r = e & 7;
  if constexpr (r == 0) {
    double2 t;
    if constexpr (q == 0) t = b;
    else if constexpr (q == 1) t = make_double2(-b.y, b.x);
    else if constexpr (q == 2) t = make_double2(-b.x, -b.y);
    else t = make_double2(b.y, -b.x);
    const double2 na = cadd(a, t), nb = csub(a, t);
    a = na;
    b = nb;
  } else {
    double u, v;
    if constexpr (r <= 4) {
      constexpr double tn = T32::t[r];
      u = fma(-tn, b.y, b.x);
      v = fma(tn, b.x, b.y);
    } else {
      constexpr double ct = T32::t[8 - r];
      u = fma(ct, b.x, -b.y);
      v = fma(ct, b.y, b.x);
    }
    constexpr double f = (r <= 4) ? C32::c[r] : C32::c[8 - r];
    double U, V;  // (u + i v) * i^q
    if constexpr (q == 0) { U = u; V = v; }
    else if constexpr (q == 1) { U = -v; V = u; }
    else if constexpr (q == 2) { U = -u; V = -v; }
    else { U = v; V = -u; }
    const double2 na = make_double2(fma(f, U, a.x), fma(f, V, a.y));
    const double2 nb = make_double2(fma(-f, U, a.x), fma(-f, V, a.y));
    a = na;
    b = nb;
  }
}
template <bool INV>
__device__ __forceinline__ void bfly_v(double2 &a, double2 &b, int e) {
  switch (e & 31) {
#define SZ_B(k) \
  case k: bfly<k, INV>(a, b); break;
    SZ_B(0) SZ_B(1) SZ_B(2) SZ_B(3) SZ_B(4) SZ_B(5) SZ_B(6) SZ_B(7)
    SZ_B(8) SZ_B(9) SZ_B(10) SZ_B(11) SZ_B(12) SZ_B(13) SZ_B(14) SZ_B(15)
#undef SZ_B
    default: break;
  }
}
// Radix-2 decimation-in-time stages on the bit-reversed view, half size H = 1..16
template <bool INV, int H>
__device__ __forceinline__ void dit32_stage(double2 (&y)[32]) {
  if constexpr (H <= 16) {
#pragma unroll
    for (int b = 0; b < 32; b += 2 * H)
#pragma unroll
      for (int j = 0; j < H; j++) bfly_v<INV>(y[b + j], y[b + j + H], j * (16 / H));
    dit32_stage<INV, 2 * H>(y);
  }
}

__host__ __device__ constexpr int bitrev5(int r) {
  return ((r & 1) << 4) | ((r & 2) << 2) | (r & 4) | ((r & 8) >> 2) | ((r & 16) >> 4);
}

// cos(pi k / 64), tan(pi k / 64), k = 0..16 (correctly rounded doubles)
struct C64 {
  static constexpr double c[17] = {
      1.0, 0.9987954562051724, 0.9951847266721969, 0.989176509964781, 0.9807852804032304, 0.970031253194544,
      0.9569403357322088, 0.9415440651830208, 0.9238795325112867, 0.9039892931234433, 0.881921264348355,
      0.8577286100002721, 0.8314696123025452, 0.8032075314806449, 0.773010453362737, 0.7409511253549591,
      0.7071067811865476};
  static constexpr double t[17] = {
      0.0, 0.049126849769467254, 0.09849140335716425, 0.14833598753834742, 0.198912367379658,
      0.25048696019130545, 0.3033466836073424, 0.3578057213145241, 0.41421356237309503, 0.4729647758913199,
      0.5345111359507917, 0.5993769336819238, 0.6681786379192989, 0.7416505462720354, 0.8206787908286604,
      0.9063471690191471, 1.0};
};
// conj(w^{32m}) = e^{-i th}, th = pi m / 64 < pi/2, written as s_m * (unscaled factor):
//   m <= 16: cos th (1 - i tan th)      m > 16: sin th (cot th - i)
// the unscaled product costs 2 FMAs; s_m folds into the rounding FMA.
__host__ __device__ constexpr double twist_scale(int m) { return m <= 16 ? C64::c[m] : C64::c[32 - m]; }
template <int M>
__device__ __forceinline__ double2 untwist_unscaled(double2 a) {
  if constexpr (M == 0) {
    return a;
  } else if constexpr (M <= 16) {
    constexpr double t = C64::t[M];
    return make_double2(fma(t, a.y, a.x), fma(-t, a.x, a.y));
  } else {
    constexpr double ct = C64::t[32 - M];
    return make_double2(fma(ct, a.x, a.y), fma(ct, a.y, -a.x));
  }
}

// inverse untwist of output m fused with the exact rounding of the limb:
// bits(s_m * u + 1.5 * 2^52) = round(x conj(w^{32m})) + bits(1.5 * 2^52), |.| < 2^51
#ifndef SZ_FFT_MARGIN
#define SZ_FFT_MARGIN 0  // 1: debug build recording the rounding margin of every limb (tools/fft_margin.py)
#endif
#if SZ_FFT_MARGIN
// per limb p: max |x - round(x)| and max |x| (f64 bits: non-negative doubles
// order like u64) and the count of values with |x - round(x)| >= 1/4 and >= 1/2
// over every rounded limb value (R20: exact while the FFT error
// stays below 1/2 and |x| < 2^51)
__device__ unsigned long long g_margin_frac[3], g_margin_abs[3], g_margin_q[3], g_margin_h[3];
// x = u * s (the untwisted limb value, never rounded on its own: the kernel
// rounds fma(u, s, 1.5 * 2^52)); |u s - round| with one rounding
__device__ __forceinline__ void margin_note(double u, double s, u64 bits, int p) {
  const double r = __longlong_as_double((long long)bits) - 6755399441055744.0;  // round(x), exact
  const double fr = fabs(fma(u, s, -r));
  unsigned long long f = (unsigned long long)__double_as_longlong(fr);
  unsigned long long a = (unsigned long long)__double_as_longlong(fabs(u * s));
  unsigned q = __popc(__ballot_sync(0xffffffffu, fr >= 0.25)), h = __popc(__ballot_sync(0xffffffffu, fr >= 0.5));
  for (int d = 16; d; d >>= 1) {  // warp-level max first (one atomic per warp)
    f = max(f, (unsigned long long)__shfl_xor_sync(0xffffffffu, f, d));
    a = max(a, (unsigned long long)__shfl_xor_sync(0xffffffffu, a, d));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&g_margin_frac[p], f);
    atomicMax(&g_margin_abs[p], a);
    if (q) atomicAdd(&g_margin_q[p], (unsigned long long)q);
    if (h) atomicAdd(&g_margin_h[p], (unsigned long long)h);
  }
}
#endif
template <int M>
__device__ __forceinline__ void untwist_round_t(double2 y, u64 &bx, u64 &by, int p) {
  const double2 u = untwist_unscaled<M>(y);
  constexpr double s = twist_scale(M);
  bx = (u64)__double_as_longlong(fma(u.x, s, 6755399441055744.0));
  by = (u64)__double_as_longlong(fma(u.y, s, 6755399441055744.0));
#if SZ_FFT_MARGIN
  margin_note(u.x, s, bx, p);
  margin_note(u.y, s, by, p);
#else
  (void)p;
#endif
}
__device__ __forceinline__ void untwist_round(double2 y, int m, u64 &bx, u64 &by, int p) {
  switch (m & 31) {
#define SZ_U(k) \
  case k: untwist_round_t<k>(y, bx, by, p); break;
    SZ_U(0) SZ_U(1) SZ_U(2) SZ_U(3) SZ_U(4) SZ_U(5) SZ_U(6) SZ_U(7)
    SZ_U(8) SZ_U(9) SZ_U(10) SZ_U(11) SZ_U(12) SZ_U(13) SZ_U(14) SZ_U(15)
    SZ_U(16) SZ_U(17) SZ_U(18) SZ_U(19) SZ_U(20) SZ_U(21) SZ_U(22) SZ_U(23)
    SZ_U(24) SZ_U(25) SZ_U(26) SZ_U(27) SZ_U(28) SZ_U(29) SZ_U(30) SZ_U(31)
#undef SZ_U
  }
}

// 32-point DFT on registers, exponent sign + (conjugate when INV), natural-order
// input and output: X[k] = sum_n x[n] e^{+-2 pi i n k / 32}; the bit reversal
// of the radix-2 DIT form is a register renaming.
template <bool INV>
__device__ __forceinline__ void dft32(double2 (&x)[32]) {
  double2 y[32];
#pragma unroll
  for (int r = 0; r < 32; r++) y[r] = x[bitrev5(r)];
  dit32_stage<INV, 1>(y);
#pragma unroll
  for (int r = 0; r < 32; r++) x[r] = y[r];
}

// Tables (host-built in long double, rounded once), w = e^{i pi / 2048}:
//   T(l, k1)   = w^{l (1 + 4 k1)}  (negacyclic twist w^l folded with the
//                four-step twiddle e^{2 pi i l k1 / M}), stored as tw[k1 * 32 + l]
//                (coalesced for lane = l)
//   c_twist32[m] = w^{32 m} = e^{i pi m / 64}
struct Tables32 {
  double2 tw[32 * 32];
};
__device__ Tables32 g_t32;
__constant__ double2 c_twist32[32];

// swizzled index of element (row, col) of a 32 x 32 block of 16-byte values:
// any 8 consecutive rows (fixed col) or cols (fixed row) hit 8 distinct 16-byte bank groups
__host__ __device__ constexpr int sw(int row, int col) { return row * 32 + (col ^ (row & 7)); }
constexpr int kXbuf = 1024;  // double2 per transposition buffer

static std::once_flag g_once[64];
static int g_status[64];

static int init_tables(int dev) {
  static Tables32 h;
  double2 tws[32];
  const long double PI = 3.141592653589793238462643383279502884L;
  for (int k1 = 0; k1 < 32; k1++)
    for (int l = 0; l < 32; l++) {
      const long double ang = PI * (long double)(l * (1 + 4 * k1)) / 2048.0L;
      h.tw[k1 * 32 + l] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
  for (int m = 0; m < 32; m++) {
    const long double ang = PI * (long double)m / 64.0L;
    tws[m] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return SILENZIO_ERR_CUDA;
  if (prev != dev && cudaSetDevice(dev) != cudaSuccess) return SILENZIO_ERR_CUDA;
  cudaError_t e = cudaMemcpyToSymbol(g_t32, &h, sizeof(Tables32));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_twist32, tws, sizeof(tws));
  if (prev != dev) cudaSetDevice(prev);
  return e == cudaSuccess ? SILENZIO_OK : SILENZIO_ERR_CUDA;
}

static int ensure_tables() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SILENZIO_ERR_CUDA;
  std::call_once(g_once[dev], [dev] { g_status[dev] = init_tables(dev); });
  return g_status[dev];
}

// twiddle T(l = lane, k1) from the global (L1-resident) table
__device__ __forceinline__ double2 tw_fwd(int l, int k1) { return __ldg(&g_t32.tw[k1 * 32 + l]); }

// Forward transform of one warp. In: x[m] = (a_j + i a_{j+1024}) at j = lane + 32 m.
// Out: x[k2] = spectrum at index lane + 32 k2 ("slot" order).
__device__ __forceinline__ void fwd_fft32(double2 (&x)[32], double2 *buf, int lane) {
#pragma unroll
  for (int m = 1; m < 32; m++) x[m] = cmul(x[m], c_twist32[m]);
  dft32<false>(x);  // x[k1] = B[l = lane][k1]
  __syncwarp();     // earlier readers of buf are done
#pragma unroll
  for (int k1 = 0; k1 < 32; k1++) buf[sw(lane, k1)] = cmul(x[k1], tw_fwd(lane, k1));
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 32; l++) x[l] = buf[sw(l, lane)];  // thread k1 = lane, natural l
  dft32<false>(x);                                        // x[k2] = Z[lane + 32 k2]
}

// Inverse transform (unnormalised). In: slot order. Out: x[m] = M (c_j + i c_{j+1024}) w^{32 m},
// j = lane + 32 m, i.e. before the final untwist conj(w^{32m}) (done by the caller:
// untwist_round fuses it with the exact rounding; UNTWIST = true applies it here).
struct NoHook32 {
  __device__ __forceinline__ void operator()() const {}
};
// `after_pass1` runs after the first radix-32 pass (pure register arithmetic): a place for
// work whose inputs were requested before the call (the stage-release atomic's result)
template <bool UNTWIST, class Hook = NoHook32>
__device__ __forceinline__ void inv_fft32(double2 (&x)[32], double2 *buf, int lane, Hook after_pass1 = Hook()) {
  dft32<true>(x);  // x[l] = 32 B'[l][k1 = lane]
  after_pass1();
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 32; l++) buf[sw(l, lane)] = x[l];
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 32; k1++) x[k1] = cmulc(buf[sw(lane, k1)], tw_fwd(lane, k1));  // thread l = lane
  dft32<true>(x);  // x[m] = M z_{lane + 32 m} w^{32 m}
  if constexpr (UNTWIST) {
#pragma unroll
    for (int m = 1; m < 32; m++) x[m] = cmulc(x[m], c_twist32[m]);
  }
}

// ------------------------------------------------------------ mbarrier / bulk copy
__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SZ_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SZ_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(mbar)),
      "r"(phase)
      : "memory");
}
// arm the barrier for `bytes` and bulk-copy them global -> shared (one thread)
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *mbar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}
// release this warp's reads of the stage and count it; returns the previous count.
// (__syncwarp orders the other lanes' reads before lane 0's release; the
// last warp's acquire then orders every warp's reads before its async-proxy
// fence and the bulk copy that overwrites the stage.)
// (the acquire-release atomic costs 1.6 % against round 1's relaxed counter:
// 207.3 vs 203.9 ms BR-only at 9 472, profiles/r02_ab_setA_micro.txt)
__device__ __forceinline__ uint32_t stage_release(uint32_t *ctr) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(ctr)) : "memory");
  return old;
}

// ------------------------------------------------------------------ kernel
struct Args {
  const u64 *lwe_small;  // [count][n+1]
  const u32 *lut_ids;    // [count] or null
  const u64 *luts;       // [num_luts][N]
  u32 num_luts;
  const double2 *fbsk;   // [n][P][2][2][32][32]
  u64 *lwe_out;          // [count][N+1]
  long count;
  int n, base_log, w;
};

__host__ __device__ constexpr size_t abar_bytes(int n) { return ((size_t)n * 2 + 15) / 16 * 16; }
// Two layouts of the same kernel:
//  SMALL = false: 4 ciphertexts, 8 warps; ciphertext s on warps s (mask) and
//    s + 4 (body), which share TMEM lane quadrant s, so the digit spectra are
//    exchanged through tensor memory (the throughput layout);
//  SMALL = true: 2 ciphertexts, 4 warps; ciphertext s on warps s and s + 2, i.e.
//    on two different schedulers (one FP64 pipe each), the spectra exchanged
//    through shared memory: a batch of <= 2 x SMs ciphertexts runs at half the
//    CMux latency of the throughput layout.
template <bool SMALL> struct Lay {
  static constexpr int cts = SMALL ? 2 : 4, warps = 2 * cts, threads = 32 * warps;
};
__host__ __device__ constexpr size_t smem_bytes(int n, bool small = false) {
  return (small ? 4 : 8) * (size_t)kXbuf * sizeof(double2)  // per-warp transposition buffers (also the ACC copy)
         + 4 * (size_t)kM * sizeof(double2)                  // BSK stage: one (i, limb), [o][row][32][32]
         + (small ? 2 * 2 * (size_t)kM * sizeof(double2) : 0)  // SMALL: digit spectra [slot][row][1024]
         + (small ? 2 : kCts) * abar_bytes(n)                // modswitched masks
         + 16;                                               // mbarrier
}

__device__ __forceinline__ u64 acc_init(const u64 *v, int j, int bt, int g) {
  const int idx = (j + bt) & (2 * kN - 1);
  const u64 vv = (idx < kN) ? v[idx] : (u64)0 - v[idx - kN];
  return g ? vv : 0ull;
}
// ACC chunk cc (16 TMEM columns) = coefficients j = lane + 32 m + 1024 h, m = kCQ cc + q (q < kCQ), h < 2
// (16-column chunks measured 3 % faster than 32, profiles/r01_warp_variants2.txt)
constexpr int kCQ = 4, kNC = 32 / kCQ;
__device__ __forceinline__ void acc_ld(uint32_t ta, int cc, u64 (&a)[kCQ][2]) {
  uint32_t r[4 * kCQ];
  tmem_ld16(ta + 16 * cc, r);
  tmem_wait_ld16(r);
#pragma unroll
  for (int q = 0; q < kCQ; q++)
#pragma unroll
    for (int h = 0; h < 2; h++) a[q][h] = (u64)r[4 * q + 2 * h] | ((u64)r[4 * q + 2 * h + 1] << 32);
}
__device__ __forceinline__ void acc_st(uint32_t ta, int cc, const u64 (&a)[kCQ][2]) {
  uint32_t r[4 * kCQ];
#pragma unroll
  for (int q = 0; q < kCQ; q++)
#pragma unroll
    for (int h = 0; h < 2; h++) {
      r[4 * q + 2 * h] = (uint32_t)a[q][h];
      r[4 * q + 2 * h + 1] = (uint32_t)(a[q][h] >> 32);
    }
  tmem_st16(ta + 16 * cc, r);
}

constexpr u64 kMagicBits = 0x4338000000000000ull;  // bits of 1.5 * 2^52

// Throughput layout: cycles the body warp of a ciphertext waits after the
// spectra exchange of every CMux, so that the two warps of a scheduler (the
// two GLWE components of one ciphertext) stop running the same phase at the
// same time: one warp's transpositions, MAC (shared-memory bound) and limb
// recombination (integer / TMEM work) then overlap the other's FP64
// butterflies. The wait costs both warps ~SZ_PAIR_SKEW idle cycles per CMux
// (the mask warp meets it again at the next exchange barrier) and still nets
// +5.9 % (profiles/r02_ab_pair_skew.txt; 0 disables).
#ifndef SZ_PAIR_SKEW
#define SZ_PAIR_SKEW 800
#endif
__device__ __forceinline__ void spin_cycles(int c) {
  const long long t0 = clock64();
  while (clock64() - t0 < c) {
  }
}

#ifndef SZ_PHASE_TIMING
#define SZ_PHASE_TIMING 0  // 1: debug build accumulating clock64 per CMux phase (CTA 0, lane 0 of each warp)
#endif
#if SZ_PHASE_TIMING
__device__ unsigned long long g_phase[8][8];
#define SZ_PT_INIT long long sz_pt_prev = clock64();
#define SZ_PT(k)                                                        \
  do {                                                                  \
    if (blockIdx.x == 0 && lane == 0) {                                 \
      const long long now = clock64();                                  \
      atomicAdd(&g_phase[wid][k], (unsigned long long)(now - sz_pt_prev)); \
      sz_pt_prev = now;                                                 \
    }                                                                   \
  } while (0)
#else
#define SZ_PT_INIT long long sz_pt_prev = 0;
#define SZ_PT(k) \
  do {           \
  } while (0)
#endif

template <int P, bool SMALL>
__global__ void __launch_bounds__(Lay<SMALL>::threads, 1) blind_rotate_warp_kernel(Args A) {
  constexpr int kC = Lay<SMALL>::cts, kW = Lay<SMALL>::warps;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ uint32_t mac_done;  // warps finished with the staged limb, monotone (the kW-th of a round re-arms)
  const int n = A.n, w = A.w, blog = A.base_log;
  double2 *xbuf_all = reinterpret_cast<double2 *>(smem);
  double2 *gbuf = xbuf_all + kW * kXbuf;
  double2 *dsm = gbuf + 4 * kM;  // SMALL: digit spectra [slot][row][32 r][32 lane]
  unsigned char *abar_base = reinterpret_cast<unsigned char *>(dsm + (SMALL ? 2 * 2 * kM : 0));
  uint64_t *mbar = reinterpret_cast<uint64_t *>(abar_base + kC * abar_bytes(n));
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int cs = wid % kC, g = wid / kC;  // ciphertext slot, GLWE component
  double2 *xbuf = xbuf_all + wid * kXbuf;
  ulonglong2 *accp = reinterpret_cast<ulonglong2 *>(xbuf);  // ACC_g copy as [1024] coefficient pairs
  unsigned short *abar = reinterpret_cast<unsigned short *>(abar_base + cs * abar_bytes(n));

  if (wid == 0) tmem_alloc(&tmem_slot, kTmemCols);
  if (tid == 32) mbar_init(mbar, 1);
  if (tid == 0) mac_done = 0;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  // TMEM: lane quadrant = warp % 4. Throughput layout: quadrant cs holds
  // ACC_0 | ACC_1 | D^_0 | D^_1 of ciphertext cs; SMALL: quadrant wid holds ACC_g.
  const uint32_t tl = tmem_slot + ((uint32_t)(32 * (wid & 3)) << 16);
  const uint32_t ta_acc = tl + (SMALL ? 0 : 128 * g), ta_d0 = tl + 256, ta_d1 = tl + 384,
                 ta_dg = tl + 256 + 128 * g;
  double2 *dsm_s = dsm + (size_t)cs * 2 * kM;  // SMALL: this slot's [row][r][lane]
  const uint32_t limb_bytes = 4 * kM * sizeof(double2);
  auto issue = [&](int i, int p) {
    bulk_load(gbuf, A.fbsk + ((size_t)i * P + p) * 4 * kM, limb_bytes, mbar);
  };
  uint32_t round = 0;  // completed bulk copies (mbarrier phase parity)
  const u64 half_q = 1ull << (63 - blog);

  const long ngroups = (A.count + kC - 1) / kC;
  for (long grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    if (tid == 0) issue(0, P - 1);
    const long c_raw = grp * kC + cs;
    const bool live = c_raw < A.count;
    const long c = live ? c_raw : A.count - 1;  // idle slots replay the last ciphertext
    const u64 *lwe = A.lwe_small + (size_t)c * (n + 1);
    // ---- modulus switch (a2)
    for (int i = g * 32 + lane; i < n; i += 64) abar[i] = (unsigned short)sz_modswitch(lwe[i], kLog2_2N);
    const int bt = (int)sz_modswitch(lwe[n], kLog2_2N);
    // ---- ACC init (a3): ACC = (0, X^{-b~} v)
    u32 id = A.lut_ids ? A.lut_ids[c] : 0u;
    if (id >= A.num_luts) id = 0;
    const u64 *v = A.luts + (size_t)id * kN;
#pragma unroll 1
    for (int cc = 0; cc < kNC; cc++) {
      u64 a4[kCQ][2];
#pragma unroll
      for (int q = 0; q < kCQ; q++)
#pragma unroll
        for (int h = 0; h < 2; h++) a4[q][h] = acc_init(v, lane + 32 * (kCQ * cc + q) + 1024 * h, bt, g);
      acc_st(ta_acc, cc, a4);
    }
    tmem_wait_st();
    __syncthreads();  // abar visible

    SZ_PT_INIT
    for (int i = 0; i < n; i++) {
      const int a = abar[i];
      // ---------------- publish ACC_g for the rotation, as coefficient pairs
      // accp[s] = (ACC_g[s], ACC_g[s + 1024]), s < 1024 (one 16-byte access serves both h)
      __syncwarp();  // previous inverse FFT's readers of xbuf are done
#pragma unroll
      for (int cc = 0; cc < kNC; cc++) {
        u64 a4[kCQ][2];
        acc_ld(ta_acc, cc, a4);
#pragma unroll
        for (int q = 0; q < kCQ; q++) accp[lane + 32 * (kCQ * cc + q)] = make_ulonglong2(a4[q][0], a4[q][1]);
      }
      __syncwarp();
      SZ_PT(0);
      // ---------------- digits of X^a ACC_g - ACC_g (a4.1-a4.2), forward FFT
      // (X^a ACC)[j] = +-ACC[(j - a) mod 2N]: for j0 = lane + 32 m and j1 = j0 + 1024,
      // src0 = (j0 - a) mod 4096 = 1024 qd + s picks the pair accp[s] for both:
      //   qd = 0: (+x, +y)   1: (+y, -x)   2: (-x, -y)   3: (-y, +x)
      double2 x[32];
#pragma unroll
      for (int cc = 0; cc < kNC; cc++) {
        u64 a4[kCQ][2];
        acc_ld(ta_acc, cc, a4);
#pragma unroll
        for (int q = 0; q < kCQ; q++) {
          const int src0 = (lane + 32 * (kCQ * cc + q) - a) & (2 * kN - 1);
          const int qd = src0 >> 10;
          const ulonglong2 pr = accp[src0 & 1023];
          u64 r0 = (qd & 1) ? pr.y : pr.x, r1 = (qd & 1) ? pr.x : pr.y;
          if (qd >= 2) r0 = (u64)0 - r0;
          if (qd == 1 || qd == 2) r1 = (u64)0 - r1;
          // level-1 balanced digit round((rot - acc) B / q) in [-B/2, B/2): the
          // arithmetic shift of the half-up-rounded value (C3; the carry out of
          // the only level is dropped, as in sz_decomp_next)
          x[kCQ * cc + q] = make_double2((double)((i64)(r0 - a4[q][0] + half_q) >> (64 - blog)),
                                         (double)((i64)(r1 - a4[q][1] + half_q) >> (64 - blog)));
        }
      }
      SZ_PT(1);
      fwd_fft32(x, xbuf, lane);
      SZ_PT(2);
      if (i > 0) {  // both warps of the ciphertext are past the previous CMux's MACs (D^ reads)
        tmem_fence_before();
        asm volatile("bar.sync %0, %1;" ::"r"(5 + cs), "r"(64) : "memory");
        tmem_fence_after();
      }
      if constexpr (SMALL) {
#pragma unroll
        for (int k2 = 0; k2 < 32; k2++) dsm_s[g * kM + 32 * k2 + lane] = x[k2];
        asm volatile("bar.sync %0, %1;" ::"r"(1 + cs), "r"(64) : "memory");  // D^_0 and D^_1 written
      } else {
#pragma unroll
        for (int jj = 0; jj < 8; jj++) {
          uint32_t r16[16];
          pack4(&x[4 * jj], r16);
          tmem_st16(ta_dg + 16 * jj, r16);
        }
        tmem_wait_st();
        tmem_fence_before();
        asm volatile("bar.sync %0, %1;" ::"r"(1 + cs), "r"(64) : "memory");  // D^_0 and D^_1 written
        tmem_fence_after();
      }
      if (!SMALL && SZ_PAIR_SKEW > 0 && g == 1) spin_cycles(SZ_PAIR_SKEW);
      SZ_PT(3);
      // ---------------- per limb: MAC with the staged BSK, inverse FFT, exact ACC update
#pragma unroll 1
      for (int p = P - 1; p >= 0; p--) {
        mbar_wait(mbar, round & 1);
        round++;
        SZ_PT(4);
        double2 (&y)[32] = x;  // the MAC output overwrites the digit-spectrum registers (now in TMEM / smem)
        const double2 *G0 = gbuf + (size_t)(2 * g) * kM + lane;  // [o = g][row 0]
        const double2 *G1 = G0 + kM;                             // [o = g][row 1]
        if constexpr (SMALL) {
#pragma unroll
          for (int r = 0; r < 32; r++) {
            double2 acc = make_double2(0.0, 0.0);
            cmac(acc, dsm_s[32 * r + lane], G0[r * 32]);
            cmac(acc, dsm_s[kM + 32 * r + lane], G1[r * 32]);
            y[r] = acc;
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 4; jj++) {
            uint32_t d0[32], d1[32];
            tmem_ld32(ta_d0 + 32 * jj, d0);
            tmem_ld32(ta_d1 + 32 * jj, d1);
            tmem_wait_ld32x2(d0, d1);
#pragma unroll
            for (int q = 0; q < 8; q++) {
              const int r = 8 * jj + q;
              double2 acc = make_double2(0.0, 0.0);
              cmac(acc, unpack1(d0, q), G0[r * 32]);
              cmac(acc, unpack1(d1, q), G1[r * 32]);
              y[r] = acc;
            }
          }
        }
        SZ_PT(5);
        // this warp is done with the stage; the last warp of the round re-arms it
        // with the next (i, limb) -- no CTA-wide barrier
        __syncwarp();
        // the release atomic's result (am I the last warp of the round?) is looked at only
        // after the inverse transform's first pass, so its latency hides behind that pass
        uint32_t rel = 0;
        if (lane == 0) rel = stage_release(&mac_done);
        constexpr bool kFusedUntwist = (P == 3);
        inv_fft32<!kFusedUntwist>(y, xbuf, lane, [&]() {
          if (lane == 0 && (rel % kW) == kW - 1) {
            if (p > 0) issue(i, p - 1);
            else if (i + 1 < n) issue(i + 1, P - 1);
          }
        });
        SZ_PT(6);
        // P = 3: bits(x + 1.5 2^52) << 22p per limb, the magic constant's share of
        // all three limbs removed once per CMux (at p = 0)
        const u64 limb_off = (p == 0) ? kMagicBits + (kMagicBits << w) + (kMagicBits << (2 * w)) : 0ull;
#pragma unroll
        for (int cc = 0; cc < kNC; cc++) {
          u64 a4[kCQ][2];
          acc_ld(ta_acc, cc, a4);
#pragma unroll
          for (int q = 0; q < kCQ; q++) {
            if constexpr (kFusedUntwist) {
              u64 bx, by;
              untwist_round(y[kCQ * cc + q], kCQ * cc + q, bx, by, p);
              a4[q][0] += (bx << (p * w)) - limb_off;
              a4[q][1] += (by << (p * w)) - limb_off;
            } else {
              a4[q][0] += limb_to_torus(y[kCQ * cc + q].x, p, P, w);
              a4[q][1] += limb_to_torus(y[kCQ * cc + q].y, p, P, w);
            }
          }
          acc_st(ta_acc, cc, a4);
        }
        tmem_wait_st();
        SZ_PT(7);
      }
    }
    // ---- sample extraction (a5): a'[0] = A[0], a'[i] = -A[N-i], b' = B[0]
    if (live) {
      u64 *out = A.lwe_out + (size_t)c * (kN + 1);
#pragma unroll 1
      for (int cc = 0; cc < kNC; cc++) {
        u64 a4[kCQ][2];
        acc_ld(ta_acc, cc, a4);
#pragma unroll
        for (int q = 0; q < kCQ; q++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int j = lane + 32 * (kCQ * cc + q) + 1024 * h;
            if (g == 0) {
              if (j == 0) out[0] = a4[q][h];
              else out[kN - j] = (u64)0 - a4[q][h];
            } else if (j == 0) {
              out[kN] = a4[q][h];
            }
          }
      }
    }
    __syncthreads();  // abar reuse
  }
  tmem_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tmem_slot, kTmemCols);
}

// ------------------------------------------------- latency kernel (small batches)
// One ciphertext per CTA (8 warps), for batches too small to fill the GPU with
// four ciphertexts per SM: the per-PBS latency, not the FP64 throughput, is
// what such a launch waits for. Same transform, tables,
// Fourier-BSK layout and arithmetic as blind_rotate_warp_kernel; the eight
// FFTs of a CMux are spread over the warps instead of two:
//   phase F  warps 0, 1 (GLWE component r = warp): ACC_r += the three limb
//            contributions of the previous CMux, digits of X^a ACC_r - ACC_r,
//            forward FFT, D^_r to shared memory;
//   phase I  warps 2..7, one per (output o, limb p): MAC of D^_0, D^_1 with
//            BSK_i[p][o] (prefetched into registers during phase F), inverse
//            FFT with the fused untwist + exact rounding, the limb's shifted
//            contribution written to the warp's own buffer.
// Two CTA barriers per CMux separate the phases.
constexpr int kLatThreads = 256;
__host__ __device__ constexpr size_t lat_smem_bytes(int n) {
  return 8 * (size_t)kXbuf * sizeof(double2)   // per-warp FFT buffers (inverse warps: + contributions)
         + 2 * (size_t)kM * sizeof(double2)    // D^_0, D^_1 in slot order
         + 2 * (size_t)kM * sizeof(ulonglong2) // ACC_0, ACC_1 as coefficient pairs (s, s + 1024)
         + abar_bytes(n);
}

// phase F of one CMux for GLWE component r (warps 0, 1)
template <int P>
__device__ __forceinline__ void lat_forward(ulonglong2 *ac, const ulonglong2 *contrib, double2 *dhat_r,
                                            double2 *xbuf, int a, bool add, int lane, u64 half_q, int blog,
                                            long long &sz_pt_prev, int wid) {
  (void)sz_pt_prev;
  (void)wid;
  if (add) {  // ACC_r += the limb contributions of the previous CMux
#pragma unroll 4
    for (int s = lane; s < kM; s += 32) {
      ulonglong2 v = ac[s];
#pragma unroll
      for (int q = 0; q < P; q++) {
        const ulonglong2 cq = contrib[q * kXbuf + s];
        v.x += cq.x;
        v.y += cq.y;
      }
      ac[s] = v;
    }
    __syncwarp();
  }
  SZ_PT(0);
  // digits of X^a ACC_r - ACC_r (a4.1-a4.2), as in blind_rotate_warp_kernel
  double2 x[32];
#pragma unroll
  for (int m = 0; m < 32; m++) {
    const int src0 = (lane + 32 * m - a) & (2 * kN - 1);
    const int qd = src0 >> 10;
    const ulonglong2 pr = ac[src0 & 1023];
    const ulonglong2 own = ac[lane + 32 * m];
    u64 r0 = (qd & 1) ? pr.y : pr.x, r1 = (qd & 1) ? pr.x : pr.y;
    if (qd >= 2) r0 = (u64)0 - r0;
    if (qd == 1 || qd == 2) r1 = (u64)0 - r1;
    x[m] = make_double2((double)((i64)(r0 - own.x + half_q) >> (64 - blog)),
                        (double)((i64)(r1 - own.y + half_q) >> (64 - blog)));
  }
  SZ_PT(1);
  fwd_fft32(x, xbuf, lane);
  SZ_PT(2);
#pragma unroll
  for (int k2 = 0; k2 < 32; k2++) dhat_r[32 * k2 + lane] = x[k2];
  SZ_PT(3);
}

template <int P>
__global__ void __launch_bounds__(kLatThreads, 1) blind_rotate_lat_kernel(Args A) {
  static_assert(P >= 1 && P <= 3, "1..3 limbs");
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = A.n, w = A.w, blog = A.base_log;
  double2 *xbuf_all = reinterpret_cast<double2 *>(smem);
  double2 *dhat = xbuf_all + 8 * kXbuf;                                  // [2][32 k2][32 lane]
  ulonglong2 *accp = reinterpret_cast<ulonglong2 *>(dhat + 2 * kM);      // [2][1024]
  unsigned short *abar = reinterpret_cast<unsigned short *>(accp + 2 * kM);
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  double2 *xbuf = xbuf_all + wid * kXbuf;
  const u64 half_q = 1ull << (63 - blog);
  for (long c = blockIdx.x; c < A.count; c += gridDim.x) {
    const u64 *lwe = A.lwe_small + (size_t)c * (n + 1);
    for (int i = tid; i < n; i += kLatThreads) abar[i] = (unsigned short)sz_modswitch(lwe[i], kLog2_2N);
    if (wid < 2) {
      // ---------------- forward warps: component r = wid
      const int r = wid;
      ulonglong2 *ac = accp + r * kM;
      const ulonglong2 *contrib = reinterpret_cast<const ulonglong2 *>(xbuf_all + (2 + 3 * r) * kXbuf);
      {  // ACC init (a3): ACC = (0, X^{-b~} v) as pairs (s, s + 1024)
        const int bt = (int)sz_modswitch(lwe[n], kLog2_2N);
        u32 id = A.lut_ids ? A.lut_ids[c] : 0u;
        if (id >= A.num_luts) id = 0;
        const u64 *v = A.luts + (size_t)id * kN;
        for (int s = lane; s < kM; s += 32)
          ac[s] = make_ulonglong2(acc_init(v, s, bt, r), acc_init(v, s + 1024, bt, r));
      }
      __syncthreads();  // abar complete
      SZ_PT_INIT
      for (int i = 0; i < n; i++) {
        lat_forward<P>(ac, contrib, dhat + r * kM, xbuf, abar[i], i > 0, lane, half_q, blog, sz_pt_prev, wid);
        __syncthreads();  // D^ published (and the previous contributions consumed)
        SZ_PT(4);
        __syncthreads();  // contributions of CMux i written
        SZ_PT(5);
      }
      // ACC += the last contributions, then sample extraction (a5)
      u64 *out = A.lwe_out + (size_t)c * (kN + 1);
      for (int s = lane; s < kM; s += 32) {
        ulonglong2 v = ac[s];
#pragma unroll
        for (int q = 0; q < P; q++) {
          const ulonglong2 cq = contrib[q * kXbuf + s];
          v.x += cq.x;
          v.y += cq.y;
        }
        if (r == 0) {  // a'[0] = A[0], a'[j] = -A[N - j]
          if (s == 0) out[0] = v.x;
          else out[kN - s] = (u64)0 - v.x;
          out[kN - (s + 1024)] = (u64)0 - v.y;
        } else if (s == 0) {
          out[kN] = v.x;  // b' = B[0]
        }
      }
    } else {
      // ---------------- inverse warps: warp 2 + 3 o + (P - 1 - p) (warps past 2 + 3 o + P - 1 idle)
      const int job = wid - 2, o = job / 3, p = P - 1 - job % 3;
      const bool active = job % 3 < P;
      const u64 limb_off =
          kMagicBits + (P >= 2 ? (kMagicBits << w) : 0ull) + (P >= 3 ? (kMagicBits << (2 * w)) : 0ull);
      double2 g0[32], g1[32];  // BSK_i[p][o] rows 0 and 1 at slots lane + 32 k2
      auto load_g = [&](int i) {
        const double2 *G = A.fbsk + (((size_t)i * P + p) * 2 + o) * 2 * kM + lane;
#pragma unroll
        for (int k2 = 0; k2 < 32; k2++) {
          g0[k2] = __ldg(G + 32 * k2);
          g1[k2] = __ldg(G + kM + 32 * k2);
        }
      };
      if (active) load_g(0);
      __syncthreads();  // abar complete
      SZ_PT_INIT
      for (int i = 0; i < n; i++) {
        __syncthreads();  // D^ published
        SZ_PT(0);
        if (active) {
          double2 (&y)[32] = g0;  // the MAC output overwrites the BSK row-0 registers
#pragma unroll
          for (int k2 = 0; k2 < 32; k2++) {
            double2 acc = make_double2(0.0, 0.0);
            cmac(acc, dhat[32 * k2 + lane], g0[k2]);
            cmac(acc, dhat[kM + 32 * k2 + lane], g1[k2]);
            y[k2] = acc;
          }
          SZ_PT(1);
          ulonglong2 *contrib = reinterpret_cast<ulonglong2 *>(xbuf);
          if constexpr (P == 3) {
            inv_fft32<false>(y, xbuf, lane);
            SZ_PT(2);
            __syncwarp();  // the transposition's readers of xbuf are done
            const u64 off = (p == 0) ? limb_off : 0ull;  // all limbs' magic share, removed once
#pragma unroll
            for (int m = 0; m < 32; m++) {
              u64 bx, by;
              untwist_round(y[m], m, bx, by, p);
              contrib[lane + 32 * m] = make_ulonglong2((bx << (p * w)) - off, (by << (p * w)) - off);
            }
          } else {
            inv_fft32<true>(y, xbuf, lane);
            __syncwarp();
#pragma unroll
            for (int m = 0; m < 32; m++)
              contrib[lane + 32 * m] =
                  make_ulonglong2(limb_to_torus(y[m].x, p, P, w), limb_to_torus(y[m].y, p, P, w));
          }
          SZ_PT(3);
          // the next BSK slice: its loads land while phase F of CMux i + 1 runs
          if (i + 1 < n) load_g(i + 1);
          SZ_PT(4);
        }
        __syncthreads();  // contributions written
        SZ_PT(5);
      }
    }
    __syncthreads();  // abar / ACC / contributions reuse by the next ciphertext
  }
}

// --------------------------------------------------------- BSK -> Fourier
struct B2FArgs {
  const u64 *bsk;  // [n][2 (rows)][2 (o)][N]
  double2 *fbsk;   // [n][P][2 (o)][2 (row)][32][32]
  int n, P, w;
};

// one warp per (i, row, o, p)
__global__ void __launch_bounds__(32) bsk_to_fourier_warp_kernel(B2FArgs A) {
  __shared__ __align__(16) double2 buf[kXbuf];
  const int lane = threadIdx.x;
  long blk = blockIdx.x;
  const int p = blk % A.P; blk /= A.P;
  const int o = blk % 2; blk /= 2;
  const int row = blk % 2; blk /= 2;
  const int i = (int)blk;
  const u64 *gsrc = A.bsk + (((size_t)i * 2 + row) * 2 + o) * kN;
  double2 x[32];
#pragma unroll
  for (int m = 0; m < 32; m++) {
    double l0[3], l1[3];
    limb_split(gsrc[lane + 32 * m], A.P, A.w, l0);
    limb_split(gsrc[lane + 32 * m + 1024], A.P, A.w, l1);
    x[m] = make_double2(l0[p], l1[p]);
  }
  fwd_fft32(x, buf, lane);
  double2 *dst = A.fbsk + ((((size_t)i * A.P + p) * 2 + o) * 2 + row) * kM;
  const double scale = 1.0 / kM;
#pragma unroll
  for (int r = 0; r < 32; r++) dst[r * 32 + lane] = make_double2(x[r].x * scale, x[r].y * scale);
}

}  // namespace w32

// ------------------------------------------------------------------ host side
bool blind_rotate_warp_supported(const silenzio_params *P) {
  return P->poly_size == 2048 && P->glwe_dim == 1 && P->pbs_level == 1 && P->fft_limbs >= 1 && P->fft_limbs <= 3 &&
         w32::smem_bytes((int)P->lwe_dim) <= 227 * 1024;
}

long blind_rotate_warp_wave() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return (long)sms * w32::kCts;  // one CTA (4 ciphertexts) per SM: 512 TMEM columns each
}

long blind_rotate_warp_launches(size_t count) { return count ? 1 : 0; }

// SZ_PHASE_TIMING debug builds: clock64 cycles per phase [warp][phase] of CTA 0
// (0 publish, 1 digits, 2 forward FFT, 3 spectra exchange, 4 stage wait, 5 MAC,
// 6 inverse FFT, 7 recombination), read and reset
extern "C" int silenzio_debug_phase_times(unsigned long long *out /* [8][8] */) {
#if SZ_PHASE_TIMING
  unsigned long long z[64] = {0};
  SZ_CUDA_OK(cudaMemcpyFromSymbol(out, w32::g_phase, sizeof(z)));
  SZ_CUDA_OK(cudaMemcpyToSymbol(w32::g_phase, z, sizeof(z)));
  return SILENZIO_OK;
#else
  (void)out;
  return SILENZIO_ERR_UNSUPPORTED;
#endif
}

// SZ_FFT_MARGIN debug builds: read-and-reset the recorded rounding margin, per
// limb p < 3: out[4 p + 0] = max |x - round(x)|, [4 p + 1] = max |x|,
// [4 p + 2] = count |x - round(x)| >= 1/4, [4 p + 3] = count >= 1/2
extern "C" int silenzio_debug_fft_margin(double *out /* [12] */) {
#if SZ_FFT_MARGIN
  unsigned long long f[3], a[3], q[3], h[3], z[3] = {0, 0, 0};
  SZ_CUDA_OK(cudaMemcpyFromSymbol(f, w32::g_margin_frac, sizeof(f)));
  SZ_CUDA_OK(cudaMemcpyFromSymbol(a, w32::g_margin_abs, sizeof(a)));
  SZ_CUDA_OK(cudaMemcpyFromSymbol(q, w32::g_margin_q, sizeof(q)));
  SZ_CUDA_OK(cudaMemcpyFromSymbol(h, w32::g_margin_h, sizeof(h)));
  SZ_CUDA_OK(cudaMemcpyToSymbol(w32::g_margin_frac, z, sizeof(z)));
  SZ_CUDA_OK(cudaMemcpyToSymbol(w32::g_margin_abs, z, sizeof(z)));
  SZ_CUDA_OK(cudaMemcpyToSymbol(w32::g_margin_q, z, sizeof(z)));
  SZ_CUDA_OK(cudaMemcpyToSymbol(w32::g_margin_h, z, sizeof(z)));
  if (out)
    for (int p = 0; p < 3; p++) {
      memcpy(&out[4 * p], &f[p], 8);
      memcpy(&out[4 * p + 1], &a[p], 8);
      out[4 * p + 2] = (double)q[p];
      out[4 * p + 3] = (double)h[p];
    }
  return SILENZIO_OK;
#else
  (void)out;
  return SILENZIO_ERR_UNSUPPORTED;
#endif
}

// Largest batch the latency kernel takes (one ciphertext per SM): one wave of
// it (8.1-8.9 ms) beats both other layouts up to SMs ciphertexts; two waves do
// not (measured, tools/ab_lat.sh). SZ_LAT_WAVES = 0 disables it.
#ifndef SZ_LAT_WAVES
#define SZ_LAT_WAVES 1
#endif
long blind_rotate_lat_max(long sms) { return SZ_LAT_WAVES * sms; }
// Largest batch the SMALL layout (two ciphertexts per CTA, four warps) takes:
// one wave of it, 2 x SMs ciphertexts (10.9 ms vs 12.6 ms for the four-
// ciphertext layout; SZ_SMALL_WAVES = 0 disables it).
#ifndef SZ_SMALL_WAVES
#define SZ_SMALL_WAVES 1
#endif
long blind_rotate_small_max(long sms) { return SZ_SMALL_WAVES * 2 * sms; }

int launch_blind_rotate_warp(const u64 *lwe_small, const u32 *lut_ids, const u64 *luts, u32 num_luts,
                             const void *fbsk, u64 *lwe_out, size_t count, const silenzio_params *P,
                             cudaStream_t stream) {
  int st = w32::ensure_tables();
  if (st != SILENZIO_OK) return st;
  void (*kern)(w32::Args) = nullptr, (*kern_s)(w32::Args) = nullptr;
  if (P->fft_limbs == 1) kern = w32::blind_rotate_warp_kernel<1, false>, kern_s = w32::blind_rotate_warp_kernel<1, true>;
  if (P->fft_limbs == 2) kern = w32::blind_rotate_warp_kernel<2, false>, kern_s = w32::blind_rotate_warp_kernel<2, true>;
  if (P->fft_limbs == 3) kern = w32::blind_rotate_warp_kernel<3, false>, kern_s = w32::blind_rotate_warp_kernel<3, true>;
  if (!kern) return SILENZIO_ERR_UNSUPPORTED;
  w32::Args A;
  A.lwe_small = lwe_small;
  A.lut_ids = lut_ids;
  A.luts = luts;
  A.num_luts = num_luts;
  A.fbsk = reinterpret_cast<const double2 *>(fbsk);
  A.lwe_out = lwe_out;
  A.count = (long)count;
  A.n = (int)P->lwe_dim;
  A.base_log = (int)P->pbs_base_log;
  A.w = (int)P->limb_bits;
  const long wave = blind_rotate_warp_wave();
  if (wave <= 0) return SILENZIO_ERR_CUDA;
  const long sms = wave / w32::kCts;
  if ((long)count <= blind_rotate_lat_max(sms) && w32::lat_smem_bytes(A.n) <= 227 * 1024) {
    // at most one ciphertext per SM: the eight FFTs of a CMux on eight warps
    void (*lk)(w32::Args) = nullptr;
    if (P->fft_limbs == 1) lk = w32::blind_rotate_lat_kernel<1>;
    if (P->fft_limbs == 2) lk = w32::blind_rotate_lat_kernel<2>;
    if (P->fft_limbs == 3) lk = w32::blind_rotate_lat_kernel<3>;
    const size_t lsmem = w32::lat_smem_bytes(A.n);
    SZ_CUDA_OK(cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsmem));
    const long grid = (long)count < sms ? (long)count : sms;
    lk<<<(unsigned)grid, w32::kLatThreads, lsmem, stream>>>(A);
    SZ_LAUNCH_OK();
    return SILENZIO_OK;
  }
  if ((long)count <= blind_rotate_small_max(sms) && w32::smem_bytes(A.n, true) <= 227 * 1024) {
    // small batch: two ciphertexts per CTA on four warps (one scheduler each)
    const size_t ssmem = w32::smem_bytes(A.n, true);
    SZ_CUDA_OK(cudaFuncSetAttribute(kern_s, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem));
    const long groups = ((long)count + 1) / 2;
    const long grid = groups < sms ? groups : sms;
    kern_s<<<(unsigned)grid, w32::Lay<true>::threads, ssmem, stream>>>(A);
    SZ_LAUNCH_OK();
    return SILENZIO_OK;
  }
  const size_t smem = w32::smem_bytes(A.n);
  SZ_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // one persistent launch, CTA b handles groups b, b + grid, ... (grid-stride).
  // CTAs drift apart in i over a long batch, but the bulk-copy stage prefetch
  // tolerates the resulting L2 misses: measured +3.8 % at 131 072 ciphertexts
  // over one launch per resident wave (which kept every CTA on the same BSK_i);
  // lock-step rounds of the grid (fewer DRAM re-reads) measured 14-28 % slower
  // (DESIGN.md §8).
  const long groups = ((long)count + w32::kCts - 1) / w32::kCts;
  const long grid = groups < wave / w32::kCts ? groups : wave / w32::kCts;
  kern<<<(unsigned)grid, w32::Lay<false>::threads, smem, stream>>>(A);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

int launch_bsk_to_fourier_warp(const u64 *bsk, void *fbsk, const silenzio_params *P, cudaStream_t stream) {
  int st = w32::ensure_tables();
  if (st != SILENZIO_OK) return st;
  w32::B2FArgs A;
  A.bsk = bsk;
  A.fbsk = reinterpret_cast<double2 *>(fbsk);
  A.n = (int)P->lwe_dim;
  A.P = (int)P->fft_limbs;
  A.w = (int)P->limb_bits;
  const long blocks = (long)A.n * 2 * 2 * A.P;
  w32::bsk_to_fourier_warp_kernel<<<(unsigned)blocks, 32, 0, stream>>>(A);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

}  // namespace sz
