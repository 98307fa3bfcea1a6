// pbs_cluster2.cu -- blind rotation at N = 8192 (parameter set C, BASELINE
// configs[2]) and N = 32768 (set B, the 8-bit stage of configs[4]) on thread-
// block clusters of R CTAs holding TWO ciphertexts per cluster.
//
// Same steps and conventions as pbs.cu / pbs_warp.cu (SURVEY.md §8(a) a2-a6,
// §8(c) C4-C7, R3-R6, R20: P = 3 exact limbs of 22/22/20 bits).
// Only the data movement differs:
//
// Transform. N = 4096 R, M = N/2 = 2048 R, w = e^{i pi / N}. The folded values
// z^_j = a_j + i a_{j+M} (j < M) are split as j = p + 2048 m' (p < 2048, m' < R);
// CTA q of the cluster owns spectral block q:
//   Z[q + R k'] = DFT_2048(x_q)[k'],   x_q[p] = F[q][p] sum_{m'} z^[p + 2048 m'] C[m'][q],
//   F[q][p] = e^{i pi p (1 + 4q) / N},  C[m'][q] = e^{i pi m' / (2R)} e^{2 pi i m' q / R},
// i.e. the negacyclic twist w^j and the first radix-R step are folded into one
// R-point DFT per position plus one twiddle per (q, p). The inverse runs it
// backwards (conjugates; 1/M is folded into the Fourier BSK).
//
// Work split. Each CTA holds block q of two ciphertexts (slot g = warp group,
// 128 threads = 4 warps each), so every SM runs two independent instruction
// streams and one BSK block load serves both:
//  * ACC: CTA s owns positions p in [s Pw, (s+1) Pw), Pw = 2048 / R, of every
//    m' and both fold halves: [comp][h][m'][Pw] u64 = 64 KiB per ciphertext;
//  * digit spectra of block q: tensor memory, one 256-column half per slot
//    (4 rows x 16 values x 4 columns per thread);
//  * the block FFT (2048 = 16 x 16 x 8, 16 values per thread, two exchanges)
//    runs in the slot's 32 KiB receive buffer.
// Exchanges between the CTAs of a cluster (per slot, point to point): st.async
// 16-byte stores that complete transaction bytes on the receiver's "full"
// mbarrier, and release-arrivals on every sender's "free" mbarrier once a
// receiver is done with its buffer (every round starts with this CTA's
// release, so the buffer stays private through the block FFTs that use it as
// scratch). Forward: the owner of position p computes
// the digits of the rotated ACC (remote 8-byte reads for sources it does not
// own) for all m', the R-point DFT, and sends x_q[p] to CTA q. Inverse: CTA q
// sends block output x'_q[p] to the owner of p, which combines the R blocks,
// rounds the limb exactly and updates its ACC.
#include <cmath>
#include <mutex>
#include <vector>

#include <cooperative_groups.h>

#include "fft.cuh"
#include "limbs.cuh"
#include "tmem.cuh"

namespace sz {
namespace c2 {

constexpr int kB = 2048;  // complex points per block
constexpr int kT = 128;   // threads per ciphertext slot
constexpr int kV = 16;    // values per thread in the block FFT
constexpr int kSlots = 2; // ciphertexts per cluster

// ---------------------------------------------------------------- tables
// block FFT: tw1[k1][t] = W_2048^{t k1} (k1 < 16, t < 128), tw2[k][s] = W_128^{s k} (k < 16, s < 8)
struct BlockTables {
  double2 tw1[16 * 128];
  double2 tw2[16 * 8];
};
__device__ BlockTables g_bt;
// radix-R step, per R in {2, 8}: F[q][p] (global), C[m'][q] (constant)
__device__ double2 g_F2[2 * kB];
__device__ double2 g_F8[8 * kB];
__constant__ double2 c_C2[2 * 2];
__constant__ double2 c_C8[8 * 8];

static std::once_flag g_once[64];
static int g_status[64];

static int init_tables(int dev) {
  const long double PI = 3.141592653589793238462643383279502884L;
  static BlockTables bt;
  for (int k1 = 0; k1 < 16; k1++)
    for (int t = 0; t < 128; t++) {
      const long double a = 2.0L * PI * (long double)(t * k1) / 2048.0L;
      bt.tw1[k1 * 128 + t] = make_double2((double)cosl(a), (double)sinl(a));
    }
  for (int k = 0; k < 16; k++)
    for (int s = 0; s < 8; s++) {
      const long double a = 2.0L * PI * (long double)(s * k) / 128.0L;
      bt.tw2[k * 8 + s] = make_double2((double)cosl(a), (double)sinl(a));
    }
  std::vector<double2> F2(2 * kB), F8(8 * kB);
  double2 C2[4], C8[64];
  for (int R : {2, 8}) {
    const long double N = 4096.0L * R;
    std::vector<double2> &F = (R == 2) ? F2 : F8;
    for (int q = 0; q < R; q++)
      for (int p = 0; p < kB; p++) {
        const long double a = PI * (long double)p * (long double)(1 + 4 * q) / N;
        F[q * kB + p] = make_double2((double)cosl(a), (double)sinl(a));
      }
    double2 *C = (R == 2) ? C2 : C8;
    for (int m = 0; m < R; m++)
      for (int q = 0; q < R; q++) {
        const long double a = PI * (long double)m / (2.0L * R) + 2.0L * PI * (long double)(m * q) / R;
        C[m * R + q] = make_double2((double)cosl(a), (double)sinl(a));
      }
  }
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return SILENZIO_ERR_CUDA;
  if (prev != dev && cudaSetDevice(dev) != cudaSuccess) return SILENZIO_ERR_CUDA;
  cudaError_t e = cudaMemcpyToSymbol(g_bt, &bt, sizeof(bt));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_F2, F2.data(), F2.size() * sizeof(double2));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_F8, F8.data(), F8.size() * sizeof(double2));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_C2, C2, sizeof(C2));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_C8, C8, sizeof(C8));
  if (prev != dev) cudaSetDevice(prev);
  return e == cudaSuccess ? SILENZIO_OK : SILENZIO_ERR_CUDA;
}

static int ensure_tables() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SILENZIO_ERR_CUDA;
  std::call_once(g_once[dev], [dev] { g_status[dev] = init_tables(dev); });
  return g_status[dev];
}

template <int R>
__device__ __forceinline__ double2 Fq(int q, int p) {
  return R == 2 ? g_F2[q * kB + p] : g_F8[q * kB + p];
}
template <int R>
__device__ __forceinline__ double2 Cmq(int m, int q) {
  return R == 2 ? c_C2[m * R + q] : c_C8[m * R + q];
}

// ---------------------------------------------------------- block FFT
// 2048 = 16 x 16 x 8 (four-step, decimation in frequency), 128 threads of one
// slot, 16 complex values per thread, exchanges through the slot's 32 KiB
// buffer with the XOR swizzle p ^ ((p >> 4) & 7) (16-byte elements: conflict
// free for all three access patterns). Positive exponent; INV = conjugate.
__device__ __forceinline__ int swz(int p) { return p ^ ((p >> 4) & 7); }
__device__ __forceinline__ void slot_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(kT) : "memory");
}

// in: x[m] = input at index t + 128 m (natural). out: x[v] = spectrum at
// k1 + 16 (k2a + 16 k2b), (k1, k2a) = pass-3 pair u = v >> 3 of this thread,
// k2b = v & 7: "slot order" (the Fourier BSK is stored in the same order).
__device__ __forceinline__ void block_fft_fwd(double2 (&x)[16], double2 *buf, int t, int g) {
  // pass 1: radix 16 over stride 128, twiddle W_2048^{t k1}
  dft<16, false>(x);  // x[r] = sum_m x_m W16^{m k1}, k1 = bitrev4(r)
  slot_sync(g);       // earlier users of buf are done
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int k1 = bitrev4(r);
    buf[swz(t + 128 * k1)] = (k1 == 0) ? x[r] : cmul(x[r], g_bt.tw1[k1 * 128 + t]);
  }
  slot_sync(g);
  // pass 2: for each (k1, s): radix 16 over m2 (t' = s + 8 m2), twiddle W_128^{s k2a}
  {
    const int k1 = t >> 3, s = t & 7;
#pragma unroll
    for (int m = 0; m < 16; m++) x[m] = buf[swz(s + 8 * m + 128 * k1)];
    dft<16, false>(x);
    slot_sync(g);
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int k2a = bitrev4(r);
      buf[swz(s + 8 * k2a + 128 * k1)] = (k2a == 0 || s == 0) ? x[r] : cmul(x[r], g_bt.tw2[k2a * 8 + s]);
    }
  }
  slot_sync(g);
  // pass 3: radix 8 over s, two (k1, k2a) pairs per thread: pair u -> c = 2 t + u
#pragma unroll
  for (int u = 0; u < 2; u++) {
    const int c = 2 * t + u, k1 = c >> 4, k2a = c & 15;
    double2 z[8];
#pragma unroll
    for (int s = 0; s < 8; s++) z[s] = buf[swz(s + 8 * k2a + 128 * k1)];
    dft<8, false>(z);  // z[r] = X[k1 + 16 (k2a + 16 bitrev3(r))]
#pragma unroll
    for (int r = 0; r < 8; r++) x[8 * u + r] = z[r];
  }
}

__host__ __device__ constexpr int bitrev3(int r) { return ((r & 1) << 2) | (r & 2) | ((r & 4) >> 2); }

// inverse of block_fft_fwd (unnormalised): slot order in, natural order out
// (x[m] = 2048 * input at t + 128 m for a forward-then-inverse round trip)
__device__ __forceinline__ void block_fft_inv(double2 (&x)[16], double2 *buf, int t, int g) {
  slot_sync(g);
#pragma unroll
  for (int u = 0; u < 2; u++) {
    const int c = 2 * t + u, k1 = c >> 4, k2a = c & 15;
    double2 z[8];
#pragma unroll
    for (int r = 0; r < 8; r++) z[bitrev3(r)] = x[8 * u + r];  // natural k2b order
    dft<8, true>(z);  // z[r'] = sum_k2b ... at s = bitrev3(r')
#pragma unroll
    for (int r = 0; r < 8; r++) buf[swz(bitrev3(r) + 8 * k2a + 128 * k1)] = z[r];
  }
  slot_sync(g);
  {
    const int k1 = t >> 3, s = t & 7;
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const double2 v = buf[swz(s + 8 * k + 128 * k1)];
      x[k] = (k == 0 || s == 0) ? v : cmulc(v, g_bt.tw2[k * 8 + s]);
    }
    dft<16, true>(x);  // x[r] = value at m2 = bitrev4(r)
    slot_sync(g);
#pragma unroll
    for (int r = 0; r < 16; r++) buf[swz(s + 8 * bitrev4(r) + 128 * k1)] = x[r];
  }
  slot_sync(g);
#pragma unroll
  for (int k1 = 0; k1 < 16; k1++) {
    const double2 v = buf[swz(t + 128 * k1)];
    x[k1] = (k1 == 0) ? v : cmulc(v, g_bt.tw1[k1 * 128 + t]);
  }
  dft<16, true>(x);  // x[r] = output at index t + 128 bitrev4(r)
  double2 o[16];
#pragma unroll
  for (int r = 0; r < 16; r++) o[bitrev4(r)] = x[r];
#pragma unroll
  for (int m = 0; m < 16; m++) x[m] = o[m];
}

// ------------------------------------------------- cluster exchange primitives
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_release_cluster() { asm volatile("fence.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void arrive_remote_relaxed(uint32_t rmbar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rmbar) : "memory");
}
__device__ __forceinline__ void wait_acq_cluster(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nSZ_C2W_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SZ_C2W_%=;\n}\n" ::"r"(mbar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_async(uint32_t raddr, double2 v, uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(v.x), "d"(v.y), "r"(rmbar)
               : "memory");
}
__device__ __forceinline__ u64 ld_remote_u64(uint32_t raddr) {
  u64 v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(raddr) : "memory");
  return v;
}

// ---------------------------------------------------------------- kernel
struct Args {
  const u64 *lwe_small;  // [count][n+1]
  const u32 *lut_ids;
  const u64 *luts;       // [num_luts][N]
  u32 num_luts;
  const double2 *fbsk;   // [n][2 o][rows][P][R q][16 v][128 t]
  u64 *lwe_out;          // [count][N+1]
  long count;
  int n, base_log, w;
};

template <int R>
struct Geo {
  static constexpr int N = 4096 * R, M = 2048 * R, log2_2N = (R == 2 ? 14 : 16);
  static constexpr int Pw = kB / R;       // owned positions per CTA
  static constexpr int PT = Pw / kT;      // owned positions per thread (R = 2: 8, R = 8: 2)
  static constexpr int ACCW = 2 * 2 * R * Pw;  // owned ACC words per ciphertext (both components)
};

__host__ __device__ constexpr size_t acc_bytes() { return (size_t)2 * 2 * kB * sizeof(u64); }  // = ACCW * 8
__host__ __device__ constexpr size_t smem_bytes(int n) {
  return kSlots * acc_bytes() + kSlots * (size_t)kB * sizeof(double2) + kSlots * (((size_t)n * 2 + 15) / 16 * 16);
}
// ACC index of (comp, h, m', loc) within a slot's 64 KiB
template <int R>
__device__ __forceinline__ int aidx(int comp, int h, int m, int loc) {
  return ((comp * 2 + h) * R + m) * Geo<R>::Pw + loc;
}

// exchange state of one slot: full (this CTA's receive buffer, one arrival +
// 32 KiB of transactions per round) and freeb (R arrivals: every receiver
// released its buffer for the next round)
struct Xch {
  uint32_t full, freeb, buf_s;
  uint32_t round;
};

template <int R>
__device__ __forceinline__ void xch_release(Xch &X, int t, int g) {
  slot_sync(g);  // every thread of this slot is done with its buffer
  if (t == 0) {
    mbar_expect(X.full, kB * sizeof(double2));
    fence_release_cluster();
#pragma unroll
    for (int r = 0; r < R; r++) arrive_remote_relaxed(mapa(X.freeb, r));
  }
}

template <int R, int L, int P>
__global__ void __launch_bounds__(kSlots * kT, 1) blind_rotate_cluster2_kernel(Args A) {
  using Gm = Geo<R>;
  extern __shared__ __align__(16) unsigned char smem[];
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  constexpr int rows = 2 * L;
  static_assert(rows * kV * 4 <= 256, "digit spectra of one slot must fit half of tensor memory");
  const int tid = threadIdx.x, wid = tid >> 5, g = tid / kT, t = tid % kT;
  const int q = (int)cl.block_rank();
  const int n = A.n, w = A.w, blog = A.base_log;
  u64 *acc = reinterpret_cast<u64 *>(smem + g * acc_bytes());
  double2 *buf = reinterpret_cast<double2 *>(smem + kSlots * acc_bytes() + g * kB * sizeof(double2));
  unsigned short *abar = reinterpret_cast<unsigned short *>(smem + kSlots * acc_bytes() +
                                                            kSlots * kB * sizeof(double2)) +
                         g * (((size_t)n * 2 + 15) / 16 * 8);
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t xbar[kSlots][2];
  if (wid == 0) tmem_alloc(&tmem_slot, 512);
  Xch X;
  X.full = smem_u32(&xbar[g][0]);
  X.freeb = smem_u32(&xbar[g][1]);
  X.buf_s = smem_u32(buf);
  X.round = 0;
  if (t == 0) {
    mbar_init(X.full, 1);
    mbar_init(X.freeb, R);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  cl.sync();  // every barrier of the cluster initialised
  // this thread's lane quadrant = wid % 4, column half = slot
  const uint32_t ta_spec = tmem_slot + ((uint32_t)(32 * (wid & 3)) << 16) + 256 * g;
  const uint32_t acc_s = smem_u32(acc);

  const long ncl = gridDim.x / R;
  for (long c0 = (long)(blockIdx.x / R) * kSlots; c0 < A.count; c0 += ncl * kSlots) {
    const long c_raw = c0 + g;
    const bool live = c_raw < A.count;
    const long c = live ? c_raw : A.count - 1;  // an idle slot replays the last ciphertext
    const u64 *lwe = A.lwe_small + (size_t)c * (n + 1);
    for (int i = t; i < n; i += kT) abar[i] = (unsigned short)sz_modswitch(lwe[i], Gm::log2_2N);
    const int bt = (int)sz_modswitch(lwe[n], Gm::log2_2N);
    u32 id = A.lut_ids ? A.lut_ids[c] : 0u;
    if (id >= A.num_luts) id = 0;
    const u64 *v = A.luts + (size_t)id * Gm::N;
    // ACC = (0, X^{-b~} v) on the owned coefficients j = h M + 2048 m' + q Pw + loc
    for (int e = t; e < 2 * R * Gm::Pw; e += kT) {
      const int loc = e % Gm::Pw, m = (e / Gm::Pw) % R, h = e / (Gm::Pw * R);
      const int j = h * Gm::M + kB * m + q * Gm::Pw + loc;
      const int idx = (j + bt) & (2 * Gm::N - 1);
      acc[aidx<R>(0, h, m, loc)] = 0;
      acc[aidx<R>(1, h, m, loc)] = (idx < Gm::N) ? v[idx] : (u64)0 - v[idx - Gm::N];
    }
    slot_sync(g);  // abar, ACC ready (this slot)
    for (int i = 0; i < n; i++) {
      const int a = abar[i];
      // ================= forward: every (component r, level lvl) row
#pragma unroll 1
      for (int r = 0; r < 2; r++) {
        // level-lvl digits of every owned position, levels 2..L kept in registers
        int dig_hi[L > 1 ? Gm::PT * R * 2 : 1];
#pragma unroll 1
        for (int lvl = 1; lvl <= L; lvl++) {
          // this CTA is done with its buffer (previous FFT / combine): release it, then
          // wait until every receiver released theirs (and every ACC slice is final)
          xch_release<R>(X, t, g);
          wait_acq_cluster(X.freeb, X.round & 1);
#pragma unroll
          for (int u = 0; u < Gm::PT; u++) {
            const int loc = t + kT * u, p = q * Gm::Pw + loc;
            double2 zz[R];
#pragma unroll
            for (int m = 0; m < R; m++) {
              double dv[2];
#pragma unroll
              for (int h = 0; h < 2; h++) {
                const int di = (u * R + m) * 2 + h;
                i64 d;
                if (lvl == 1) {
                  // rotated coefficient X^a ACC_r at j: +-ACC_r[(j - a) mod 2N]
                  const int j = h * Gm::M + kB * m + p;
                  const int src = (j - a) & (2 * Gm::N - 1);
                  const int sj = src & (Gm::N - 1);
                  const int sh = sj / Gm::M, sm = (sj / kB) % R, sp = sj % kB;
                  const int owner = sp / Gm::Pw, sloc = sp % Gm::Pw;
                  const uint32_t sa = acc_s + 8 * aidx<R>(r, sh, sm, sloc);
                  const u64 rv = (owner == q) ? acc[aidx<R>(r, sh, sm, sloc)] : ld_remote_u64(mapa(sa, owner));
                  const u64 rot = (src < Gm::N) ? rv : (u64)0 - rv;
                  u64 rr = sz_decomp_round(rot - acc[aidx<R>(r, h, m, loc)], blog, L);
                  d = sz_decomp_next(rr, blog);  // level L (least significant) first
                  if constexpr (L > 1) {
                    // C3: digits peeled from level L up to 1; level 1 is the last
                    i64 dl[L];
                    dl[L - 1] = d;
#pragma unroll
                    for (int tt = L - 2; tt >= 0; tt--) dl[tt] = sz_decomp_next(rr, blog);
                    d = dl[0];
                    dig_hi[di] = (int)dl[1];  // L = 2 (static_assert below)
                  }
                } else {
                  d = dig_hi[di];
                }
                dv[h] = (double)d;
              }
              zz[m] = make_double2(dv[0], dv[1]);
            }
            // x_q'[p] = F[q'][p] DFT_R(z^[m'] e^{i pi m' / 2R})[q']  via the C table
#pragma unroll
            for (int qq = 0; qq < R; qq++) {
              double2 s = make_double2(0.0, 0.0);
#pragma unroll
              for (int m = 0; m < R; m++) cmac(s, zz[m], Cmq<R>(m, qq));
              const double2 xv = cmul(s, Fq<R>(qq, p));
              st_async(mapa(X.buf_s + p * 16, qq), xv, mapa(X.full, qq));
            }
          }
          wait_acq_cluster(X.full, X.round & 1);  // block inputs delivered
          X.round++;
          double2 x[16];
#pragma unroll
          for (int m = 0; m < 16; m++) x[m] = buf[t + kT * m];
          block_fft_fwd(x, buf, t, g);
          const int row = r * L + (lvl - 1);
#pragma unroll
          for (int jj = 0; jj < 4; jj++) {
            uint32_t r16[16];
            pack4(&x[4 * jj], r16);
            tmem_st16(ta_spec + 64 * row + 16 * jj, r16);
          }
        }
      }
      tmem_wait_st();
      // ================= inverse: per output o and limb p
#pragma unroll 1
      for (int o = 0; o < 2; o++) {
#pragma unroll 1
        for (int pl = P - 1; pl >= 0; pl--) {
          double2 y[16];
#pragma unroll
          for (int sl = 0; sl < 16; sl++) y[sl] = make_double2(0.0, 0.0);
#pragma unroll 1
          for (int row = 0; row < rows; row++) {
            const double2 *G = A.fbsk + (((((size_t)i * 2 + o) * rows + row) * P + pl) * R + q) * kB + t;
#pragma unroll
            for (int qq = 0; qq < 4; qq += 2) {
              double2 gg[8];
#pragma unroll
              for (int k = 0; k < 8; k++) gg[k] = __ldg(&G[(4 * qq + k) * kT]);
              uint32_t d0[16], d1[16];
              tmem_ld16(ta_spec + 64 * row + 16 * qq, d0);
              tmem_ld16(ta_spec + 64 * row + 16 * (qq + 1), d1);
              tmem_wait_ld16x2(d0, d1);
#pragma unroll
              for (int k = 0; k < 4; k++) {
                cmac(y[4 * qq + k], unpack1(d0, k), gg[k]);
                cmac(y[4 * qq + 4 + k], unpack1(d1, k), gg[4 + k]);
              }
            }
          }
          block_fft_inv(y, buf, t, g);  // scratch: this CTA's buffer, released only below
          xch_release<R>(X, t, g);
          wait_acq_cluster(X.freeb, X.round & 1);
          // block output at p -> owner of p, slot q of its buffer: buf[q Pw + (p mod Pw)]
#pragma unroll
          for (int m = 0; m < 16; m++) {
            const int p = t + kT * m, owner = p / Gm::Pw;
            st_async(mapa(X.buf_s + (q * Gm::Pw + (p % Gm::Pw)) * 16, owner), y[m], mapa(X.full, owner));
          }
          wait_acq_cluster(X.full, X.round & 1);  // the R block outputs of my positions delivered
          X.round++;
          // combine: z^[p + 2048 m'] = conj(e^{i pi m'/2R}) IDFT_R(conj(F[q'][p]) x'_q'[p])[m']
#pragma unroll
          for (int u = 0; u < Gm::PT; u++) {
            const int loc = t + kT * u, p = q * Gm::Pw + loc;
            double2 uq[R];
#pragma unroll
            for (int qq = 0; qq < R; qq++) uq[qq] = cmulc(buf[qq * Gm::Pw + loc], Fq<R>(qq, p));
#pragma unroll
            for (int m = 0; m < R; m++) {
              double2 s = make_double2(0.0, 0.0);
#pragma unroll
              for (int qq = 0; qq < R; qq++) s = cadd(s, cmulc(uq[qq], Cmq<R>(m, qq)));
              acc[aidx<R>(o, 0, m, loc)] += limb_to_torus(s.x, pl, P, w);
              acc[aidx<R>(o, 1, m, loc)] += limb_to_torus(s.y, pl, P, w);
            }
          }
        }
      }
    }
    // ---- sample extraction of the owned coefficients: a'[0] = A[0], a'[j] = -A[N-j], b' = B[0]
    if (live) {
      u64 *out = A.lwe_out + (size_t)c * (Gm::N + 1);
      for (int e = t; e < 2 * R * Gm::Pw; e += kT) {
        const int loc = e % Gm::Pw, m = (e / Gm::Pw) % R, h = e / (Gm::Pw * R);
        const int j = h * Gm::M + kB * m + q * Gm::Pw + loc;
        const u64 a0 = acc[aidx<R>(0, h, m, loc)];
        if (j == 0) {
          out[0] = a0;
          out[Gm::N] = acc[aidx<R>(1, h, m, loc)];
        } else {
          out[Gm::N - j] = (u64)0 - a0;
        }
      }
    }
    // The next ciphertext's ACC init rewrites owned words; every remote reader
    // read them in a forward row long before (its sends of the inverse rounds
    // depend on those reads), and its next reads follow the next round's
    // release of this CTA (made after the init).
    slot_sync(g);
  }
  cl.sync();  // no CTA leaves while its shared memory may still be accessed
  tmem_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tmem_slot, 512);
}

// ---------------------------------------------------------- BSK -> Fourier
struct B2FArgs {
  const u64 *bsk;  // [n][rows][2 o][N]
  double2 *fbsk;   // [n][2 o][rows][P][R q][16 v][128 t]
  int n, rows, P, w;
};

// one 128-thread CTA per (i, row, o, limb p, block q): x_q, block FFT, * 1/M
template <int R>
__global__ void __launch_bounds__(kT) bsk_to_fourier_cluster2_kernel(B2FArgs A) {
  using Gm = Geo<R>;
  __shared__ __align__(16) double2 buf[kB];
  const int t = threadIdx.x;
  long blk = blockIdx.x;
  const int q = blk % R; blk /= R;
  const int p = blk % A.P; blk /= A.P;
  const int o = blk % 2; blk /= 2;
  const int row = blk % A.rows; blk /= A.rows;
  const int i = (int)blk;
  const u64 *src = A.bsk + (((size_t)i * A.rows + row) * 2 + o) * Gm::N;
  double2 x[16];
#pragma unroll
  for (int mm = 0; mm < 16; mm++) {
    const int pp = t + kT * mm;
    double2 s = make_double2(0.0, 0.0);
#pragma unroll
    for (int m = 0; m < R; m++) {
      double l0[3], l1[3];
      limb_split(src[kB * m + pp], A.P, A.w, l0);
      limb_split(src[Gm::M + kB * m + pp], A.P, A.w, l1);
      cmac(s, make_double2(l0[p], l1[p]), Cmq<R>(m, q));
    }
    x[mm] = cmul(s, Fq<R>(q, pp));
  }
  block_fft_fwd(x, buf, t, 0);
  double2 *dst = A.fbsk + ((((size_t)i * 2 + o) * A.rows + row) * A.P + p) * R * kB + (size_t)q * kB;
  const double scale = 1.0 / Gm::M;
#pragma unroll
  for (int vv = 0; vv < 16; vv++) dst[vv * kT + t] = make_double2(x[vv].x * scale, x[vv].y * scale);
}

}  // namespace c2

// ------------------------------------------------------------------ host side
#ifndef SZ_CLUSTER2
#define SZ_CLUSTER2 1  // 0: the one-ciphertext-per-SM (set C) / per-4-SM-cluster (set B) kernels
#endif
bool blind_rotate_cluster2_supported(const silenzio_params *P) {
  return SZ_CLUSTER2 && (P->poly_size == 8192 || P->poly_size == 32768) && P->glwe_dim == 1 &&
         P->pbs_level == 2 && P->fft_limbs == 3 && c2::smem_bytes((int)P->lwe_dim) <= 227 * 1024;
}

template <int R>
static long cluster2_grid(void (*kern)(c2::Args), size_t smem) {
  struct Entry { int dev; void (*kern)(c2::Args); size_t smem; long ncl; };
  static std::mutex m;
  static std::vector<Entry> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  {
    std::lock_guard<std::mutex> lk(m);
    for (const Entry &e : cache)
      if (e.dev == dev && e.kern == kern && e.smem == smem) return e.ncl;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(R * 32, 1, 1);
  cfg.blockDim = dim3(c2::kSlots * c2::kT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = R;
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

template <int R>
static int launch_cluster2_R(const c2::Args &A, size_t count, cudaStream_t stream) {
  void (*kern)(c2::Args) = c2::blind_rotate_cluster2_kernel<R, 2, 3>;
  const size_t smem = c2::smem_bytes(A.n);
  SZ_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long ncl = cluster2_grid<R>(kern, smem);
  if (ncl <= 0) return SILENZIO_ERR_CUDA;
  const long need = ((long)count + c2::kSlots - 1) / c2::kSlots;
  const long grid = need < ncl ? need : ncl;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(grid * R), 1, 1);
  cfg.blockDim = dim3(c2::kSlots * c2::kT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = R;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  SZ_CUDA_OK(cudaLaunchKernelEx(&cfg, kern, A));
  return SILENZIO_OK;
}

int launch_blind_rotate_cluster2(const u64 *lwe_small, const u32 *lut_ids, const u64 *luts, u32 num_luts,
                                 const void *fbsk, u64 *lwe_out, size_t count, const silenzio_params *P,
                                 cudaStream_t stream) {
  int st = c2::ensure_tables();
  if (st) return st;
  c2::Args A;
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
  return P->poly_size == 8192 ? launch_cluster2_R<2>(A, count, stream) : launch_cluster2_R<8>(A, count, stream);
}

int launch_bsk_to_fourier_cluster2(const u64 *bsk, void *fbsk, const silenzio_params *P, cudaStream_t stream) {
  int st = c2::ensure_tables();
  if (st) return st;
  c2::B2FArgs A;
  A.bsk = bsk;
  A.fbsk = reinterpret_cast<double2 *>(fbsk);
  A.n = (int)P->lwe_dim;
  A.rows = 2 * (int)P->pbs_level;
  A.P = (int)P->fft_limbs;
  A.w = (int)P->limb_bits;
  const int R = (int)P->poly_size / 4096;
  const long blocks = (long)A.n * A.rows * 2 * A.P * R;
  if (R == 2) c2::bsk_to_fourier_cluster2_kernel<2><<<(unsigned)blocks, c2::kT, 0, stream>>>(A);
  else c2::bsk_to_fourier_cluster2_kernel<8><<<(unsigned)blocks, c2::kT, 0, stream>>>(A);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

}  // namespace sz
