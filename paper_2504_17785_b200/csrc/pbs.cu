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
// Design: CTAs of 128 threads = two teams of 64; team g
// owns GLWE component g (mask / body) of one ciphertext. The accumulator lives
// in tensor memory (TMEM, each thread its own lane: the 32 coefficients its
// inverse FFT produces), which frees the registers to prefetch the next
// limb's Fourier-BSK operands during the current limb's inverse FFT -- the
// L2 latency of the BSK stream is then hidden behind FFT arithmetic. The
// decomposed digits' spectra are staged in shared memory (one 16 KiB array per
// GGSW row); every transform is register resident (16 complex per thread) with
// two shared-memory exchanges.
#include <cmath>
#include <mutex>

#include "fft.cuh"
#include "limbs.cuh"
#include "tmem.cuh"

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

// Forward transform. In: x[m] = folded value at j = t + 64 m (natural m).
// Out: x[4u + r] = spectrum at position 4 (t + 64 u) + bitrev2(r) ("slot" order).
// `buf` (16 KiB) is the exchange buffer; on return the caller must team_sync
// before overwriting it (other threads may still be reading pass-3 data).
// Pass-1 twiddles w^{t(4k+1)} of register r (k = bitrev4(r)) either from the
// global table (L1) or, with TW_TM, from this thread's TMEM lane at columns
// tw_ta + 4r .. 4r + 3 (four registers per chunk of 16 columns, one round trip).
template <bool TW_TM>
__device__ __forceinline__ void fwd_fft(double2 (&x)[16], double2 *buf, int t, int team, uint32_t tw_ta = 0) {
  const Tables &T = g_tables;
  // negacyclic twist, part 1: w^{64 m} (the w^t part is folded into tw1)
#pragma unroll
  for (int m = 1; m < 16; m++) x[m] = cmul(x[m], c_twist[m]);
  // pass 1: radix 16 over stride 64 (thread owns offset s = t)
  dft<16, false>(x);
  const int c1 = t ^ ((t >> 3) & 3);  // swz(t + 64 k) = 64 k + (c1 ^ 4 (k & 1))
  team_sync(team);
  if constexpr (TW_TM) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      uint32_t r16[16];
      tmem_ld16(tw_ta + 16 * j, r16);
      tmem_wait_ld16(r16);
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int r = 4 * j + q, k = bitrev4(r);
        buf[64 * k + (c1 ^ ((k & 1) << 2))] = cmul(x[r], unpack1(r16, q));
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int k = bitrev4(r);
      buf[64 * k + (c1 ^ ((k & 1) << 2))] = cmul(x[r], __ldg(&T.tw1[k * 64 + t]));
    }
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
    buf[swz(64 * b + s + 4 * k)] = (k == 0) ? y[r] : cmul(y[r], __ldg(&T.tw2[k * 4 + s]));
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
template <bool TW_TM>
__device__ __forceinline__ void inv_fft(double2 (&x)[16], double2 *buf, int t, int team, uint32_t tw_ta = 0) {
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
  if constexpr (TW_TM) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      uint32_t r16[16];
      tmem_ld16(tw_ta + 16 * j, r16);
      tmem_wait_ld16(r16);
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int k = bitrev4(4 * j + q);
        x[k] = cmulc(buf[64 * k + (c1 ^ ((k & 1) << 2))], unpack1(r16, q));
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = cmulc(buf[64 * k + (c1 ^ ((k & 1) << 2))], __ldg(&T.tw1[k * 64 + t]));
  }
  dft<16, true>(x);
  // x[q] now holds m = bitrev4(q); reorder to natural m and untwist
  double2 o[16];
#pragma unroll
  for (int q = 0; q < 16; q++) o[bitrev4(q)] = x[q];
  x[0] = o[0];
#pragma unroll
  for (int m = 1; m < 16; m++) x[m] = cmulc(o[m], c_twist[m]);
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

// Shared memory per CTA: two 16 KiB transient buffers (team g's ACC copy the
// rotation reads, later its inverse-FFT exchange) + one 16 KiB spectrum per
// GGSW row (also the forward exchange buffer) + the modswitched mask.
__host__ __device__ constexpr size_t br_smem_bytes(int rows, int n) {
  return 2 * kM * sizeof(double2) + (size_t)rows * kM * sizeof(double2) +
         ((size_t)n * sizeof(unsigned short) + 15) / 16 * 16;
}

// ACC init value of coefficient j: (X^{-b} v)[j] = v[j + b] (negacyclic), body only
__device__ __forceinline__ u64 acc_init(const u64 *v, int j, int bt, int team) {
  const int idx = (j + bt) & (2 * kN - 1);
  const u64 vv = (idx < kN) ? v[idx] : (u64)0 - v[idx - kN];
  return team ? vv : 0ull;
}

// ---- ACC in TMEM. Thread t of team g (warp 2g + t/32, TMEM lanes of its warp's
// quadrant) keeps ACC_g[j], j = t + 64 m + 1024 h, in its own lane: u64 (m, h)
// at columns 4m + 2h (low word) and 4m + 2h + 1 (high word), 64 columns per CTA.
// Chunk c (16 columns) holds m = 4c .. 4c + 3.
constexpr uint32_t kAccCols = 64;
constexpr uint32_t kTmemCols = 128;  // ACC [0, 64) + pass-1 twiddles [64, 128)

__device__ __forceinline__ void acc_load(uint32_t ta, int c, u64 (&a)[4][2]) {
  uint32_t r[16];
  tmem_ld16(ta + 16 * c, r);
  tmem_wait_ld16(r);
#pragma unroll
  for (int q = 0; q < 4; q++)
#pragma unroll
    for (int h = 0; h < 2; h++) a[q][h] = (u64)r[4 * q + 2 * h] | ((u64)r[4 * q + 2 * h + 1] << 32);
}
__device__ __forceinline__ void acc_store(uint32_t ta, int c, const u64 (&a)[4][2]) {
  uint32_t r[16];
#pragma unroll
  for (int q = 0; q < 4; q++)
#pragma unroll
    for (int h = 0; h < 2; h++) {
      r[4 * q + 2 * h] = (uint32_t)a[q][h];
      r[4 * q + 2 * h + 1] = (uint32_t)(a[q][h] >> 32);
    }
  tmem_st16(ta + 16 * c, r);
}

// Fourier-BSK operands of one row pair (rows 2 rp, 2 rp + 1) for this thread's
// 16 slots: the MAC's whole global-memory input for that pair (128 registers).
__device__ __forceinline__ void load_g(double2 (&g)[2][16], const double2 *G0, const double2 *G1) {
#pragma unroll
  for (int sl = 0; sl < 16; sl++) {
    g[0][sl] = __ldg(&G0[sl * 64]);
    g[1][sl] = __ldg(&G1[sl * 64]);
  }
}

template <int L, int P>
__global__ void __launch_bounds__(128, 3) blind_rotate_kernel(BRArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t tmem_slot;
  constexpr int rows = 2 * L;
  double2 *tbuf_all = reinterpret_cast<double2 *>(smem);  // [2 teams][1024]
  double2 *dsm = tbuf_all + 2 * kM;                       // [rows][16][64]
  unsigned short *abar = reinterpret_cast<unsigned short *>(dsm + (size_t)rows * kM);
  const int tid = threadIdx.x, team = tid >> 6, t = tid & 63, wid = tid >> 5;
  double2 *tbuf = tbuf_all + team * kM;
  u64 *accs = reinterpret_cast<u64 *>(tbuf);  // ACC_g copy [2048] for the rotation
  const int n = A.n, w = A.w, blog = A.base_log;

  if (wid == 0) tmem_alloc(&tmem_slot, kTmemCols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t ta = tmem_slot + ((uint32_t)(32 * wid) << 16);
  const uint32_t ta_tw = ta + kAccCols;
  // pass-1 twiddles of this thread's t, register order r (k = bitrev4(r))
#pragma unroll
  for (int j = 0; j < 4; j++) {
    double2 tw[4];
#pragma unroll
    for (int q = 0; q < 4; q++) tw[q] = g_tables.tw1[bitrev4(4 * j + q) * 64 + t];
    uint32_t r16[16];
    pack4(tw, r16);
    tmem_st16(ta_tw + 16 * j, r16);
  }
  tmem_wait_st();

  // Fourier-BSK pointer of (i, output component team, row, limb p), thread offset t
  auto gptr = [&](int i, int row, int p) {
    return A.fbsk + ((((size_t)i * 2 + team) * rows + row) * P + p) * kM + t;
  };

  for (long c = blockIdx.x; c < A.count; c += gridDim.x) {
    const u64 *lwe = A.lwe_small + (size_t)c * (n + 1);
    // ---- modulus switch (a2)
    for (int i = tid; i < n; i += 128) abar[i] = (unsigned short)sz_modswitch(lwe[i], kLog2_2N);
    const int bt = (int)sz_modswitch(lwe[n], kLog2_2N);
    // ---- ACC init (a3): ACC = (0, X^{-b~} v)
    u32 id = A.lut_ids ? A.lut_ids[c] : 0u;
    if (id >= A.num_luts) id = 0;
    const u64 *v = A.luts + (size_t)id * kN;
#pragma unroll
    for (int cc = 0; cc < 4; cc++) {
      u64 a4[4][2];
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int h = 0; h < 2; h++) a4[q][h] = acc_init(v, t + 64 * (4 * cc + q) + 1024 * h, bt, team);
      acc_store(ta, cc, a4);
    }
    tmem_wait_st();
    __syncthreads();  // abar visible

    for (int i = 0; i < n; i++) {
      const int a = abar[i];
      // ---------------- publish ACC_g for the rotation
#pragma unroll
      for (int cc = 0; cc < 4; cc++) {
        u64 a4[4][2];
        acc_load(ta, cc, a4);
#pragma unroll
        for (int q = 0; q < 4; q++)
#pragma unroll
          for (int h = 0; h < 2; h++) accs[t + 64 * (4 * cc + q) + 1024 * h] = a4[q][h];
      }
      team_sync(team);
      // ---------------- forward: digits of X^a ACC_g - ACC_g, one FFT per level
#pragma unroll 1
      for (int lvl = 1; lvl <= L; lvl++) {
        double2 x[16];
#pragma unroll
        for (int cc = 0; cc < 4; cc++) {
          u64 a4[4][2];
          acc_load(ta, cc, a4);
#pragma unroll
          for (int q = 0; q < 4; q++) {
            double dv[2];
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int j = t + 64 * (4 * cc + q) + 1024 * h;
              const int src = (j - a) & (2 * kN - 1);
              const u64 rv = accs[src & (kN - 1)];
              const u64 rot = (src < kN) ? rv : (u64)0 - rv;
              u64 r = sz_decomp_round(rot - a4[q][h], blog, L);
              i64 d = 0;
              // peel digits t = l, l-1, ..., lvl  (level lvl has weight q/B^lvl)
#pragma unroll
              for (int tt = L; tt >= 1; tt--) {
                const i64 dd = sz_decomp_next(r, blog);
                if (tt == lvl) d = dd;
              }
              dv[h] = (double)d;
            }
            x[4 * cc + q] = make_double2(dv[0], dv[1]);
          }
        }
        double2 *drow = dsm + (size_t)(team * L + (lvl - 1)) * kM;
        fwd_fft<1>(x, drow, t, team, ta_tw);  // the row's own spectrum buffer is the exchange buffer
        team_sync(team);
#pragma unroll
        for (int sl = 0; sl < 16; sl++) drow[sl * 64 + t] = x[sl];
      }
      __syncthreads();  // every row's spectrum is complete
      // ---------------- inverse: output component o = team, limbs top -> 0
#pragma unroll 1
      for (int p = P - 1; p >= 0; p--) {
        double2 y[16];
#pragma unroll
        for (int sl = 0; sl < 16; sl++) y[sl] = make_double2(0.0, 0.0);
#pragma unroll 1
        for (int row = 0; row < rows; row++) {
          const double2 *G = gptr(i, row, p);
          const double2 *D = dsm + (size_t)row * kM + t;
#pragma unroll
          for (int qq = 0; qq < 4; qq++) {
            double2 gg[4], dd[4];
#pragma unroll
            for (int q = 0; q < 4; q++) gg[q] = __ldg(&G[(4 * qq + q) * 64]);
#pragma unroll
            for (int q = 0; q < 4; q++) dd[q] = D[(4 * qq + q) * 64];
#pragma unroll
            for (int q = 0; q < 4; q++) cmac(y[4 * qq + q], dd[q], gg[q]);
          }
        }
        inv_fft<1>(y, tbuf, t, team, ta_tw);
#pragma unroll
        for (int cc = 0; cc < 4; cc++) {
          u64 a4[4][2];
          acc_load(ta, cc, a4);
#pragma unroll
          for (int q = 0; q < 4; q++) {
            a4[q][0] += limb_to_torus(y[4 * cc + q].x, p, P, w);
            a4[q][1] += limb_to_torus(y[4 * cc + q].y, p, P, w);
          }
          acc_store(ta, cc, a4);
        }
        tmem_wait_st();
      }
      __syncthreads();  // spectra and transient buffers free for the next CMux
    }
    // ---- sample extraction (a5): a'[0] = A[0], a'[i] = -A[N-i], b' = B[0]
    u64 *out = A.lwe_out + (size_t)c * (kN + 1);
#pragma unroll
    for (int cc = 0; cc < 4; cc++) {
      u64 a4[4][2];
      acc_load(ta, cc, a4);
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int j = t + 64 * (4 * cc + q) + 1024 * h;
          if (team == 0) {
            if (j == 0) out[0] = a4[q][h];
            else out[kN - j] = (u64)0 - a4[q][h];
          } else if (j == 0) {
            out[kN] = a4[q][h];
          }
        }
    }
    __syncthreads();  // abar reuse
  }
  tmem_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tmem_slot, kTmemCols);
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
  fwd_fft<false>(x, buf, t, 0);
  double2 *dst = A.fbsk + ((((size_t)i * 2 + o) * A.rows + row) * A.P + p) * kM;
  const double scale = 1.0 / kM;
#pragma unroll
  for (int sl = 0; sl < 16; sl++) dst[sl * 64 + t] = make_double2(x[sl].x * scale, x[sl].y * scale);
}

// ------------------------------------------------------------ host launch
// Kernel variant, shared memory and resident ciphertexts per wave for these params.
struct BRPlan {
  void (*kern)(BRArgs);
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
  const size_t smem = br_smem_bytes(2 * level, n);
  if (smem > 227 * 1024) return SILENZIO_ERR_UNSUPPORTED;
  SZ_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 0, per_sm = 0;
  SZ_CUDA_OK(cudaGetDevice(&dev));
  SZ_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SZ_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
  // The occupancy API under-reports residency for this (TMEM-allocating) kernel
  // (1 CTA/SM where ncu's "Block Limit" registers/shared memory give 2): size
  // the wave from registers, shared memory and TMEM columns instead.
  {
    cudaFuncAttributes fa;
    int smem_sm = 0;
    SZ_CUDA_OK(cudaFuncGetAttributes(&fa, kern));
    SZ_CUDA_OK(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    const int by_regs = 65536 / (128 * ((fa.numRegs + 7) / 8 * 8));  // 64K registers per SM
    const int by_smem = smem_sm / (int)(smem + fa.sharedSizeBytes + 1024);
    const int by_tmem = 512 / (int)kTmemCols;
    per_sm = by_regs < by_smem ? by_regs : by_smem;
    if (per_sm > by_tmem) per_sm = by_tmem;
    if (per_sm < 1) per_sm = 1;
  }
  if (per_sm < 1) return SILENZIO_ERR_UNSUPPORTED;
  plan->kern = kern;
  plan->smem = smem;
  plan->wave = (long)sms * per_sm;
  return SILENZIO_OK;
}

// N = 2048, level-1 gadget: the warp-FFT kernel of pbs_warp.cu (own Fourier-BSK layout)
bool blind_rotate_warp_supported(const silenzio_params *P);
long blind_rotate_warp_wave();
long blind_rotate_warp_launches(size_t count);
long blind_rotate_wave(const silenzio_params *P);
int launch_blind_rotate_warp(const u64 *lwe_small, const u32 *lut_ids, const u64 *luts, u32 num_luts,
                             const void *fbsk, u64 *lwe_out, size_t count, const silenzio_params *P,
                             cudaStream_t stream);
int launch_bsk_to_fourier_warp(const u64 *bsk, void *fbsk, const silenzio_params *P, cudaStream_t stream);
#ifdef SZ_NO_WARP_BR
static bool use_warp(const silenzio_params *) { return false; }
#else
static bool use_warp(const silenzio_params *P) { return blind_rotate_warp_supported(P); }
#endif

// number of blind-rotation kernel launches for `count` ciphertexts
long blind_rotate_launches(const silenzio_params *P, size_t count) {
  if (use_warp(P)) return blind_rotate_warp_launches(count);
  const long wave = blind_rotate_wave(P);
  return wave <= 0 ? -1 : (long)((count + wave - 1) / wave);
}

long blind_rotate_wave(const silenzio_params *P) {
  if (use_warp(P)) return blind_rotate_warp_wave();
  BRPlan plan;
  if (ensure_tables() != SILENZIO_OK || plan_blind_rotate(P, &plan) != SILENZIO_OK) return -1;
  return plan.wave;
}

int launch_blind_rotate(const u64 *lwe_small, const u32 *lut_ids, const u64 *luts, u32 num_luts,
                        const void *fbsk, u64 *lwe_out, size_t count, const silenzio_params *P,
                        cudaStream_t stream) {
  if (use_warp(P)) return launch_blind_rotate_warp(lwe_small, lut_ids, luts, num_luts, fbsk, lwe_out, count, P, stream);
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
  BRPlan plan;
  if ((st = plan_blind_rotate(P, &plan))) return st;
  // One launch per resident wave: every CTA of a wave sweeps BSK_0..BSK_{n-1}
  // at the same pace, so the streamed Fourier BSK (146 MB at set A, > L2)
  // is fetched from HBM about once per wave instead of once per drifting CTA.
  for (long c0 = 0; c0 < (long)count; c0 += plan.wave) {
    BRArgs W = A;
    const long cnt = ((long)count - c0 < plan.wave) ? (long)count - c0 : plan.wave;
    W.lwe_small = A.lwe_small + (size_t)c0 * (A.n + 1);
    W.lut_ids = A.lut_ids ? A.lut_ids + c0 : nullptr;
    W.lwe_out = A.lwe_out + (size_t)c0 * (kN + 1);
    W.count = cnt;
    plan.kern<<<(unsigned)cnt, 128, plan.smem, stream>>>(W);
    SZ_LAUNCH_OK();
  }
  return SILENZIO_OK;
}

int launch_bsk_to_fourier(const u64 *bsk, void *fbsk, const silenzio_params *P, cudaStream_t stream) {
  if (use_warp(P)) return launch_bsk_to_fourier_warp(bsk, fbsk, P, stream);
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
