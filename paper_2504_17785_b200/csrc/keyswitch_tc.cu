// keyswitch_tc.cu -- batched LWE keyswitch on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM), SURVEY.md §8(a) a1, §8(c) C3:
//     out = (0,...,0,b) - sum_j sum_t Dec_t(a_j) * KSK[j][t]   mod 2^64.
//
// As a matrix product over the batch: D [count x K] (signed gadget digits,
// K = in_dim * l, k = j l + t - 1) times KSK [K x (n+1)] (u64). Each KSK entry
// is split into its 8 bytes, KSK = sum_b 2^{8b} P_b with P_b in [0, 255], so
//     D x KSK = sum_b 2^{8b} (D x P_b)          (mod 2^64)
// and every D x P_b is an exact int8 x uint8 -> int32 product
// (|sum| <= K 2^{B-1} 255 < 2^31, checked on the host). The 8 byte planes of
// 32 output columns form one N = 256 MMA operand, so a CTA owns a 128-row x
// 32-output tile and recombines the planes in its epilogue.
//
// Per CTA (128 ciphertexts x 32 outputs, 256 threads):
//   * B (byte planes) is pre-arranged once per call (ks_planes_kernel) in the
//     tensor-core core-matrix layout, so each K-stage is one contiguous bulk
//     copy (cp.async.bulk, mbarrier completion);
//   * A (signed digits) is decomposed once per call (ks_digits_kernel) into the
//     same core-matrix layout, per 128-row tile and K-stage, so each stage of
//     both operands is two contiguous bulk copies; the 24 column-block CTAs of a
//     row tile (adjacent in launch order) re-read it from L2;
//   * one thread streams the stages (mbarrier expect-tx) and issues the l MMAs
//     of each (M=128, N=256, K=32 each), committing them to the stage's "empty"
//     mbarrier; 3 stages in flight;
//   * the epilogue reads the int32 accumulators from TMEM (thread = ciphertext
//     row), recombines sum_b C_b << 8b, subtracts from the body column.
//
// Shared-memory operand layout (K-major, no swizzle; the canonical UMMA
// "interleave" layout): 8-row x 16-byte core matrices, core matrix (row group
// i, 16-byte K chunk kc) at i * SBO + kc * LBO, LBO = 128 B, SBO = 2 l * 128 B.
#include "common.cuh"
#include "tmem.cuh"

namespace sz {
namespace kst {

constexpr int kRows = 128;    // ciphertexts per CTA (MMA M)
constexpr int kCols = 32;     // output columns per CTA
constexpr int kN = 8 * kCols;  // MMA N: 8 byte planes x 32 columns
constexpr int kStages = 3;
constexpr int kThreads = 256;
constexpr int kJ = 32;  // input coefficients per K-stage (K_stage = 32 l)

__host__ __device__ constexpr int stage_k(int level) { return kJ * level; }           // bytes of K per stage
__host__ __device__ constexpr int a_tile(int level) { return kRows * stage_k(level); }  // A bytes per stage
__host__ __device__ constexpr int b_tile(int level) { return kN * stage_k(level); }     // B bytes per stage
__host__ __device__ constexpr size_t smem_bytes(int level) {
  return (size_t)kStages * (a_tile(level) + b_tile(level)) + 8 * (2 * kStages + 1) + 1024;
}
// byte offset of (row, k) in a core-matrix tile with K extent kst bytes
__host__ __device__ constexpr int cm_off(int row, int k, int kst) {
  return (row >> 3) * (kst / 16) * 128 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}

// ---------------------------------------------------------- plane preparation
// planes[cb][stage][b_tile]: row = b * 32 + c (byte b of column 32 cb + c),
// K index k (within the stage) = row k0 + k of the flat KSK [K][n+1].
// One thread per (cb, stage, c, 16-byte K chunk): reads 16 u64, writes 8 x 16 bytes.
__global__ void ks_planes_kernel(const u64 *ksk, unsigned char *planes, int K, int n1, int level, int ncb) {
  const int kst = stage_k(level), chunks = kst / 16, nst = K / kst;
  const long total = (long)ncb * nst * kCols * chunks;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    long r = e;
    const int kc = (int)(r % chunks); r /= chunks;
    const int c = (int)(r % kCols); r /= kCols;
    const int st = (int)(r % nst); r /= nst;
    const int cb = (int)r;
    const int col = cb * kCols + c;
    u64 v[16];
#pragma unroll
    for (int q = 0; q < 16; q++) {
      const long k = (long)st * kst + kc * 16 + q;
      v[q] = (col < n1) ? __ldg(&ksk[k * n1 + col]) : 0ull;
    }
    unsigned char *tile = planes + ((size_t)cb * nst + st) * b_tile(level);
#pragma unroll
    for (int b = 0; b < 8; b++) {
      uint32_t w[4];
#pragma unroll
      for (int q4 = 0; q4 < 4; q4++) {
        uint32_t x = 0;
#pragma unroll
        for (int q = 0; q < 4; q++) x |= (uint32_t)((v[4 * q4 + q] >> (8 * b)) & 0xff) << (8 * q);
        w[q4] = x;
      }
      *reinterpret_cast<uint4 *>(tile + cm_off(b * kCols + c, kc * 16, kst)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// ------------------------------------------------------------ digit matrix
// digits[row_tile][stage][a_tile]: row r of the tile = ciphertext 128 rt + r,
// K index k = jj l + t - 1 for coefficient j = 32 stage + jj (signed digit of
// level t, C3 decomposition). One thread per (ciphertext, stage, half of the
// stage's 32 coefficients): 16 coefficients -> 16 l digit bytes.
// Optional linear prologue (SURVEY.md §8(a) a0 fused into a1): with lin.idx set,
// row r of the keyswitch input is sum_t coef[r][t] * in[idx[r][t]] + (0,..,0,cst[r])
// mod 2^64, formed on the fly (the combination never goes through HBM); its
// body is written to bodies[r] for the GEMM epilogue.
struct Lin {
  const u32 *idx;   // [count][terms] rows of `in`, or null (row r is in[r])
  const i64 *coef;  // [count][terms]
  const u64 *cst;   // [count] or null
  int terms;
};
__device__ __forceinline__ u64 lin_value(const u64 *in, const Lin &lin, long row, int in_dim, int j) {
  if (!lin.idx) return __ldg(in + (size_t)row * (in_dim + 1) + j);
  u64 v = 0;
  for (int t = 0; t < lin.terms; t++) {
    const size_t o = (size_t)row * lin.terms + t;
    v += (u64)__ldg(lin.coef + o) * __ldg(in + (size_t)__ldg(lin.idx + o) * (in_dim + 1) + j);
  }
  return v;
}
template <int L>
__global__ void ks_digits_kernel(const u64 *in, Lin lin, u64 *bodies, unsigned char *digits, long count,
                                 int rows_padded, int in_dim, int base_log) {
  constexpr int KST = stage_k(L);
  const int nst = in_dim / kJ;
  const long total = (long)rows_padded * nst * 2;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int h = (int)(e & 1);
    long rest = e >> 1;
    const long row = rest % rows_padded;
    const int st = (int)(rest / rows_padded);
    const bool live = row < count;
    const int j0 = kJ * st + 16 * h;
    uint32_t w[4 * L];
#pragma unroll
    for (int q = 0; q < 4 * L; q++) w[q] = 0;
#pragma unroll
    for (int jj = 0; jj < 16; jj++) {
      u64 rr = sz_decomp_round(live ? lin_value(in, lin, row, in_dim, j0 + jj) : 0ull, base_log, L);
#pragma unroll
      for (int t = L; t >= 1; t--) {
        const int d = (int)sz_decomp_next(rr, base_log);
        const int k = jj * L + (t - 1);
        w[k >> 2] |= (uint32_t)(d & 0xff) << (8 * (k & 3));
      }
    }
    if (bodies && live && st == 0 && h == 0)
      bodies[row] = lin_value(in, lin, row, in_dim, in_dim) + (lin.cst ? __ldg(lin.cst + row) : 0ull);
    unsigned char *tile = digits + ((size_t)(row / kRows) * nst + st) * a_tile(L);
    const int r = (int)(row % kRows);
#pragma unroll
    for (int c = 0; c < L; c++)
      *reinterpret_cast<uint4 *>(tile + cm_off(r, 16 * (h * L + c), KST)) =
          make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
  }
}

// --------------------------------------------------------------- primitives
__device__ __forceinline__ void mbar_init(uint64_t *m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SZ_KW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SZ_KW_%=;\n"
      "}\n" ::"r"(smem_u32(m)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, uint32_t bytes, uint64_t *m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *m) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
// shared-memory matrix descriptor: K-major, no swizzle (sm_100 descriptor version 1)
__device__ __forceinline__ uint64_t smem_desc(const void *p, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((smem_u32(p) >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
// instruction descriptor: D s32, A s8 (signed digits), B u8 (key bytes), K-major both, M = 128, N = 256
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(kRows >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *m) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(m))
               : "memory");
}

// ------------------------------------------------------------------ kernel
struct Args {
  const u64 *in;                // [count][in_dim+1]
  const unsigned char *planes;  // [ncb][nst][b_tile]
  const unsigned char *digits;  // [row tiles][nst][a_tile]
  const u64 *bodies;            // [count] input bodies (linear prologue), or null: in[row][in_dim]
  u64 *out;                     // [count][n+1]
  long count;
  int in_dim, n1, base_log, level;
};

template <int L>
__global__ void __launch_bounds__(kThreads, 1) keyswitch_tc_kernel(Args A) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  constexpr int KST = stage_k(L);
  unsigned char *As = smem;                               // [kStages][a_tile]
  unsigned char *Bs = smem + kStages * a_tile(L);         // [kStages][b_tile]
  uint64_t *full = reinterpret_cast<uint64_t *>(Bs + kStages * b_tile(L));
  uint64_t *empty = full + kStages;
  uint64_t *done = empty + kStages;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  // column blocks of one row tile are adjacent in launch order, so the tile's
  // input rows are fetched from HBM once and re-read from L2
  const long row0 = (long)blockIdx.y * kRows;
  const int cb = blockIdx.x;
  const int nst = A.in_dim * L / KST;

  if (wid == 0) tmem_alloc(&tmem_slot, 256);
  if (tid == 32) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem_d = tmem_slot;
  const unsigned char *Bg = A.planes + (size_t)cb * nst * b_tile(L);

  const unsigned char *Ag = A.digits + (size_t)blockIdx.y * nst * a_tile(L);
  if (tid == 0) {
    // one thread streams both operands stage by stage and issues the MMAs,
    // kStages - 1 stages ahead of the tensor core
    for (int it = 0; it < nst + kStages - 1; it++) {
      if (it < nst) {
        const int s = it % kStages;
        if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);  // MMAs of stage it - kStages done
        mbar_expect_tx(&full[s], a_tile(L) + b_tile(L));
        bulk_copy(As + s * a_tile(L), Ag + (size_t)it * a_tile(L), a_tile(L), &full[s]);
        bulk_copy(Bs + s * b_tile(L), Bg + (size_t)it * b_tile(L), b_tile(L), &full[s]);
      }
      const int kc = it - (kStages - 1);
      if (kc >= 0) {
        const int s = kc % kStages;
        mbar_wait(&full[s], (kc / kStages) & 1);
        tmem_fence_after();
        const unsigned char *at = As + s * a_tile(L);
        const unsigned char *bt = Bs + s * b_tile(L);
#pragma unroll
        for (int q = 0; q < L; q++) {  // K = 32 per MMA: core-matrix chunks 2q, 2q + 1
          const uint64_t ad = smem_desc(at + q * 256, 128, (KST / 16) * 128);
          const uint64_t bd = smem_desc(bt + q * 256, 128, (KST / 16) * 128);
          mma_i8(tmem_d, ad, bd, (kc > 0 || q > 0) ? 1u : 0u);
        }
        mma_commit(&empty[s]);
        if (kc == nst - 1) mma_commit(done);
      }
    }
  }
  __syncwarp();
  // ---- epilogue: thread (warp w, lane) owns ciphertext row 32 (w % 4) + lane,
  // output columns 16 (w / 4) .. + 15 of this CTA's 32
  mbar_wait(done, 0);
  tmem_fence_after();
  const int er = 32 * (wid & 3) + lane, half = wid >> 2;
  const long ecrow = row0 + er;
  u64 acc[16];
#pragma unroll
  for (int c = 0; c < 16; c++) acc[c] = 0;
#pragma unroll
  for (int b = 0; b < 8; b++) {
    uint32_t v[16];
    tmem_ld16(tmem_d + ((uint32_t)(32 * (wid & 3)) << 16) + b * kCols + 16 * half, v);
    tmem_wait_ld16(v);
#pragma unroll
    for (int c = 0; c < 16; c++) acc[c] += (u64)(i64)(int32_t)v[c] << (8 * b);
  }
  if (ecrow < A.count) {
    u64 *orow = A.out + (size_t)ecrow * A.n1;
#pragma unroll
    for (int c = 0; c < 16; c++) {
      const int col = cb * kCols + 16 * half + c;
      if (col < A.n1) {
        u64 body = 0;
        if (col == A.n1 - 1) body = A.bodies ? A.bodies[ecrow] : A.in[(size_t)ecrow * (A.in_dim + 1) + A.in_dim];
        orow[col] = body - acc[c];
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tmem_slot, 256);
}

}  // namespace kst

// ------------------------------------------------------------------ host side
static bool ks_tc_applicable(int in_dim, int level, int base_log) {
  if (level < 1 || level > 8 || base_log < 1 || base_log > 7) return false;  // digits must fit int8
  if (in_dim % kst::kJ) return false;
  const double bound = (double)in_dim * level * (double)(1 << (base_log - 1)) * 255.0;
  if (bound >= 2147483648.0) return false;  // int32 accumulation must stay exact
  return kst::smem_bytes(level) <= 227 * 1024;
}

// workspace: KSK byte planes [ncb][nst][b_tile], then the digit matrix [row tiles][nst][a_tile]
static size_t ks_planes_bytes(int in_dim, int n, int level) {
  const size_t ncb = (size_t)(n + 1 + kst::kCols - 1) / kst::kCols;
  return ncb * (size_t)in_dim * level * kst::kN;
}
size_t keyswitch_tc_workspace_bytes(int in_dim, int n, int level, int base_log, size_t count) {
  if (!ks_tc_applicable(in_dim, level, base_log)) return 0;
  const size_t rows = (count + kst::kRows - 1) / kst::kRows * kst::kRows;
  return ks_planes_bytes(in_dim, n, level) + rows * (size_t)in_dim * level;
}

// KSK -> byte planes in the tensor-core operand layout (once per key, or per call by launch_keyswitch_tc)
size_t keyswitch_tc_planes_bytes(int in_dim, int n, int level, int base_log) {
  return ks_tc_applicable(in_dim, level, base_log) ? ks_planes_bytes(in_dim, n, level) : 0;
}
int launch_ks_planes(const u64 *ksk, void *planes_, int in_dim, int n, int base_log, int level, cudaStream_t stream) {
  if (!ks_tc_applicable(in_dim, level, base_log)) return SILENZIO_ERR_UNSUPPORTED;
  const int n1 = n + 1, K = in_dim * level;
  const int ncb = (n1 + kst::kCols - 1) / kst::kCols;
  const long total = (long)ncb * (K / kst::stage_k(level)) * kst::kCols * (kst::stage_k(level) / 16);
  const int threads = 256;
  const long blocks = (total + threads - 1) / threads;
  kst::ks_planes_kernel<<<(unsigned)(blocks < 65535 * 16 ? blocks : 65535 * 16), threads, 0, stream>>>(
      ksk, reinterpret_cast<unsigned char *>(planes_), K, n1, level, ncb);
  SZ_LAUNCH_OK();
  return SILENZIO_OK;
}

// scratch of the product itself: digit matrix, then (linear prologue only) the input bodies
size_t keyswitch_tc_scratch_bytes(int in_dim, int level, size_t count) {
  const size_t rows = (count + kst::kRows - 1) / kst::kRows * kst::kRows;
  return rows * (size_t)in_dim * level + rows * sizeof(u64);
}

// out = keyswitch of (the linear combinations of) `in` with prepared byte planes.
// idx == null: row r = in[r]. scratch: keyswitch_tc_scratch_bytes, 16-byte aligned.
int launch_keyswitch_tc_planes(const u64 *in, const u32 *idx, const i64 *coef, const u64 *cst, int terms,
                               const void *planes_, void *scratch, u64 *out, size_t count, int in_dim, int n,
                               int base_log, int level, cudaStream_t stream) {
  if (!ks_tc_applicable(in_dim, level, base_log)) return SILENZIO_ERR_UNSUPPORTED;
  if (((uintptr_t)planes_ & 15) != 0 || ((uintptr_t)scratch & 15) != 0) return SILENZIO_ERR_MISALIGNED;
  const int n1 = n + 1;
  const int ncb = (n1 + kst::kCols - 1) / kst::kCols;
  const unsigned char *planes = reinterpret_cast<const unsigned char *>(planes_);
  unsigned char *digits = reinterpret_cast<unsigned char *>(scratch);
  const size_t rows_all = (count + kst::kRows - 1) / kst::kRows * kst::kRows;
  u64 *bodies = idx ? reinterpret_cast<u64 *>(digits + rows_all * (size_t)in_dim * level) : nullptr;
  void (*kern)(kst::Args) = nullptr;
  switch (level) {
    case 1: kern = kst::keyswitch_tc_kernel<1>; break;
    case 2: kern = kst::keyswitch_tc_kernel<2>; break;
    case 3: kern = kst::keyswitch_tc_kernel<3>; break;
    case 4: kern = kst::keyswitch_tc_kernel<4>; break;
    case 5: kern = kst::keyswitch_tc_kernel<5>; break;
    case 6: kern = kst::keyswitch_tc_kernel<6>; break;
    default: return SILENZIO_ERR_UNSUPPORTED;
  }
  const size_t smem = kst::smem_bytes(level);
  SZ_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void (*dkern)(const u64 *, kst::Lin, u64 *, unsigned char *, long, int, int, int) = nullptr;
  switch (level) {
    case 1: dkern = kst::ks_digits_kernel<1>; break;
    case 2: dkern = kst::ks_digits_kernel<2>; break;
    case 3: dkern = kst::ks_digits_kernel<3>; break;
    case 4: dkern = kst::ks_digits_kernel<4>; break;
    case 5: dkern = kst::ks_digits_kernel<5>; break;
    case 6: dkern = kst::ks_digits_kernel<6>; break;
    default: return SILENZIO_ERR_UNSUPPORTED;
  }
  const size_t max_rows = (size_t)65535 * kst::kRows;  // grid.y limit per launch
  for (size_t c0 = 0; c0 < count; c0 += max_rows) {
    const size_t cnt = count - c0 < max_rows ? count - c0 : max_rows;
    const int rows_padded = (int)((cnt + kst::kRows - 1) / kst::kRows * kst::kRows);
    // with the prologue, rows address `in` through idx (not offset by c0); without it, row r is in[c0 + r]
    const u64 *in_c = idx ? in : in + c0 * (size_t)(in_dim + 1);
    kst::Lin lin{idx ? idx + c0 * (size_t)terms : nullptr, idx ? coef + c0 * (size_t)terms : nullptr,
                 (idx && cst) ? cst + c0 : nullptr, terms};
    {
      const long total = (long)rows_padded * (in_dim / kst::kJ) * 2;
      const long blocks = (total + 255) / 256;
      dkern<<<(unsigned)(blocks < 65535L * 64 ? blocks : 65535L * 64), 256, 0, stream>>>(
          in_c, lin, bodies ? bodies + c0 : nullptr, digits, (long)cnt, rows_padded, in_dim, base_log);
      SZ_LAUNCH_OK();
    }
    kst::Args A{in_c, planes, digits, bodies ? bodies + c0 : nullptr, out + c0 * (size_t)n1, (long)cnt, in_dim, n1,
                base_log, level};
    dim3 grid((unsigned)ncb, (unsigned)((cnt + kst::kRows - 1) / kst::kRows));
    kern<<<grid, kst::kThreads, smem, stream>>>(A);
    SZ_LAUNCH_OK();
  }
  return SILENZIO_OK;
}

// planes re-derived from the KSK into the workspace on every call (silenzio_keyswitch_batch, silenzio_pbs_batch)
int launch_keyswitch_tc(const u64 *in, const u64 *ksk, u64 *out, size_t count, int in_dim, int n, int base_log,
                        int level, void *workspace, cudaStream_t stream) {
  if (!ks_tc_applicable(in_dim, level, base_log)) return SILENZIO_ERR_UNSUPPORTED;
  if (((uintptr_t)workspace & 15) != 0) return SILENZIO_ERR_MISALIGNED;
  unsigned char *planes = reinterpret_cast<unsigned char *>(workspace);
  int rc = launch_ks_planes(ksk, planes, in_dim, n, base_log, level, stream);
  if (rc) return rc;
  return launch_keyswitch_tc_planes(in, nullptr, nullptr, nullptr, 1, planes, planes + ks_planes_bytes(in_dim, n, level),
                                    out, count, in_dim, n, base_log, level, stream);
}

}  // namespace sz
