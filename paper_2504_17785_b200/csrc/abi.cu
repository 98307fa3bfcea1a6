// abi.cu -- the extern "C" boundary of libsilenzio (include/silenzio.h):
// argument validation, workspace sizing and kernel dispatch. No computation
// happens on the host; no CPU fallback exists.
#include <cstring>

#include "common.cuh"
#include "nvtx.cuh"

namespace sz {
int launch_blind_rotate(const u64 *, const u32 *, const u64 *, u32, const void *, u64 *, size_t,
                        const silenzio_params *, cudaStream_t);
int launch_bsk_to_fourier(const u64 *, void *, const silenzio_params *, cudaStream_t);
long blind_rotate_wave(const silenzio_params *);
long blind_rotate_launches(const silenzio_params *, size_t);
int launch_blind_rotate_large(const u64 *, const u32 *, const u64 *, u32, const void *, u64 *, size_t,
                              const silenzio_params *, cudaStream_t);
int launch_bsk_to_fourier_large(const u64 *, void *, const silenzio_params *, cudaStream_t);
long blind_rotate_large_wave(const silenzio_params *);
int launch_blind_rotate_huge(const u64 *, const u32 *, const u64 *, u32, const void *, u64 *, size_t,
                             const silenzio_params *, void *, cudaStream_t);
int launch_bsk_to_fourier_huge(const u64 *, void *, const silenzio_params *, cudaStream_t);
size_t blind_rotate_huge_ws_bytes(const silenzio_params *, size_t);
long blind_rotate_huge_wave(const silenzio_params *);
int launch_keyswitch(const u64 *, const u64 *, u64 *, size_t, int, int, int, int, cudaStream_t);
size_t keyswitch_tc_workspace_bytes(int in_dim, int n, int level, int base_log, size_t count);
int launch_keyswitch_tc(const u64 *, const u64 *, u64 *, size_t, int, int, int, int, void *, cudaStream_t);
size_t keyswitch_tc_planes_bytes(int in_dim, int n, int level, int base_log);
size_t keyswitch_tc_scratch_bytes(int in_dim, int level, size_t count);
int launch_ks_planes(const u64 *, void *, int, int, int, int, cudaStream_t);
int launch_keyswitch_tc_planes(const u64 *, const u32 *, const i64 *, const u64 *, int, const void *, void *, u64 *,
                               size_t, int, int, int, int, cudaStream_t);
int launch_lwe_encrypt(const u64 *, const i64 *, const u64 *, const u64 *, int, size_t, u64 *, cudaStream_t);
int launch_lwe_phase(const u64 *, const u64 *, int, size_t, u64 *, cudaStream_t);
int launch_bsk_generate(const u64 *, const u64 *, const u64 *, const i64 *, u64 *, int, int, int, int, int,
                        cudaStream_t);
int launch_bsk_generate_huge(const u64 *, const u64 *, const u64 *, const i64 *, u64 *, int, int, int, int, void *,
                             cudaStream_t);
size_t glwe_body_huge_ws_bytes();
int launch_ksk_generate(const u64 *, const u64 *, const u64 *, const i64 *, u64 *, int, int, int, int,
                        cudaStream_t);
int launch_testpoly(const u64 *, int, int, int, u64 *, cudaStream_t);
int launch_lwe_linear(const u64 *, const u32 *, const i64 *, const u64 *, int, int, size_t, u64 *, cudaStream_t);
}  // namespace sz

using namespace sz;

namespace {

bool is_pow2(uint32_t x) { return x && !(x & (x - 1)); }

// Parameter validity (independent of which kernels exist).
int check_params(const silenzio_params *P) {
  if (!P) return SILENZIO_ERR_NULL_POINTER;
  if (P->glwe_dim < 1 || P->lwe_dim < 1 || !is_pow2(P->poly_size) || P->poly_size < 64) return SILENZIO_ERR_INVALID_PARAM;
  if (P->pbs_base_log < 1 || P->pbs_level < 1 || P->pbs_base_log * P->pbs_level > 64 || P->pbs_base_log > 32)
    return SILENZIO_ERR_INVALID_PARAM;
  if (P->ks_base_log < 1 || P->ks_level < 1 || P->ks_base_log * P->ks_level > 64 || P->ks_base_log > 32)
    return SILENZIO_ERR_INVALID_PARAM;
  if (P->fft_limbs < 1 || P->fft_limbs > 3) return SILENZIO_ERR_INVALID_PARAM;
  if (P->fft_limbs > 1) {
    const uint32_t w = P->limb_bits, top = 64 - (P->fft_limbs - 1) * w;
    if (w < 8 || w > 52 || top < 8 || top > 52) return SILENZIO_ERR_INVALID_PARAM;
  }
  return SILENZIO_OK;
}

// Shapes the blind-rotation kernel implements (DESIGN.md §Kernels / §Scope).
int check_br_supported(const silenzio_params *P) {
  if (P->glwe_dim != 1) return SILENZIO_ERR_UNSUPPORTED;
  if (P->poly_size == 2048) {
    if (P->pbs_level > 4 || P->pbs_level == 3 || P->lwe_dim > 4096) return SILENZIO_ERR_UNSUPPORTED;
    return SILENZIO_OK;
  }
  if (P->poly_size == 8192) {
    if (P->pbs_level > 4 || P->lwe_dim > 4096) return SILENZIO_ERR_UNSUPPORTED;
    return SILENZIO_OK;
  }
  if (P->poly_size == 32768) {
    if (!(P->pbs_level == 1 || P->pbs_level == 2 || P->pbs_level == 4) || P->fft_limbs != 3 || P->lwe_dim > 8192)
      return SILENZIO_ERR_UNSUPPORTED;
    return SILENZIO_OK;
  }
  return SILENZIO_ERR_UNSUPPORTED;
}

int check_ks_params(const silenzio_params *P) {
  if (P->ks_in_dim < 1) return SILENZIO_ERR_INVALID_PARAM;
  return SILENZIO_OK;
}

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

const char *kVersion = "libsilenzio 0.3 (sm_100a; blind rotation N=2048, 8192, 32768; P-limb exact FFT)";

}  // namespace

extern "C" {

const char *silenzio_status_string(int s) {
  switch (s) {
    case SILENZIO_OK: return "ok";
    case SILENZIO_ERR_INVALID_PARAM: return "invalid parameter";
    case SILENZIO_ERR_UNSUPPORTED: return "unsupported parameter set (no kernel for this shape)";
    case SILENZIO_ERR_NULL_POINTER: return "null pointer";
    case SILENZIO_ERR_MISALIGNED: return "pointer not 16-byte aligned";
    case SILENZIO_ERR_COUNT: return "invalid count";
    case SILENZIO_ERR_WINDOW: return "value window too large for one PBS";
    case SILENZIO_ERR_CUDA: return "CUDA error";
    case SILENZIO_ERR_WORKSPACE: return "workspace missing or too small";
    default: return "unknown status";
  }
}

const char *silenzio_version(void) { return kVersion; }

size_t silenzio_fourier_bsk_bytes(const silenzio_params *P) {
  if (check_params(P) != SILENZIO_OK) return 0;
  const size_t rows = (size_t)(P->glwe_dim + 1) * P->pbs_level;
  return (size_t)P->lwe_dim * rows * (P->glwe_dim + 1) * P->fft_limbs * (P->poly_size / 2) * 16;
}

size_t silenzio_blind_rotate_workspace_bytes(const silenzio_params *P, size_t count) {
  if (check_params(P) != SILENZIO_OK) return 0;
  if (P->poly_size == 32768) return round_up(blind_rotate_huge_ws_bytes(P, count), 256);
  return 0;
}

size_t silenzio_keyswitch_workspace_bytes(const silenzio_params *P, size_t count) {
  if (check_params(P) != SILENZIO_OK || check_ks_params(P) != SILENZIO_OK) return 0;
  return round_up(keyswitch_tc_workspace_bytes((int)P->ks_in_dim, (int)P->lwe_dim, (int)P->ks_level,
                                               (int)P->ks_base_log, count), 256);
}

size_t silenzio_pbs_workspace_bytes(const silenzio_params *P, size_t count) {
  if (check_params(P) != SILENZIO_OK) return 0;
  return round_up(count * (size_t)(P->lwe_dim + 1) * sizeof(u64), 256) + silenzio_blind_rotate_workspace_bytes(P, count) +
         silenzio_keyswitch_workspace_bytes(P, count);
}

// tensor-core keyswitch when the parameters allow it and a workspace is given,
// else the CUDA-core kernel (both exact)
static int run_keyswitch(const u64 *in, const u64 *ksk, u64 *out, size_t count, const silenzio_params *P,
                         void *ks_ws, cudaStream_t st) {
  if (ks_ws && silenzio_keyswitch_workspace_bytes(P, count) > 0)
    return launch_keyswitch_tc(in, ksk, out, count, (int)P->ks_in_dim, (int)P->lwe_dim, (int)P->ks_base_log,
                               (int)P->ks_level, ks_ws, st);
  return launch_keyswitch(in, ksk, out, count, (int)P->ks_in_dim, (int)P->lwe_dim, (int)P->ks_base_log,
                          (int)P->ks_level, st);
}

int silenzio_bsk_to_fourier(const uint64_t *bsk, void *fbsk, const silenzio_params *P, void *stream) {
  SZ_RANGE("bsk_to_fourier");
  int st = check_params(P);
  if (st) return st;
  if (!bsk || !fbsk) return SILENZIO_ERR_NULL_POINTER;
  if (!sz_aligned16(bsk) || !sz_aligned16(fbsk)) return SILENZIO_ERR_MISALIGNED;
  if ((st = check_br_supported(P))) return st;
  if (P->poly_size == 8192) return launch_bsk_to_fourier_large(bsk, fbsk, P, sz_stream(stream));
  if (P->poly_size == 32768) return launch_bsk_to_fourier_huge(bsk, fbsk, P, sz_stream(stream));
  return launch_bsk_to_fourier(bsk, fbsk, P, sz_stream(stream));
}

int silenzio_keyswitch_batch(const uint64_t *in, const uint64_t *ksk, uint64_t *out, size_t count,
                             const silenzio_params *P, void *workspace, void *stream) {
  SZ_RANGE("keyswitch_batch");
  int st = check_params(P);
  if (st) return st;
  if ((st = check_ks_params(P))) return st;
  if (count == 0) return SILENZIO_OK;
  if (!in || !ksk || !out) return SILENZIO_ERR_NULL_POINTER;
  if (count > (1ull << 36)) return SILENZIO_ERR_COUNT;
  if (workspace && !sz_aligned16(workspace)) return SILENZIO_ERR_MISALIGNED;
  return run_keyswitch(in, ksk, out, count, P, workspace, sz_stream(stream));
}

int silenzio_blind_rotate_batch(const uint64_t *lwe_small, const uint32_t *lut_ids, const uint64_t *luts,
                                uint32_t num_luts, const void *fbsk, uint64_t *out, size_t count,
                                const silenzio_params *P, void *workspace, void *stream) {
  SZ_RANGE("blind_rotate_batch");
  int st = check_params(P);
  if (st) return st;
  if ((st = check_br_supported(P))) return st;
  if (count == 0) return SILENZIO_OK;
  if (!lwe_small || !luts || !fbsk || !out) return SILENZIO_ERR_NULL_POINTER;
  if (num_luts == 0) return SILENZIO_ERR_INVALID_PARAM;
  if (!sz_aligned16(fbsk) || !sz_aligned(lwe_small, 8) || !sz_aligned(out, 8) || !sz_aligned(luts, 8) ||
      (lut_ids && !sz_aligned(lut_ids, 4)))
    return SILENZIO_ERR_MISALIGNED;
  if (count > (1ull << 31)) return SILENZIO_ERR_COUNT;
  if (P->poly_size == 8192)
    return launch_blind_rotate_large(lwe_small, lut_ids, luts, num_luts, fbsk, out, count, P, sz_stream(stream));
  if (P->poly_size == 32768)
    return launch_blind_rotate_huge(lwe_small, lut_ids, luts, num_luts, fbsk, out, count, P, workspace,
                                    sz_stream(stream));
  return launch_blind_rotate(lwe_small, lut_ids, luts, num_luts, fbsk, out, count, P, sz_stream(stream));
}

int silenzio_pbs_batch(const uint64_t *in, const uint32_t *lut_ids, const uint64_t *luts, uint32_t num_luts,
                       const void *fbsk, const uint64_t *ksk, uint64_t *out, size_t count,
                       const silenzio_params *P, void *workspace, void *stream) {
  SZ_RANGE("pbs_batch");
  int st = check_params(P);
  if (st) return st;
  if ((st = check_ks_params(P))) return st;
  if ((st = check_br_supported(P))) return st;
  if (P->ks_in_dim != P->glwe_dim * P->poly_size) return SILENZIO_ERR_INVALID_PARAM;
  if (count == 0) return SILENZIO_OK;
  if (!in || !luts || !fbsk || !ksk || !out) return SILENZIO_ERR_NULL_POINTER;
  if (!sz_aligned(in, 8) || !sz_aligned(out, 8) || !sz_aligned(luts, 8) || !sz_aligned(ksk, 8) ||
      (lut_ids && !sz_aligned(lut_ids, 4)))
    return SILENZIO_ERR_MISALIGNED;
  if (count > (1ull << 31)) return SILENZIO_ERR_COUNT;  // the blind rotation's limit, checked before the keyswitch runs
  if (!workspace) return SILENZIO_ERR_WORKSPACE;
  if (in == out) return SILENZIO_ERR_INVALID_PARAM;
  if (!sz_aligned16(workspace)) return SILENZIO_ERR_MISALIGNED;
  u64 *small = reinterpret_cast<u64 *>(workspace);
  unsigned char *br_ws = reinterpret_cast<unsigned char *>(workspace) + round_up(count * (size_t)(P->lwe_dim + 1) * sizeof(u64), 256);
  unsigned char *ks_ws = br_ws + silenzio_blind_rotate_workspace_bytes(P, count);
  {
    SZ_RANGE("pbs.keyswitch");
    if ((st = run_keyswitch(in, ksk, small, count, P, ks_ws, sz_stream(stream)))) return st;
  }
  return silenzio_blind_rotate_batch(small, lut_ids, luts, num_luts, fbsk, out, count, P, br_ws, stream);
}

size_t silenzio_ksk_planes_bytes(const silenzio_params *P) {
  if (check_params(P) != SILENZIO_OK || check_ks_params(P) != SILENZIO_OK) return 0;
  return round_up(keyswitch_tc_planes_bytes((int)P->ks_in_dim, (int)P->lwe_dim, (int)P->ks_level, (int)P->ks_base_log),
                  256);
}

int silenzio_ksk_to_planes(const uint64_t *ksk, void *planes, const silenzio_params *P, void *stream) {
  SZ_RANGE("ksk_to_planes");
  int st = check_params(P);
  if (st) return st;
  if ((st = check_ks_params(P))) return st;
  if (!ksk || !planes) return SILENZIO_ERR_NULL_POINTER;
  if (!sz_aligned(ksk, 8) || !sz_aligned16(planes)) return SILENZIO_ERR_MISALIGNED;
  if (silenzio_ksk_planes_bytes(P) == 0) return SILENZIO_ERR_UNSUPPORTED;
  return launch_ks_planes(ksk, planes, (int)P->ks_in_dim, (int)P->lwe_dim, (int)P->ks_base_log, (int)P->ks_level,
                          sz_stream(stream));
}

size_t silenzio_pbs_linear_workspace_bytes(const silenzio_params *P, size_t count) {
  if (check_params(P) != SILENZIO_OK || silenzio_ksk_planes_bytes(P) == 0) return 0;
  return round_up(count * (size_t)(P->lwe_dim + 1) * sizeof(u64), 256) + silenzio_blind_rotate_workspace_bytes(P, count) +
         round_up(keyswitch_tc_scratch_bytes((int)P->ks_in_dim, (int)P->ks_level, count), 256);
}

int silenzio_pbs_linear_batch(const uint64_t *in, const uint32_t *idx, const int64_t *coef, const uint64_t *cst,
                              uint32_t terms, const uint32_t *lut_ids, const uint64_t *luts, uint32_t num_luts,
                              const void *fbsk, const void *planes, uint64_t *out, size_t count,
                              const silenzio_params *P, void *workspace, void *stream) {
  SZ_RANGE("pbs_linear_batch");
  int st = check_params(P);
  if (st) return st;
  if ((st = check_ks_params(P))) return st;
  if ((st = check_br_supported(P))) return st;
  if (P->ks_in_dim != P->glwe_dim * P->poly_size) return SILENZIO_ERR_INVALID_PARAM;
  if (silenzio_ksk_planes_bytes(P) == 0) return SILENZIO_ERR_UNSUPPORTED;
  if (count == 0) return SILENZIO_OK;
  if (!in || !luts || !fbsk || !planes || !out) return SILENZIO_ERR_NULL_POINTER;
  if (idx ? (!coef || terms == 0) : (coef || cst)) return SILENZIO_ERR_INVALID_PARAM;
  if (!sz_aligned(in, 8) || !sz_aligned(out, 8) || !sz_aligned(luts, 8) || !sz_aligned16(planes) ||
      !sz_aligned16(fbsk) || (lut_ids && !sz_aligned(lut_ids, 4)) || (idx && !sz_aligned(idx, 4)) ||
      (coef && !sz_aligned(coef, 8)) || (cst && !sz_aligned(cst, 8)))
    return SILENZIO_ERR_MISALIGNED;
  if (count > (1ull << 31)) return SILENZIO_ERR_COUNT;
  if (!workspace) return SILENZIO_ERR_WORKSPACE;
  if (!sz_aligned16(workspace)) return SILENZIO_ERR_MISALIGNED;
  u64 *small = reinterpret_cast<u64 *>(workspace);
  unsigned char *br_ws = reinterpret_cast<unsigned char *>(workspace) + round_up(count * (size_t)(P->lwe_dim + 1) * sizeof(u64), 256);
  unsigned char *ks_ws = br_ws + silenzio_blind_rotate_workspace_bytes(P, count);
  {
    SZ_RANGE("pbs.linear+keyswitch");
    if ((st = launch_keyswitch_tc_planes(in, idx, coef, cst, (int)terms, planes, ks_ws, small, count, (int)P->ks_in_dim,
                                         (int)P->lwe_dim, (int)P->ks_base_log, (int)P->ks_level, sz_stream(stream))))
      return st;
  }
  return silenzio_blind_rotate_batch(small, lut_ids, luts, num_luts, fbsk, out, count, P, br_ws, stream);
}

long silenzio_pbs_launch_count(const silenzio_params *P, size_t count) {
  if (check_params(P) != SILENZIO_OK || check_br_supported(P) != SILENZIO_OK) return -1;
  if (count == 0) return 0;
  long br;
  if (P->poly_size == 2048) {
    br = blind_rotate_launches(P, count);  // one persistent launch (set A) or one per wave
  } else {
    const long wave = P->poly_size == 8192 ? blind_rotate_large_wave(P) : blind_rotate_huge_wave(P);
    br = wave <= 0 ? -1 : (long)((count + wave - 1) / wave);  // one per resident wave
  }
  if (br < 0) return -1;
  // keyswitch: byte-plane preparation + (digit matrix + GEMM) per 65535 row tiles (tensor cores), else one launch
  const long ks = silenzio_keyswitch_workspace_bytes(P, count) > 0 ? 1 + 2 * (long)((count + 65535L * 128 - 1) / (65535L * 128)) : 1;
  return ks + br;
}

size_t silenzio_pbs_host_workspace_bytes(const silenzio_params *P, size_t chunk) {
  if (check_params(P) != SILENZIO_OK) return 0;
  if (chunk == 0) chunk = 16384;
  const size_t big = (size_t)P->glwe_dim * P->poly_size + 1;
  // per stage (2 stages): input chunk + output chunk + ids + KS workspace
  const size_t per = round_up(chunk * big * 8, 256) * 2 + round_up(chunk * 4, 256) +
                     silenzio_pbs_workspace_bytes(P, chunk);
  return 2 * per;
}

int silenzio_pbs_batch_host(const uint64_t *in_h, const uint32_t *ids_h, const uint64_t *luts, uint32_t num_luts,
                            const void *fbsk, const uint64_t *ksk, uint64_t *out_h, size_t count, size_t chunk,
                            const silenzio_params *P, void *workspace, void *stream) {
  SZ_RANGE("pbs_batch_host");
  int st = check_params(P);
  if (st) return st;
  if (count == 0) return SILENZIO_OK;
  if (!in_h || !out_h || !luts || !fbsk || !ksk) return SILENZIO_ERR_NULL_POINTER;
  if (!workspace) return SILENZIO_ERR_WORKSPACE;
  if (chunk == 0) chunk = 16384;
  const size_t big = (size_t)P->glwe_dim * P->poly_size + 1;
  const size_t in_b = round_up(chunk * big * 8, 256), id_b = round_up(chunk * 4, 256);
  const size_t ws_b = silenzio_pbs_workspace_bytes(P, chunk);
  const size_t per = in_b * 2 + id_b + ws_b;
  cudaStream_t s[2] = {nullptr, nullptr};
  if (cudaStreamCreateWithFlags(&s[0], cudaStreamNonBlocking) != cudaSuccess) return SILENZIO_ERR_CUDA;
  if (cudaStreamCreateWithFlags(&s[1], cudaStreamNonBlocking) != cudaSuccess) {
    cudaStreamDestroy(s[0]);
    return SILENZIO_ERR_CUDA;
  }
  int rc = SILENZIO_OK;
  // The internal streams start after everything already queued on the
  // caller's stream (keys, LUTs or workspace written there, or memory the
  // caching allocator recycled), and the caller's stream is ordered after
  // the last internal chunk before returning.
  cudaEvent_t ready = nullptr;
  if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(ready, sz_stream(stream)) != cudaSuccess ||
      cudaStreamWaitEvent(s[0], ready, 0) != cudaSuccess || cudaStreamWaitEvent(s[1], ready, 0) != cudaSuccess)
    rc = SILENZIO_ERR_CUDA;
  // Two stages alternate; each chunk: H2D in, PBS, D2H out on its stage's
  // stream, so chunk c+1's copies overlap chunk c's compute.
  for (size_t c0 = 0, it = 0; c0 < count && rc == SILENZIO_OK; c0 += chunk, it++) {
    const int sidx = (int)(it & 1);
    const size_t cnt = (count - c0 < chunk) ? count - c0 : chunk;
    unsigned char *base = reinterpret_cast<unsigned char *>(workspace) + sidx * per;
    u64 *d_in = reinterpret_cast<u64 *>(base);
    u64 *d_out = reinterpret_cast<u64 *>(base + in_b);
    u32 *d_ids = reinterpret_cast<u32 *>(base + 2 * in_b);
    void *ws = base + 2 * in_b + id_b;
    if (cudaMemcpyAsync(d_in, in_h + c0 * big, cnt * big * 8, cudaMemcpyHostToDevice, s[sidx]) != cudaSuccess) {
      rc = SILENZIO_ERR_CUDA;
      break;
    }
    if (ids_h && cudaMemcpyAsync(d_ids, ids_h + c0, cnt * 4, cudaMemcpyHostToDevice, s[sidx]) != cudaSuccess) {
      rc = SILENZIO_ERR_CUDA;
      break;
    }
    rc = silenzio_pbs_batch(d_in, ids_h ? d_ids : nullptr, luts, num_luts, fbsk, ksk, d_out, cnt, P, ws, s[sidx]);
    if (rc) break;
    if (cudaMemcpyAsync(out_h + c0 * big, d_out, cnt * big * 8, cudaMemcpyDeviceToHost, s[sidx]) != cudaSuccess)
      rc = SILENZIO_ERR_CUDA;
  }
  for (int i = 0; i < 2; i++) {
    if (cudaStreamSynchronize(s[i]) != cudaSuccess) rc = SILENZIO_ERR_CUDA;
    cudaStreamDestroy(s[i]);
  }
  if (ready) cudaEventDestroy(ready);
  return rc;
}

int silenzio_lwe_linear_batch(const uint64_t *in, const uint32_t *idx, const int64_t *coef, const uint64_t *cst,
                              uint32_t terms, uint32_t dim, size_t count, uint64_t *out, void *stream) {
  SZ_RANGE("lwe_linear_batch");
  if (count == 0) return SILENZIO_OK;
  if (!in || !idx || !coef || !out) return SILENZIO_ERR_NULL_POINTER;
  if (terms == 0 || dim == 0) return SILENZIO_ERR_INVALID_PARAM;
  if (count > (1ull << 31)) return SILENZIO_ERR_COUNT;
  return launch_lwe_linear(in, idx, reinterpret_cast<const i64 *>(coef), cst, (int)terms, (int)dim, count, out,
                           sz_stream(stream));
}

int silenzio_build_testpoly(const uint64_t *tables, uint32_t num, uint32_t p, uint32_t N, uint64_t *polys,
                            void *stream) {
  if (!tables || !polys) return SILENZIO_ERR_NULL_POINTER;
  if (num == 0 || !is_pow2(N) || p > 16 || (N >> p) < 2) return SILENZIO_ERR_INVALID_PARAM;
  return launch_testpoly(tables, (int)num, (int)p, (int)N, polys, sz_stream(stream));
}

int silenzio_lwe_encrypt_batch(const uint64_t *mask, const int64_t *noise, const uint64_t *pt, const uint64_t *key,
                               uint32_t dim, size_t count, uint64_t *out, void *stream) {
  if (count == 0) return SILENZIO_OK;
  if (!mask || !noise || !pt || !key || !out) return SILENZIO_ERR_NULL_POINTER;
  if (dim == 0) return SILENZIO_ERR_INVALID_PARAM;
  return launch_lwe_encrypt(mask, reinterpret_cast<const i64 *>(noise), pt, key, (int)dim, count, out,
                            sz_stream(stream));
}

int silenzio_lwe_phase_batch(const uint64_t *ct, const uint64_t *key, uint32_t dim, size_t count, uint64_t *phase,
                             void *stream) {
  if (count == 0) return SILENZIO_OK;
  if (!ct || !key || !phase) return SILENZIO_ERR_NULL_POINTER;
  if (dim == 0) return SILENZIO_ERR_INVALID_PARAM;
  return launch_lwe_phase(ct, key, (int)dim, count, phase, sz_stream(stream));
}

size_t silenzio_bsk_generate_workspace_bytes(const silenzio_params *P) {
  if (check_params(P) != SILENZIO_OK) return 0;
  return P->poly_size == 32768 ? glwe_body_huge_ws_bytes() : 0;
}

int silenzio_bsk_generate(const uint64_t *lwe_key, const uint64_t *glwe_key, const uint64_t *mask,
                          const int64_t *noise, uint64_t *bsk, const silenzio_params *P, void *workspace,
                          void *stream) {
  int st = check_params(P);
  if (st) return st;
  if (!lwe_key || !glwe_key || !mask || !noise || !bsk) return SILENZIO_ERR_NULL_POINTER;
  if (P->poly_size == 32768) {
    if (P->glwe_dim != 1) return SILENZIO_ERR_UNSUPPORTED;
    return launch_bsk_generate_huge(lwe_key, glwe_key, mask, reinterpret_cast<const i64 *>(noise), bsk,
                                    (int)P->lwe_dim, (int)P->poly_size, (int)P->pbs_base_log, (int)P->pbs_level,
                                    workspace, sz_stream(stream));
  }
  return launch_bsk_generate(lwe_key, glwe_key, mask, reinterpret_cast<const i64 *>(noise), bsk, (int)P->lwe_dim,
                             (int)P->glwe_dim, (int)P->poly_size, (int)P->pbs_base_log, (int)P->pbs_level,
                             sz_stream(stream));
}

int silenzio_ksk_generate(const uint64_t *in_key, const uint64_t *lwe_key, const uint64_t *mask, const int64_t *noise,
                          uint64_t *ksk, uint32_t in_dim, uint32_t n, uint32_t base_log, uint32_t level, void *stream) {
  if (!in_key || !lwe_key || !mask || !noise || !ksk) return SILENZIO_ERR_NULL_POINTER;
  if (in_dim == 0 || n == 0 || base_log == 0 || level == 0 || base_log * level > 64) return SILENZIO_ERR_INVALID_PARAM;
  return launch_ksk_generate(in_key, lwe_key, mask, reinterpret_cast<const i64 *>(noise), ksk, (int)in_dim, (int)n,
                             (int)base_log, (int)level, sz_stream(stream));
}

}  // extern "C"
