// gadget_util.cuh -- host-side helpers shared by the gadget drivers: LUT
// tables for 16-value windows of Z_32 (SURVEY toolbox T1), staging of index
// arrays and chunked PBS calls. Every ciphertext operation runs in a kernel.
#pragma once
#include <cstring>
#include <vector>

#include "common.cuh"

extern "C" {
int silenzio_pbs_batch(const uint64_t *, const uint32_t *, const uint64_t *, uint32_t, const void *,
                       const uint64_t *, uint64_t *, size_t, const silenzio_params *, void *, void *);
int silenzio_lwe_linear_batch(const uint64_t *, const uint32_t *, const int64_t *, const uint64_t *, uint32_t,
                              uint32_t, size_t, uint64_t *, void *);
int silenzio_build_testpoly(const uint64_t *, uint32_t, uint32_t, uint32_t, uint64_t *, void *);
int silenzio_pbs_linear_batch(const uint64_t *, const uint32_t *, const int64_t *, const uint64_t *, uint32_t,
                              const uint32_t *, const uint64_t *, uint32_t, const void *, const void *, uint64_t *,
                              size_t, const silenzio_params *, void *, void *);
size_t silenzio_pbs_linear_workspace_bytes(const silenzio_params *, size_t);
size_t silenzio_ksk_planes_bytes(const silenzio_params *);
int silenzio_ksk_to_planes(const uint64_t *, void *, const silenzio_params *, void *);
size_t silenzio_pbs_workspace_bytes(const silenzio_params *, size_t);
}

namespace sz {
// trace.cu: sampled-PBS recording for oracle replays (no-op unless a trace is active)
bool trace_active(int kind);
void trace_pbs(int kind, const u64 *in, size_t in_words, const u64 *out, size_t out_words, const u64 *luts,
               size_t lut_words, const u32 *ids_host, size_t count, cudaStream_t st);
int launch_lwe_axpy3(u64 *out, const u64 *A, i64 ca, const u64 *B, i64 cb, const u64 *C, i64 cc, u64 cst,
                     size_t count, int dim, cudaStream_t st);
int launch_lwe_axpy_bcast(u64 *out, const u64 *A, i64 ca, const u64 *B, i64 cb, const u64 *C, i64 cc, size_t count,
                          int dim, cudaStream_t st);
}

namespace szg {
using namespace sz;
constexpr int kP = 4;                   // message bits (set A)
constexpr u64 kDelta = 1ull << 59;      // 2^(64 - (p+1))
constexpr u64 kDelta16 = 1ull << 60;    // scale of the native mod-16 channel

inline u64 enc(i64 v, u64 scale) { return (u64)v * scale; }

inline int inv4(int m) {
  for (int x = 1; x < m; x++)
    if ((4 * x) % m == 1) return x;
  return -1;
}

inline int pmod(long v, int m) { return (int)(((v % m) + m) % m); }

// 16-entry tables of torus values for window [w0, w0 + 16) of Z_32 (SURVEY
// toolbox T1): T[x mod 16] = f(x) for x in [0,16); inputs x in [16,32) return
// -T[x - 16], so a negative input x in [-8,0) needs T[x + 16] = -f(x).
template <class F>
inline std::vector<u64> table_window(int w0, F f) {
  std::vector<u64> T(16, 0);
  for (int x = w0; x < w0 + 16; x++) {
    const int xm = ((x % 32) + 32) % 32;
    if (xm < 16) T[xm] = f(x);
    else T[xm - 16] = (u64)0 - f(x);
  }
  return T;
}

struct Dev {
  cudaStream_t st;
  const silenzio_params *P;
  const void *fbsk;
  const u64 *ksk;
  const void *planes = nullptr;  // KSK byte planes prepared once per driver call (null: silenzio_pbs_batch per lookup)
  size_t big;  // k N + 1
  // scratch
  u64 *luts;           // [kMaxLuts][N]
  u64 *tables;         // [kMaxLuts][16]
  u32 *idx;            // linear-op index scratch
  i64 *coef;
  u64 *cst;
  u32 *ids;            // lut ids
  void *pbs_ws;
  size_t idx_cap, ids_cap, pbs_cap;
};

constexpr int kMaxLuts = 4;

inline int upload_luts(Dev &D, const std::vector<std::vector<u64>> &tabs) {
  std::vector<u64> flat;
  for (auto &t : tabs) flat.insert(flat.end(), t.begin(), t.end());
  SZ_CUDA_OK(cudaMemcpyAsync(D.tables, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, D.st));
  return silenzio_build_testpoly(D.tables, (u32)tabs.size(), kP, D.P->poly_size, D.luts, D.st);
}

// out[i] = sum_t coef[i][t] * in[idx[i][t]] + cst[i]
inline int linear(Dev &D, const u64 *in, u64 *out, size_t count, int terms, const std::vector<u32> &idx,
           const std::vector<i64> &coef, const std::vector<u64> &cst) {
  if (count == 0) return SILENZIO_OK;
  if (count * terms > D.idx_cap || count > D.idx_cap) return SILENZIO_ERR_WORKSPACE;
  SZ_CUDA_OK(cudaMemcpyAsync(D.idx, idx.data(), count * terms * 4, cudaMemcpyHostToDevice, D.st));
  SZ_CUDA_OK(cudaMemcpyAsync(D.coef, coef.data(), count * terms * 8, cudaMemcpyHostToDevice, D.st));
  SZ_CUDA_OK(cudaMemcpyAsync(D.cst, cst.data(), count * 8, cudaMemcpyHostToDevice, D.st));
  // the staging buffers are reused by the next call: keep host vectors alive
  // until the copies have been consumed
  SZ_CUDA_OK(cudaStreamSynchronize(D.st));
  return silenzio_lwe_linear_batch(in, D.idx, D.coef, D.cst, (u32)terms, (u32)(D.big - 1), count, out, D.st);
}

// PBS of `count` ciphertexts; lut id per ciphertext (empty = all 0)
inline int lookup(Dev &D, const u64 *in, u64 *out, size_t count, const std::vector<u32> &ids, u32 num_luts) {
  if (count == 0) return SILENZIO_OK;
  const size_t chunk = D.pbs_cap;
  for (size_t c0 = 0; c0 < count; c0 += chunk) {
    const size_t cnt = count - c0 < chunk ? count - c0 : chunk;
    const u32 *idp = nullptr;
    if (!ids.empty()) {
      if (cnt > D.ids_cap) return SILENZIO_ERR_WORKSPACE;
      SZ_CUDA_OK(cudaMemcpyAsync(D.ids, ids.data() + c0, cnt * 4, cudaMemcpyHostToDevice, D.st));
      SZ_CUDA_OK(cudaStreamSynchronize(D.st));
      idp = D.ids;
    }
    int rc = D.planes ? silenzio_pbs_linear_batch(in + c0 * D.big, nullptr, nullptr, nullptr, 1, idp, D.luts, num_luts,
                                                  D.fbsk, D.planes, out + c0 * D.big, cnt, D.P, D.pbs_ws, D.st)
                      : silenzio_pbs_batch(in + c0 * D.big, idp, D.luts, num_luts, D.fbsk, D.ksk, out + c0 * D.big,
                                           cnt, D.P, D.pbs_ws, D.st);
    if (rc) return rc;
    if (trace_active(0))
      trace_pbs(0, in + c0 * D.big, D.big, out + c0 * D.big, D.big, D.luts, D.P->poly_size,
                ids.empty() ? nullptr : ids.data() + c0, cnt, D.st);
  }
  return SILENZIO_OK;
}


// out[i] = PBS(sum_t coef[i][t] * in[idx[i][t]] + cst[i]; luts[ids[i]]): the linear op runs inside the
// keyswitch (silenzio_pbs_linear_batch, needs D.planes). `trace_tmp` (count ciphertexts, may be null)
// receives the combinations only while a PBS trace is recording them.
inline int linear_lookup(Dev &D, const u64 *in, u64 *out, size_t count, int terms, const std::vector<u32> &idx,
                         const std::vector<i64> &coef, const std::vector<u64> &cst, const std::vector<u32> &ids,
                         u32 num_luts, u64 *trace_tmp) {
  if (count == 0) return SILENZIO_OK;
  if (!D.planes || (trace_active(0) && trace_tmp)) {  // unfused: the trace records the PBS inputs
    if (!trace_tmp) return SILENZIO_ERR_WORKSPACE;
    int rc = linear(D, in, trace_tmp, count, terms, idx, coef, cst);
    if (rc) return rc;
    return lookup(D, trace_tmp, out, count, ids, num_luts);
  }
  if (count * terms > D.idx_cap || count > D.idx_cap) return SILENZIO_ERR_WORKSPACE;
  SZ_CUDA_OK(cudaMemcpyAsync(D.idx, idx.data(), count * terms * 4, cudaMemcpyHostToDevice, D.st));
  SZ_CUDA_OK(cudaMemcpyAsync(D.coef, coef.data(), count * terms * 8, cudaMemcpyHostToDevice, D.st));
  SZ_CUDA_OK(cudaMemcpyAsync(D.cst, cst.data(), count * 8, cudaMemcpyHostToDevice, D.st));
  const size_t chunk = D.pbs_cap;
  for (size_t c0 = 0; c0 < count; c0 += chunk) {
    const size_t cnt = count - c0 < chunk ? count - c0 : chunk;
    const u32 *idp = nullptr;
    if (!ids.empty()) {
      if (cnt > D.ids_cap) return SILENZIO_ERR_WORKSPACE;
      SZ_CUDA_OK(cudaMemcpyAsync(D.ids, ids.data() + c0, cnt * 4, cudaMemcpyHostToDevice, D.st));
      idp = D.ids;
    }
    int rc = silenzio_pbs_linear_batch(in, D.idx + c0 * terms, D.coef + c0 * terms, D.cst + c0, (u32)terms, idp, D.luts,
                                       num_luts, D.fbsk, D.planes, out + c0 * D.big, cnt, D.P, D.pbs_ws, D.st);
    if (rc) return rc;
  }
  // the staging buffers are reused by the next call and the host vectors die with the caller
  SZ_CUDA_OK(cudaStreamSynchronize(D.st));
  return SILENZIO_OK;
}

// out[e] = ca A[e] + cb B[e] + cc C[e] + cst (elementwise over `count` ciphertexts; null arrays skipped)
inline int axpy3(Dev &D, u64 *out, const u64 *A, i64 ca, const u64 *B, i64 cb, const u64 *C, i64 cc, u64 cst,
                 size_t count) {
  return launch_lwe_axpy3(out, A, ca, B, cb, C, cc, cst, count, (int)(D.big - 1), D.st);
}

// carve the scratch a Dev needs out of a workspace pointer (advances p)
inline void dev_init(Dev &D, unsigned char *&p, const silenzio_params *P, const void *fbsk, const u64 *ksk,
                     cudaStream_t st, size_t idx_cap) {
  auto carve = [&](size_t bytes) {
    unsigned char *r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  D.st = st;
  D.P = P;
  D.fbsk = fbsk;
  D.ksk = ksk;
  D.big = (size_t)P->glwe_dim * P->poly_size + 1;
  D.idx_cap = idx_cap;
  D.idx = reinterpret_cast<u32 *>(carve(idx_cap * 4));
  D.coef = reinterpret_cast<i64 *>(carve(idx_cap * 8));
  D.cst = reinterpret_cast<u64 *>(carve(idx_cap * 8));
  D.pbs_cap = 65536;
  D.ids_cap = D.pbs_cap;
  D.ids = reinterpret_cast<u32 *>(carve(D.ids_cap * 4));
  D.tables = reinterpret_cast<u64 *>(carve(kMaxLuts * 16 * 8));
  D.luts = reinterpret_cast<u64 *>(carve((size_t)kMaxLuts * P->poly_size * 8));
  D.pbs_ws = carve(silenzio_pbs_workspace_bytes(P, D.pbs_cap));
}

inline size_t dev_bytes(const silenzio_params *P, size_t idx_cap) {
  return idx_cap * (4 + 8 + 8) + 65536 * 4 + kMaxLuts * (P->poly_size + 16) * 8 +
         silenzio_pbs_workspace_bytes(P, 65536) + 8 * 256;
}

}  // namespace szg
