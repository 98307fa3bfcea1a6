// gadgets_shift.cu -- silenzio_shift2msbs_pm: the whole Shift2MSBs+- gadget
// (Alg. 4, with Alg. 3 Shift2MSBs+) behind one
// C-ABI call, composed from the config-4 drivers (DESIGN.md §6b', §6d):
//   digits = RNS2MRNS(x)                                   (stream A)
//   e, |x| = Sign_(-1,1,1) / abs;  RNS2MRNS(|x|);  bit lengths + block max
//                                                          (stream B, concurrently)
//   Y, maxBit = 8-bit MRNS digit combine (set B) of the top digit of x, the
//               digits of |x| and the block maxima          (stream A, after both)
// The two chains are independent; each driver blocks on its own stream, so the
// |x| chain runs in a second host thread on a second stream. Every ciphertext
// sees exactly the operations of the sequential composition.
#include <thread>

#include "common.cuh"
#include "nvtx.cuh"

extern "C" {
size_t silenzio_gadget_workspace_bytes(const silenzio_params *, uint32_t, size_t);
size_t silenzio_mrns_combine_workspace_bytes(const silenzio_params *, const silenzio_params *, uint32_t, size_t);
int silenzio_rns2mrns(const uint64_t *, const uint32_t *, uint32_t, size_t, uint64_t *, const void *, const uint64_t *,
                      const silenzio_params *, void *, size_t, void *);
int silenzio_rns_sign_abs(const uint64_t *, const uint32_t *, uint32_t, size_t, uint64_t *, uint64_t *, const void *,
                          const uint64_t *, const silenzio_params *, void *, size_t, void *);
int silenzio_mrns_bitlen_max(const uint64_t *, uint32_t, size_t, uint64_t *, uint64_t *, const void *,
                             const uint64_t *, const silenzio_params *, void *, size_t, void *);
int silenzio_mrns_digit_combine(const uint64_t *, const uint64_t *, const uint64_t *, uint32_t, size_t, uint32_t,
                                uint32_t, uint32_t, uint64_t *, uint64_t *, const void *, const uint64_t *,
                                const silenzio_params *, const void *, const silenzio_params *, const uint64_t *,
                                const silenzio_params *, const uint64_t *, const silenzio_params *, void *, size_t,
                                void *);
}

namespace {
size_t rup256(size_t x) { return (x + 255) / 256 * 256; }
size_t ctw(const silenzio_params *P) { return (size_t)P->glwe_dim * P->poly_size + 1; }
}  // namespace

extern "C" {

size_t silenzio_shift2msbs_workspace_bytes(const silenzio_params *pa, const silenzio_params *pb, uint32_t k,
                                           size_t count) {
  if (!pa || !pb || k < 1) return 0;
  const size_t kc = rup256((size_t)k * count * ctw(pa) * 8);
  const size_t g = silenzio_gadget_workspace_bytes(pa, k, count);
  // digits, |x|, digits of |x|, bit lengths [k][count]; sign [count]; maxima [k];
  // two gadget workspaces (one per chain); the combine workspace
  return 4 * kc + rup256(count * ctw(pa) * 8) + rup256((size_t)k * ctw(pa) * 8) + 2 * rup256(g) +
         silenzio_mrns_combine_workspace_bytes(pa, pb, k, count) + 4096;
}

int silenzio_shift2msbs_pm(const uint64_t *residues, const uint32_t *moduli_host, uint32_t k, size_t count,
                           uint32_t w, uint32_t gamma, uint64_t *out, uint64_t *maxbit_out, const void *fbsk_a,
                           const uint64_t *ksk_a, const silenzio_params *pa, const void *fbsk_b,
                           const silenzio_params *pb, const uint64_t *ksk_ab, const silenzio_params *pab,
                           const uint64_t *ksk_ba, const silenzio_params *pba, void *workspace,
                           size_t workspace_bytes, void *stream) {
  SZ_RANGE("shift2msbs_pm");
  if (!residues || !moduli_host || !out || !maxbit_out || !fbsk_a || !ksk_a || !pa || !fbsk_b || !pb || !ksk_ab ||
      !pab || !ksk_ba || !pba)
    return SILENZIO_ERR_NULL_POINTER;
  if (k < 1) return SILENZIO_ERR_COUNT;
  if (!workspace || workspace_bytes < silenzio_shift2msbs_workspace_bytes(pa, pb, k, count))
    return SILENZIO_ERR_WORKSPACE;
  if (count == 0) return SILENZIO_OK;
  const size_t cw = ctw(pa);
  const size_t kc = rup256((size_t)k * count * cw * 8);
  const size_t g = silenzio_gadget_workspace_bytes(pa, k, count);
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  u64 *digits = reinterpret_cast<u64 *>(p);
  p += kc;
  u64 *absr = reinterpret_cast<u64 *>(p);
  p += kc;
  u64 *dabs = reinterpret_cast<u64 *>(p);
  p += kc;
  u64 *bl = reinterpret_cast<u64 *>(p);
  p += kc;
  u64 *sign = reinterpret_cast<u64 *>(p);
  p += rup256(count * cw * 8);
  u64 *mx = reinterpret_cast<u64 *>(p);
  p += rup256((size_t)k * cw * 8);
  void *ws_a = p;
  p += rup256(g);
  void *ws_b = p;
  p += rup256(g);
  void *ws_c = p;
  const size_t ws_c_bytes = silenzio_mrns_combine_workspace_bytes(pa, pb, k, count);

  cudaStream_t sa = sz_stream(stream);
  cudaStream_t sb = nullptr;
  cudaEvent_t ready = nullptr;
  SZ_CUDA_OK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
  // the second stream and its event are released on every return path below
  auto finish = [&](int code) {
    if (sb) cudaStreamSynchronize(sb);
    if (ready) cudaEventDestroy(ready);
    cudaStreamDestroy(sb);
    return code;
  };
  if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess) return finish(SILENZIO_ERR_CUDA);
  // stream B starts after everything already queued on the caller's stream
  if (cudaEventRecord(ready, sa) != cudaSuccess || cudaStreamWaitEvent(sb, ready, 0) != cudaSuccess)
    return finish(SILENZIO_ERR_CUDA);
  int rc_b = SILENZIO_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  std::thread chain_b([&] {
    cudaSetDevice(dev);
    rc_b = silenzio_rns_sign_abs(residues, moduli_host, k, count, sign, absr, fbsk_a, ksk_a, pa, ws_b, g, sb);
    if (!rc_b) rc_b = silenzio_rns2mrns(absr, moduli_host, k, count, dabs, fbsk_a, ksk_a, pa, ws_b, g, sb);
    if (!rc_b) rc_b = silenzio_mrns_bitlen_max(dabs, k, count, bl, mx, fbsk_a, ksk_a, pa, ws_b, g, sb);
  });
  int rc = silenzio_rns2mrns(residues, moduli_host, k, count, digits, fbsk_a, ksk_a, pa, ws_a, g, sa);
  chain_b.join();
  if (!rc) rc = rc_b;
  if (!rc && (cudaEventRecord(ready, sb) != cudaSuccess || cudaStreamWaitEvent(sa, ready, 0) != cudaSuccess))
    rc = SILENZIO_ERR_CUDA;
  if (!rc) {
    rc = silenzio_mrns_digit_combine(digits + (size_t)(k - 1) * count * cw, dabs, mx, k, count, moduli_host[k - 1],
                                     w, gamma, out, maxbit_out, fbsk_a, ksk_a, pa, fbsk_b, pb, ksk_ab, pab, ksk_ba,
                                     pba, ws_c, ws_c_bytes, sa);
  }
  return finish(rc);
}

}  // extern "C"
