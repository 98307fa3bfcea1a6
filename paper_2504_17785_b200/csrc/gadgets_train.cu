// gadgets_train.cu -- the 4-bit gadgets one encrypted training step (PAPER.md
// Alg. 6) adds to the config-3/4 drivers,
// at parameter set A (plaintext Z_32, Delta = 2^59). Thin drivers: they build
// LUT tables and sequence linear LWE ops and PBS calls; every ciphertext
// operation runs in a kernel. Schedules and readings: DESIGN.md §6b'' (R23-R26).
//   silenzio_channel16      the m = 16 residue Matmul^RNS keeps at 2^60 -> Delta
//   silenzio_rns_sign3      Sign^RNS_(-1,0,1) (zero test P:313)
//   silenzio_relu_cap       ReLU_x
//   silenzio_relu_mask      error sign times the ReLU_x derivative (R25)
//   silenzio_weight_update  clip(W - G) for G in {-1, 0, 1} (Alg. 6 last line, R23)
#include "gadget_util.cuh"
#include "nvtx.cuh"

extern "C" int silenzio_rns2mrns(const uint64_t *, const uint32_t *, uint32_t, size_t, uint64_t *, const void *,
                                 const uint64_t *, const silenzio_params *, void *, size_t, void *);
extern "C" size_t silenzio_gadget_workspace_bytes(const silenzio_params *, uint32_t, size_t);

using namespace szg;

namespace {

size_t ctb(const silenzio_params *P) { return ((size_t)P->glwe_dim * P->poly_size + 1) * 8; }
size_t rup(size_t x) { return (x + 255) / 256 * 256; }
constexpr u64 kHalfDelta = kDelta >> 1;

// a single-table PBS of `count` ciphertexts
int lut1(Dev &D, const u64 *in, u64 *out, size_t count, const std::vector<u64> &table) {
  int rc = upload_luts(D, {table});
  if (rc) return rc;
  return lookup(D, in, out, count, {}, 1);
}

int check_common(const void *a, const void *b, const void *fbsk, const void *ksk, const silenzio_params *P,
                 void *ws, size_t ws_bytes, size_t need) {
  if (!a || !b || !fbsk || !ksk || !P) return SILENZIO_ERR_NULL_POINTER;
  if (!ws || ws_bytes < need) return SILENZIO_ERR_WORKSPACE;
  if (P->poly_size != 2048 || P->glwe_dim != 1) return SILENZIO_ERR_UNSUPPORTED;
  return SILENZIO_OK;
}

}  // namespace

extern "C" {

size_t silenzio_train_workspace_bytes(const silenzio_params *P, uint32_t k, size_t count) {
  if (!P) return 0;
  const size_t ct = ctb(P);
  const size_t kk = k < 1 ? 1 : k;
  // sign3: digits [k][count] + rns2mrns workspace + (k + 2) temporaries; others: <= 6 temporaries
  const size_t sign3 = rup(kk * count * ct) + silenzio_gadget_workspace_bytes(P, (uint32_t)kk, count) +
                       (kk + 2) * rup(count * ct);
  const size_t rest = 6 * rup(count * ct);
  return (sign3 > rest ? sign3 : rest) + dev_bytes(P, 4 * count + 64) + 4096;
}

int silenzio_channel16(const uint64_t *in, size_t count, uint64_t *out, const void *fbsk, const uint64_t *ksk,
                       const silenzio_params *P, void *workspace, size_t workspace_bytes, void *stream) {
  SZ_RANGE("channel16");
  int rc = check_common(in, out, fbsk, ksk, P, workspace, workspace_bytes, silenzio_train_workspace_bytes(P, 1, count));
  if (rc) return rc;
  if (count == 0) return SILENZIO_OK;
  const size_t cw = ctb(P) / 8;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  u64 *sp = reinterpret_cast<u64 *>(p);
  p += rup(count * cw * 8);
  u64 *x = reinterpret_cast<u64 *>(p);
  p += rup(count * cw * 8);
  u64 *hi = reinterpret_cast<u64 *>(p);
  p += 4 * rup(count * cw * 8);
  Dev D;
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  // z reads index 2r of Z_32: s' = PBS(z; -4) = -4 (r < 8) / +4 (r >= 8, negacyclic)
  if ((rc = lut1(D, in, sp, count, table_window(0, [](int) { return (u64)0 - 4 * kDelta; })))) return rc;
  // x = z - 2 s' - 8 = 2 (r mod 8); r = PBS(x; x/2 + 4) + s' (toolbox T4, e = [r >= 8])
  if ((rc = axpy3(D, x, in, 1, sp, -2, nullptr, 0, (u64)0 - 8 * kDelta, count))) return rc;
  if ((rc = lut1(D, x, hi, count, table_window(0, [](int v) { return enc(v / 2 + 4, kDelta); })))) return rc;
  return axpy3(D, out, hi, 1, sp, 1, nullptr, 0, 0, count);
}

int silenzio_rns_sign3(const uint64_t *residues, const uint32_t *moduli_host, uint32_t k, size_t count,
                       uint64_t *out, const void *fbsk, const uint64_t *ksk, const silenzio_params *P,
                       void *workspace, size_t workspace_bytes, void *stream) {
  SZ_RANGE("rns_sign3");
  int rc = check_common(residues, out, fbsk, ksk, P, workspace, workspace_bytes,
                        silenzio_train_workspace_bytes(P, k, count));
  if (rc) return rc;
  if (!moduli_host) return SILENZIO_ERR_NULL_POINTER;
  if (k < 1 || k > 7) return SILENZIO_ERR_WINDOW;                       // packed sum + 8 [neg] < 16
  if (moduli_host[k - 1] != 16) return SILENZIO_ERR_WINDOW;             // top radix 16: neg = [top >= 8]
  if (count == 0) return SILENZIO_OK;
  const size_t cw = ctb(P) / 8;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  u64 *digits = reinterpret_cast<u64 *>(p);
  p += rup((size_t)k * count * cw * 8);
  void *r2m_ws = p;
  const size_t r2m_bytes = silenzio_gadget_workspace_bytes(P, k, count);
  p += r2m_bytes;
  u64 *nz = reinterpret_cast<u64 *>(p);  // [k][count] indicators [d_i != 0]
  p += (size_t)k * rup(count * cw * 8);
  u64 *packed = reinterpret_cast<u64 *>(p);
  p += 2 * rup(count * cw * 8);
  Dev D;
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  // MRNS digits (Alg. 1), least significant first
  if ((rc = silenzio_rns2mrns(residues, moduli_host, k, count, digits, fbsk, ksk, P, r2m_ws, r2m_bytes, D.st)))
    return rc;
  // [d_i != 0] for every digit (one batch: the digit slabs are consecutive)
  if ((rc = lut1(D, digits, nz, (size_t)k * count, table_window(0, [](int v) { return enc(v ? 1 : 0, kDelta); }))))
    return rc;
  // packed = 8 [top digit >= 8] + sum_i [d_i != 0], in [0, 15]
  if ((rc = lut1(D, digits + (size_t)(k - 1) * count * cw, packed, count,
                 table_window(0, [](int v) { return enc(v >= 8 ? 8 : 0, kDelta); }))))
    return rc;
  for (uint32_t i = 0; i < k; i++)
    if ((rc = axpy3(D, packed, packed, 1, nz + (size_t)i * count * cw, 1, nullptr, 0, 0, count))) return rc;
  // 0 if no digit is nonzero, else -1 (negative) / +1
  return lut1(D, packed, out, count,
              table_window(0, [](int v) { return v % 8 == 0 ? (u64)0 : (v >= 8 ? (u64)0 - kDelta : kDelta); }));
}

int silenzio_relu_cap(const uint64_t *in, size_t count, int32_t cap, uint64_t *out, const void *fbsk,
                      const uint64_t *ksk, const silenzio_params *P, void *workspace, size_t workspace_bytes,
                      void *stream) {
  SZ_RANGE("relu_cap");
  int rc = check_common(in, out, fbsk, ksk, P, workspace, workspace_bytes, silenzio_train_workspace_bytes(P, 1, count));
  if (rc) return rc;
  if (cap < 0 || cap > 7) return SILENZIO_ERR_WINDOW;
  if (count == 0) return SILENZIO_OK;
  Dev D;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace) + 6 * rup(count * ctb(P));
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  return lut1(D, in, out, count,
              table_window(-8, [cap](int v) { return enc(v < 0 ? 0 : (v > cap ? cap : v), kDelta); }));
}

int silenzio_relu_mask(const uint64_t *e, const uint64_t *s, size_t count, int32_t cap, uint64_t *out,
                       const void *fbsk, const uint64_t *ksk, const silenzio_params *P, void *workspace,
                       size_t workspace_bytes, void *stream) {
  SZ_RANGE("relu_mask");
  int rc = check_common(e, s, fbsk, ksk, P, workspace, workspace_bytes, silenzio_train_workspace_bytes(P, 1, count));
  if (rc) return rc;
  if (!out) return SILENZIO_ERR_NULL_POINTER;
  if (cap < 0 || cap > 7) return SILENZIO_ERR_WINDOW;
  if (count == 0) return SILENZIO_OK;
  const size_t cw = ctb(P) / 8;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  u64 *m4 = reinterpret_cast<u64 *>(p);
  p += rup(count * cw * 8);
  u64 *packed = reinterpret_cast<u64 *>(p);
  p += 5 * rup(count * cw * 8);
  Dev D;
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  // 4 [0 < s < cap]; packed = (e + 1) + 4 [mask] in [0, 6]; out = packed - 5 if packed >= 4 else 0
  if ((rc = lut1(D, s, m4, count, table_window(-8, [cap](int v) { return enc(v > 0 && v < cap ? 4 : 0, kDelta); }))))
    return rc;
  if ((rc = axpy3(D, packed, e, 1, m4, 1, nullptr, 0, kDelta, count))) return rc;
  return lut1(D, packed, out, count, table_window(0, [](int v) { return enc(v >= 4 ? v - 5 : 0, kDelta); }));
}

int silenzio_weight_update(const uint64_t *w, const uint64_t *g, size_t count, int32_t wmin, int32_t wmax,
                           uint64_t *out, const void *fbsk, const uint64_t *ksk, const silenzio_params *P,
                           void *workspace, size_t workspace_bytes, void *stream) {
  SZ_RANGE("weight_update");
  int rc = check_common(w, g, fbsk, ksk, P, workspace, workspace_bytes, silenzio_train_workspace_bytes(P, 1, count));
  if (rc) return rc;
  if (!out) return SILENZIO_ERR_NULL_POINTER;
  if (wmin < -8 || wmax > 7 || wmin >= wmax) return SILENZIO_ERR_WINDOW;
  if (count == 0) return SILENZIO_OK;
  const size_t cw = ctb(P) / 8;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  u64 *T[6];
  for (int i = 0; i < 6; i++) {
    T[i] = reinterpret_cast<u64 *>(p);
    p += rup(count * cw * 8);
  }
  Dev D;
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  // clip(W - G) = W - e+ [W != wmin] + e- [W != wmax], e+- = [G = +-1]; each
  // product a bit x 4-bit T4: f(e, W) = PBS(W; (g0+g1)/2) + PBS(16 e + W; (g0-g1)/2)
  u64 *ep = T[0], *em = T[1], *s = T[2], *t = T[3], *u = T[4];
  if ((rc = lut1(D, g, ep, count, table_window(-8, [](int v) { return enc(v == 1 ? 1 : 0, kDelta); })))) return rc;
  if ((rc = lut1(D, g, em, count, table_window(-8, [](int v) { return enc(v == -1 ? 1 : 0, kDelta); })))) return rc;
  // s = W + A1 + B1 + A2 + B2 accumulated term by term (half-step outputs, units of Delta / 2)
  if ((rc = lut1(D, w, t, count, table_window(-8, [wmin](int v) { return (u64)0 - (u64)(v != wmin) * kHalfDelta; }))))
    return rc;
  if ((rc = axpy3(D, s, w, 1, t, 1, nullptr, 0, 0, count))) return rc;
  if ((rc = axpy3(D, u, ep, 16, w, 1, nullptr, 0, 0, count))) return rc;
  if ((rc = lut1(D, u, t, count, table_window(-8, [wmin](int v) { return (u64)(v != wmin) * kHalfDelta; }))))
    return rc;
  if ((rc = axpy3(D, s, s, 1, t, 1, nullptr, 0, 0, count))) return rc;
  if ((rc = lut1(D, w, t, count, table_window(-8, [wmax](int v) { return (u64)(v != wmax) * kHalfDelta; }))))
    return rc;
  if ((rc = axpy3(D, s, s, 1, t, 1, nullptr, 0, 0, count))) return rc;
  if ((rc = axpy3(D, u, em, 16, w, 1, nullptr, 0, 0, count))) return rc;
  if ((rc = lut1(D, u, t, count, table_window(-8, [wmax](int v) { return (u64)0 - (u64)(v != wmax) * kHalfDelta; }))))
    return rc;
  if ((rc = axpy3(D, s, s, 1, t, 1, nullptr, 0, 0, count))) return rc;
  // refreshing identity PBS: the new weights are fresh ciphertexts (R26)
  return lut1(D, s, out, count, table_window(-8, [](int v) { return enc(v, kDelta); }));
}

}  // extern "C"
