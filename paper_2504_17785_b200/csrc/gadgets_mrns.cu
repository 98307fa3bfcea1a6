// gadgets_mrns.cu -- config-4 gadget drivers at parameter set A (4-bit PBS):
//   silenzio_rns2mrns          Alg. 1 RNS2MRNS          (g4)
//   silenzio_rns_sign_abs      Sign_(-1,1,1) and |x| in RNS (l.309-323, Alg. 4 l.414-415) (g5)
//   silenzio_mrns_bitlen_max   bit length of MRNS digits + tensor-wide max (Alg. 3 step 2) (g6)
//   silenzio_int_ce_grad       IntCELossDeriv at Gamma = 4, kappa = 0 (Alg. 5, R10/R12) (g8)
// Thin drivers: they sequence linear LWE ops and PBS calls; every ciphertext
// operation runs in a kernel. Schedule: DESIGN.md §Config 4.
#include "gadget_util.cuh"

using namespace szg;

namespace {

int inv_mod(int a, int m) {
  a %= m;
  for (int x = 1; x < m; x++)
    if ((a * x) % m == 1) return x;
  return -1;
}

int bitlen(int d) {
  int b = 0;
  while (d > 0) {
    b++;
    d >>= 1;
  }
  return b;
}

long rhe(double x) { return (long)nearbyint(x); }  // round half to even (default FE_TONEAREST)

// Alg. 1 on device buffers; `out` may not alias `in`. tmp*: count ciphertexts each.
int rns2mrns_impl(Dev &D, const u64 *in, const uint32_t *moduli, int k, size_t count, u64 *out, u64 *tmp,
                  u64 *tmp2, u64 *tmp3) {
  const size_t cw = D.big;
  SZ_CUDA_OK(cudaMemcpyAsync(out, in, (size_t)k * count * cw * 8, cudaMemcpyDeviceToDevice, D.st));
  int rc;
  for (int i = 1; i < k; i++) {
    const int mp = (int)moduli[i - 1];
    const u64 *pivot = out + (size_t)(i - 1) * count * cw;
    for (int j = i; j < k; j++) {
      const int mj = (int)moduli[j];
      const int t = inv_mod(mp, mj);
      u64 *yj = out + (size_t)j * count * cw;
      // d = y_j - y_{i-1} in [-(mp-1), mj-1]
      if ((rc = axpy3(D, tmp, yj, 1, pivot, -1, nullptr, 0, 0, count))) return rc;
      if (mp + mj - 1 <= 16) {
        std::vector<std::vector<u64>> tabs = {
            table_window(-(mp - 1), [mj, t](int d) { return enc(pmod((long)d * t, mj), kDelta); })};
        if ((rc = upload_luts(D, tabs))) return rc;
        if ((rc = lookup(D, tmp, yj, count, {}, 1))) return rc;
      } else {
        // T3: u = d mod mj = d + mj Delta/2 - sign(d) mj Delta/2 ; then T1 on [0,16)
        const u64 half = (u64)mj * (kDelta >> 1);
        std::vector<std::vector<u64>> tabs = {std::vector<u64>(16, half)};
        if ((rc = upload_luts(D, tabs))) return rc;
        if ((rc = lookup(D, tmp, tmp2, count, {}, 1))) return rc;
        if ((rc = axpy3(D, tmp3, tmp, 1, tmp2, -1, nullptr, 0, half, count))) return rc;
        std::vector<std::vector<u64>> tabs2 = {
            table_window(0, [mj, t](int u) { return enc(pmod((long)u * t, mj), kDelta); })};
        if ((rc = upload_luts(D, tabs2))) return rc;
        if ((rc = lookup(D, tmp3, yj, count, {}, 1))) return rc;
      }
    }
  }
  return SILENZIO_OK;
}

int check_moduli(const uint32_t *moduli, uint32_t k) {
  for (uint32_t i = 0; i < k; i++) {
    if (moduli[i] < 2 || moduli[i] > 16) return SILENZIO_ERR_WINDOW;
    if (i > 0 && moduli[i] < moduli[i - 1]) return SILENZIO_ERR_WINDOW;  // T3 needs m_{i-1} - 1 <= m_j
  }
  return SILENZIO_OK;
}

size_t ct_bytes(const silenzio_params *P) { return ((size_t)P->glwe_dim * P->poly_size + 1) * 8; }
size_t rup(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

extern "C" {

size_t silenzio_gadget_workspace_bytes(const silenzio_params *P, uint32_t k, size_t count) {
  if (!P) return 0;
  const size_t ct = ct_bytes(P);
  // digits [k][count] + 6 temporaries of `count` + index scratch for row sums
  return rup((size_t)k * count * ct) + 6 * rup(count * ct) + dev_bytes(P, 4 * count + 64) + 4096;
}

int silenzio_rns2mrns(const uint64_t *in, const uint32_t *moduli_host, uint32_t k, size_t count, uint64_t *out,
                      const void *fbsk, const uint64_t *ksk, const silenzio_params *P, void *workspace,
                      size_t workspace_bytes, void *stream) {
  if (!in || !moduli_host || !out || !fbsk || !ksk || !P) return SILENZIO_ERR_NULL_POINTER;
  if (!workspace || workspace_bytes < silenzio_gadget_workspace_bytes(P, k, count)) return SILENZIO_ERR_WORKSPACE;
  if (P->poly_size != 2048 || k < 1) return SILENZIO_ERR_UNSUPPORTED;
  int rc = check_moduli(moduli_host, k);
  if (rc) return rc;
  if (count == 0) return SILENZIO_OK;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  const size_t ct = ct_bytes(P);
  p += rup((size_t)k * count * ct);  // (digits slot unused here)
  u64 *t0 = reinterpret_cast<u64 *>(p);
  p += rup(count * ct);
  u64 *t1 = reinterpret_cast<u64 *>(p);
  p += rup(count * ct);
  u64 *t2 = reinterpret_cast<u64 *>(p);
  p += 4 * rup(count * ct);
  Dev D;
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  return rns2mrns_impl(D, in, moduli_host, (int)k, count, out, t0, t1, t2);
}

int silenzio_rns_sign_abs(const uint64_t *in, const uint32_t *moduli_host, uint32_t k, size_t count,
                          uint64_t *sign_out, uint64_t *abs_out, const void *fbsk, const uint64_t *ksk,
                          const silenzio_params *P, void *workspace, size_t workspace_bytes, void *stream) {
  if (!in || !moduli_host || !sign_out || !abs_out || !fbsk || !ksk || !P) return SILENZIO_ERR_NULL_POINTER;
  if (!workspace || workspace_bytes < silenzio_gadget_workspace_bytes(P, k, count)) return SILENZIO_ERR_WORKSPACE;
  if (P->poly_size != 2048 || k < 1) return SILENZIO_ERR_UNSUPPORTED;
  int rc = check_moduli(moduli_host, k);
  if (rc) return rc;
  if (moduli_host[k - 1] % 2) return SILENZIO_ERR_WINDOW;  // sign needs an even top radix
  if (count == 0) return SILENZIO_OK;
  const size_t cw = ct_bytes(P) / 8;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  u64 *digits = reinterpret_cast<u64 *>(p);
  p += rup((size_t)k * count * cw * 8);
  u64 *t[6];
  for (int i = 0; i < 6; i++) {
    t[i] = reinterpret_cast<u64 *>(p);
    p += rup(count * cw * 8);
  }
  Dev D;
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  if ((rc = rns2mrns_impl(D, in, moduli_host, (int)k, count, digits, t[0], t[1], t[2]))) return rc;
  // e = [top digit >= r_k / 2]  (0 or 1 at Delta)
  const int rk = (int)moduli_host[k - 1];
  std::vector<std::vector<u64>> st = {table_window(0, [rk](int y) { return enc(2 * y >= rk ? 1 : 0, kDelta); })};
  if ((rc = upload_luts(D, st))) return rc;
  if ((rc = lookup(D, digits + (size_t)(k - 1) * count * cw, sign_out, count, {}, 1))) return rc;
  // |x| per residue with the bit x 4-bit construction (T4): g0 = x, g1 = -x mod m
  for (uint32_t j = 0; j < k; j++) {
    const int m = (int)moduli_host[j];
    const u64 *xj = in + (size_t)j * count * cw;
    const u64 hd = kDelta >> 1;  // Delta / 2
    std::vector<std::vector<u64>> ta = {table_window(0, [m, hd](int x) { return x == 0 ? (u64)0 : (u64)m * hd; })};
    if ((rc = upload_luts(D, ta))) return rc;
    if ((rc = lookup(D, xj, t[0], count, {}, 1))) return rc;                         // A
    if ((rc = axpy3(D, t[1], sign_out, 16, xj, 1, nullptr, 0, 0, count))) return rc;   // 16 e + x
    std::vector<std::vector<u64>> tb = {
        table_window(0, [m, hd](int x) { return x == 0 ? (u64)0 : (u64)(2 * x - m) * hd; })};
    if ((rc = upload_luts(D, tb))) return rc;
    if ((rc = lookup(D, t[1], t[2], count, {}, 1))) return rc;                        // B
    if ((rc = axpy3(D, abs_out + (size_t)j * count * cw, t[0], 1, t[2], 1, nullptr, 0, 0, count))) return rc;
  }
  return SILENZIO_OK;
}

int silenzio_mrns_bitlen_max(const uint64_t *digits, uint32_t k, size_t count, uint64_t *bitlen_out,
                             uint64_t *max_out, const void *fbsk, const uint64_t *ksk, const silenzio_params *P,
                             void *workspace, size_t workspace_bytes, void *stream) {
  if (!digits || !bitlen_out || !max_out || !fbsk || !ksk || !P) return SILENZIO_ERR_NULL_POINTER;
  if (!workspace || workspace_bytes < silenzio_gadget_workspace_bytes(P, k, count)) return SILENZIO_ERR_WORKSPACE;
  if (P->poly_size != 2048) return SILENZIO_ERR_UNSUPPORTED;
  if (count == 0) return SILENZIO_OK;
  const size_t cw = ct_bytes(P) / 8;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  p += rup((size_t)k * count * cw * 8);
  u64 *buf = reinterpret_cast<u64 *>(p);
  p += rup(count * cw * 8);
  u64 *tmp = reinterpret_cast<u64 *>(p);
  p += rup(count * cw * 8);
  u64 *tmp2 = reinterpret_cast<u64 *>(p);
  p += 4 * rup(count * cw * 8);
  Dev D;
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  int rc;
  std::vector<std::vector<u64>> tb = {table_window(0, [](int d) { return enc(bitlen(d), kDelta); })};
  if ((rc = upload_luts(D, tb))) return rc;
  if ((rc = lookup(D, digits, bitlen_out, (size_t)k * count, {}, 1))) return rc;
  std::vector<std::vector<u64>> trelu = {table_window(-8, [](int d) { return enc(d > 0 ? d : 0, kDelta); })};
  for (uint32_t i = 0; i < k; i++) {
    // max tree (T7): max(a, b) = b + ReLU(a - b), first half against second half
    SZ_CUDA_OK(cudaMemcpyAsync(buf, bitlen_out + (size_t)i * count * cw, count * cw * 8, cudaMemcpyDeviceToDevice, D.st));
    size_t cur = count;
    while (cur > 1) {
      const size_t half = cur / 2;
      if ((rc = axpy3(D, tmp, buf, 1, buf + half * cw, -1, nullptr, 0, 0, half))) return rc;
      if ((rc = upload_luts(D, trelu))) return rc;
      if ((rc = lookup(D, tmp, tmp2, half, {}, 1))) return rc;
      if ((rc = axpy3(D, buf, buf + half * cw, 1, tmp2, 1, nullptr, 0, 0, half))) return rc;
      if (cur & 1)
        SZ_CUDA_OK(cudaMemcpyAsync(buf + half * cw, buf + (cur - 1) * cw, cw * 8, cudaMemcpyDeviceToDevice, D.st));
      cur = half + (cur & 1);
    }
    SZ_CUDA_OK(cudaMemcpyAsync(max_out + (size_t)i * cw, buf, cw * 8, cudaMemcpyDeviceToDevice, D.st));
  }
  return SILENZIO_OK;
}

int silenzio_int_ce_grad(const uint64_t *Yhat, const uint64_t *Y, uint32_t a, uint32_t b, uint64_t *out,
                         const void *fbsk, const uint64_t *ksk, const silenzio_params *P, void *workspace,
                         size_t workspace_bytes, void *stream) {
  if (!Yhat || !Y || !out || !fbsk || !ksk || !P) return SILENZIO_ERR_NULL_POINTER;
  const size_t count = (size_t)a * b;
  if (!workspace || workspace_bytes < silenzio_gadget_workspace_bytes(P, 1, count)) return SILENZIO_ERR_WORKSPACE;
  if (P->poly_size != 2048) return SILENZIO_ERR_UNSUPPORTED;
  if (b == 0 || b > 13) return SILENZIO_ERR_WINDOW;  // row sums and E'' must fit 16-value windows
  if (a == 0) return SILENZIO_OK;
  const size_t cw = ct_bytes(P) / 8;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  p += rup(count * cw * 8);
  u64 *T[6];
  for (int i = 0; i < 6; i++) {
    T[i] = reinterpret_cast<u64 *>(p);
    p += rup(count * cw * 8);
  }
  Dev D;
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  int rc;
  const u64 hd = kDelta >> 1;
  // row sum (idx i*b + j) and broadcast (idx e / b) index arrays
  std::vector<u32> sidx(count), bidx(count);
  std::vector<i64> ones(count, 1), one1(count, 1);
  std::vector<u64> zero_a(a, 0), zero_c(count, 0);
  for (size_t e = 0; e < count; e++) {
    sidx[e] = (u32)e;
    bidx[e] = (u32)(e / b);
  }
  u64 *E = T[0], *S = T[1], *Sb = T[2], *Ep = T[3], *X = T[4], *Z = T[5];
  // E = round(e^{ReLU(v) - 7}) = [v == 7]   (exp LUT, kappa = 0, gamma = 3)
  std::vector<std::vector<u64>> t_exp = {table_window(-8, [](int v) { return enc(v == 7 ? 1 : 0, kDelta); })};
  if ((rc = upload_luts(D, t_exp))) return rc;
  if ((rc = lookup(D, Yhat, E, count, {}, 1))) return rc;
  // S = row sums, broadcast
  if ((rc = linear(D, E, S, a, (int)b, sidx, ones, zero_a))) return rc;
  if ((rc = linear(D, S, Sb, count, 1, bidx, one1, zero_c))) return rc;
  // E' = round((E 2^kappa + 1) / (S + 1)) = T4(E, S): g0(S) = round(1/(S+1)), g1(S) = round(2/(S+1))
  auto g0 = [](int s) { return rhe(1.0 / (s + 1)); };
  auto g1 = [](int s) { return rhe(2.0 / (s + 1)); };
  std::vector<std::vector<u64>> tA = {table_window(0, [&](int s) { return (u64)(g0(s) + g1(s)) * hd; })};
  std::vector<std::vector<u64>> tB = {table_window(0, [&](int s) { return (u64)(g0(s) - g1(s)) * hd; })};
  if ((rc = upload_luts(D, tA))) return rc;
  if ((rc = lookup(D, Sb, X, count, {}, 1))) return rc;                          // A (per element)
  if ((rc = axpy3(D, Z, E, 16, Sb, 1, nullptr, 0, 0, count))) return rc;          // 16 E + S
  if ((rc = upload_luts(D, tB))) return rc;
  if ((rc = lookup(D, Z, Ep, count, {}, 1))) return rc;                          // B
  if ((rc = axpy3(D, Ep, Ep, 1, X, 1, nullptr, 0, 0, count))) return rc;          // E' = A + B
  // F = Y * rowsum(E') = T4(Y, R): g0 = 0, g1 = R
  if ((rc = linear(D, Ep, S, a, (int)b, sidx, ones, zero_a))) return rc;         // R
  if ((rc = linear(D, S, Sb, count, 1, bidx, one1, zero_c))) return rc;         // R broadcast
  std::vector<std::vector<u64>> tA2 = {table_window(0, [&](int r) { return (u64)r * hd; })};
  std::vector<std::vector<u64>> tB2 = {table_window(0, [&](int r) { return (u64)0 - (u64)r * hd; })};
  if ((rc = upload_luts(D, tA2))) return rc;
  if ((rc = lookup(D, Sb, X, count, {}, 1))) return rc;
  if ((rc = axpy3(D, Z, Y, 16, Sb, 1, nullptr, 0, 0, count))) return rc;
  if ((rc = upload_luts(D, tB2))) return rc;
  if ((rc = lookup(D, Z, E, count, {}, 1))) return rc;
  // E'' = E' - F = E' - A2 - B2 ; sign on window [-13, 3)
  if ((rc = axpy3(D, Z, Ep, 1, X, -1, E, -1, 0, count))) return rc;
  std::vector<std::vector<u64>> tsg = {table_window(-13, [](int v) { return enc((v > 0) - (v < 0), kDelta); })};
  if ((rc = upload_luts(D, tsg))) return rc;
  return lookup(D, Z, out, count, {}, 1);
}

}  // extern "C"
