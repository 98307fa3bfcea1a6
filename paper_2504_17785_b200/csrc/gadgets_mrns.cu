// gadgets_mrns.cu -- config-4 gadget drivers at parameter set A (4-bit PBS):
//   silenzio_rns2mrns          Alg. 1 RNS2MRNS          (g4)
//   silenzio_rns_sign_abs      Sign_(-1,1,1) and |x| in RNS (l.309-323, Alg. 4 l.414-415) (g5)
//   silenzio_mrns_bitlen_max   bit length of MRNS digits + tensor-wide max (Alg. 3 step 2) (g6)
//   silenzio_int_ce_grad       IntCELossDeriv at Gamma = 4, kappa = 0 (Alg. 5, R10/R12) (g8)
// Thin drivers: they sequence linear LWE ops and PBS calls; every ciphertext
// operation runs in a kernel. Schedule: DESIGN.md §Config 4.
#include "gadget_util.cuh"
#include "nvtx.cuh"

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

// Alg. 1 on device buffers; `out` may not alias `in`. tmp holds tcap,
// tmp2 / tmp3 hold tcap2 ciphertexts (each >= count). For pivot i the targets
// j >= i are independent: consecutive targets are evaluated together (one PBS
// batch per group, one LUT per target via lut ids), as many as the scratch and
// the kMaxLuts test polynomials allow. Every ciphertext sees exactly the
// operations of the one-target-at-a-time schedule.
int rns2mrns_impl(Dev &D, const u64 *in, const uint32_t *moduli, int k, size_t count, u64 *out, u64 *tmp,
                  u64 *tmp2, u64 *tmp3, size_t tcap, size_t tcap2) {
  const size_t cw = D.big;
  SZ_CUDA_OK(cudaMemcpyAsync(out, in, (size_t)k * count * cw * 8, cudaMemcpyDeviceToDevice, D.st));
  int rc;
  for (int i = 1; i < k; i++) {
    const int mp = (int)moduli[i - 1];
    const u64 *pivot = out + (size_t)(i - 1) * count * cw;
    int j0 = i;
    while (j0 < k) {
      // group [j0, j1): same kind (direct window or T3), within scratch and LUT capacity
      const bool direct = mp + (int)moduli[j0] - 1 <= 16;
      const size_t cap = direct ? tcap : tcap2;
      int j1 = j0 + 1;
      while (j1 < k && j1 - j0 < kMaxLuts && (size_t)(j1 - j0 + 1) * count <= cap &&
             (mp + (int)moduli[j1] - 1 <= 16) == direct)
        j1++;
      const int ng = j1 - j0;
      std::vector<u32> ids((size_t)ng * count);
      for (int g = 0; g < ng; g++) std::fill(ids.begin() + (size_t)g * count, ids.begin() + (size_t)(g + 1) * count, (u32)g);
      // d = y_j - y_{i-1} in [-(mp-1), mj-1]
      for (int g = 0; g < ng; g++) {
        u64 *yj = out + (size_t)(j0 + g) * count * cw;
        if ((rc = axpy3(D, tmp + (size_t)g * count * cw, yj, 1, pivot, -1, nullptr, 0, 0, count))) return rc;
      }
      u64 *yout = out + (size_t)j0 * count * cw;  // targets j0.. are consecutive in out
      if (direct) {
        std::vector<std::vector<u64>> tabs;
        for (int g = 0; g < ng; g++) {
          const int mj = (int)moduli[j0 + g], t = inv_mod(mp, mj);
          tabs.push_back(table_window(-(mp - 1), [mj, t](int d) { return enc(pmod((long)d * t, mj), kDelta); }));
        }
        if ((rc = upload_luts(D, tabs))) return rc;
        if ((rc = lookup(D, tmp, yout, (size_t)ng * count, ids, (u32)ng))) return rc;
      } else {
        // T3: u = d mod mj = d + mj Delta/2 - sign(d) mj Delta/2 ; then T1 on [0,16)
        std::vector<std::vector<u64>> tabs;
        for (int g = 0; g < ng; g++) tabs.push_back(std::vector<u64>(16, (u64)moduli[j0 + g] * (kDelta >> 1)));
        if ((rc = upload_luts(D, tabs))) return rc;
        if ((rc = lookup(D, tmp, tmp2, (size_t)ng * count, ids, (u32)ng))) return rc;
        for (int g = 0; g < ng; g++) {
          const u64 half = (u64)moduli[j0 + g] * (kDelta >> 1);
          const size_t o = (size_t)g * count * cw;
          if ((rc = axpy3(D, tmp3 + o, tmp + o, 1, tmp2 + o, -1, nullptr, 0, half, count))) return rc;
        }
        std::vector<std::vector<u64>> tabs2;
        for (int g = 0; g < ng; g++) {
          const int mj = (int)moduli[j0 + g], t = inv_mod(mp, mj);
          tabs2.push_back(table_window(0, [mj, t](int u) { return enc(pmod((long)u * t, mj), kDelta); }));
        }
        if ((rc = upload_luts(D, tabs2))) return rc;
        if ((rc = lookup(D, tmp3, yout, (size_t)ng * count, ids, (u32)ng))) return rc;
      }
      j0 = j1;
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
  SZ_RANGE("rns2mrns");
  if (!in || !moduli_host || !out || !fbsk || !ksk || !P) return SILENZIO_ERR_NULL_POINTER;
  if (!workspace || workspace_bytes < silenzio_gadget_workspace_bytes(P, k, count)) return SILENZIO_ERR_WORKSPACE;
  if (P->poly_size != 2048 || k < 1) return SILENZIO_ERR_UNSUPPORTED;
  int rc = check_moduli(moduli_host, k);
  if (rc) return rc;
  if (count == 0) return SILENZIO_OK;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  const size_t ct = ct_bytes(P);
  u64 *t0 = reinterpret_cast<u64 *>(p);  // k count (the digits slot is free here)
  p += rup((size_t)k * count * ct);
  u64 *t1 = reinterpret_cast<u64 *>(p);  // 3 count
  p += 3 * rup(count * ct);
  u64 *t2 = reinterpret_cast<u64 *>(p);  // 3 count
  p += 3 * rup(count * ct);
  Dev D;
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  return rns2mrns_impl(D, in, moduli_host, (int)k, count, out, t0, t1, t2, (size_t)k * count, 3 * count);
}

int silenzio_rns_sign_abs(const uint64_t *in, const uint32_t *moduli_host, uint32_t k, size_t count,
                          uint64_t *sign_out, uint64_t *abs_out, const void *fbsk, const uint64_t *ksk,
                          const silenzio_params *P, void *workspace, size_t workspace_bytes, void *stream) {
  SZ_RANGE("rns_sign_abs");
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
  if ((rc = rns2mrns_impl(D, in, moduli_host, (int)k, count, digits, t[0], t[2], t[4], 2 * count, 2 * count))) return rc;
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
  SZ_RANGE("mrns_bitlen_max");
  if (!digits || !bitlen_out || !max_out || !fbsk || !ksk || !P) return SILENZIO_ERR_NULL_POINTER;
  if (!workspace || workspace_bytes < silenzio_gadget_workspace_bytes(P, k, count)) return SILENZIO_ERR_WORKSPACE;
  if (P->poly_size != 2048) return SILENZIO_ERR_UNSUPPORTED;
  if (count == 0) return SILENZIO_OK;
  const size_t cw = ct_bytes(P) / 8;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  u64 *buf = reinterpret_cast<u64 *>(p);   // [k][count] working copy of the bit lengths
  p += rup((size_t)k * count * cw * 8);
  u64 *tmp = reinterpret_cast<u64 *>(p);   // [k][count / 2] (k <= 6 fits the 3 count reserved)
  p += 3 * rup(count * cw * 8);
  u64 *tmp2 = reinterpret_cast<u64 *>(p);  // [k][count / 2]
  p += 3 * rup(count * cw * 8);
  if (k > 6) return SILENZIO_ERR_UNSUPPORTED;
  Dev D;
  dev_init(D, p, P, fbsk, ksk, sz_stream(stream), 4 * count + 64);
  int rc;
  std::vector<std::vector<u64>> tb = {table_window(0, [](int d) { return enc(bitlen(d), kDelta); })};
  if ((rc = upload_luts(D, tb))) return rc;
  if ((rc = lookup(D, digits, bitlen_out, (size_t)k * count, {}, 1))) return rc;
  std::vector<std::vector<u64>> trelu = {table_window(-8, [](int d) { return enc(d > 0 ? d : 0, kDelta); })};
  if ((rc = upload_luts(D, trelu))) return rc;
  // max tree (T7) per digit position: max(a, b) = b + ReLU(a - b), first half
  // against second half; the k positions advance level by level together (one
  // PBS batch per level, positions at stride `count` in buf)
  SZ_CUDA_OK(cudaMemcpyAsync(buf, bitlen_out, (size_t)k * count * cw * 8, cudaMemcpyDeviceToDevice, D.st));
  size_t cur = count;
  while (cur > 1) {
    const size_t half = cur / 2;
    for (uint32_t i = 0; i < k; i++) {
      u64 *bi = buf + (size_t)i * count * cw;
      if ((rc = axpy3(D, tmp + (size_t)i * half * cw, bi, 1, bi + half * cw, -1, nullptr, 0, 0, half))) return rc;
    }
    if ((rc = lookup(D, tmp, tmp2, (size_t)k * half, {}, 1))) return rc;
    for (uint32_t i = 0; i < k; i++) {
      u64 *bi = buf + (size_t)i * count * cw;
      if ((rc = axpy3(D, bi, bi + half * cw, 1, tmp2 + (size_t)i * half * cw, 1, nullptr, 0, 0, half))) return rc;
      if (cur & 1)
        SZ_CUDA_OK(cudaMemcpyAsync(bi + half * cw, bi + (cur - 1) * cw, cw * 8, cudaMemcpyDeviceToDevice, D.st));
    }
    cur = half + (cur & 1);
  }
  for (uint32_t i = 0; i < k; i++)
    SZ_CUDA_OK(cudaMemcpyAsync(max_out + (size_t)i * cw, buf + (size_t)i * count * cw, cw * 8, cudaMemcpyDeviceToDevice,
                               D.st));
  return SILENZIO_OK;
}

int silenzio_int_ce_grad(const uint64_t *Yhat, const uint64_t *Y, uint32_t a, uint32_t b, uint64_t *out,
                         const void *fbsk, const uint64_t *ksk, const silenzio_params *P, void *workspace,
                         size_t workspace_bytes, void *stream) {
  SZ_RANGE("int_ce_grad");
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

// ---------------------------------------------------------------------------
// g7: Shift2MSBs+- digit combine with the 8-bit stage (parameter set B).
// Alg. 3 steps 2-6 + Alg. 4 re-sign (l.419): per digit
// position i, digitShift_i = (gamma - (maxBit - w i)) * anyShift (clamped to
// [-4, gamma-1], output-equivalent for 4-bit digits); per element and digit one
// 8-bit PBS evaluates +-((d << lshift) >> rshift) on the packed index
// neg * 128 + (S_i + 4) * 16 + d; the digit results are summed.
// A set-B PBS here = KS (set-A big key -> set-B small key) -> BR at N = 32768
// -> SE (set-B big key) -> KS (set-B big key -> set-A big key).
extern "C" {
int silenzio_keyswitch_batch(const uint64_t *, const uint64_t *, uint64_t *, size_t, const silenzio_params *, void *,
                             void *);
int silenzio_blind_rotate_batch(const uint64_t *, const uint32_t *, const uint64_t *, uint32_t, const void *,
                                uint64_t *, size_t, const silenzio_params *, void *, void *);
size_t silenzio_blind_rotate_workspace_bytes(const silenzio_params *, size_t);
}

namespace {

constexpr u64 kDeltaB = 1ull << 55;  // set B: p = 8 + padding
constexpr size_t kBChunk = 2048;

template <class F>
std::vector<u64> table_window_b(int w0, F f) {  // 256-value window of Z_512
  std::vector<u64> T(256, 0);
  for (int x = w0; x < w0 + 256; x++) {
    const int xm = ((x % 512) + 512) % 512;
    if (xm < 256) T[xm] = f(x);
    else T[xm - 256] = (u64)0 - f(x);
  }
  return T;
}

struct DevB {
  const void *fbsk;
  const silenzio_params *pb, *pab, *pba;
  const u64 *ksk_ab, *ksk_ba;
  u64 *small, *big, *tables, *luts;
  u32 *ids;
  void *brws;
  cudaStream_t st;
};

size_t devb_bytes(const silenzio_params *pb, uint32_t nluts) {
  return rup(kBChunk * (pb->lwe_dim + 1) * 8) + rup(kBChunk * ((size_t)pb->glwe_dim * pb->poly_size + 1) * 8) +
         rup((size_t)nluts * 256 * 8) + rup((size_t)nluts * pb->poly_size * 8) + rup(kBChunk * 4) +
         rup(silenzio_blind_rotate_workspace_bytes(pb, kBChunk));
}

int upload_luts_b(DevB &B, const std::vector<std::vector<u64>> &tabs) {
  std::vector<u64> flat;
  for (auto &t : tabs) flat.insert(flat.end(), t.begin(), t.end());
  SZ_CUDA_OK(cudaMemcpyAsync(B.tables, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, B.st));
  SZ_CUDA_OK(cudaStreamSynchronize(B.st));
  return silenzio_build_testpoly(B.tables, (u32)tabs.size(), 8, B.pb->poly_size, B.luts, B.st);
}

// set-A big-key in -> set-A big-key out through the 8-bit PBS
int pbs_b(DevB &B, const u64 *in, u64 *out, size_t count, u32 num_luts, const std::vector<u32> &ids) {
  const size_t ca = (size_t)B.pab->ks_in_dim + 1;  // set-A big LWE words
  for (size_t c0 = 0; c0 < count; c0 += kBChunk) {
    const size_t cnt = count - c0 < kBChunk ? count - c0 : kBChunk;
    const u32 *idp = nullptr;
    if (!ids.empty()) {
      SZ_CUDA_OK(cudaMemcpyAsync(B.ids, ids.data() + c0, cnt * 4, cudaMemcpyHostToDevice, B.st));
      SZ_CUDA_OK(cudaStreamSynchronize(B.st));
      idp = B.ids;
    }
    int rc = silenzio_keyswitch_batch(in + c0 * ca, B.ksk_ab, B.small, cnt, B.pab, nullptr, B.st);
    if (rc) return rc;
    if ((rc = silenzio_blind_rotate_batch(B.small, idp, B.luts, num_luts, B.fbsk, B.big, cnt, B.pb, B.brws, B.st)))
      return rc;
    if (trace_active(1))
      trace_pbs(1, B.small, (size_t)B.pb->lwe_dim + 1, B.big, (size_t)B.pb->glwe_dim * B.pb->poly_size + 1, B.luts,
                B.pb->poly_size, ids.empty() ? nullptr : ids.data() + c0, cnt, B.st);
    if ((rc = silenzio_keyswitch_batch(B.big, B.ksk_ba, out + c0 * ca, cnt, B.pba, nullptr, B.st))) return rc;
  }
  return SILENZIO_OK;
}

}  // namespace

extern "C" {

size_t silenzio_mrns_combine_workspace_bytes(const silenzio_params *pa, const silenzio_params *pb, uint32_t k,
                                             size_t count) {
  if (!pa || !pb) return 0;
  const size_t ct = ct_bytes(pa);
  return 3 * rup((size_t)k * count * ct) + rup(count * ct) + 4 * rup((size_t)k * ct) +
         dev_bytes(pa, 4 * count + 64) + devb_bytes(pb, k) + 4096;
}

int silenzio_mrns_digit_combine(const uint64_t *top_digit, const uint64_t *abs_digits, const uint64_t *maxes,
                                uint32_t k, size_t count, uint32_t top_radix, uint32_t w, uint32_t gamma,
                                uint64_t *out, uint64_t *maxbit_out, const void *fbsk_a, const uint64_t *ksk_a,
                                const silenzio_params *pa, const void *fbsk_b, const silenzio_params *pb,
                                const uint64_t *ksk_ab, const silenzio_params *pab, const uint64_t *ksk_ba,
                                const silenzio_params *pba, void *workspace, size_t workspace_bytes, void *stream) {
  SZ_RANGE("mrns_digit_combine");
  if (!top_digit || !abs_digits || !maxes || !out || !maxbit_out || !fbsk_a || !ksk_a || !pa || !fbsk_b || !pb ||
      !ksk_ab || !pab || !ksk_ba || !pba)
    return SILENZIO_ERR_NULL_POINTER;
  if (!workspace || workspace_bytes < silenzio_mrns_combine_workspace_bytes(pa, pb, k, count))
    return SILENZIO_ERR_WORKSPACE;
  if (pa->poly_size != 2048 || pb->poly_size != 32768) return SILENZIO_ERR_UNSUPPORTED;
  if (pab->ks_in_dim != pa->glwe_dim * pa->poly_size || pab->lwe_dim != pb->lwe_dim ||
      pba->ks_in_dim != pb->glwe_dim * pb->poly_size || pba->lwe_dim != pa->glwe_dim * pa->poly_size)
    return SILENZIO_ERR_INVALID_PARAM;
  if (k == 0 || w * (k - 1) + w > 127 || gamma < 1 || gamma > 4 || top_radix % 2) return SILENZIO_ERR_WINDOW;
  if (count == 0) return SILENZIO_OK;
  const size_t cw = ct_bytes(pa) / 8;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  auto carve = [&](size_t bytes) {
    unsigned char *r = p;
    p += rup(bytes);
    return r;
  };
  u64 *dB = reinterpret_cast<u64 *>(carve((size_t)k * count * cw * 8));
  u64 *packed = reinterpret_cast<u64 *>(carve((size_t)k * count * cw * 8));
  u64 *R = reinterpret_cast<u64 *>(carve((size_t)k * count * cw * 8));
  u64 *eB = reinterpret_cast<u64 *>(carve(count * cw * 8));
  u64 *v = reinterpret_cast<u64 *>(carve((size_t)k * cw * 8));
  u64 *mbk = reinterpret_cast<u64 *>(carve((size_t)k * cw * 8));
  u64 *S = reinterpret_cast<u64 *>(carve((size_t)k * cw * 8));
  u64 *tmp = reinterpret_cast<u64 *>(carve((size_t)k * cw * 8));
  Dev D;
  dev_init(D, p, pa, fbsk_a, ksk_a, sz_stream(stream), 4 * count + 64);
  DevB B;
  B.fbsk = fbsk_b;
  B.pb = pb;
  B.pab = pab;
  B.pba = pba;
  B.ksk_ab = ksk_ab;
  B.ksk_ba = ksk_ba;
  B.st = sz_stream(stream);
  B.small = reinterpret_cast<u64 *>(carve(kBChunk * (pb->lwe_dim + 1) * 8));
  B.big = reinterpret_cast<u64 *>(carve(kBChunk * ((size_t)pb->glwe_dim * pb->poly_size + 1) * 8));
  B.tables = reinterpret_cast<u64 *>(carve((size_t)k * 256 * 8));
  B.luts = reinterpret_cast<u64 *>(carve((size_t)k * pb->poly_size * 8));
  B.ids = reinterpret_cast<u32 *>(carve(kBChunk * 4));
  B.brws = carve(silenzio_blind_rotate_workspace_bytes(pb, kBChunk));
  int rc;
  const int rk = (int)top_radix, W = (int)w, g = (int)gamma;
  // (1) sign bit at 128 Delta_B = 2^62, fresh
  std::vector<std::vector<u64>> ts = {table_window(0, [rk](int y) { return 2 * y >= rk ? (1ull << 62) : 0ull; })};
  if ((rc = upload_luts(D, ts))) return rc;
  if ((rc = lookup(D, top_digit, eB, count, {}, 1))) return rc;
  // (2) digits rescaled to Delta_B
  std::vector<std::vector<u64>> td = {table_window(0, [](int d) { return enc(d, kDeltaB); })};
  if ((rc = upload_luts(D, td))) return rc;
  if ((rc = lookup(D, abs_digits, dB, (size_t)k * count, {}, 1))) return rc;
  // (3) v_i = M_i > 0 ? M_i + w i : 0 at Delta_B (one LUT per position)
  {
    std::vector<std::vector<u64>> tv;
    std::vector<u32> ids(k);
    for (uint32_t i = 0; i < k; i++) {
      tv.push_back(table_window(0, [i, W](int M) { return enc(M > 0 ? M + W * (int)i : 0, kDeltaB); }));
      ids[i] = i;
    }
    // the Dev holds kMaxLuts (4) test polynomials: evaluate in groups
    for (uint32_t i0 = 0; i0 < k; i0 += kMaxLuts) {
      const uint32_t ng = (k - i0 < (uint32_t)kMaxLuts) ? k - i0 : (uint32_t)kMaxLuts;
      std::vector<std::vector<u64>> grp(tv.begin() + i0, tv.begin() + i0 + ng);
      std::vector<u32> gids(ids.begin() + i0, ids.begin() + i0 + ng);
      for (auto &x : gids) x -= i0;
      if ((rc = upload_luts(D, grp))) return rc;
      if ((rc = lookup(D, maxes + (size_t)i0 * cw, v + (size_t)i0 * cw, ng, gids, ng))) return rc;
    }
  }
  // (4) maxBit = fold of max(x, y) = y + ReLU_B(x - y) over v_0..v_{k-1} (8-bit window [-128, 128))
  SZ_CUDA_OK(cudaMemcpyAsync(maxbit_out, v, cw * 8, cudaMemcpyDeviceToDevice, D.st));
  {
    std::vector<std::vector<u64>> trelu = {table_window_b(-128, [](int t) { return enc(t > 0 ? t : 0, kDeltaB); })};
    if ((rc = upload_luts_b(B, trelu))) return rc;
    for (uint32_t i = 1; i < k; i++) {
      const u64 *y = v + (size_t)i * cw;
      if ((rc = axpy3(D, tmp, maxbit_out, 1, y, -1, nullptr, 0, 0, 1))) return rc;        // x - y
      if ((rc = pbs_b(B, tmp, tmp + cw, 1, 1, {}))) return rc;                             // ReLU
      if ((rc = axpy3(D, maxbit_out, y, 1, tmp + cw, 1, nullptr, 0, 0, 1))) return rc;    // y + ReLU
    }
  }
  // (5) S'_i = (clamp(digitShift_i, -4, gamma-1) + 4) * 16 * Delta_B
  {
    std::vector<std::vector<u64>> tsh;
    std::vector<u32> ids(k);
    for (uint32_t i = 0; i < k; i++) {
      tsh.push_back(table_window_b(0, [i, W, g](int mb) {
        int ds = (mb > W) ? (g + W * (int)i - mb) : 0;
        ds = ds < -4 ? -4 : (ds > g - 1 ? g - 1 : ds);
        return enc((ds + 4) * 16, kDeltaB);
      }));
      ids[i] = i;
      SZ_CUDA_OK(cudaMemcpyAsync(mbk + (size_t)i * cw, maxbit_out, cw * 8, cudaMemcpyDeviceToDevice, D.st));
    }
    if ((rc = upload_luts_b(B, tsh))) return rc;
    if ((rc = pbs_b(B, mbk, S, k, k, ids))) return rc;
  }
  // (6) packed index and (7) the 8-bit digit PBS
  for (uint32_t i = 0; i < k; i++)
    if ((rc = launch_lwe_axpy_bcast(packed + (size_t)i * count * cw, eB, 1, dB + (size_t)i * count * cw, 1,
                                    S + (size_t)i * cw, 1, count, (int)(cw - 1), D.st)))
      return rc;
  {
    std::vector<std::vector<u64>> tc = {table_window_b(0, [g](int x) {
      const int neg = x >> 7, s = ((x >> 4) & 7) - 4, d = x & 15;
      const int l = s < 0 ? 0 : (s > g - 1 ? g - 1 : s), r = s < 0 ? -s : 0;
      const int val = (d << l) >> r;
      return enc(neg ? -val : val, kDelta);
    })};
    if ((rc = upload_luts_b(B, tc))) return rc;
    if ((rc = pbs_b(B, packed, R, (size_t)k * count, 1, {}))) return rc;
  }
  // (8) sum over digits
  SZ_CUDA_OK(cudaMemcpyAsync(out, R, count * cw * 8, cudaMemcpyDeviceToDevice, D.st));
  for (uint32_t i = 1; i < k; i++)
    if ((rc = axpy3(D, out, out, 1, R + (size_t)i * count * cw, 1, nullptr, 0, 0, count))) return rc;
  return SILENZIO_OK;
}

}  // extern "C"
