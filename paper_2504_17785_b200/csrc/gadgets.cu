// gadgets.cu -- silenzio_rns_matmul: the encrypted Matmul^RNS gadget
// (Alg. 2, l.280-307) at 4-bit PBS precision (parameter set A).
//
// The driver only composes linear LWE ops (silenzio_lwe_linear_batch) and
// PBS (silenzio_pbs_batch); every ciphertext operation runs in the CUDA
// kernels. Host code here builds LUT tables and index arrays and sequences
// the batched calls. The schedule (DESIGN.md §Config 3) realises the paper's
// three steps with 16-value windows (plaintext Z_32, Delta = 2^59):
//   g1 RNS conversion   one PBS per (element, modulus) on the signed window
//                       [-8, 8); modulus 16 directly as two 2-bit digits.
//   g2 residue products quarter squares ab = 4^{-1}((a+b)^2 - (a-b)^2) mod m:
//                       m in {5,7}: 2 PBS; m in {9,11,13}: a+b, a-b first
//                       reduced mod m with the sign trick (T3) -> 4 PBS;
//                       m = 16: 2-bit digit products a0b0 + 4(a0b1 + a1b0)
//                       as 3 packed-index PBS emitted at scale 2^60.
//   g3 modular sums     m = 16: native wrap at 2^60; m in {5,7}: clean groups
//                       of 3 / 2 reduced by a fresh mod-m PBS; m >= 9: pair
//                       tree of T3 reductions.

#include "gadget_util.cuh"
#include "nvtx.cuh"

namespace szg {

// Pairwise/grouped reduction tree over `groups` independent groups of `terms`
// consecutive ciphertexts in buf (in place). Returns the group results in
// buf[0..groups).
int sum_tree(Dev &D, int m, u64 *buf, u64 *tmp, u64 *tmp2, size_t groups, size_t terms) {
  const u64 half_m = (u64)m * (kDelta >> 1);  // m * Delta / 2
  size_t cur = terms;
  while (cur > 1) {
    if (m <= 8) {
      // clean groups of g terms (g (m-1) <= 15) -> fresh mod-m PBS
      const size_t g = (m == 5) ? 3 : 2;
      const size_t next = (cur + g - 1) / g;
      std::vector<u32> idx(groups * next * g);
      std::vector<i64> coef(groups * next * g);
      std::vector<u64> cst(groups * next, 0);
      for (size_t q = 0; q < groups; q++)
        for (size_t o = 0; o < next; o++)
          for (size_t t = 0; t < g; t++) {
            const size_t src = o * g + t;
            idx[(q * next + o) * g + t] = (u32)(q * cur + (src < cur ? src : 0));
            coef[(q * next + o) * g + t] = src < cur ? 1 : 0;
          }
      std::vector<std::vector<u64>> tabs = {table_window(0, [m](int s) { return enc(pmod(s, m), kDelta); })};
      int rc = upload_luts(D, tabs);
      if (rc) return rc;
      // in place: the keyswitch stage consumes every input before the blind rotation writes buf
      if ((rc = linear_lookup(D, buf, buf, groups * next, (int)g, idx, coef, cst, {}, 1, tmp))) return rc;
      cur = next;
    } else {
      // pair tree with the sign trick T3: t = x + y - m; s = sign PBS(t) * m Delta/2;
      // z = t + m Delta/2 - s = x + y - m Delta/2 - s  in [0, m)
      const size_t next = (cur + 1) / 2;
      std::vector<u32> idx(groups * next * 2);
      std::vector<i64> coef(groups * next * 2);
      std::vector<u64> cst(groups * next);
      for (size_t q = 0; q < groups; q++)
        for (size_t o = 0; o < next; o++) {
          const size_t a = o * 2, b = o * 2 + 1;
          const bool pair = b < cur;
          idx[(q * next + o) * 2] = (u32)(q * cur + a);
          idx[(q * next + o) * 2 + 1] = (u32)(q * cur + (pair ? b : a));
          coef[(q * next + o) * 2] = 1;
          coef[(q * next + o) * 2 + 1] = pair ? 1 : 0;
          // singles pass through the same T3 (t = x - m, exact mod m too)
          cst[q * next + o] = (u64)0 - (u64)m * kDelta;
        }
      int rc = linear(D, buf, tmp, groups * next, 2, idx, coef, cst);  // t
      if (rc) return rc;
      std::vector<std::vector<u64>> tabs = {std::vector<u64>(16, half_m)};  // T2 sign
      if ((rc = upload_luts(D, tabs))) return rc;
      // s lands right after t in tmp, so the second linear op addresses both through one base
      if ((rc = lookup(D, tmp, tmp + groups * next * D.big, groups * next, {}, 1))) return rc;  // s
      // z = t + m Delta/2 - s
      std::vector<u32> idx2(groups * next * 2);
      std::vector<i64> coef2(groups * next * 2);
      std::vector<u64> cst2(groups * next, half_m);
      for (size_t e = 0; e < groups * next; e++) {
        idx2[e * 2] = (u32)e;
        idx2[e * 2 + 1] = (u32)(groups * next + e);
        coef2[e * 2] = 1;
        coef2[e * 2 + 1] = -1;
      }
      if ((rc = linear(D, tmp, buf, groups * next, 2, idx2, coef2, cst2))) return rc;
      cur = next;
    }
  }
  return SILENZIO_OK;
}

}  // namespace szg

using namespace szg;

extern "C" {

// Rows of X processed per pass: enough products per PBS batch to fill the GPU
// (a PBS launch costs one full blind rotation of latency whatever its size), at
// most one row when a single row already gives >= kPassProducts products.
constexpr size_t kPassProducts = 4096;
static uint32_t rows_per_pass(uint32_t a, uint32_t b, uint32_t c) {
  const size_t per_row = (size_t)b * c;
  size_t r = (kPassProducts + per_row - 1) / per_row;
  if (r < 1) r = 1;
  return (uint32_t)(r < a ? r : a);
}

size_t silenzio_rns_matmul_workspace_bytes(const silenzio_params *P, uint32_t a, uint32_t b, uint32_t c) {
  if (!P || a == 0) return 0;
  const size_t big = (size_t)P->glwe_dim * P->poly_size + 1;
  const size_t ct = big * 8;
  const size_t R = rows_per_pass(a, b, c);
  const size_t xr = 2 * (size_t)a * b, wr = 2 * (size_t)b * c;   // residues / digits of one modulus
  const size_t prod = 4 * R * b * c;                               // per pass of R rows: up to 4 ciphertexts per product
  const size_t bufs = xr + wr + 4 * prod;                          // X', W', 4 row buffers
  const size_t idx_cap = 2 * prod;
  const size_t pbs_cap = 65536;
  return bufs * ct + idx_cap * (4 + 8) + idx_cap * 8 + pbs_cap * 4 + kMaxLuts * (P->poly_size + 16) * 8 +
         silenzio_pbs_workspace_bytes(P, pbs_cap) + silenzio_ksk_planes_bytes(P) + 4096;
}

int silenzio_rns_matmul(const uint64_t *X, const uint64_t *W, uint32_t a, uint32_t b, uint32_t c,
                        const uint32_t *moduli, uint32_t k, uint64_t *out, const void *fbsk, const uint64_t *ksk,
                        const silenzio_params *P, void *workspace, size_t workspace_bytes, void *stream) {
  SZ_RANGE("rns_matmul");
  if (!X || !W || !moduli || !out || !fbsk || !ksk || !P) return SILENZIO_ERR_NULL_POINTER;
  if (!workspace) return SILENZIO_ERR_WORKSPACE;
  if (a == 0 || b == 0 || c == 0 || k == 0) return SILENZIO_ERR_COUNT;
  if (P->poly_size != 2048 || P->glwe_dim != 1) return SILENZIO_ERR_UNSUPPORTED;
  if (workspace_bytes < silenzio_rns_matmul_workspace_bytes(P, a, b, c)) return SILENZIO_ERR_WORKSPACE;
  for (uint32_t i = 0; i < k; i++) {
    const int m = (int)moduli[i];
    // window checks (the SPEC guard analogue): every LUT input window <= 16 values
    if (!(m == 5 || m == 7 || m == 9 || m == 11 || m == 13 || m == 16)) return SILENZIO_ERR_WINDOW;
  }
  Dev D;
  D.st = sz_stream(stream);
  D.P = P;
  D.fbsk = fbsk;
  D.ksk = ksk;
  D.big = (size_t)P->glwe_dim * P->poly_size + 1;
  const size_t ctw = D.big;  // words per ciphertext
  const uint32_t RP = rows_per_pass(a, b, c);
  const size_t xr = 2 * (size_t)a * b, wr = 2 * (size_t)b * c, prod = 4 * (size_t)RP * b * c;
  unsigned char *p = reinterpret_cast<unsigned char *>(workspace);
  auto carve = [&](size_t bytes) {
    unsigned char *r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  u64 *Xr = reinterpret_cast<u64 *>(carve(xr * ctw * 8));
  u64 *Wr = reinterpret_cast<u64 *>(carve(wr * ctw * 8));
  u64 *T0 = reinterpret_cast<u64 *>(carve(prod * ctw * 8));
  u64 *T1 = reinterpret_cast<u64 *>(carve(prod * ctw * 8));
  u64 *T2 = reinterpret_cast<u64 *>(carve(prod * ctw * 8));
  u64 *T3 = reinterpret_cast<u64 *>(carve(prod * ctw * 8));
  D.idx_cap = 2 * prod;
  D.idx = reinterpret_cast<u32 *>(carve(D.idx_cap * 4));
  D.coef = reinterpret_cast<i64 *>(carve(D.idx_cap * 8));
  D.cst = reinterpret_cast<u64 *>(carve(D.idx_cap * 8));
  D.pbs_cap = 65536;
  D.ids_cap = D.pbs_cap;
  D.ids = reinterpret_cast<u32 *>(carve(D.ids_cap * 4));
  D.tables = reinterpret_cast<u64 *>(carve(kMaxLuts * 16 * 8));
  D.luts = reinterpret_cast<u64 *>(carve((size_t)kMaxLuts * P->poly_size * 8));
  D.pbs_ws = carve(silenzio_pbs_workspace_bytes(P, D.pbs_cap));
  // KSK byte planes once per call (not once per PBS launch); every "linear op, then lookup"
  // below is then one silenzio_pbs_linear_batch (a0 fused into a1)
  if (const size_t pb = silenzio_ksk_planes_bytes(P)) {
    void *planes = carve(pb);
    int prc = silenzio_ksk_to_planes(ksk, planes, P, D.st);
    if (prc) return prc;
    D.planes = planes;
  }

  const size_t nX = (size_t)a * b, nW = (size_t)b * c;
  int rc;
  for (uint32_t mi = 0; mi < k; mi++) {
    const int m = (int)moduli[mi];
    // ---------------- g1: RNS conversion of X and W (signed window [-8, 8))
    if (m != 16) {
      std::vector<std::vector<u64>> tabs = {table_window(-8, [m](int x) { return enc(pmod(x, m), kDelta); })};
      if ((rc = upload_luts(D, tabs))) return rc;
      if ((rc = lookup(D, X, Xr, nX, {}, 1))) return rc;
      if ((rc = lookup(D, W, Wr, nW, {}, 1))) return rc;
    } else {
      // 2-bit digits of x mod 16: d0 = x mod 4 at [0, nX), d1 = (x mod 16) div 4 at [nX, 2 nX)
      std::vector<std::vector<u64>> tabs = {
          table_window(-8, [](int x) { return enc(pmod(x, 16) & 3, kDelta); }),
          table_window(-8, [](int x) { return enc(pmod(x, 16) >> 2, kDelta); })};
      if ((rc = upload_luts(D, tabs))) return rc;
      std::vector<u32> idsx(nX, 0u);
      if ((rc = lookup(D, X, Xr, nX, idsx, 2))) return rc;
      std::fill(idsx.begin(), idsx.end(), 1u);
      if ((rc = lookup(D, X, Xr + nX * ctw, nX, idsx, 2))) return rc;
      std::vector<u32> idsw(nW, 0u);
      if ((rc = lookup(D, W, Wr, nW, idsw, 2))) return rc;
      std::fill(idsw.begin(), idsw.end(), 1u);
      if ((rc = lookup(D, W, Wr + nW * ctw, nW, idsw, 2))) return rc;
    }
    // ---------------- per pass of R rows i0.. of X: products over (r, j, kk), then
    // the sum tree per output (r, j)
    for (uint32_t i0 = 0; i0 < a; i0 += RP) {
      const uint32_t R = (a - i0 < RP) ? a - i0 : RP;
      const uint32_t i = i0;
      // Linear inputs address one array: gather the rows of X' and all of W'
      // as [X'(i0..i0+R, 0..b) | W'(0..b, 0..c)] (digits doubled for m = 16).
      const size_t xw = (m == 16) ? 2 : 1;
      const size_t nrow = xw * R * b, nw = xw * nW;
      // stage rows i0.. of X' (and their digit plane) into T3, W' after them
      for (size_t d = 0; d < xw; d++)
        SZ_CUDA_OK(cudaMemcpyAsync(T3 + d * R * b * ctw, Xr + (d * nX + (size_t)i0 * b) * ctw, R * b * ctw * 8,
                                   cudaMemcpyDeviceToDevice, D.st));
      SZ_CUDA_OK(cudaMemcpyAsync(T3 + nrow * ctw, Wr, nw * ctw * 8, cudaMemcpyDeviceToDevice, D.st));
      // product index e = (r c + j) b + kk  (products of one output are contiguous)
      const size_t np = (size_t)R * c * b;
      auto xi = [&](size_t d, size_t r, size_t kk) { return (u32)(d * R * b + r * b + kk); };
      auto wi = [&](size_t d, size_t kk, size_t j) { return (u32)(nrow + d * nW + kk * c + j); };
      size_t terms_per_product;
      if (m == 5 || m == 7) {
        // s = x + w (window [0,16)), d = x - w (window [-8,8))
        std::vector<u32> idx(2 * np * 2);
        std::vector<i64> coef(2 * np * 2);
        std::vector<u64> cst(2 * np, 0);
        std::vector<u32> ids(2 * np);
        for (size_t r = 0; r < R; r++)
        for (size_t j = 0; j < c; j++)
          for (size_t kk = 0; kk < b; kk++) {
            const size_t e = (r * c + j) * b + kk;
            for (int h = 0; h < 2; h++) {
              const size_t o = 2 * e + h;
              idx[2 * o] = xi(0, r, kk);
              idx[2 * o + 1] = wi(0, kk, j);
              coef[2 * o] = 1;
              coef[2 * o + 1] = h ? -1 : 1;
              ids[o] = (u32)h;
            }
          }
        const int i4 = inv4(m);
        std::vector<std::vector<u64>> tabs = {
            table_window(0, [m, i4](int s) { return enc(pmod((long)i4 * s * s, m), kDelta); }),
            table_window(-8, [m, i4](int d) { return enc(pmod(-(long)i4 * d * d, m), kDelta); })};
        if ((rc = upload_luts(D, tabs))) return rc;
        if ((rc = linear_lookup(D, T3, T1, 2 * np, 2, idx, coef, cst, ids, 2, T0))) return rc;
        terms_per_product = 2;
      } else if (m == 16) {
        // q00 = 4 a0 + b0, q01 = 4 a0 + b1, q10 = 4 a1 + b0; digit products at 2^60
        std::vector<u32> idx(3 * np * 2);
        std::vector<i64> coef(3 * np * 2);
        std::vector<u64> cst(3 * np, 0);
        std::vector<u32> ids(3 * np);
        for (size_t r = 0; r < R; r++)
        for (size_t j = 0; j < c; j++)
          for (size_t kk = 0; kk < b; kk++) {
            const size_t e = (r * c + j) * b + kk;
            const size_t da[3] = {0, 0, 1}, db[3] = {0, 1, 0};
            for (int h = 0; h < 3; h++) {
              const size_t o = 3 * e + h;
              idx[2 * o] = xi(da[h], r, kk);
              idx[2 * o + 1] = wi(db[h], kk, j);
              coef[2 * o] = 4;
              coef[2 * o + 1] = 1;
              ids[o] = h == 0 ? 0u : 1u;
            }
          }
        std::vector<std::vector<u64>> tabs = {
            table_window(0, [](int q) { return enc(((q >> 2) * (q & 3)) & 15, kDelta16); }),
            table_window(0, [](int q) { return enc((4 * (q >> 2) * (q & 3)) & 15, kDelta16); })};
        if ((rc = upload_luts(D, tabs))) return rc;
        if ((rc = linear_lookup(D, T3, T1, 3 * np, 2, idx, coef, cst, ids, 2, T0))) return rc;
        terms_per_product = 3;
      } else {
        // m in {9, 11, 13}: t1 = x + w - m, t2 = x - w; sigma = sign PBS; u, v = T3(t);
        // P1 = qs+(u), P2 = qs-(v), both on [0, 16)
        const u64 half_m = (u64)m * (kDelta >> 1);
        std::vector<u32> idx(2 * np * 2);
        std::vector<i64> coef(2 * np * 2);
        std::vector<u64> cst(2 * np);
        for (size_t r = 0; r < R; r++)
        for (size_t j = 0; j < c; j++)
          for (size_t kk = 0; kk < b; kk++) {
            const size_t e = (r * c + j) * b + kk;
            for (int h = 0; h < 2; h++) {
              const size_t o = 2 * e + h;
              idx[2 * o] = xi(0, r, kk);
              idx[2 * o + 1] = wi(0, kk, j);
              coef[2 * o] = 1;
              coef[2 * o + 1] = h ? -1 : 1;
              cst[o] = h ? 0 : (u64)0 - (u64)m * kDelta;
            }
          }
        if ((rc = linear(D, T3, T0, 2 * np, 2, idx, coef, cst))) return rc;  // t
        std::vector<std::vector<u64>> tabs = {std::vector<u64>(16, half_m)};
        if ((rc = upload_luts(D, tabs))) return rc;
        if ((rc = lookup(D, T0, T0 + 2 * np * ctw, 2 * np, {}, 1))) return rc;  // sigma after t
        // u/v = t + m Delta/2 - sigma
        std::vector<u32> idx2(2 * np * 2);
        std::vector<i64> coef2(2 * np * 2);
        std::vector<u64> cst2(2 * np, half_m);
        for (size_t o = 0; o < 2 * np; o++) {
          idx2[2 * o] = (u32)o;
          idx2[2 * o + 1] = (u32)(2 * np + o);
          coef2[2 * o] = 1;
          coef2[2 * o + 1] = -1;
        }
        const int i4 = inv4(m);
        std::vector<std::vector<u64>> tabs2 = {
            table_window(0, [m, i4](int s) { return enc(pmod((long)i4 * s * s, m), kDelta); }),
            table_window(0, [m, i4](int d) { return enc(pmod(-(long)i4 * d * d, m), kDelta); })};
        if ((rc = upload_luts(D, tabs2))) return rc;
        std::vector<u32> ids(2 * np);
        for (size_t o = 0; o < 2 * np; o++) ids[o] = (u32)(o & 1);
        if ((rc = linear_lookup(D, T0, T1, 2 * np, 2, idx2, coef2, cst2, ids, 2, T2))) return rc;
        terms_per_product = 2;
      }
      // ---------------- g3: modular summation of the b * terms_per_product terms of each output j
      const size_t terms = b * terms_per_product;
      const size_t outs = (size_t)R * c;
      u64 *dst = out + ((size_t)mi * a + i) * c * ctw;
      if (m == 16) {
        // native wrap at scale 2^60: one linear op sums all terms
        std::vector<u32> idx(outs * terms);
        std::vector<i64> coef(outs * terms, 1);
        std::vector<u64> cst(outs, 0);
        for (size_t j = 0; j < outs; j++)
          for (size_t t = 0; t < terms; t++) idx[j * terms + t] = (u32)(j * terms + t);
        if ((rc = linear(D, T1, dst, outs, (int)terms, idx, coef, cst))) return rc;
      } else {
        if ((rc = sum_tree(D, m, T1, T0, T2, outs, terms))) return rc;
        SZ_CUDA_OK(cudaMemcpyAsync(dst, T1, outs * ctw * 8, cudaMemcpyDeviceToDevice, D.st));
      }
    }
  }
  return SILENZIO_OK;
}

}  // extern "C"
