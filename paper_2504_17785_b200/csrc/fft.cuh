// fft.cuh -- negacyclic f64 FFT building blocks for N = 2048 (M = N/2 = 1024).
//
// The negacyclic transform of a real polynomial a of length N (SURVEY.md
// §8(a) a4.3): fold z_j = (a_j + i a_{j+N/2}) * w^j, w = e^{i pi / N},
// j < N/2, then an M-point DFT with POSITIVE exponent:
//     Z_k = sum_j z_j e^{+2 pi i jk / M} = A(zeta_k),  zeta_k = w^{4k+1},
// the evaluations of A at half of the roots of X^N + 1 (the other half are
// conjugates because A is real). Products in Z[X]/(X^N+1) become pointwise.
// The inverse runs the same passes backwards with conjugate twiddles; 1/M is
// folded into the Fourier BSK.
//
// Decomposition M = 1024 = 16 x 16 x 4 (four-step, decimation in frequency,
// in place, digit-reversed output). One "team" of T = 64 threads owns one
// transform; every thread holds 16 complex values in registers per pass:
//   pass 1: radix-16 over stride 64   (positions t + 64 m)
//   pass 2: radix-16 over stride 4    (positions 64 b + s + 4 m, b = t/4, s = t%4)
//   pass 3: radix-4  over stride 1    (positions 4 (t + 64 u) + m, u < 4)
// Passes exchange through a 16 KiB shared buffer with an XOR swizzle that makes
// all three access patterns bank-conflict free for 16-byte elements.
#pragma once
#include "common.cuh"

namespace sz {

constexpr int kM = 1024;      // complex points per transform (N = 2048)
constexpr int kTeam = 64;     // threads per transform
constexpr int kPts = 16;      // complex values per thread

// e^{+2 pi i j / 16}, j = 0..15 (literal values, correctly rounded doubles)
struct C16 {
  static constexpr double c[16] = {
      1.0, 0.92387953251128673848, 0.70710678118654757274, 0.38268343236508978178,
      0.0, -0.38268343236508978178, -0.70710678118654757274, -0.92387953251128673848,
      -1.0, -0.92387953251128673848, -0.70710678118654757274, -0.38268343236508978178,
      0.0, 0.38268343236508978178, 0.70710678118654757274, 0.92387953251128673848};
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// acc += a * b
__device__ __forceinline__ void cmac(double2 &acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}

// multiply by W_16^E (E taken mod 16), conjugated when INV.
template <int E, bool INV>
__device__ __forceinline__ double2 mulw16(double2 a) {
  constexpr int e = INV ? ((16 - (E & 15)) & 15) : (E & 15);
  if constexpr (e == 0) {
    return a;
  } else if constexpr (e == 4) {
    return make_double2(-a.y, a.x);
  } else if constexpr (e == 8) {
    return make_double2(-a.x, -a.y);
  } else if constexpr (e == 12) {
    return make_double2(a.y, -a.x);
  } else {
    constexpr double c = C16::c[e];
    constexpr double s = C16::c[(e + 12) & 15];  // sin(2 pi e/16) = cos(2 pi (e-4)/16)
    return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
  }
}

// In-place radix-2 DIF DFT of size R (R | 16) on registers, exponent sign +
// (conjugate when INV). Natural-order input, bit-reversed output: x[r] holds
// X[bitrev_R(r)].
template <int R, bool INV, int H = R / 2>
__device__ __forceinline__ void dft_stage(double2 (&x)[R]) {
  if constexpr (H >= 1) {
#pragma unroll
    for (int b = 0; b < R; b += 2 * H) {
#pragma unroll
      for (int j = 0; j < H; j++) {
        const double2 a = x[b + j], c = x[b + j + H];
        x[b + j] = cadd(a, c);
        const double2 d = csub(a, c);
        // twiddle W_{2H}^j = W_16^{j * 16 / (2H)}
        switch ((j * (16 / (2 * H))) & 15) {
          case 0: x[b + j + H] = mulw16<0, INV>(d); break;
          case 1: x[b + j + H] = mulw16<1, INV>(d); break;
          case 2: x[b + j + H] = mulw16<2, INV>(d); break;
          case 3: x[b + j + H] = mulw16<3, INV>(d); break;
          case 4: x[b + j + H] = mulw16<4, INV>(d); break;
          case 5: x[b + j + H] = mulw16<5, INV>(d); break;
          case 6: x[b + j + H] = mulw16<6, INV>(d); break;
          case 7: x[b + j + H] = mulw16<7, INV>(d); break;
          default: break;
        }
      }
    }
    dft_stage<R, INV, H / 2>(x);
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft(double2 (&x)[R]) {
  dft_stage<R, INV, R / 2>(x);
}

// ---- FMA-form radix-2 decimation-in-time butterflies (6 FP64 instructions when
// the twiddle is nontrivial, against 8 for "add, subtract, multiply"): with
// W^e = i^q e^{i theta}, |theta| <= pi/4 after pulling out i^q,
//   e^{i theta} b = cos (b.x - tan b.y, b.y + tan b.x) = sin (cot b.x - b.y, cot b.y + b.x)
// and the cos / sin factor folds into the four output FMAs. W = e^{+2 pi i / 32}.
struct FmaTw32 {
  // cos(2 pi r / 32), tan(2 pi r / 32), r = 0..4 (correctly rounded doubles)
  static constexpr double c[5] = {1.0, 0.9807852804032304, 0.9238795325112867, 0.8314696123025452,
                                  0.7071067811865476};
  static constexpr double t[5] = {0.0, 0.198912367379658, 0.41421356237309503, 0.6681786379192989, 1.0};
};
template <int E, bool INV>
__device__ __forceinline__ void bfly32(double2 &a, double2 &b) {
  constexpr int e = INV ? ((32 - (E & 31)) & 31) : (E & 31);
  constexpr int q = e >> 3, r = e & 7;
  if constexpr (r == 0) {
    double2 t;
    if constexpr (q == 0) t = b;
    else if constexpr (q == 1) t = make_double2(-b.y, b.x);
    else if constexpr (q == 2) t = make_double2(-b.x, -b.y);
    else t = make_double2(b.y, -b.x);
    const double2 na = cadd(a, t), nb = csub(a, t);
    a = na;
    b = nb;
  } else {
    double u, v;
    if constexpr (r <= 4) {
      constexpr double tn = FmaTw32::t[r];
      u = fma(-tn, b.y, b.x);
      v = fma(tn, b.x, b.y);
    } else {
      constexpr double ct = FmaTw32::t[8 - r];
      u = fma(ct, b.x, -b.y);
      v = fma(ct, b.y, b.x);
    }
    constexpr double f = (r <= 4) ? FmaTw32::c[r] : FmaTw32::c[8 - r];
    double U, V;  // (u + i v) * i^q
    if constexpr (q == 0) { U = u; V = v; }
    else if constexpr (q == 1) { U = -v; V = u; }
    else if constexpr (q == 2) { U = -u; V = -v; }
    else { U = v; V = -u; }
    const double2 na = make_double2(fma(f, U, a.x), fma(f, V, a.y));
    const double2 nb = make_double2(fma(-f, U, a.x), fma(-f, V, a.y));
    a = na;
    b = nb;
  }
}
template <bool INV>
__device__ __forceinline__ void bfly32_v(double2 &a, double2 &b, int e) {
  switch (e & 31) {
#define SZ_B32(k) \
  case k: bfly32<k, INV>(a, b); break;
    SZ_B32(0) SZ_B32(2) SZ_B32(4) SZ_B32(6) SZ_B32(8) SZ_B32(10) SZ_B32(12) SZ_B32(14)
#undef SZ_B32
    default: break;
  }
}
template <bool INV, int H>
__device__ __forceinline__ void dit16_stage(double2 (&y)[16]) {
  if constexpr (H <= 8) {
#pragma unroll
    for (int b = 0; b < 16; b += 2 * H)
#pragma unroll
      for (int j = 0; j < H; j++) bfly32_v<INV>(y[b + j], y[b + j + H], j * (16 / H));
    dit16_stage<INV, 2 * H>(y);
  }
}

__host__ __device__ constexpr int bitrev4_(int r) {
  return ((r & 1) << 3) | ((r & 2) << 1) | ((r & 4) >> 1) | ((r & 8) >> 3);
}
#ifndef SZ_DFT16_FMA
#define SZ_DFT16_FMA 1  // 1: dft<16> in FMA-form decimation in time (same contract: natural in, bit-reversed out)
#endif
#if SZ_DFT16_FMA
template <>
__device__ __forceinline__ void dft<16, false>(double2 (&x)[16]) {
  double2 y[16];
#pragma unroll
  for (int r = 0; r < 16; r++) y[r] = x[bitrev4_(r)];
  dit16_stage<false, 1>(y);
#pragma unroll
  for (int r = 0; r < 16; r++) x[r] = y[bitrev4_(r)];
}
template <>
__device__ __forceinline__ void dft<16, true>(double2 (&x)[16]) {
  double2 y[16];
#pragma unroll
  for (int r = 0; r < 16; r++) y[r] = x[bitrev4_(r)];
  dit16_stage<true, 1>(y);
#pragma unroll
  for (int r = 0; r < 16; r++) x[r] = y[bitrev4_(r)];
}
#endif

__host__ __device__ constexpr int bitrev4(int r) {
  return ((r & 1) << 3) | ((r & 2) << 1) | ((r & 4) >> 1) | ((r & 8) >> 3);
}
__host__ __device__ constexpr int bitrev2(int r) { return ((r & 1) << 1) | ((r & 2) >> 1); }

// XOR swizzle of a 16-byte-element index p in [0, 1024) (see header comment).
__device__ __forceinline__ int swz(int p) { return p ^ (((p >> 3) & 3) | (((p >> 6) & 1) << 2)); }

// Twiddle tables in global memory (built once per device, see fft_tables.cu):
//   tw1[k][t] = w^{t (4k+1)}     = e^{i pi t (4k+1) / 2048}, k < 16, t < 64
//   tw2[k][s] = W_64^{s k}       = e^{2 pi i s k / 64},      k < 16, s < 4
//   twist[m]  = w^{64 m}         = e^{i pi m / 32},          m < 16
struct Tables {
  double2 tw1[16 * 64];
  double2 tw2[16 * 4];
  double2 twist[16];
};

}  // namespace sz
