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
