// limbs.cuh -- exact P-limb split of u64 torus values and exact recombination
// of integer-valued inverse-FFT outputs (R20: P = 3 limbs of 22 bits
// keep every limb product sum below 2^53, so rounding is exact).
#pragma once
#include "common.cuh"

namespace sz {

__device__ __forceinline__ i64 sext(i64 x, int bits) {
  return (bits >= 64) ? x : (i64)((u64)x << (64 - bits)) >> (64 - bits);
}

// Split a u64 torus coefficient into P signed limbs, limb p weighted 2^{p*w};
// the top limb is reduced mod 2^{64-(P-1)w} (its weight makes higher bits vanish).
__device__ __forceinline__ void limb_split(u64 g, int P, int w, double (&l)[3]) {
  if (P == 1) {
    l[0] = (double)(i64)g;
    return;
  }
  const i64 l0 = sext((i64)g, w);
  const u64 rem = (g - (u64)l0) >> w;  // exact: g - l0 = 0 mod 2^w
  l[0] = (double)l0;
  if (P == 2) {
    l[1] = (double)sext((i64)rem, 64 - w);
    return;
  }
  const i64 l1 = sext((i64)rem, w);
  const i64 rem2 = ((i64)rem - l1) >> w;
  l[1] = (double)l1;
  l[2] = (double)sext(rem2, 64 - 2 * w);
}

// double (integer-valued up to rounding) -> round to nearest, mod 2^64
__device__ __forceinline__ u64 f64_to_torus(double x) {
  const double hi = floor(x * 0x1p-32);
  const double lo = fma(hi, -0x1p32, x);  // exact
  return ((u64)__double2ll_rn(hi) << 32) + (u64)__double2ll_rn(lo);
}

// limb p of the inverse transform -> its exact contribution round(x) * 2^{p w} mod 2^64
__device__ __forceinline__ u64 limb_to_torus(double x, int p, int P, int w) {
  if (P == 3 || p > 0) return (u64)__double2ll_rn(x) << (p * w);  // |x| < 2^53: exact
  return f64_to_torus(x);                                          // P <= 2, low limb may exceed 2^53
}

// Exact round-to-nearest (ties to even, as F2I.RN) of a double with |x| < 2^51,
// as a two's-complement u64, on the FP64 pipe: adding 1.5 * 2^52 leaves
// round(x) in the low mantissa bits. The P = 3 limb sums stay below 2^51 with
// overwhelming margin (R20: sigma ~ 2^47.4, 2^51 is > 11 sigma).
__device__ __forceinline__ u64 rint_small(double x) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  return (u64)(__double_as_longlong(x + magic) - __double_as_longlong(magic));
}

}  // namespace sz
