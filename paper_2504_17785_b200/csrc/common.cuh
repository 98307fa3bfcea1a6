// common.cuh -- shared device/host helpers of libsilenzio (sm_100a).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "silenzio.h"

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;

#define SZ_CUDA_OK(expr)                                   \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return SILENZIO_ERR_CUDA;       \
  } while (0)

#define SZ_LAUNCH_OK()                                     \
  do {                                                     \
    cudaError_t _e = cudaGetLastError();                   \
    if (_e != cudaSuccess) return SILENZIO_ERR_CUDA;       \
  } while (0)

static inline cudaStream_t sz_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

static inline bool sz_aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
static inline bool sz_aligned(const void *p, uintptr_t bytes) { return (reinterpret_cast<uintptr_t>(p) & (bytes - 1)) == 0; }

// Signed gadget decomposition (R3/R4): rounds a to
// the top l*beta bits (half up), then extracts l balanced digits in [-B/2, B/2)
// from least to most significant, propagating carries; the final carry is
// dropped. digit(t) has weight 2^{64 - t*beta}, t = 1..l. Returns the rounded
// value r (l*beta bits) -- callers peel digits themselves.
__device__ __forceinline__ u64 sz_decomp_round(u64 a, int base_log, int level) {
  const int lb = base_log * level;
  if (lb >= 64) return a;
  return (a + (1ull << (63 - lb))) >> (64 - lb);
}

// Peel the least-significant remaining digit from r (in/out).
__device__ __forceinline__ i64 sz_decomp_next(u64 &r, int base_log) {
  const u64 mask = (1ull << base_log) - 1;
  i64 d = (i64)(r & mask);
  r >>= base_log;
  const i64 half = 1ll << (base_log - 1);
  // branch-free carry: if d >= half { d -= B; r += 1 }
  const i64 carry = (d >= half) ? 1 : 0;
  d -= carry << base_log;
  r += (u64)carry;
  return d;
}

// Modulus switch to 2N (C4): round(a * 2N / 2^64) half up, wrapping mod 2N.
__device__ __forceinline__ u32 sz_modswitch(u64 a, int log2_2N) {
  return (u32)((a + (1ull << (63 - log2_2N))) >> (64 - log2_2N));
}
