// TMEM round-trip latency: one warp (or W warps) per SM doing
// tcgen05.ld.32x32b.x16 -> tcgen05.wait::ld -> use, serially; and the same
// for an LDS.128 chain for comparison. Prints cycles per round trip.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void tmem_lat(long long *cyc, uint32_t *out, int iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&taddr_s)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t ta = taddr_s + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 16;
  uint32_t acc = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(ta + (acc & 0)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int i = 0; i < 16; i++) acc += r[i];
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr_s), "r"(128));
}

__global__ void tmem_st_lat(long long *cyc, uint32_t *out, int iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&taddr_s)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t ta = taddr_s + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 16;
  uint32_t acc = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    uint32_t r[16];
    // st then ld of the same columns (read-after-write round trip)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(ta), "r"(acc), "r"(acc + 1), "r"(acc + 2), "r"(acc + 3), "r"(acc + 4), "r"(acc + 5), "r"(acc + 6), "r"(acc + 7),
                 "r"(acc + 8), "r"(acc + 9), "r"(acc + 10), "r"(acc + 11), "r"(acc + 12), "r"(acc + 13), "r"(acc + 14), "r"(acc + 15));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int i = 0; i < 16; i++) acc += r[i];
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr_s), "r"(128));
}

__global__ void lds_lat(long long *cyc, uint32_t *out, int iters) {
  __shared__ uint4 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  uint32_t idx = threadIdx.x & 31, acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    uint4 v = buf[(idx + acc) & 1023];
    acc += v.x + v.y + v.z + v.w;
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + (threadIdx.x >> 5)] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  long long *cyc;
  uint32_t *out;
  cudaMalloc(&cyc, 148 * 32 * 8);
  cudaMalloc(&out, 148 * 1024 * 4);
  const int iters = 4096;
  for (int which = 0; which < 3; which++)
    for (int warps : {1, 4, 8}) {
      if (which == 0) tmem_lat<<<148, 32 * warps>>>(cyc, out, iters);
      if (which == 1) tmem_st_lat<<<148, 32 * warps>>>(cyc, out, iters);
      if (which == 2) lds_lat<<<148, 32 * warps>>>(cyc, out, iters);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[32];
      cudaMemcpy(h, cyc, 8 * 32, cudaMemcpyDeviceToHost);
      const char *nm[] = {"tcgen05.ld x16 + wait", "tcgen05.st x16 + wait + ld + wait", "LDS.128 chain"};
      printf("%-36s warps/SM=%d: %.1f cycles per round trip (warp 0)  err=%s\n", nm[which], warps,
             (double)h[0] / iters, cudaGetErrorString(e));
    }
  return 0;
}
