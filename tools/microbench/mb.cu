// Micro-benchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
// FP64 DFMA peak, shared-memory LDS.128 bandwidth, SHFL throughput, L2 read bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
  #pragma unroll
  for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < 16; i++) s += x[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void lds_kernel(double* out, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int j = 0; j < 8; j++) {
      double2 v = buf[(idx + j * 128 + it) & 2047];
      acc.x += v.x; acc.y += v.y;
    }
  }
  if (acc.x == 1234.5) out[0] = acc.y;
}

__global__ void shfl_kernel(double* out, int iters) {
  unsigned v[8];
  #pragma unroll
  for (int i = 0; i < 8; i++) v[i] = threadIdx.x + i;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) v[i] = __shfl_xor_sync(0xffffffff, v[i], (i + 1) & 31);
  }
  unsigned s = 0;
  #pragma unroll
  for (int i = 0; i < 8; i++) s += v[i];
  if (s == 12345) out[0] = s;
}

__global__ void l2_kernel(const double2* __restrict__ src, size_t n_elems, double* out, int reps) {
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < reps; r++)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_elems; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = src[i]; acc.x += v.x; acc.y += v.y;
    }
  if (acc.x == 1234.5) out[0] = acc.y;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d L2 %d MB smemPerSM %zu regsPerSM %d clock %d kHz\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor, p.clockRate);
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // FP64 DFMA: 16 chains/thread, 256 threads, 4 blocks per SM
  for (int rep = 0; rep < 2; rep++) {
    int iters = 20000; int blocks = sms * 4, threads = 256;
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 2; rep++) {
    int iters = 20000; int blocks = sms * 4, threads = 256;
    cudaEventRecord(e0); lds_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 16.0 * 8 * iters * (double)blocks * threads;
    printf("LDS.128: %.2f TB/s chip, %.1f B/clk/SM at %d MHz nominal\n", bytes / ms / 1e9, bytes / (ms * 1e-3) / sms / (p.clockRate * 1e3), p.clockRate / 1000);
  }
  for (int rep = 0; rep < 2; rep++) {
    int iters = 20000; int blocks = sms * 4, threads = 256;
    cudaEventRecord(e0); shfl_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = 8.0 * iters * (double)blocks * threads / 32;  // warp-level shfl instrs
    printf("SHFL: %.3f warp-instr/clk/SM (nominal clock)\n", n / (ms * 1e-3) / sms / (p.clockRate * 1e3));
  }
  // L2 read: 64 MB buffer read repeatedly
  size_t nbytes = 64ull << 20; double2* src; CK(cudaMalloc(&src, nbytes)); CK(cudaMemset(src, 0, nbytes));
  for (int rep = 0; rep < 2; rep++) {
    int reps = 20;
    cudaEventRecord(e0); l2_kernel<<<sms * 8, 512>>>(src, nbytes / 16, out, reps); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("L2 read (64MB x%d): %.2f TB/s\n", reps, nbytes * (double)reps / ms / 1e9);
  }
  size_t big = 4ull << 30; double2* src2; CK(cudaMalloc(&src2, big)); CK(cudaMemset(src2, 0, big));
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0); l2_kernel<<<sms * 8, 512>>>(src2, big / 16, out, 1); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("HBM read (4GB): %.2f TB/s\n", big / ms / 1e9);
  }
  return 0;
}
