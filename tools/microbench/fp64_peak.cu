// FP64 roofline denominator for bench.py (MEASURED_PEAKS.json has no FP64 entry).
// DFMA chains on every SM, measured two ways (mirroring how the driver measures
// bf16 in MEASURED_PEAKS.json):
//   burst     : best of 10 launches of ~20 ms each (CUDA events);
//   sustained : back-to-back launches for >= 4 s, total flops / total time.
// Several shapes (chains per thread x threads per SM) are tried and the best is
// reported, so the number is the pipe's, not one configuration's.
// Prints one JSON object on stdout; tools/fp64_peak.py adds the clock log.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; i++) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int i = 0; i < CHAINS; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) s += x[i];
  if (s == 1234.5) out[0] = s;
}

struct Shape { int chains, threads, blocks_per_sm; };

template <int C>
static void launch(int blocks, int threads, double* out, int iters, cudaStream_t st) {
  dfma_kernel<C><<<blocks, threads, 0, st>>>(out, iters, 1.0000001, 1e-7);
}

static void launch_shape(const Shape& s, int sms, double* out, int iters, cudaStream_t st) {
  int blocks = sms * s.blocks_per_sm;
  if (s.chains == 8) launch<8>(blocks, s.threads, out, iters, st);
  else if (s.chains == 16) launch<16>(blocks, s.threads, out, iters, st);
  else launch<32>(blocks, s.threads, out, iters, st);
}

int main(int argc, char** argv) {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<Shape> shapes = {{8, 256, 4}, {16, 256, 4}, {16, 512, 2}, {32, 128, 4}, {16, 128, 8}, {8, 512, 4}};
  const int iters = 6000;  // x4 x chains DFMAs per thread per launch
  double best_burst = 0;
  Shape best_shape = shapes[0];
  printf("{\"device\": \"%s\", \"sms\": %d, \"shapes\": [", p.name, sms);
  for (size_t si = 0; si < shapes.size(); si++) {
    const Shape& s = shapes[si];
    double flops = 2.0 * 4 * s.chains * (double)iters * sms * s.blocks_per_sm * s.threads;
    launch_shape(s, sms, out, iters, st);  // warm-up
    CK(cudaStreamSynchronize(st));
    double best = 0;
    for (int rep = 0; rep < 10; rep++) {
      cudaEventRecord(e0, st);
      launch_shape(s, sms, out, iters, st);
      cudaEventRecord(e1, st);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double tf = flops / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
    }
    printf("%s{\"chains\": %d, \"threads\": %d, \"blocks_per_sm\": %d, \"burst_tflops\": %.3f}",
           si ? ", " : "", s.chains, s.threads, s.blocks_per_sm, best);
    if (best > best_burst) { best_burst = best; best_shape = s; }
  }
  // sustained: the best shape back to back for >= 4 s
  const Shape& s = best_shape;
  double flops = 2.0 * 4 * s.chains * (double)iters * sms * s.blocks_per_sm * s.threads;
  fprintf(stderr, "SUSTAINED_START\n");
  fflush(stderr);
  int n = 0;
  float total_ms = 0;
  cudaEventRecord(e0, st);
  while (total_ms < 4000.f) {
    for (int i = 0; i < 20; i++) launch_shape(s, sms, out, iters, st);
    n += 20;
    cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&total_ms, e0, e1);
  }
  fprintf(stderr, "SUSTAINED_END\n");
  double sustained = flops * n / (total_ms * 1e-3) / 1e12;
  printf("], \"burst_tflops\": %.3f, \"sustained_tflops\": %.3f, \"sustained_seconds\": %.3f, "
         "\"sustained_launches\": %d, \"best_shape\": {\"chains\": %d, \"threads\": %d, \"blocks_per_sm\": %d}, "
         "\"launch_ms\": %.3f}\n",
         best_burst, sustained, total_ms * 1e-3, n, s.chains, s.threads, s.blocks_per_sm, total_ms / n);
  return 0;
}
