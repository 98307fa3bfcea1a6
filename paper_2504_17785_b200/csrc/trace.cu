// trace.cu -- PBS sampling inside the gadget drivers (test / debug facility).
//
// The gadget drivers (silenzio_rns_matmul, silenzio_shift2msbs_pm, ...) issue
// their PBS internally, so an oracle replay of "sampled PBS calls of config 3
// and 4" needs their inputs and outputs. While a trace of a
// kind is active, every `stride`-th PBS (global element counter, offset
// `phase`) evaluated by that kind of call site is copied, stream-ordered, into
// the caller's device buffer as one record:
//   [input ciphertext][output ciphertext][test polynomial][global index, lut id]
// kind 0: set-A PBS of the gadget drivers (szg::lookup): big-key LWE in/out;
// kind 1: set-B blind rotation + sample extraction of the 8-bit stage
//         (pbs_b): set-B small-key LWE in, set-B big-key LWE out.
// Nothing is recorded (and nothing changes) while no trace is active.
#include <atomic>
#include <mutex>

#include "common.cuh"

namespace sz {

struct TraceKind {
  std::mutex m;
  std::atomic<bool> on{false};
  u64 *rec = nullptr;
  size_t max = 0, in_words = 0, out_words = 0, lut_words = 0;
  u64 stride = 1, phase = 0, seen = 0, written = 0;
  int status = SILENZIO_OK;
};
static TraceKind g_trace[2];

bool trace_active(int kind) { return kind >= 0 && kind < 2 && g_trace[kind].on.load(std::memory_order_acquire); }

// record the sampled elements of one batched PBS call (luts: [num][lut_words],
// ids: host array or null = lut 0)
void trace_pbs(int kind, const u64 *in, size_t in_words, const u64 *out, size_t out_words, const u64 *luts,
               size_t lut_words, const u32 *ids_host, size_t count, cudaStream_t st) {
  if (!trace_active(kind)) return;
  TraceKind &T = g_trace[kind];
  std::lock_guard<std::mutex> lk(T.m);
  if (!T.on.load() || in_words != T.in_words || out_words != T.out_words || lut_words != T.lut_words) {
    T.seen += count;
    return;
  }
  const size_t words = T.in_words + T.out_words + T.lut_words + 2;
  for (size_t e = 0; e < count; e++) {
    const u64 gi = T.seen + e;
    if (gi % T.stride != T.phase || T.written >= T.max) continue;
    u64 *r = T.rec + T.written * words;
    const u32 id = ids_host ? ids_host[e] : 0u;
    const u64 meta[2] = {gi, id};
    cudaError_t err = cudaMemcpyAsync(r, in + e * in_words, in_words * 8, cudaMemcpyDeviceToDevice, st);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(r + T.in_words, out + e * out_words, out_words * 8, cudaMemcpyDeviceToDevice, st);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(r + T.in_words + T.out_words, luts + (size_t)id * lut_words, lut_words * 8,
                            cudaMemcpyDeviceToDevice, st);
    // meta words are tiny: synchronous host -> device copy on the same stream
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(r + words - 2, meta, sizeof(meta), cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);  // `meta` lives on this stack frame
    if (err != cudaSuccess) T.status = SILENZIO_ERR_CUDA;
    T.written++;
  }
  T.seen += count;
}

}  // namespace sz

extern "C" {

int silenzio_pbs_trace_begin(int kind, uint64_t *records, size_t max_records, uint64_t stride, uint64_t phase,
                             size_t in_words, size_t out_words, size_t lut_words) {
  if (kind < 0 || kind > 1) return SILENZIO_ERR_INVALID_PARAM;
  if (!records && max_records) return SILENZIO_ERR_NULL_POINTER;
  if (stride == 0 || phase >= stride || !in_words || !out_words || !lut_words) return SILENZIO_ERR_INVALID_PARAM;
  sz::TraceKind &T = sz::g_trace[kind];
  std::lock_guard<std::mutex> lk(T.m);
  T.rec = records;
  T.max = max_records;
  T.stride = stride;
  T.phase = phase;
  T.in_words = in_words;
  T.out_words = out_words;
  T.lut_words = lut_words;
  T.seen = 0;
  T.written = 0;
  T.status = SILENZIO_OK;
  T.on.store(true, std::memory_order_release);
  return SILENZIO_OK;
}

long silenzio_pbs_trace_end(int kind, uint64_t *elements_seen) {
  if (kind < 0 || kind > 1) return SILENZIO_ERR_INVALID_PARAM;
  sz::TraceKind &T = sz::g_trace[kind];
  std::lock_guard<std::mutex> lk(T.m);
  T.on.store(false, std::memory_order_release);
  if (elements_seen) *elements_seen = T.seen;
  if (T.status != SILENZIO_OK) return T.status;
  return (long)T.written;
}

}  // extern "C"
