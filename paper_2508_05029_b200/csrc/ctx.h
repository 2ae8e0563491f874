// ctx.h — internal host-side state of a tq context (one per GPU).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tq_gpu.h"

struct tq_ctx {
  int device = 0;
  int sms = 148;
  uint32_t ctas_per_sm = 0;
  cudaStream_t stream = nullptr;
  cudaMemPool_t pool = nullptr;
  uint64_t budget = 0;                 // Device-tier capacity (0 = unlimited)
  std::atomic<uint64_t> in_use{0};     // ledger: allocated bytes
  std::atomic<uint32_t> launches{0};   // kernels launched by this context
  void* pinned = nullptr;              // small pinned readback area (4 KiB)
  std::vector<cudaStream_t> exec_streams;  // engine executor streams (exec_stream)
  std::mutex mu;                       // guards pinned + program cache
  std::map<std::string, void*> prog_cache;  // program bytes -> device copy
  // optional per-kernel CUDA-event timing (tq_profile_*): events recorded on
  // the launching stream around each pipeline kernel
  bool jit = true;                      // NVRTC-specialised pipeline kernels (jit.cu)
  // Host tier kept across engine runs (pinning GBs of memory takes seconds)
  void* host_pool = nullptr;
  uint64_t host_pool_buffers = 0, host_pool_buffer_size = 0;
  void (*host_pool_free)(void*) = nullptr;
  std::atomic<uint64_t> jit_launches{0};
  bool profiling = false;
  struct Ev {
    std::string name;
    cudaEvent_t a, b;
    double bytes;
  };
  std::vector<Ev> evs;
};

namespace tq {

struct Fail {
  int status;
  std::string msg;
};
[[noreturn]] void fail(int status, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define TQ_CUDA(x) ::tq::cuda_check((x), #x)

inline cudaStream_t pick(tq_ctx* c, void* s) { return s ? (cudaStream_t)s : c->stream; }
inline uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

void* dalloc(tq_ctx* c, uint64_t bytes, cudaStream_t st);
void dfree(tq_ctx* c, void* p, uint64_t bytes, cudaStream_t st);

// Ownership record stored in tq_batch.owner for batches this library allocated.
struct Owner {
  tq_ctx* ctx;
  cudaStream_t stream;
  std::vector<std::pair<void*, uint64_t>> bufs;
};

size_t width_of(uint8_t kind);
// Allocate a device batch: per column values (+ zeroed bitmap when want_valid[c]).
void alloc_batch(tq_ctx* c, uint64_t rows, const std::vector<tq_column>& schema, const std::vector<bool>& want_valid,
                 tq_batch* out, cudaStream_t st, const std::vector<uint64_t>* utf8_bytes = nullptr);
void counted_launch(tq_ctx* c);
// begin/end an event-timed region for kernel `name` (no-op unless profiling)
// This thread's small pinned read-back area (4 KiB, portable, device-visible):
// data-dependent counts are copied here and read after a stream sync, with
// no context-wide lock held across the sync (concurrent operators on other
// threads' streams — and a peer rank's collectives — never wait on it).
void* pinned_scratch(tq_ctx* c);
// The context's executor stream `idx` (created on first use, kept for the
// context's lifetime: the engine's Compute / Memory / Pre-loading threads of
// every query reuse them, so stream-ordered pool memory freed by one query is
// reused by the next without new mappings).
cudaStream_t exec_stream(tq_ctx* c, int idx);
int prof_begin(tq_ctx* c, const char* name, cudaStream_t st);
void prof_end(tq_ctx* c, int h, cudaStream_t st);

extern thread_local std::string g_err;

// Host-side phase timing (TQ_HOST_TIMING=1: totals printed at exit).
bool host_timing_on();
void host_timing_add(const char* name, double us);
struct HostTimer {
  const char* name;
  long long t0;
  explicit HostTimer(const char* n);
  ~HostTimer();
};
#define TQ_HT_CAT2(a, b) a##b
#define TQ_HT_CAT(a, b) TQ_HT_CAT2(a, b)
#define TQ_HT(name) ::tq::HostTimer TQ_HT_CAT(_ht_, __LINE__)(name)

template <typename F>
tq_status guard(F&& f) {
  try {
    f();
    return TQ_OK;
  } catch (const Fail& e) {
    g_err = e.msg;
    return e.status;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return TQ_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TQ_INTERNAL;
  }
}

}  // namespace tq
