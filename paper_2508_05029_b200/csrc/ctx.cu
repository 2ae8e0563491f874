// ctx.cu — context, Device-tier ledger/allocator and batch movement.
//
// Device memory comes from a per-device stream-ordered pool
// (cudaMallocFromPoolAsync) with the release threshold at "never", so a
// steady-state query reuses its buffers without driver calls.  Every
// allocation is charged to the context ledger (SPEC.md:240-276,
// MemoryLedger / alloc_within); exceeding the configured Device capacity
// returns ReservationExceeded, the signal the Compute Executor's on_oom
// retry path consumes.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>

#include "ctx.h"

namespace tq {

thread_local std::string g_err;

namespace {
struct HostTiming {
  std::mutex mu;
  std::map<std::string, std::pair<uint64_t, double>> acc;
  bool on = false;
  HostTiming() {
    const char* e = getenv("TQ_HOST_TIMING");
    on = e && e[0] == '1';
  }
  std::string report() {
    std::lock_guard<std::mutex> g(mu);
    std::string r;
    char line[160];
    for (auto& kv : acc) {
      snprintf(line, sizeof line, "%-28s %8llu calls %10.1f us total %8.2f us/call\n", kv.first.c_str(),
               (unsigned long long)kv.second.first, kv.second.second,
               kv.second.second / std::max<uint64_t>(1, kv.second.first));
      r += line;
    }
    acc.clear();
    return r;
  }
};
HostTiming& host_timing() {
  static HostTiming* h = new HostTiming;  // never destroyed: frees can run during interpreter teardown
  return *h;
}
long long now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
}  // namespace

bool host_timing_on() { return host_timing().on; }
std::string host_timing_report() { return host_timing().report(); }
void host_timing_add(const char* name, double us) {
  HostTiming& h = host_timing();
  std::lock_guard<std::mutex> g(h.mu);
  auto& e = h.acc[name];
  e.first++;
  e.second += us;
}
HostTimer::HostTimer(const char* n) : name(n), t0(host_timing_on() ? now_ns() : 0) {}
HostTimer::~HostTimer() {
  if (t0) host_timing_add(name, (now_ns() - t0) / 1e3);
}

void fail(int status, const std::string& msg) { throw Fail{status, msg}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(TQ_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

namespace {
// Pinned read-back slots are recycled process-wide: a thread takes one on
// first use and hands it back when it exits (the engine starts executor
// threads per query; a cudaHostAlloc / cudaFreeHost pair per thread would
// pin memory and synchronise the device every time).
std::mutex g_pinned_mu;
std::vector<void*>* g_pinned_free = new std::vector<void*>;  // never destroyed
struct PinnedScratch {
  void* p = nullptr;
  ~PinnedScratch() {
    if (!p) return;
    std::lock_guard<std::mutex> g(g_pinned_mu);
    g_pinned_free->push_back(p);
  }
};
thread_local PinnedScratch t_pinned;
}  // namespace

void* pinned_scratch(tq_ctx* c) {
  (void)c;
  if (!t_pinned.p) {
    {
      std::lock_guard<std::mutex> g(g_pinned_mu);
      if (!g_pinned_free->empty()) {
        t_pinned.p = g_pinned_free->back();
        g_pinned_free->pop_back();
      }
    }
    if (!t_pinned.p) TQ_CUDA(cudaHostAlloc(&t_pinned.p, 4096, cudaHostAllocPortable));
  }
  return t_pinned.p;
}

cudaStream_t exec_stream(tq_ctx* c, int idx) {
  std::lock_guard<std::mutex> g(c->mu);
  while ((int)c->exec_streams.size() <= idx) {
    cudaStream_t s;
    TQ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    c->exec_streams.push_back(s);
  }
  return c->exec_streams[idx];
}

void counted_launch(tq_ctx* c) { c->launches.fetch_add(1, std::memory_order_relaxed); }

int prof_begin(tq_ctx* c, const char* name, cudaStream_t st) {
  if (!c->profiling) return -1;
  std::lock_guard<std::mutex> g(c->mu);
  tq_ctx::Ev e{name, nullptr, nullptr, 0};
  cudaEventCreate(&e.a);
  cudaEventCreate(&e.b);
  cudaEventRecord(e.a, st);
  c->evs.push_back(e);
  return (int)c->evs.size() - 1;
}
void prof_end(tq_ctx* c, int h, cudaStream_t st) {
  if (h < 0) return;
  std::lock_guard<std::mutex> g(c->mu);
  cudaEventRecord(c->evs[h].b, st);
}

size_t width_of(uint8_t kind) {
  switch (kind) {
    case TQ_INT64: return 8;
    case TQ_FLOAT64: return 8;
    case TQ_BOOL: return 1;
    case TQ_DECIMAL: return 16;
    default: return 0;
  }
}

void* dalloc(tq_ctx* c, uint64_t bytes, cudaStream_t st) {
  TQ_HT("dalloc");
  uint64_t b = round_up(bytes ? bytes : 1, 256) + 256;  // tail pad: 16-B bulk copies never run off the end
  uint64_t now = c->in_use.fetch_add(b) + b;
  if (c->budget && now > c->budget) {
    c->in_use.fetch_sub(b);
    fail(TQ_RESERVATION_EXCEEDED, "device budget exceeded: need " + std::to_string(now) + " of " +
                                      std::to_string(c->budget) + " bytes");
  }
  void* p = nullptr;
  const long long t0 = host_timing_on() ? now_ns() : 0;
  cudaError_t e = cudaMallocFromPoolAsync(&p, b, c->pool, st);
  if (t0 && now_ns() - t0 > 1000000) {
    unsigned long long res = 0, used = 0;
    cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrReservedMemCurrent, &res);
    cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrUsedMemCurrent, &used);
    fprintf(stderr, "[tq] slow dalloc %.3f ms: %llu bytes on stream %p (pool reserved %.2f GB, used %.2f GB)\n",
            (now_ns() - t0) / 1e6, (unsigned long long)b, (void*)st, res / 1e9, used / 1e9);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    c->in_use.fetch_sub(b);
    fail(TQ_RESERVATION_EXCEEDED, std::string("device allocation failed: ") + cudaGetErrorString(e));
  }
  return p;
}

void dfree(tq_ctx* c, void* p, uint64_t bytes, cudaStream_t st) {
  TQ_HT("dfree");
  if (!p) return;
  uint64_t b = round_up(bytes ? bytes : 1, 256) + 256;
  cudaFreeAsync(p, st);
  c->in_use.fetch_sub(b);
}

void alloc_batch(tq_ctx* c, uint64_t rows, const std::vector<tq_column>& schema, const std::vector<bool>& want_valid,
                 tq_batch* out, cudaStream_t st, const std::vector<uint64_t>* utf8_bytes) {
  Owner* own = new Owner{c, st, {}};
  out->rows = rows;
  out->ncols = (uint32_t)schema.size();
  out->mem = TQ_MEM_DEVICE;
  out->owner = own;
  out->cols = (tq_column*)std::calloc(schema.size() ? schema.size() : 1, sizeof(tq_column));
  try {
    for (size_t i = 0; i < schema.size(); ++i) {
      tq_column& d = out->cols[i];
      d.kind = schema[i].kind;
      d.precision = schema[i].precision;
      d.scale = schema[i].scale;
      uint64_t vb = d.kind == TQ_UTF8 ? (utf8_bytes ? (*utf8_bytes)[i] : 0) : rows * width_of(d.kind);
      d.values_bytes = vb;
      d.values = dalloc(c, vb, st);
      own->bufs.push_back({d.values, vb});
      if (d.kind == TQ_UTF8) {
        uint64_t ob = (rows + 1) * 4;
        d.offsets = (int32_t*)dalloc(c, ob, st);
        own->bufs.push_back({d.offsets, ob});
      }
      if (want_valid[i] && rows > 0) {
        uint64_t bb = (rows + 7) / 8;
        d.validity = (uint8_t*)dalloc(c, bb, st);
        own->bufs.push_back({d.validity, bb});
        TQ_CUDA(cudaMemsetAsync(d.validity, 0, round_up(bb, 4), st));
      }
    }
  } catch (...) {
    tq_batch_free(c, out);
    throw;
  }
}

}  // namespace tq

using namespace tq;

extern "C" {

const char* tq_last_error(void) { return tq::g_err.c_str(); }

const char* tq_errc_name(tq_status s) {
  static const char* names[] = {"OK", "PoolExhausted", "CorruptLayout", "MalformedBatch", "SchemaMismatch", "NotTcf",
                                "CorruptFooter", "UnknownColumn", "CorruptRowGroup", "IoError",
                                "ReservationImpossible", "ReservationExceeded", "NoEligibleVictims",
                                "OutOfMemoryUnsplittable", "CorruptFrame", "PeerDisconnected", "InvalidPlan",
                                "WorkerFailure", "Internal"};
  if (s < 0 || s > TQ_INTERNAL) return "Unknown";
  return names[s];
}

tq_status tq_ctx_create(const tq_opts* opts, tq_ctx** out) {
  return guard([&] {
    int dev = opts ? opts->device : 0;
    int n = 0;
    TQ_CUDA(cudaGetDeviceCount(&n));
    if (dev < 0 || dev >= n) fail(TQ_INTERNAL, "no such CUDA device");
    TQ_CUDA(cudaSetDevice(dev));
    cudaDeviceProp prop;
    TQ_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10) fail(TQ_INTERNAL, "libtq_gpu.so is built for sm_100a (B200) only");
    tq_ctx* c = new tq_ctx();
    c->device = dev;
    c->sms = prop.multiProcessorCount;
    c->ctas_per_sm = opts ? opts->ctas_per_sm : 0;
    c->budget = opts ? opts->device_budget_bytes : 0;
    TQ_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    // a pool of our own (not the device's default pool, which other libraries
    // in the process — NCCL, PyTorch — may trim or reconfigure): memory it has
    // mapped stays mapped (release threshold = never), so steady-state
    // allocations are reuse, never a new physical mapping (~25 ms per GB)
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    TQ_CUDA(cudaMemPoolCreate(&c->pool, &props));
    uint64_t thresh = ~0ull;
    TQ_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thresh));
    int on = 1;
    TQ_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowOpportunistic, &on));
    TQ_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowInternalDependencies, &on));
    TQ_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseFollowEventDependencies, &on));
    TQ_CUDA(cudaHostAlloc(&c->pinned, 4096, cudaHostAllocPortable));
    if (opts && opts->pool_reserve_bytes) {
      void* p = nullptr;
      if (cudaMallocFromPoolAsync(&p, opts->pool_reserve_bytes, c->pool, c->stream) == cudaSuccess) {
        cudaFreeAsync(p, c->stream);
        TQ_CUDA(cudaStreamSynchronize(c->stream));
      } else {
        cudaGetLastError();
      }
    }
    *out = c;
  });
}

void tq_ctx_destroy(tq_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& kv : c->prog_cache) cudaFree(kv.second);
  if (c->host_pool && c->host_pool_free) c->host_pool_free(c->host_pool);
  cudaFreeHost(c->pinned);
  for (cudaStream_t s : c->exec_streams) {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  cudaStreamDestroy(c->stream);
  cudaMemPoolDestroy(c->pool);  // (outstanding allocations keep it alive until freed)
  delete c;
}

tq_status tq_sync(tq_ctx* c, void* stream) {
  return guard([&] { TQ_CUDA(cudaStreamSynchronize(pick(c, stream))); });
}

uint64_t tq_device_bytes_in_use(tq_ctx* c) { return c->in_use.load(); }

uint64_t tq_device_bytes_reserved(tq_ctx* c) {
  unsigned long long v = 0;
  cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrReservedMemCurrent, &v);
  return (uint64_t)v;
}

void tq_profile_enable(tq_ctx* c, int on) {
  std::lock_guard<std::mutex> g(c->mu);
  c->profiling = on != 0;
}

// Synchronise, then write "name count total_ms\n" lines (summed per kernel
// name) into buf and clear the recorded events.  Returns bytes written.
uint64_t tq_profile_report(tq_ctx* c, char* buf, uint64_t cap) {
  cudaStreamSynchronize(c->stream);
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> g(c->mu);
  std::map<std::string, std::pair<int, double>> agg;
  for (auto& e : c->evs) {
    float ms = 0;
    cudaEventElapsedTime(&ms, e.a, e.b);
    auto& x = agg[e.name];
    x.first += 1;
    x.second += ms;
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  c->evs.clear();
  std::string out;
  for (auto& kv : agg)
    out += kv.first + " " + std::to_string(kv.second.first) + " " + std::to_string(kv.second.second) + "\n";
  uint64_t n = std::min<uint64_t>(out.size(), cap ? cap - 1 : 0);
  if (cap) {
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return n;
}

void* tq_ctx_stream(tq_ctx* c) { return (void*)c->stream; }

tq_status tq_pinned_alloc(uint64_t bytes, void** out) {
  return guard([&] { TQ_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable)); });
}
void tq_pinned_free(void* p) {
  if (p) cudaFreeHost(p);
}
uint32_t tq_kernel_launches(tq_ctx* c) { return c->launches.load(); }

tq_status tq_batch_alloc(tq_ctx* c, const tq_batch* like, uint64_t rows, tq_batch* out, void* stream) {
  return guard([&] {
    std::vector<tq_column> sch(like->cols, like->cols + like->ncols);
    std::vector<bool> wv;
    for (uint32_t i = 0; i < like->ncols; ++i) {
      if (like->cols[i].kind == TQ_UTF8) fail(TQ_INVALID_PLAN, "tq_batch_alloc: utf8 needs byte sizes");
      wv.push_back(like->cols[i].validity != nullptr);
    }
    alloc_batch(c, rows, sch, wv, out, pick(c, stream));
  });
}

tq_status tq_batch_upload(tq_ctx* c, const tq_batch* h, tq_batch* out, void* stream) {
  return guard([&] {
    cudaStream_t st = pick(c, stream);
    std::vector<tq_column> sch(h->cols, h->cols + h->ncols);
    std::vector<bool> wv;
    std::vector<uint64_t> ub;
    for (uint32_t i = 0; i < h->ncols; ++i) {
      wv.push_back(h->cols[i].validity != nullptr);
      ub.push_back(h->cols[i].values_bytes);
      if (h->cols[i].kind != TQ_UTF8 && h->cols[i].values_bytes != h->rows * width_of(h->cols[i].kind))
        fail(TQ_MALFORMED_BATCH, "values length mismatch");
    }
    alloc_batch(c, h->rows, sch, wv, out, st, &ub);
    for (uint32_t i = 0; i < h->ncols; ++i) {
      const tq_column& s = h->cols[i];
      tq_column& d = out->cols[i];
      if (s.values_bytes) TQ_CUDA(cudaMemcpyAsync(d.values, s.values, s.values_bytes, cudaMemcpyHostToDevice, st));
      if (d.validity && h->rows)
        TQ_CUDA(cudaMemcpyAsync(d.validity, s.validity, (h->rows + 7) / 8, cudaMemcpyHostToDevice, st));
      if (s.kind == TQ_UTF8)
        TQ_CUDA(cudaMemcpyAsync(d.offsets, s.offsets, (h->rows + 1) * 4, cudaMemcpyHostToDevice, st));
    }
  });
}

tq_status tq_batch_download(tq_ctx* c, const tq_batch* d, tq_batch* out, void* stream) {
  return guard([&] {
    cudaStream_t st = pick(c, stream);
    out->rows = d->rows;
    out->ncols = d->ncols;
    out->mem = TQ_MEM_HOST;
    out->owner = nullptr;
    out->cols = (tq_column*)std::calloc(d->ncols ? d->ncols : 1, sizeof(tq_column));
    for (uint32_t i = 0; i < d->ncols; ++i) {
      const tq_column& s = d->cols[i];
      tq_column& h = out->cols[i];
      h.kind = s.kind;
      h.precision = s.precision;
      h.scale = s.scale;
      h.values_bytes = s.values_bytes;
      h.values = std::malloc(s.values_bytes ? s.values_bytes : 1);
      if (s.values_bytes) TQ_CUDA(cudaMemcpyAsync(h.values, s.values, s.values_bytes, cudaMemcpyDeviceToHost, st));
      if (s.validity && d->rows) {
        h.validity = (uint8_t*)std::malloc((d->rows + 7) / 8);
        TQ_CUDA(cudaMemcpyAsync(h.validity, s.validity, (d->rows + 7) / 8, cudaMemcpyDeviceToHost, st));
      }
      if (s.kind == TQ_UTF8) {
        h.offsets = (int32_t*)std::malloc((d->rows + 1) * 4);
        TQ_CUDA(cudaMemcpyAsync(h.offsets, s.offsets, (d->rows + 1) * 4, cudaMemcpyDeviceToHost, st));
      }
    }
    TQ_CUDA(cudaStreamSynchronize(st));
  });
}

void tq_batch_free(tq_ctx* c, tq_batch* b) {
  if (!b) return;
  if (b->owner) {
    // Released in the context stream's order: work on other streams that
    // still reads the batch must be synchronised by the caller first (the
    // producing stream may be gone by now, e.g. an executor thread's).
    Owner* o = (Owner*)b->owner;
    for (auto& pb : o->bufs) dfree(o->ctx, pb.first, pb.second, o->ctx->stream);
    delete o;
  }
  (void)c;
  std::free(b->cols);
  b->cols = nullptr;
  b->ncols = 0;
  b->rows = 0;
  b->owner = nullptr;
}

void tq_host_batch_free(tq_batch* b) {
  if (!b || !b->cols) return;
  for (uint32_t i = 0; i < b->ncols; ++i) {
    std::free(b->cols[i].values);
    std::free(b->cols[i].validity);
    std::free(b->cols[i].offsets);
  }
  std::free(b->cols);
  b->cols = nullptr;
}

}  // extern "C"

extern "C" uint64_t tq_host_timing_report(char* buf, uint64_t cap) {
  std::string r = tq::host_timing_report();
  uint64_t n = std::min<uint64_t>(r.size(), cap ? cap - 1 : 0);
  if (cap) {
    std::memcpy(buf, r.data(), n);
    buf[n] = 0;
  }
  return n;
}
