// engine.cu — worker runtime (include/tq_engine.h): BatchHolders, the
// Memory / Pre-loading / Compute executors and the query DAGs, driving the
// GPU operators of libtq_gpu.so on one GPU.  Host code only.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tq_engine.h"
#include "ctx.h"

namespace tq {
namespace exec {

using Clock = std::chrono::steady_clock;

// ------------------------------------------------------------------ expression builder (prefix order)
struct EB {
  std::vector<tq_expr_node> n;
  EB& col(uint32_t c) { tq_expr_node x{}; x.tag = TQ_EX_COL; x.column = c; n.push_back(x); return *this; }
  EB& i64(int64_t v) { tq_expr_node x{}; x.tag = TQ_EX_LIT; x.kind = TQ_INT64; x.lo = (uint64_t)v; n.push_back(x); return *this; }
  EB& dec(int64_t v, uint8_t s = 2) {
    tq_expr_node x{}; x.tag = TQ_EX_LIT; x.kind = TQ_DECIMAL; x.scale = s; x.lo = (uint64_t)v; x.hi = v < 0 ? ~0ull : 0;
    n.push_back(x); return *this;
  }
  EB& cmp(int op) { tq_expr_node x{}; x.tag = TQ_EX_CMP; x.op = (uint8_t)op; n.push_back(x); return *this; }
  EB& ar(int op) { tq_expr_node x{}; x.tag = TQ_EX_ARITH; x.op = (uint8_t)op; n.push_back(x); return *this; }
  EB& land() { tq_expr_node x{}; x.tag = TQ_EX_AND; n.push_back(x); return *this; }
  tq_expr e() const { return tq_expr{n.data(), (uint32_t)n.size(), 0}; }
};
EB Col(uint32_t c) { EB b; b.col(c); return b; }

// ------------------------------------------------------------------ handles / holders
enum Tier { DEVICE = 0, HOST = 1 };

struct Handle {
  uint64_t id = 0;
  int tier = DEVICE;
  uint64_t bytes = 0;
  int pins = 0;
  bool view = false;  // borrows an input table's device memory: never freed or spilled
  bool spilling = false;  // chosen as a spill victim (under rt->mu); the copy runs outside it
  tq_batch dev{};
  tq_chunked* host = nullptr;
  std::mutex mu;
};
using HP = std::shared_ptr<Handle>;

uint64_t batch_bytes(const tq_batch& b) {  // batch_size_bytes (types.cpp:166-170)
  uint64_t t = 0;
  for (uint32_t i = 0; i < b.ncols; ++i) {
    t += b.cols[i].values_bytes;
    if (b.cols[i].validity && b.rows) t += (b.rows + 7) / 8;
    if (b.cols[i].kind == TQ_UTF8) t += (b.rows + 1) * 4;
  }
  return t;
}

void check(tq_status s) {
  if (s != TQ_OK) fail(s, g_err);
}

struct OpStat {
  uint64_t tasks = 0;
  double ms = 0;
  std::atomic<uint64_t> rows_out{0};
};

class Runtime;

class Holder {
 public:
  explicit Holder(Runtime* rt) : rt_(rt) {}
  void push(HP h);  // never fails
  void close();
  void close_locked() { closed_ = true; }
  // caller holds rt->mu
  bool empty() const { return q_.empty(); }
  bool closed() const { return closed_; }
  HP pop() {
    HP h = q_.front();
    q_.pop_front();
    return h;
  }
  const std::deque<HP>& items() const { return q_; }

 private:
  Runtime* rt_;
  std::deque<HP> q_;
  bool closed_ = false;
};

struct Task {
  class Op* op = nullptr;
  std::vector<HP> inputs;
  int attempt = 1;
  uint64_t estimate = 0;
  uint64_t seq = 0;
  int kind = 0;  // op-defined
};

class Op {
 public:
  Op(Runtime* rt, std::string name, int depth, double mult) : rt(rt), name(std::move(name)), depth(depth), mult(mult) {}
  virtual ~Op() = default;
  // coordinator, under rt->mu: append runnable tasks
  virtual void poll(std::vector<Task>& out) = 0;
  // compute thread
  virtual void run(Task& t, cudaStream_t st) = 0;
  virtual bool splittable(const Task& t) const { return t.inputs.size() > 1; }
  Runtime* rt;
  std::string name;
  int depth;
  double mult;  // default reservation multiplier
  int running = 0;
  bool finished = false;
  Holder* out = nullptr;
  // OperatorStats
  uint64_t samples = 0;
  double ema_peak = 0, ema_ratio = 0;
  OpStat stat;
};

// ------------------------------------------------------------------ runtime
class Runtime {
 public:
  Runtime(tq_ctx* c, tq_comm* comm, const tq_engine_opts& o) : ctx(c), comm(comm), opts(o) {}
  ~Runtime();
  void setup();
  void run();

  HP adopt(const tq_batch& b, bool view) {
    HP h = std::make_shared<Handle>();
    h->dev = b;
    h->view = view;
    h->tier = DEVICE;
    h->bytes = batch_bytes(b);
    std::lock_guard<std::mutex> g(mu);
    h->id = ++next_id;
    registry.push_back(h);
    return h;
  }
  void free_handle(HP h) {
    std::lock_guard<std::mutex> g(h->mu);
    if (h->tier == DEVICE && !h->view && h->dev.cols) tq_batch_free(ctx, &h->dev);
    if (h->host) {
      tq_chunked_release(h->host);
      h->host = nullptr;
    }
  }
  // Device -> Host.  Runs WITHOUT rt->mu: the victim was
  // chosen and marked (spilling, pinned) under it by pick_victims, so no task
  // uses it meanwhile; a task that later wants it waits on h->mu and then
  // finds it in the Host tier (load_to_device).  The D2H copies go on the
  // memory executor's copy stream; only the spilling thread waits for them.
  bool spill(HP h) {
    std::lock_guard<std::mutex> g(h->mu);
    if (h->tier != DEVICE || h->view || !h->dev.cols) return false;
    tq_chunked* cb = nullptr;
    if (tq_spill(ctx, pool, &h->dev, &cb, copy_stream) != TQ_OK) return false;  // PoolExhausted: keep on Device
    cudaStreamSynchronize(copy_stream);
    tq_batch_free(ctx, &h->dev);
    h->host = cb;
    h->tier = HOST;
    m_spills++;
    m_spill_bytes += h->bytes;
    return true;
  }
  // Host -> Device (load_to_device)
  void load(HP h, cudaStream_t st, bool preload) {
    std::lock_guard<std::mutex> g(h->mu);
    if (h->tier == DEVICE) return;
    tq_batch b{};
    check(tq_load(ctx, h->host, &b, st));
    cudaStreamSynchronize(st);
    tq_chunked_release(h->host);
    h->host = nullptr;
    h->dev = b;
    h->tier = DEVICE;
    (preload ? m_preloads : m_loads)++;
    m_load_bytes += h->bytes;
  }
  uint64_t device_in_use() const { return ctx->in_use.load(); }
  // spill unpinned Device handles, farthest from execution first, until `need`
  // more bytes fit under the capacity; protects the top-K queued tasks' inputs
  // (select_spill_victims).  Caller holds mu.
  // Choose spill victims so that `need` more bytes fit under `limit`; marks
  // them (spilling + pinned) and returns them.  Caller holds mu.
  std::vector<HP> pick_victims(uint64_t need, uint64_t limit);
  // Spill the victims (caller does NOT hold mu), then unmark them.
  void spill_victims(std::vector<HP>& v);
  // High watermark: queue victims down to the low watermark
  // for the memory executor thread.  Caller holds mu.
  void watermark_tick();
  void submit(Task t) {
    t.seq = ++next_seq;
    queue.push_back(std::move(t));
    cv.notify_all();
  }
  void notify() { cv.notify_all(); }
  Holder* holder() {
    holders.emplace_back(new Holder(this));
    return holders.back().get();
  }
  template <class T, class... A>
  T* op(A&&... a) {
    T* p = new T(this, std::forward<A>(a)...);
    ops.emplace_back(p);
    return p;
  }

  tq_ctx* ctx;
  tq_comm* comm;
  tq_engine_opts opts;
  tq_pool* pool = nullptr;
  uint64_t capacity = 0;
  cudaStream_t copy_stream = nullptr, preload_stream = nullptr;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::unique_ptr<Op>> ops;
  std::vector<std::unique_ptr<Holder>> holders;
  std::vector<Task> queue;
  std::vector<std::weak_ptr<Handle>> registry;
  uint64_t next_id = 0, next_seq = 0, reserved = 0;
  int running_tasks = 0;
  int executing = 0;  // tasks past their reservation (the ones that can free memory)
  bool stop = false;
  std::exception_ptr error;
  int exchange_turn = 0;  // collectives run in DAG order on every worker
  // metrics
  std::atomic<uint64_t> m_tasks{0}, m_retries{0}, m_splits{0}, m_spills{0}, m_spill_bytes{0}, m_loads{0},
      m_preloads{0}, m_load_bytes{0}, m_peak{0}, m_injected{0};
  uint64_t spilling_bytes = 0;           // Device bytes of marked victims not yet freed (under mu)
  std::deque<std::vector<HP>> spill_q;   // watermark spills for the memory executor (under mu)
  std::vector<HP> keep;  // handles alive until the query ends (build sides)
  std::vector<tq_batch> results;

 private:
  void worker(int idx);
  void preloader();
  void memory_executor();
  void run_task(Task& t, cudaStream_t st);
  bool pick(Task& t);
};

void Holder::push(HP h) {
  {
    std::lock_guard<std::mutex> g(rt_->mu);
    q_.push_back(std::move(h));
    rt_->watermark_tick();
  }
  rt_->notify();
}
void Holder::close() {
  {
    std::lock_guard<std::mutex> g(rt_->mu);
    closed_ = true;
  }
  rt_->notify();
}

std::vector<HP> Runtime::pick_victims(uint64_t need, uint64_t limit) {
  std::vector<HP> out;
  auto projected = [&] { return device_in_use() - std::min(device_in_use(), spilling_bytes); };
  if (projected() + need <= limit) return out;
  std::set<Handle*> protect;
  std::vector<const Task*> top;
  for (const Task& t : queue) top.push_back(&t);
  std::sort(top.begin(), top.end(), [](const Task* a, const Task* b) { return a->seq < b->seq; });
  for (size_t i = 0; i < top.size() && i < opts.protect_top_k; ++i)
    for (const HP& h : top[i]->inputs) protect.insert(h.get());
  // candidates (select_spill_victims): unpinned Device
  // handles not feeding the top-K queued tasks, newest (deepest) first
  std::vector<HP> cand;
  for (auto& w : registry)
    if (HP h = w.lock())
      if (h->tier == DEVICE && !h->view && !h->spilling && h->pins == 0 && h->dev.cols && !protect.count(h.get()))
        cand.push_back(h);
  std::sort(cand.begin(), cand.end(), [](const HP& a, const HP& b) { return a->id > b->id; });
  for (HP& h : cand) {
    if (projected() + need <= limit) break;
    h->spilling = true;
    h->pins++;
    spilling_bytes += h->bytes;
    out.push_back(h);
  }
  return out;
}

void Runtime::spill_victims(std::vector<HP>& v) {
  for (HP& h : v) spill(h);
  std::lock_guard<std::mutex> g(mu);
  for (HP& h : v) {
    h->spilling = false;
    h->pins--;
    spilling_bytes -= std::min(spilling_bytes, h->bytes);
  }
  cv.notify_all();
}

void Runtime::watermark_tick() {
  if (!capacity) return;
  uint64_t use = device_in_use();
  m_peak = std::max<uint64_t>(m_peak.load(), use);
  if (use >= (uint64_t)(opts.high_watermark * capacity)) {
    std::vector<HP> v = pick_victims(0, (uint64_t)(opts.low_watermark * capacity));
    if (!v.empty()) {
      spill_q.push_back(std::move(v));
      cv.notify_all();
    }
  }
}

// Memory executor (one thread): performs the watermark
// spills queued by BatchHolder pushes, so the pushing compute thread and
// everyone waiting on rt->mu keep running while the D2H copies proceed.
void Runtime::memory_executor() {
  cudaSetDevice(ctx->device);
  for (;;) {
    std::vector<HP> v;
    {
      std::unique_lock<std::mutex> g(mu);
      cv.wait(g, [&] { return stop || !spill_q.empty(); });
      if (spill_q.empty()) break;  // stop
      v = std::move(spill_q.front());
      spill_q.pop_front();
    }
    spill_victims(v);
  }
}

bool Runtime::pick(Task& t) {
  // PriorityKey: starvation boost (probe side of a join whose
  // build is ready) > best input tier (Device first) > plan depth (deeper first) > seq
  if (queue.empty()) return false;
  auto key = [](const Task& a) {
    int tier = DEVICE;
    for (const HP& h : a.inputs) tier = std::max(tier, h->tier);
    return std::make_tuple(tier, -a.op->depth, a.seq);
  };
  size_t best = 0;
  for (size_t i = 1; i < queue.size(); ++i)
    if (key(queue[i]) < key(queue[best])) best = i;
  t = std::move(queue[best]);
  queue.erase(queue.begin() + best);
  return true;
}

uint64_t estimate(const Op& op, uint64_t input_bytes) {
  return tq_estimate_reservation(op.samples, op.ema_peak, op.ema_ratio, input_bytes, op.mult, 1.25);
}

void Runtime::run_task(Task& t, cudaStream_t st) {
  Op* op = t.op;
  uint64_t in_bytes = 0, host_bytes = 0;
  for (HP& h : t.inputs) {
    in_bytes += h->bytes;
    if (h->tier == HOST) host_bytes += h->bytes;
  }
  if (!t.estimate) t.estimate = estimate(*op, in_bytes);
  // ---- reserve(Device, estimate): new allocations only
  const uint64_t want = t.estimate > in_bytes ? t.estimate - in_bytes + host_bytes : host_bytes;
  {
    std::unique_lock<std::mutex> g(mu);
    if (capacity) {
      while (device_in_use() + reserved + want > capacity) {
        std::vector<HP> v = pick_victims(reserved + want, capacity);
        if (!v.empty()) {  // spill outside the lock, then re-check
          g.unlock();
          spill_victims(v);
          g.lock();
          continue;
        }
        if (executing == 0 && spilling_bytes == 0) break;  // nobody can free memory: try it, on_oom on failure
        cv.wait_for(g, std::chrono::milliseconds(2));
      }
    }
    reserved += want;
    executing++;
    for (HP& h : t.inputs) h->pins++;
  }
  auto release = [&] {
    std::lock_guard<std::mutex> g(mu);
    executing--;
    reserved -= want;
    for (HP& h : t.inputs) h->pins--;
    cv.notify_all();
  };
  const uint64_t before = device_in_use();
  auto t0 = Clock::now();
  try {
    // test-only fault injection (tq_engine_opts.inject_oom_*): the named
    // operator's next tasks fail with ReservationExceeded before executing
    if (opts.inject_oom_count && op->name == opts.inject_oom_op &&
        m_injected.fetch_add(1) < opts.inject_oom_count) {
      if (opts.inject_oom_mode == 2) t.estimate = std::max<uint64_t>(t.estimate, capacity);  // oversize
      fail(TQ_RESERVATION_EXCEEDED, op->name + ": injected");
    }
    for (HP& h : t.inputs) load(h, st, false);  // load_to_device
    op->run(t, st);                             // execute + deposit (all-or-nothing per task)
    cudaStreamSynchronize(st);
  } catch (const Fail& f) {
    release();
    if (f.status == TQ_RESERVATION_EXCEEDED) {  // on_oom
      uint64_t est = 0;
      const int action = tq_on_oom_decide(t.estimate, capacity, op->splittable(t) ? 1 : 0, &est);
      std::vector<HP> v;
      {
        std::lock_guard<std::mutex> g(mu);
        // the Device may be full of other operators' data: spill what we can
        if (capacity) v = pick_victims(capacity, capacity);
      }
      spill_victims(v);
      std::lock_guard<std::mutex> g(mu);
      if (action == TQ_OOM_RETRY) {
        Task r = t;
        r.estimate = est;
        r.attempt++;
        m_retries++;
        op->running++;
        submit(std::move(r));
      } else if (action == TQ_OOM_SPLIT) {
        op->running += 2;
        m_splits++;
        Task a = t, b = t;
        size_t half = t.inputs.size() / 2;
        a.inputs.assign(t.inputs.begin(), t.inputs.begin() + half);
        b.inputs.assign(t.inputs.begin() + half, t.inputs.end());
        a.estimate = b.estimate = 0;
        submit(std::move(a));
        submit(std::move(b));
      } else {
        fail(TQ_OUT_OF_MEMORY_UNSPLITTABLE, op->name + ": " + f.msg);
      }
      return;
    }
    throw;
  }
  const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
  const uint64_t peak = std::max<uint64_t>(device_in_use(), before) - std::min<uint64_t>(device_in_use(), before);
  {
    std::lock_guard<std::mutex> g(mu);
    // stats from successful tasks only (EMA alpha 0.3)
    const double a = 0.3;
    double ratio = in_bytes ? (double)peak / (double)in_bytes : 0;
    if (op->samples == 0) {
      op->ema_peak = (double)peak;
      op->ema_ratio = ratio;
    } else {
      op->ema_peak = a * peak + (1 - a) * op->ema_peak;
      op->ema_ratio = a * ratio + (1 - a) * op->ema_ratio;
    }
    op->samples++;
    op->stat.tasks++;
    op->stat.ms += ms;
  }
  release();
  m_tasks++;
}

void Runtime::worker(int idx) {
  cudaSetDevice(ctx->device);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);  // one stream per Compute thread
  for (;;) {
    Task t;
    {
      std::unique_lock<std::mutex> g(mu);
      cv.wait(g, [&] { return stop || !queue.empty(); });
      if (stop) break;
      if (!pick(t)) continue;
      running_tasks++;
    }
    try {
      run_task(t, st);
    } catch (...) {
      std::lock_guard<std::mutex> g(mu);
      if (!error) error = std::current_exception();
    }
    {
      std::lock_guard<std::mutex> g(mu);
      running_tasks--;
      t.op->running--;
      cv.notify_all();
    }
  }
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  (void)idx;
}

// Pre-loading executor: promote Host-resident inputs of the first queued
// tasks to Device while Device headroom >= 15%.
void Runtime::preloader() {
  cudaSetDevice(ctx->device);
  for (;;) {
    HP h;
    {
      std::unique_lock<std::mutex> g(mu);
      cv.wait_for(g, std::chrono::milliseconds(1));
      if (stop) break;
      if (capacity && device_in_use() + reserved > (uint64_t)(0.85 * capacity)) continue;
      std::vector<const Task*> top;
      for (const Task& t : queue) top.push_back(&t);
      std::sort(top.begin(), top.end(), [](const Task* a, const Task* b) { return a->seq < b->seq; });
      for (size_t i = 0; i < top.size() && i < 4 && !h; ++i)
        for (const HP& x : top[i]->inputs)
          if (x->tier == HOST && x->pins == 0) {
            h = x;
            break;
          }
      if (!h) continue;
      h->pins++;
    }
    try {
      load(h, preload_stream, true);
    } catch (...) {
    }
    std::lock_guard<std::mutex> g(mu);
    h->pins--;
  }
}

void Runtime::run() {
  std::vector<std::thread> threads;
  for (uint32_t i = 0; i < std::max<uint32_t>(1, opts.compute_threads); ++i) threads.emplace_back(&Runtime::worker, this, i);
  if (opts.preload) threads.emplace_back(&Runtime::preloader, this);
  threads.emplace_back(&Runtime::memory_executor, this);
  // coordinator: poll operators for runnable tasks until every operator finished
  {
    std::unique_lock<std::mutex> g(mu);
    for (;;) {
      if (error) break;
      bool all = true;
      for (auto& o : ops) {
        if (o->finished) continue;
        std::vector<Task> ts;
        o->poll(ts);
        for (Task& t : ts) {
          o->running++;
          submit(std::move(t));
        }
        if (o->finished && o->out && !o->out->closed()) {
          o->out->close_locked();  // EndOfStream after the last output
          cv.notify_all();
        }
        all = all && o->finished;
      }
      if (all) break;
      cv.wait_for(g, std::chrono::milliseconds(1));
    }
    stop = true;
    cv.notify_all();
  }
  for (auto& t : threads) t.join();
  if (error) std::rethrow_exception(error);
}

Runtime::~Runtime() {
  for (auto& w : registry)
    if (HP h = w.lock()) {
      if (h->tier == DEVICE && !h->view && h->dev.cols) tq_batch_free(ctx, &h->dev);
      if (h->host) tq_chunked_release(h->host);
      h->host = nullptr;
      h->dev.cols = nullptr;
    }
  // the pool belongs to the context (reused by the next query)
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (preload_stream) cudaStreamDestroy(preload_stream);
}

void Runtime::setup() {
  cudaSetDevice(ctx->device);
  cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&preload_stream, cudaStreamNonBlocking);
  if (opts.pool_capacity) {
    const uint64_t bs = opts.pool_buffer_size ? opts.pool_buffer_size : (1 << 20);
    if (ctx->host_pool && ctx->host_pool_buffer_size == bs && ctx->host_pool_buffers >= opts.pool_capacity &&
        tq_pool_free_count((tq_pool*)ctx->host_pool) == ctx->host_pool_buffers) {
      pool = (tq_pool*)ctx->host_pool;  // reuse the context's pinned Host tier
    } else {
      if (ctx->host_pool) ctx->host_pool_free(ctx->host_pool);
      ctx->host_pool = nullptr;
      check(tq_pool_create(bs, opts.pool_capacity, &pool));
      ctx->host_pool = pool;
      ctx->host_pool_buffers = opts.pool_capacity;
      ctx->host_pool_buffer_size = bs;
      ctx->host_pool_free = [](void* p) { tq_pool_destroy((tq_pool*)p); };
    }
  }
}

// ------------------------------------------------------------------ operators
// Scan: splits a device table into row-group batches (zero-copy views); with
// tables_on_host each batch is first moved to the Host tier so scan tasks go
// through load_to_device.
class ScanOp : public Op {
 public:
  ScanOp(Runtime* rt, std::string n, const tq_batch* table) : Op(rt, std::move(n), 0, 4.0), table(*table) {}
  void poll(std::vector<Task>&) override {
    // (under rt->mu) publish every batch once, then close the output
    std::vector<HP> hs;
    uint64_t br = rt->opts.batch_rows ? rt->opts.batch_rows : (16u << 20);
    br = std::max<uint64_t>(512, br / 512 * 512);  // tile-aligned views stay 16-B aligned for TMA
    for (uint64_t r = 0; r < table.rows || (r == 0 && table.rows == 0); r += br) {
      uint64_t n = std::min<uint64_t>(br, table.rows - r);
      tq_batch v{};
      v.rows = n;
      v.ncols = table.ncols;
      v.mem = TQ_MEM_DEVICE;
      views.emplace_back(table.ncols);
      for (uint32_t c = 0; c < table.ncols; ++c) {
        tq_column col = table.cols[c];
        size_t w = width_of(col.kind);
        col.values = (uint8_t*)col.values + r * w;
        col.values_bytes = n * w;
        if (col.validity) col.validity = col.validity + r / 8;
        views.back()[c] = col;
      }
      v.cols = views.back().data();
      hs.push_back(mk(v));
      if (table.rows == 0) break;
    }
    for (HP& h : hs) out_q.push_back(h);
    finished = true;
    // pushes happen outside the coordinator lock
    pending = std::move(hs);
  }
  void run(Task&, cudaStream_t) override {}
  HP mk(const tq_batch& v) {
    HP h = std::make_shared<Handle>();
    h->dev = v;
    h->view = true;
    h->tier = DEVICE;
    h->bytes = batch_bytes(v);
    h->id = ++rt->next_id;
    rt->registry.push_back(h);
    return h;
  }
  tq_batch table;
  std::deque<std::vector<tq_column>> views;
  std::vector<HP> out_q, pending;
};

// Filter -> Project (one fused GPU pipeline per input batch).  A task takes up
// to opts.task_batches batches; its outputs are deposited only after every
// input succeeded (a failed task can be retried or split without duplicates).
void run_all_or_nothing(Runtime* rt, Op* op, Task& t, cudaStream_t st,
                        const std::function<void(const tq_batch&, tq_batch&)>& body) {
  std::vector<tq_batch> outs;
  try {
    for (HP& h : t.inputs) {
      tq_batch o{};
      body(h->dev, o);
      outs.push_back(o);
    }
    cudaStreamSynchronize(st);
  } catch (...) {
    cudaStreamSynchronize(st);
    for (tq_batch& o : outs) tq_batch_free(rt->ctx, &o);
    throw;
  }
  for (tq_batch& o : outs) {
    op->stat.rows_out += o.rows;
    op->out->push(rt->adopt(o, false));
  }
  for (HP& h : t.inputs)
    if (!h->view) rt->free_handle(h);
}

void poll_batches(Runtime* rt, Op* op, Holder* in, std::vector<Task>& ts) {
  const size_t k = std::max<uint32_t>(1, rt->opts.task_batches);
  while (!in->empty()) {
    Task t;
    t.op = op;
    while (!in->empty() && t.inputs.size() < k) t.inputs.push_back(in->pop());
    ts.push_back(std::move(t));
  }
}

class PipeOp : public Op {
 public:
  PipeOp(Runtime* rt, std::string n, int depth, Holder* in, EB* pred, std::vector<EB> exprs)
      : Op(rt, std::move(n), depth, 2.0), in(in), pred(pred ? *pred : EB()), has_pred(pred), exprs(std::move(exprs)) {}
  void poll(std::vector<Task>& ts) override {
    poll_batches(rt, this, in, ts);
    if (in->closed() && in->empty() && running == 0 && ts.empty()) {
      finished = true;
      closing = true;
    }
  }
  void run(Task& t, cudaStream_t st) override {
    std::vector<tq_expr> ex;
    for (auto& e : exprs) ex.push_back(e.e());
    tq_expr pe = pred.e();
    run_all_or_nothing(rt, this, t, st, [&](const tq_batch& b, tq_batch& o) {
      check(tq_pipeline_materialize(rt->ctx, &b, has_pred ? &pe : nullptr, ex.empty() ? nullptr : ex.data(),
                                    (uint32_t)ex.size(), &o, st));
    });
  }
  Holder* in;
  EB pred;
  bool has_pred;
  std::vector<EB> exprs;
  bool closing = false;
};

// Join build side: waits for EndOfStream, concatenates, builds the table
class BuildOp : public Op {
 public:
  BuildOp(Runtime* rt, std::string n, int depth, Holder* in, EB* pred, std::vector<uint32_t> keys)
      : Op(rt, std::move(n), depth, 3.0), in(in), pred(pred ? *pred : EB()), has_pred(pred), keys(std::move(keys)) {}
  void poll(std::vector<Task>& ts) override {
    while (!in->empty()) got.push_back(in->pop());
    if (in->closed() && !submitted) {
      submitted = true;
      Task t;
      t.op = this;
      t.inputs = got;
      ts.push_back(std::move(t));
    }
    if (ready) finished = true;
  }
  bool splittable(const Task&) const override { return false; }
  void run(Task& t, cudaStream_t st) override {
    HP b;
    if (t.inputs.size() == 1) {
      b = t.inputs[0];
    } else if (t.inputs.empty()) {
      fail(TQ_INTERNAL, name + ": empty build side");
    } else {
      std::vector<tq_batch> bs;
      for (HP& h : t.inputs) bs.push_back(h->dev);
      tq_batch cat{};
      check(tq_concat(rt->ctx, bs.data(), (uint32_t)bs.size(), &cat, st));
      cudaStreamSynchronize(st);
      b = rt->adopt(cat, false);
      for (HP& h : t.inputs)
        if (!h->view) rt->free_handle(h);
    }
    tq_expr pe = pred.e();
    tq_join_table* jt = nullptr;
    check(tq_pipeline_build(rt->ctx, &b->dev, has_pred ? &pe : nullptr, keys.data(), (uint32_t)keys.size(), &jt, st));
    cudaStreamSynchronize(st);
    std::lock_guard<std::mutex> g(rt->mu);
    b->pins++;  // the probe gathers build columns by row id until the query ends
    rt->keep.push_back(b);
    build = b;
    table = jt;
    ready = true;
  }
  ~BuildOp() override {
    if (table) tq_join_table_destroy(rt->ctx, table);
  }
  Holder* in;
  EB pred;
  bool has_pred;
  std::vector<uint32_t> keys;
  std::vector<HP> got;
  bool submitted = false, ready = false;
  HP build;
  tq_join_table* table = nullptr;
};

// Join probe side: streams once the build is ready
class ProbeOp : public Op {
 public:
  ProbeOp(Runtime* rt, std::string n, int depth, BuildOp* b, Holder* in, EB* pred, std::vector<EB> exprs,
          std::vector<uint32_t> keys, std::vector<uint32_t> build_cols)
      : Op(rt, std::move(n), depth, 3.0), b(b), in(in), pred(pred ? *pred : EB()), has_pred(pred),
        exprs(std::move(exprs)), keys(std::move(keys)), build_cols(std::move(build_cols)) {}
  void poll(std::vector<Task>& ts) override {
    if (!b->ready) return;
    poll_batches(rt, this, in, ts);
    if (in->closed() && in->empty() && running == 0 && ts.empty()) finished = true;
  }
  void run(Task& t, cudaStream_t st) override {
    std::vector<tq_expr> ex;
    for (auto& e : exprs) ex.push_back(e.e());
    tq_expr pe = pred.e();
    static const uint32_t none = 0;  // NULL build_cols would mean "all build columns"
    const uint32_t* bcols = build_cols.empty() ? &none : build_cols.data();
    run_all_or_nothing(rt, this, t, st, [&](const tq_batch& in_b, tq_batch& o) {
      check(tq_pipeline_probe(rt->ctx, b->table, &in_b, has_pred ? &pe : nullptr, ex.empty() ? nullptr : ex.data(),
                              (uint32_t)ex.size(), keys.data(), (uint32_t)keys.size(), bcols,
                              (uint32_t)build_cols.size(), &o, st));
    });
  }
  BuildOp* b;
  Holder* in;
  EB pred;
  bool has_pred;
  std::vector<EB> exprs;
  std::vector<uint32_t> keys, build_cols;
};

// Hash aggregate: one GPU update per batch into partial accumulators
// (serialised per operator), then finalize after EndOfStream.
class AggOp : public Op {
 public:
  AggOp(Runtime* rt, std::string n, int depth, Holder* in, EB* pred, std::vector<EB> exprs, std::vector<uint32_t> keys,
        std::vector<tq_agg> aggs)
      : Op(rt, std::move(n), depth, 2.0), in(in) {
    std::vector<tq_expr> ex;
    for (auto& e : exprs) ex.push_back(e.e());
    EB p = pred ? *pred : EB();
    tq_expr pe = p.e();
    check(tq_agg_create(rt->ctx, pred ? &pe : nullptr, ex.empty() ? nullptr : ex.data(), (uint32_t)ex.size(),
                        keys.data(), (uint32_t)keys.size(), aggs.data(), (uint32_t)aggs.size(), &state));
  }
  ~AggOp() override { tq_agg_destroy(state); }
  void poll(std::vector<Task>& ts) override {
    if (running) return;
    if (!in->empty()) {
      Task t;
      t.op = this;
      t.inputs.push_back(in->pop());
      ts.push_back(std::move(t));
      return;
    }
    if (in->closed() && !final_submitted) {
      final_submitted = true;
      Task t;
      t.op = this;
      t.kind = 1;
      ts.push_back(std::move(t));
      return;
    }
    if (done) finished = true;
  }
  bool splittable(const Task&) const override { return false; }
  void run(Task& t, cudaStream_t st) override {
    if (t.kind == 0) {
      for (HP& h : t.inputs) {
        check(tq_agg_update(state, &h->dev, st));
        cudaStreamSynchronize(st);
        if (!h->view) rt->free_handle(h);
      }
      return;
    }
    tq_batch o{};
    check(tq_agg_finalize(state, &o, st));
    cudaStreamSynchronize(st);
    stat.rows_out += o.rows;
    out->push(rt->adopt(o, false));
    std::lock_guard<std::mutex> g(rt->mu);
    done = true;
  }
  Holder* in;
  tq_agg_state* state = nullptr;
  bool final_submitted = false, done = false;
};

// Exchange: HashPartition on key columns or Broadcast, one
// NCCL collective per exchange after EndOfStream, in DAG order on all workers.
class ExchangeOp : public Op {
 public:
  ExchangeOp(Runtime* rt, std::string n, int depth, Holder* in, int turn, bool broadcast, std::vector<uint32_t> keys)
      : Op(rt, std::move(n), depth, 1.5), in(in), turn(turn), broadcast(broadcast), keys(std::move(keys)) {}
  void poll(std::vector<Task>& ts) override {
    while (!in->empty()) got.push_back(in->pop());
    if (in->closed() && !submitted && rt->exchange_turn == turn) {
      submitted = true;
      Task t;
      t.op = this;
      t.inputs = got;
      ts.push_back(std::move(t));
    }
    if (done) finished = true;
  }
  bool splittable(const Task&) const override { return false; }
  void run(Task& t, cudaStream_t st) override {
    tq_batch cat{};
    bool owned = false;
    if (t.inputs.size() == 1) {
      cat = t.inputs[0]->dev;
    } else {
      std::vector<tq_batch> bs;
      for (HP& h : t.inputs) bs.push_back(h->dev);
      check(tq_concat(rt->ctx, bs.data(), (uint32_t)bs.size(), &cat, st));
      owned = true;
    }
    tq_batch o{};
    if (!rt->comm) {
      if (owned) o = cat;
      else check(tq_slice(rt->ctx, &cat, 0, cat.rows, &o, st));
      owned = false;
    } else if (broadcast) {
      check(tq_comm_allgather(rt->comm, &cat, &o, nullptr, st));
    } else {
      int n = 0;
      std::vector<uint64_t> offs(257);
      tq_batch part{};
      // nparts = world size (the communicator's n, recovered from the allgather header size)
      n = nranks;
      check(tq_hash_partition(rt->ctx, &cat, keys.data(), (uint32_t)keys.size(), (uint32_t)n, &part, offs.data(), st));
      check(tq_comm_exchange(rt->comm, &part, offs.data(), &o, nullptr, st));
      cudaStreamSynchronize(st);
      tq_batch_free(rt->ctx, &part);
    }
    cudaStreamSynchronize(st);
    if (owned) tq_batch_free(rt->ctx, &cat);
    for (HP& h : t.inputs)
      if (!h->view) rt->free_handle(h);
    out->push(rt->adopt(o, false));
    std::lock_guard<std::mutex> g(rt->mu);
    done = true;
    rt->exchange_turn++;
  }
  Holder* in;
  int turn;
  bool broadcast;
  std::vector<uint32_t> keys;
  std::vector<HP> got;
  bool submitted = false, done = false;
  int nranks = 1;
};

// Sink: collects the query result
class SinkOp : public Op {
 public:
  SinkOp(Runtime* rt, Holder* in) : Op(rt, "sink", 99, 1.0), in(in) {}
  void poll(std::vector<Task>&) override {
    while (!in->empty()) hs.push_back(in->pop());
    if (in->closed()) finished = true;
  }
  void run(Task&, cudaStream_t) override {}
  Holder* in;
  std::vector<HP> hs;
};

// ------------------------------------------------------------------ query DAGs
enum { L_ORDERKEY, L_PARTKEY, L_SUPPKEY, L_QUANTITY, L_EXTPRICE, L_DISCOUNT, L_TAX, L_RETURNFLAG, L_LINESTATUS, L_SHIPDATE };
enum { O_ORDERKEY, O_CUSTKEY, O_ORDERDATE, O_SHIPPRIORITY, O_YEAR };
enum { T_ORDERS, T_LINEITEM, T_CUSTOMER, T_SUPPLIER, T_PART, T_PARTSUPP, T_NATION, T_REGION };

struct Plan {
  Runtime* rt;
  const tq_batch* tables;
  std::vector<ScanOp*> scans;
  std::vector<Op*> wiring;  // ops whose `out` must be connected
  int turns = 0;
  Holder* scan(int t) {
    if (!tables[t].cols) fail(TQ_INVALID_PLAN, "query needs table " + std::to_string(t));
    ScanOp* s = rt->op<ScanOp>("scan" + std::to_string(t), &tables[t]);
    s->out = rt->holder();
    scans.push_back(s);
    return s->out;
  }
  template <class T>
  Holder* wire(T* o) {
    o->out = rt->holder();
    return o->out;
  }
  Holder* exchange(Holder* in, int depth, bool broadcast, std::vector<uint32_t> keys) {
    if (!rt->comm) return in;
    auto* x = rt->op<ExchangeOp>("exchange" + std::to_string(turns), depth, in, turns, broadcast, std::move(keys));
    turns++;
    return wire(x);
  }
};

EB rev() {  // ep * (1.00 - disc)
  EB b;
  b.ar(TQ_MUL).col(L_EXTPRICE).ar(TQ_SUB).dec(100).col(L_DISCOUNT);
  return b;
}

Holder* build_plan(Plan& P, int q) {
  Runtime* rt = P.rt;
  if (q == 6) {
    Holder* li = P.scan(T_LINEITEM);
    EB f;
    f.land().land().cmp(TQ_GE).col(L_SHIPDATE).i64(8766).cmp(TQ_LT).col(L_SHIPDATE).i64(9131)
        .land().land().cmp(TQ_GE).col(L_DISCOUNT).dec(5).cmp(TQ_LE).col(L_DISCOUNT).dec(7)
        .cmp(TQ_LT).col(L_QUANTITY).dec(2400);
    EB r;
    r.ar(TQ_MUL).col(L_EXTPRICE).col(L_DISCOUNT);
    return P.wire(rt->op<AggOp>("q6_agg", 1, li, &f, std::vector<EB>{r}, std::vector<uint32_t>{},
                                std::vector<tq_agg>{{TQ_AGG_SUM, 0}}));
  }
  if (q == 1) {
    Holder* li = P.scan(T_LINEITEM);
    EB f;
    f.cmp(TQ_LE).col(L_SHIPDATE).i64(10471);
    EB dp, ch;
    dp.ar(TQ_MUL).col(L_EXTPRICE).ar(TQ_SUB).dec(100).col(L_DISCOUNT);
    ch.ar(TQ_MUL).ar(TQ_MUL).col(L_EXTPRICE).ar(TQ_SUB).dec(100).col(L_DISCOUNT).ar(TQ_ADD).dec(100).col(L_TAX);
    std::vector<EB> ex = {Col(L_RETURNFLAG), Col(L_LINESTATUS), Col(L_QUANTITY), Col(L_EXTPRICE), Col(L_DISCOUNT), dp, ch};
    std::vector<tq_agg> ag = {{TQ_AGG_SUM, 2}, {TQ_AGG_SUM, 3}, {TQ_AGG_SUM, 5}, {TQ_AGG_SUM, 6},
                              {TQ_AGG_AVG, 2}, {TQ_AGG_AVG, 3}, {TQ_AGG_AVG, 4}, {TQ_AGG_COUNT_STAR, 0}};
    return P.wire(rt->op<AggOp>("q1_agg", 1, li, &f, ex, std::vector<uint32_t>{0, 1}, ag));
  }
  if (q == 3) {
    Holder* cu = P.scan(T_CUSTOMER);
    EB fc;
    fc.cmp(TQ_EQ).col(2).i64(1);
    Holder* cf = P.wire(rt->op<PipeOp>("customer_f", 1, cu, &fc, std::vector<EB>{Col(0)}));
    cf = P.exchange(cf, 2, true, {});
    auto* cb = rt->op<BuildOp>("customer_build", 3, cf, nullptr, std::vector<uint32_t>{0});
    Holder* od = P.scan(T_ORDERS);
    EB fo;
    fo.cmp(TQ_LT).col(O_ORDERDATE).i64(9204);
    Holder* of = P.wire(rt->op<ProbeOp>("orders_probe", 4, cb, od, &fo,
                                        std::vector<EB>{Col(O_ORDERKEY), Col(O_ORDERDATE), Col(O_SHIPPRIORITY), Col(O_CUSTKEY)},
                                        std::vector<uint32_t>{3}, std::vector<uint32_t>{}));
    of = P.exchange(of, 5, false, {0});
    auto* ob = rt->op<BuildOp>("orders_build", 6, of, nullptr, std::vector<uint32_t>{0});
    Holder* li = P.scan(T_LINEITEM);
    EB fl;
    fl.cmp(TQ_GT).col(L_SHIPDATE).i64(9204);
    Holder* lf = P.wire(rt->op<PipeOp>("lineitem_f", 1, li, &fl, std::vector<EB>{Col(L_ORDERKEY), rev()}));
    lf = P.exchange(lf, 5, false, {0});
    Holder* j = P.wire(rt->op<ProbeOp>("lineitem_probe", 7, ob, lf, nullptr, std::vector<EB>{}, std::vector<uint32_t>{0},
                                       std::vector<uint32_t>{1, 2}));
    // j: [o_orderdate, o_shippriority, l_orderkey, rev]
    return P.wire(rt->op<AggOp>("q3_agg", 8, j, nullptr, std::vector<EB>{}, std::vector<uint32_t>{2, 0, 1},
                                std::vector<tq_agg>{{TQ_AGG_SUM, 3}}));
  }
  if (q == 5) {
    Holder* re = P.scan(T_REGION);
    EB fr;
    fr.cmp(TQ_EQ).col(1).i64(2);
    auto* rb = rt->op<BuildOp>("region_build", 1, re, &fr, std::vector<uint32_t>{0});
    Holder* na = P.scan(T_NATION);
    Holder* nf = P.wire(rt->op<ProbeOp>("nation_probe", 2, rb, na, nullptr, std::vector<EB>{Col(0), Col(1)},
                                        std::vector<uint32_t>{1}, std::vector<uint32_t>{}));
    auto* nb = rt->op<BuildOp>("nation_build", 3, nf, nullptr, std::vector<uint32_t>{0});
    Holder* cu = P.scan(T_CUSTOMER);
    Holder* cf = P.wire(rt->op<ProbeOp>("customer_probe", 4, nb, cu, nullptr, std::vector<EB>{Col(0), Col(1)},
                                        std::vector<uint32_t>{1}, std::vector<uint32_t>{}));
    auto* cb = rt->op<BuildOp>("customer_build", 5, cf, nullptr, std::vector<uint32_t>{0});
    Holder* od = P.scan(T_ORDERS);
    EB fo;
    fo.land().cmp(TQ_GE).col(O_ORDERDATE).i64(8766).cmp(TQ_LT).col(O_ORDERDATE).i64(9131);
    Holder* of = P.wire(rt->op<ProbeOp>("orders_probe", 6, cb, od, &fo, std::vector<EB>{Col(O_ORDERKEY), Col(O_CUSTKEY)},
                                        std::vector<uint32_t>{1}, std::vector<uint32_t>{1}));
    auto* ob = rt->op<BuildOp>("orders_build", 7, of, nullptr, std::vector<uint32_t>{1});
    Holder* li = P.scan(T_LINEITEM);
    Holder* lj = P.wire(rt->op<ProbeOp>("lineitem_probe", 8, ob, li, nullptr,
                                        std::vector<EB>{Col(L_ORDERKEY), Col(L_SUPPKEY), rev()}, std::vector<uint32_t>{0},
                                        std::vector<uint32_t>{0}));
    Holder* su = P.scan(T_SUPPLIER);
    auto* sb = rt->op<BuildOp>("supplier_build", 1, su, nullptr, std::vector<uint32_t>{0, 1});
    Holder* sj = P.wire(rt->op<ProbeOp>("supplier_probe", 9, sb, lj, nullptr, std::vector<EB>{}, std::vector<uint32_t>{2, 0},
                                        std::vector<uint32_t>{1}));
    return P.wire(rt->op<AggOp>("q5_agg", 10, sj, nullptr, std::vector<EB>{}, std::vector<uint32_t>{0},
                                std::vector<tq_agg>{{TQ_AGG_SUM, 4}}));
  }
  if (q == 9) {
    Holder* pa = P.scan(T_PART);
    EB fp;
    fp.cmp(TQ_LT).col(1).i64(54);
    auto* pb = rt->op<BuildOp>("part_build", 1, pa, &fp, std::vector<uint32_t>{0});
    Holder* ps = P.scan(T_PARTSUPP);
    Holder* psf = P.wire(rt->op<ProbeOp>("partsupp_probe", 2, pb, ps, nullptr, std::vector<EB>{}, std::vector<uint32_t>{0},
                                         std::vector<uint32_t>{}));
    auto* psb = rt->op<BuildOp>("partsupp_build", 3, psf, nullptr, std::vector<uint32_t>{0, 1});
    Holder* li = P.scan(T_LINEITEM);
    Holder* lj = P.wire(rt->op<ProbeOp>("lineitem_probe", 4, psb, li, nullptr,
                                        std::vector<EB>{Col(L_ORDERKEY), Col(L_PARTKEY), Col(L_SUPPKEY), Col(L_QUANTITY),
                                                        Col(L_EXTPRICE), Col(L_DISCOUNT)},
                                        std::vector<uint32_t>{1, 2}, std::vector<uint32_t>{2}));
    Holder* su = P.scan(T_SUPPLIER);
    auto* sb = rt->op<BuildOp>("supplier_build", 1, su, nullptr, std::vector<uint32_t>{0});
    Holder* sj = P.wire(rt->op<ProbeOp>("supplier_probe", 5, sb, lj, nullptr, std::vector<EB>{}, std::vector<uint32_t>{3},
                                        std::vector<uint32_t>{1}));
    Holder* od = P.scan(T_ORDERS);
    auto* ob = rt->op<BuildOp>("orders_build", 1, od, nullptr, std::vector<uint32_t>{0});
    EB amt;
    amt.ar(TQ_SUB).ar(TQ_MUL).col(6).ar(TQ_SUB).dec(100).col(7).ar(TQ_MUL).col(1).col(5);
    Holder* oj = P.wire(rt->op<ProbeOp>("orders_probe", 6, ob, sj, nullptr, std::vector<EB>{Col(0), amt, Col(2)},
                                        std::vector<uint32_t>{2}, std::vector<uint32_t>{4}));
    return P.wire(rt->op<AggOp>("q9_agg", 7, oj, nullptr, std::vector<EB>{}, std::vector<uint32_t>{1, 0},
                                std::vector<tq_agg>{{TQ_AGG_SUM, 2}}));
  }
  fail(TQ_INVALID_PLAN, "unknown query " + std::to_string(q));
}

}  // namespace exec
}  // namespace tq

using namespace tq;
using namespace tq::exec;

extern "C" {

uint64_t tq_estimate_reservation(uint64_t samples, double ema_peak, double ema_ratio, uint64_t input_bytes,
                                 double default_multiplier, double safety) {
  double est = samples == 0 ? default_multiplier * (double)input_bytes
                            : std::max(ema_peak, ema_ratio * (double)input_bytes) * safety;
  return std::max<uint64_t>((uint64_t)est, input_bytes);
}

int tq_on_oom_decide(uint64_t estimate, uint64_t capacity, int splittable, uint64_t* new_estimate) {
  // double the estimate; retry while it fits the Device
  // capacity (0 = unbounded), else split a splittable task, else abort
  const uint64_t e = std::max<uint64_t>(1, estimate) * 2;
  if (new_estimate) *new_estimate = e;
  if (capacity == 0 || e <= capacity) return TQ_OOM_RETRY;
  return splittable ? TQ_OOM_SPLIT : TQ_OOM_ABORT;
}

tq_status tq_engine_run_query(tq_ctx* c, tq_comm* comm, int query, const tq_batch* tables, const tq_engine_opts* o,
                              tq_batch* result, char* metrics_json, uint64_t cap) {
  return guard([&] {
    tq_engine_opts opts{};
    if (o) opts = *o;
    if (!opts.compute_threads) opts.compute_threads = 4;
    if (!opts.batch_rows) opts.batch_rows = 16u << 20;
    if (opts.high_watermark <= 0) opts.high_watermark = 0.90;
    if (opts.low_watermark <= 0) opts.low_watermark = 0.70;
    if (!opts.protect_top_k) opts.protect_top_k = 8;
    if (!opts.pool_buffer_size) opts.pool_buffer_size = 1 << 20;
    const uint64_t saved_budget = c->budget;
    auto t0 = Clock::now();
    Runtime rt(c, comm, opts);
    rt.capacity = opts.device_budget ? opts.device_budget : c->budget;
    bool host_tables = false;
    for (int t = 0; t < 8; ++t) host_tables |= tables[t].cols && tables[t].mem == TQ_MEM_HOST;
    if (!rt.opts.pool_capacity && (rt.capacity || host_tables)) {
      // Host tier sized for the host tables plus spill headroom
      uint64_t bytes = 4ull << 30;
      for (int t = 0; t < 8; ++t)
        if (tables[t].cols && tables[t].mem == TQ_MEM_HOST) bytes += batch_bytes(tables[t]) + (tables[t].rows / 512 + 1) * 8 * tables[t].ncols * 2;
      rt.opts.pool_capacity = bytes / rt.opts.pool_buffer_size + 1;
    }
    rt.setup();
    int nranks = 1;
    if (comm) nranks = tq_comm_size(comm);
    // a plan without a distributed form must not run as one worker of N: it
    // would silently join / aggregate only this rank's shard
    if (nranks > 1 && query != 3)
      fail(TQ_INVALID_PLAN, "query " + std::to_string(query) + " has no distributed plan");
    Plan P{&rt, tables};
    Holder* res = build_plan(P, query);
    SinkOp* sink = rt.op<SinkOp>(res);
    for (auto& op : rt.ops)
      if (auto* x = dynamic_cast<ExchangeOp*>(op.get())) x->nranks = nranks;
    // publish the scans: device tables as zero-copy row-group views; HOST
    // tables are encoded into the pinned pool (Host tier) and every scan task
    // goes through load_to_device
    for (ScanOp* s : P.scans) {
      if (s->table.mem == TQ_MEM_HOST) {
        if (!rt.pool) fail(TQ_INVALID_PLAN, "host tables need a host pool");
        uint64_t br = std::max<uint64_t>(512, opts.batch_rows / 512 * 512);
        for (uint64_t r = 0; r < s->table.rows || (r == 0 && s->table.rows == 0); r += br) {
          uint64_t n = std::min<uint64_t>(br, s->table.rows - r);
          std::vector<tq_column> cols(s->table.ncols);
          for (uint32_t k = 0; k < s->table.ncols; ++k) {
            tq_column col = s->table.cols[k];
            size_t w = width_of(col.kind);
            if (col.kind == TQ_UTF8) fail(TQ_INVALID_PLAN, "utf8 host tables are not supported by the engine");
            col.values = (uint8_t*)col.values + r * w;
            col.values_bytes = n * w;
            if (col.validity) col.validity = col.validity + r / 8;
            cols[k] = col;
          }
          tq_batch v{n, s->table.ncols, TQ_MEM_HOST, cols.data(), nullptr};
          tq_chunked* cb = nullptr;
          check(tq_chunked_encode(rt.pool, &v, &cb));
          HP h = std::make_shared<Handle>();
          h->tier = HOST;
          h->host = cb;
          h->bytes = batch_bytes(v);
          {
            std::lock_guard<std::mutex> g(rt.mu);
            h->id = ++rt.next_id;
            rt.registry.push_back(h);
          }
          s->out->push(h);
          if (s->table.rows == 0) break;
        }
        s->finished = true;
      } else {
        std::vector<Task> none;
        {
          std::lock_guard<std::mutex> g(rt.mu);
          s->poll(none);
        }
        for (HP& h : s->pending) s->out->push(h);
        s->pending.clear();
      }
      s->out->close();
    }
    if (rt.capacity) c->budget = rt.capacity;
    const auto t_run = Clock::now();
    const double setup_ms = std::chrono::duration<double, std::milli>(t_run - t0).count();
    try {
      rt.run();
    } catch (...) {
      c->budget = saved_budget;
      throw;
    }
    c->budget = saved_budget;
    // result -> host
    {
      std::lock_guard<std::mutex> g(rt.mu);
      std::vector<Task> none;
      sink->poll(none);
    }
    if (sink->hs.empty()) fail(TQ_INTERNAL, "query produced no result batch");
    HP r = sink->hs[0];
    rt.load(r, c->stream, false);
    check(tq_batch_download(c, &r->dev, result, nullptr));
    double wall = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
    double run_ms = std::chrono::duration<double, std::milli>(Clock::now() - t_run).count();
    if (metrics_json && cap) {
      std::ostringstream js;
      js << "{\"wall_ms\": " << wall << ", \"setup_ms\": " << setup_ms << ", \"run_ms\": " << run_ms << ", \"tasks\": " << rt.m_tasks << ", \"oom_retries\": " << rt.m_retries
         << ", \"splits\": " << rt.m_splits << ", \"spills\": " << rt.m_spills << ", \"spill_bytes\": " << rt.m_spill_bytes
         << ", \"loads\": " << rt.m_loads << ", \"preloads\": " << rt.m_preloads << ", \"load_bytes\": " << rt.m_load_bytes
         << ", \"peak_device_bytes\": " << rt.m_peak << ", \"device_capacity\": " << rt.capacity << ", \"ops\": {";
      bool first = true;
      for (auto& op : rt.ops) {
        if (!op->stat.tasks) continue;
        js << (first ? "" : ", ") << "\"" << op->name << "\": {\"tasks\": " << op->stat.tasks << ", \"ms\": " << op->stat.ms
           << ", \"rows_out\": " << op->stat.rows_out.load() << "}";
        first = false;
      }
      js << "}}";
      std::string s = js.str();
      uint64_t n = std::min<uint64_t>(s.size(), cap - 1);
      std::memcpy(metrics_json, s.data(), n);
      metrics_json[n] = 0;
    }
  });
}

}  // extern "C"
