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
#include "../../include/tq_storage.h"
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
enum Tier { DEVICE = 0, HOST = 1, STORAGE = 2 };

struct Handle {
  uint64_t id = 0;
  int tier = DEVICE;
  uint64_t bytes = 0;
  int pins = 0;
  bool view = false;  // borrows an input table's device memory: never freed or spilled
  bool spilling = false;  // chosen as a spill victim (under rt->mu); the copy runs outside it
  tq_batch dev{};
  tq_chunked* host = nullptr;
  tq_tcf* file = nullptr;  // STORAGE tier: a row group of a TCF file
  uint32_t row_group = 0;
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
  double gpu_ms = 0;       // stream time between events around the operator calls (Filter/Project/Probe)
  double first_call_ms = 0;  // host time of the first operator call's return (launch + host syncs inside)
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

struct XPair {
  int decide_turn = 0;
  // the sides' phase-1 estimates start once the previous pair decided: they
  // are off the critical path then, instead of competing with the first
  // pair's estimates at the start of the query
  int est_turn = 0;
  bool est_ready[2] = {false, false};
  uint64_t est[2] = {0, 0};
  bool decide_submitted = false, decided = false;
  int strategy = TQ_XCHG_HASH_PARTITION, bcast_side = -1;
  uint64_t totals[2] = {0, 0};
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
thread_local int tl_worker = -1;  // compute thread index (watchdog phases)

class Runtime {
 public:
  Runtime(tq_ctx* c, tq_comm* comm, const tq_engine_opts& o) : ctx(c), comm(comm), opts(o) {}
  ~Runtime();
  void setup();
  void start_threads();
  void stop_threads();
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
    if (h->tier == STORAGE) {
      // Storage -> Host: the row group's column ranges read straight into the
      // pinned pool (byte-range preload), then on to Device
      std::vector<uint32_t> cols(tq_tcf_ncols(h->file));
      for (uint32_t k = 0; k < cols.size(); ++k) cols[k] = k;
      check(tq_tcf_fetch(h->file, pool, h->row_group, cols.data(), (uint32_t)cols.size(), 4, &h->host));
      h->tier = HOST;
      m_storage_reads++;
    }
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
  std::vector<std::thread> threads;  // executor threads (start_threads .. stop_threads)
  // TQ_ENGINE_WATCHDOG=<seconds> (diagnostics): per compute thread, what it is
  // doing (0 idle, 1 reserving, 2 waiting for an input's spill, 3 loading,
  // 4 executing) and for which operator, dumped when a query runs that long
  std::atomic<int> phase[64]{};
  std::atomic<int> mem_phase{0}, pre_phase{0};  // 0 waiting, 1 spilling / loading, 2 exited
  std::atomic<const char*> phase_op[64]{};
  void dump_state();
  uint64_t next_id = 0, next_seq = 0, reserved = 0;
  int running_tasks = 0;
  int executing = 0;  // tasks past their reservation (the ones that can free memory)
  bool stop = false;
  std::exception_ptr error;
  int exchange_turn = 0;  // collectives run in DAG order on every worker
  bool poll_changed = false;  // the current coordination pass changed some operator's state
  bool all_done = false;      // every operator finished (a pass saw it)
  bool poll_all();            // one coordination pass; caller holds mu
  // metrics
  std::atomic<uint64_t> m_tasks{0}, m_retries{0}, m_splits{0}, m_spills{0}, m_spill_bytes{0}, m_loads{0},
      m_preloads{0}, m_load_bytes{0}, m_peak{0}, m_injected{0}, m_storage_reads{0};
  uint64_t spilling_bytes = 0;           // Device bytes of marked victims not yet freed (under mu)
  std::deque<std::vector<HP>> spill_q;   // watermark spills for the memory executor (under mu)
  struct Decision {
    std::string name;
    int strategy, side;
    uint64_t total0, total1;
  };
  std::vector<Decision> decisions;  // exchange_decide outcomes (metrics)
  struct Span {
    std::string op;
    int kind;
    double t0, t1;  // ms since the run phase started
  };
  std::vector<Span> timeline;  // every task's [start, end) (metrics)
  Clock::time_point run_start = Clock::now();
  std::vector<std::unique_ptr<XPair>> pairs;
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
  if (use >= (uint64_t)(opts.high_watermark * capacity) && !stop) {
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
      if (spill_q.empty()) break;  // stop (queued victims are drained first)
      v = std::move(spill_q.front());
      spill_q.pop_front();
    }
    mem_phase = 1;
    spill_victims(v);
    mem_phase = 0;
  }
  mem_phase = 2;
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
  uint64_t in_bytes = 0, host_bytes = 0, want = 0;
  for (HP& h : t.inputs) in_bytes += h->bytes;
  if (!t.estimate) t.estimate = estimate(*op, in_bytes);
  // ---- reserve(Device, estimate): new allocations only
  {
    std::unique_lock<std::mutex> g(mu);
    // pin the inputs first so this task's own reservation never picks them as
    // victims; an input chosen as a victim before it was pinned is being
    // copied out by another thread: let that finish (load() then brings it
    // back) rather than run on a batch that is about to be freed
    for (HP& h : t.inputs) h->pins++;
    if (tl_worker >= 0 && tl_worker < 64) phase[tl_worker] = 2;
    cv.wait(g, [&] {
      if (stop) return true;
      for (HP& h : t.inputs)
        if (h->spilling) return false;
      return true;
    });
    if (stop) {  // the query is being torn down (another task failed): leave
      for (HP& h : t.inputs) h->pins--;
      fail(TQ_INTERNAL, op->name + ": query aborted");
    }
    for (HP& h : t.inputs)  // inputs not on the Device are loaded into the reservation
      if (h->tier != DEVICE) host_bytes += h->bytes;
    want = t.estimate > in_bytes ? t.estimate - in_bytes + host_bytes : host_bytes;
    if (tl_worker >= 0 && tl_worker < 64) phase[tl_worker] = 1;
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
        if (stop) {  // torn down: queued spills will not run
          for (HP& h : t.inputs) h->pins--;
          fail(TQ_INTERNAL, op->name + ": query aborted");
        }
        cv.wait_for(g, std::chrono::milliseconds(2));
      }
    }
    reserved += want;
    executing++;
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
    if (tl_worker >= 0 && tl_worker < 64) phase[tl_worker] = 3;
    for (HP& h : t.inputs) load(h, st, false);  // load_to_device
    if (tl_worker >= 0 && tl_worker < 64) phase[tl_worker] = 4;
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
    const double s0 = std::chrono::duration<double, std::milli>(t0 - run_start).count();
    timeline.push_back({op->name, t.kind, s0, s0 + ms});
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
  // one stream per Compute thread, kept by the context across queries
  cudaStream_t st = exec_stream(ctx, 2 + idx);
  {  // TQ_ENGINE_ONE_STREAM=1 (experiments): every task on the context stream
    static const bool one = [] { const char* e = getenv("TQ_ENGINE_ONE_STREAM"); return e && e[0] == '1'; }();
    if (one) st = ctx->stream;
  }
  for (;;) {
    Task t;
    {
      std::unique_lock<std::mutex> g(mu);
      cv.wait(g, [&] { return stop || !queue.empty(); });
      if (stop) break;
      if (!pick(t)) continue;
      running_tasks++;
    }
    if (idx < 64) {
      tl_worker = idx;
      phase_op[idx] = t.op->name.c_str();
    }
    try {
      run_task(t, st);
    } catch (...) {
      std::lock_guard<std::mutex> g(mu);
      if (!error) error = std::current_exception();
    }
    if (idx < 64) phase[idx] = 0;
    {
      std::lock_guard<std::mutex> g(mu);
      running_tasks--;
      t.op->running--;
      // the finishing worker polls the DAG itself: the follow-up task is
      // queued (and often picked by this same thread) without a wake-up of
      // the coordinator in between
      if (!error && !all_done) poll_all();
      cv.notify_all();
    }
  }
  cudaStreamSynchronize(st);
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
          if (x->tier != DEVICE && x->pins == 0) {
            h = x;
            break;
          }
      if (!h) continue;
      h->pins++;
    }
    pre_phase = 1;
    try {
      load(h, preload_stream, true);
    } catch (...) {
    }
    pre_phase = 0;
    std::lock_guard<std::mutex> g(mu);
    h->pins--;
  }
}

// One coordination pass (caller holds mu): poll every unfinished operator for
// runnable tasks, close the outputs of finished ones (EndOfStream), and go
// again while a pass changed something — a poll can make an op polled earlier
// in the pass runnable (an exchange side's estimate readies its decide, an
// EndOfStream its consumer).  Returns true when every operator finished.
bool Runtime::poll_all() {
  for (;;) {
    bool all = true;
    poll_changed = false;
    for (auto& o : ops) {
      if (o->finished) continue;
      std::vector<Task> ts;
      o->poll(ts);
      poll_changed |= !ts.empty();
      for (Task& t : ts) {
        o->running++;
        submit(std::move(t));
      }
      if (o->finished && o->out && !o->out->closed()) {
        o->out->close_locked();  // EndOfStream after the last output
        cv.notify_all();
      }
      poll_changed |= o->finished;
      all = all && o->finished;
    }
    if (all) {
      all_done = true;
      cv.notify_all();
      return true;
    }
    if (!poll_changed) return false;
  }
}

// Executor threads are started before the run phase (they wait for tasks):
// starting them is setup, not query work.
void Runtime::start_threads() {
  for (uint32_t i = 0; i < std::max<uint32_t>(1, opts.compute_threads); ++i) threads.emplace_back(&Runtime::worker, this, i);
  if (opts.preload) threads.emplace_back(&Runtime::preloader, this);
  threads.emplace_back(&Runtime::memory_executor, this);
}

void Runtime::stop_threads() {
  {
    std::lock_guard<std::mutex> g(mu);
    stop = true;
    cv.notify_all();
  }
  for (auto& t : threads)
    if (t.joinable()) t.join();
  threads.clear();
}

void Runtime::dump_state() {
  fprintf(stderr, "[tq watchdog] in_use %.3f GB capacity %.3f GB memexec %d preloader %d stop %d error %d\n",
          device_in_use() / 1e9, capacity / 1e9, mem_phase.load(), pre_phase.load(), (int)stop, (int)(bool)error);
  for (uint32_t i = 0; i < std::max<uint32_t>(1, opts.compute_threads) && i < 64; ++i) {
    const char* n = phase_op[i].load();
    fprintf(stderr, "[tq watchdog] worker %u phase %d op %s\n", i, phase[i].load(), n ? n : "-");
  }
  std::unique_lock<std::mutex> g(mu, std::defer_lock);
  for (int k = 0; k < 200 && !g.try_lock(); ++k) std::this_thread::sleep_for(std::chrono::milliseconds(5));
  if (!g.owns_lock()) {
    fprintf(stderr, "[tq watchdog] runtime lock held\n");
    return;
  }
  fprintf(stderr, "[tq watchdog] queue %zu executing %d reserved %.3f GB running %d spilling %.3f GB spill_q %zu\n",
          queue.size(), executing, reserved / 1e9, running_tasks, spilling_bytes / 1e9, spill_q.size());
  for (auto& o : ops)
    if (!o->finished)
      fprintf(stderr, "[tq watchdog] op %s running %d\n", o->name.c_str(), o->running);
  int n_spilling = 0, n_pinned = 0;
  for (auto& w : registry)
    if (HP h = w.lock()) {
      n_spilling += h->spilling;
      n_pinned += h->pins > 0;
    }
  fprintf(stderr, "[tq watchdog] handles spilling %d pinned %d\n", n_spilling, n_pinned);
}

void Runtime::run() {
  run_start = Clock::now();
  if (threads.empty()) start_threads();
  std::atomic<bool> finished_run{false};
  std::thread watchdog;
  static const int wd_s = [] { const char* e = getenv("TQ_ENGINE_WATCHDOG"); return e ? atoi(e) : 0; }();
  if (wd_s > 0)
    watchdog = std::thread([this, &finished_run] {
      for (int s = 0; !finished_run.load(); ++s) {
        std::this_thread::sleep_for(std::chrono::seconds(1));
        if (s + 1 >= wd_s && (s + 1) % wd_s == 0 && !finished_run.load()) dump_state();
      }
    });
  struct Join {
    std::thread& t;
    std::atomic<bool>& f;
    ~Join() {
      f = true;
      if (t.joinable()) t.join();
    }
  } join_wd{watchdog, finished_run};
  // coordinator: poll operators for runnable tasks until every operator finished
  {
    std::unique_lock<std::mutex> g(mu);
    for (;;) {
      if (error) break;
      if (poll_all()) break;
      cv.wait_for(g, std::chrono::milliseconds(1));
    }
    stop = true;
    cv.notify_all();
  }
  stop_threads();
  if (error) std::rethrow_exception(error);
}

Runtime::~Runtime() {
  stop_threads();
  for (auto& w : registry)
    if (HP h = w.lock()) {
      if (h->tier == DEVICE && !h->view && h->dev.cols) tq_batch_free(ctx, &h->dev);
      if (h->host) tq_chunked_release(h->host);
      h->host = nullptr;
      h->dev.cols = nullptr;
    }
  // the pool belongs to the context (reused by the next query)
  // (copy / preload streams belong to the context)
}

void Runtime::setup() {
  cudaSetDevice(ctx->device);
  copy_stream = exec_stream(ctx, 0);
  preload_stream = exec_stream(ctx, 1);
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
  ScanOp(Runtime* rt, std::string n, const tq_batch* table)
      : Op(rt, std::move(n), 0, 4.0), table(*table), src(table) {}
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
    nbatches = hs.size();
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
  const tq_batch* src;  // the caller's table entry (identifies a TCF-backed table)
  std::deque<std::vector<tq_column>> views;
  std::vector<HP> out_q, pending;
  uint64_t nbatches = 0;  // batches this scan publishes (phase-1 progress of the exchanges it drives)
};

// Filter -> Project (one fused GPU pipeline per input batch).  A task takes up
// to opts.task_batches batches; its outputs are deposited only after every
// input succeeded (a failed task can be retried or split without duplicates).
void run_all_or_nothing(Runtime* rt, Op* op, Task& t, cudaStream_t st,
                        const std::function<void(const tq_batch&, tq_batch&)>& body) {
  std::vector<tq_batch> outs;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  try {
    cudaEventRecord(e0, st);
    auto h0 = Clock::now();
    for (HP& h : t.inputs) {
      tq_batch o{};
      body(h->dev, o);
      outs.push_back(o);
    }
    const double call_ms = std::chrono::duration<double, std::milli>(Clock::now() - h0).count();
    cudaEventRecord(e1, st);
    cudaStreamSynchronize(st);
    float g = 0;
    cudaEventElapsedTime(&g, e0, e1);
    op->stat.gpu_ms += g;
    op->stat.first_call_ms += call_ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  } catch (...) {
    cudaStreamSynchronize(st);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
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
class XSideOp;
uint64_t side_capacity(const XSideOp* x);

class BuildOp : public Op {
 public:
  // semi: a semi-join build (no build columns are taken); bloom_from: the
  // exchange side that produced this build's input — its agreed window
  // capacity sizes the table's Bloom filter so the workers' filters can be
  // all-gathered as one partitioned LIP filter (tq_comm_gather_table_blooms)
  BuildOp(Runtime* rt, std::string n, int depth, Holder* in, EB* pred, std::vector<uint32_t> keys, bool semi = false,
          XSideOp* bloom_from = nullptr)
      : Op(rt, std::move(n), depth, 3.0), in(in), pred(pred ? *pred : EB()), has_pred(pred), keys(std::move(keys)),
        semi(semi), bloom_from(bloom_from) {}
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
      {
        // pinned before anything reads it: an unpinned handle in the registry
        // is a spill victim, and the build and every probe read its columns
        std::lock_guard<std::mutex> g(rt->mu);
        b->pins++;
      }
      for (HP& h : t.inputs)
        if (!h->view) rt->free_handle(h);
    }
    tq_expr pe = pred.e();
    tq_join_table* jt = nullptr;
    const uint64_t bloom_keys = bloom_from ? side_capacity(bloom_from) : 0;
    check(tq_pipeline_build_ex(rt->ctx, &b->dev, has_pred ? &pe : nullptr, keys.data(), (uint32_t)keys.size(),
                               bloom_keys, semi ? 1 : 0, &jt, st));
    cudaStreamSynchronize(st);
    std::lock_guard<std::mutex> g(rt->mu);
    if (t.inputs.size() == 1) b->pins++;  // the probe gathers build columns by row id until the query ends
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
  bool semi;
  XSideOp* bloom_from;
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

bool pair_hash_partitioned(const XPair* x);

// Hash aggregate: one GPU update per batch into partial accumulators
// (serialised per operator), then finalize after EndOfStream.
// Distributed (dist): the aggregate's input must be partitioned on the group
// keys.  When it is — the join feeding it was hash-partitioned
// on a group key (copart decided HashPartition) — each worker's finalize is
// final; otherwise the worker's partial (keys + raw accumulators) is
// hash-partitioned on the group keys over the fused exchange and the
// received partials are merged (local pre-aggregation).
class AggOp : public Op {
 public:
  AggOp(Runtime* rt, std::string n, int depth, Holder* in, EB* pred, std::vector<EB> exprs, std::vector<uint32_t> keys,
        std::vector<tq_agg> aggs, bool dist = false, const XPair* copart = nullptr, int turn = -1)
      : Op(rt, std::move(n), depth, 2.0), in(in), nkeys((uint32_t)keys.size()), dist(dist), copart(copart), turn(turn),
        pred(pred ? *pred : EB()), has_pred(pred), exprs(exprs), keys(keys), aggs(aggs) {
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
    // the first batch is held back: a single-batch input is aggregated and
    // finalised in one call (no partial state + merge pass)
    if (!in->empty() && !first && !updated) {
      first = in->pop();
      return;
    }
    if (!in->empty()) {
      // one batch per update task: an update that fails (on_oom) is retried
      // as a whole, so a task must never hold an already-aggregated batch
      Task t;
      t.op = this;
      if (first) {
        t.inputs.push_back(first);  // the next batch stays queued for the next task
        first = nullptr;
      } else {
        t.inputs.push_back(in->pop());
      }
      updated = true;
      ts.push_back(std::move(t));
      return;
    }
    // (distributed: the final step is a collective, taken in DAG order)
    if (in->closed() && !final_submitted && (!dist || rt->exchange_turn == turn)) {
      final_submitted = true;
      Task t;
      t.op = this;
      t.kind = 1;
      if (first) t.inputs.push_back(first);
      first = nullptr;
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
    const bool local = !dist || (copart && pair_hash_partitioned(copart));
    if (local && !updated && t.inputs.size() == 1) {  // the whole input in one batch: one call
      std::vector<tq_expr> ex;
      for (auto& e : exprs) ex.push_back(e.e());
      tq_expr pe = pred.e();
      tq_batch o{};
      check(tq_pipeline_aggregate(rt->ctx, &t.inputs[0]->dev, has_pred ? &pe : nullptr, ex.empty() ? nullptr : ex.data(),
                                  (uint32_t)ex.size(), keys.data(), (uint32_t)keys.size(), aggs.data(),
                                  (uint32_t)aggs.size(), &o, st));
      cudaStreamSynchronize(st);
      if (!t.inputs[0]->view) rt->free_handle(t.inputs[0]);
      stat.rows_out += o.rows;
      out->push(rt->adopt(o, false));
      std::lock_guard<std::mutex> g(rt->mu);
      done = true;
      if (dist) rt->exchange_turn++;
      return;
    }
    for (HP& h : t.inputs) {  // a held-back first batch
      check(tq_agg_update(state, &h->dev, st));
      cudaStreamSynchronize(st);
      if (!h->view) rt->free_handle(h);
    }
    if (!local) {
      tq_batch part{}, recv{};
      check(tq_agg_take_partial(state, &part, st));
      std::vector<uint32_t> kk(nkeys);
      for (uint32_t k = 0; k < nkeys; ++k) kk[k] = k;
      tq_status r = tq_pipeline_partition_exchange(rt->comm, &part, nullptr, nullptr, 0, kk.data(), nkeys, nullptr,
                                                   &recv, st);
      tq_batch_free(rt->ctx, &part);
      check(r);
      r = tq_agg_add_partial(state, &recv, st);
      cudaStreamSynchronize(st);
      tq_batch_free(rt->ctx, &recv);
      check(r);
    }
    tq_batch o{};
    check(tq_agg_finalize(state, &o, st));
    cudaStreamSynchronize(st);
    stat.rows_out += o.rows;
    out->push(rt->adopt(o, false));
    std::lock_guard<std::mutex> g(rt->mu);
    done = true;
    if (dist) rt->exchange_turn++;
  }
  Holder* in;
  uint32_t nkeys;
  bool dist;
  const XPair* copart;
  int turn;
  EB pred;
  bool has_pred;
  std::vector<EB> exprs;
  std::vector<uint32_t> keys;
  std::vector<tq_agg> aggs;
  tq_agg_state* state = nullptr;
  HP first;              // held-back first input batch
  bool updated = false;  // some batch went through tq_agg_update
  bool final_submitted = false, done = false;
};

// ------------------------------------------------------------------ AdaptiveExchange
// One exchange PAIR per distributed join: side 0 and side 1 feed the join's
// two inputs.  Phase 1: each side, once its driving scan passed
// TQ_SAMPLE_FRACTION (or ended), estimates its total bytes
// (tq_exchange_phase1); the DecideOp all-gathers both sides' estimates of every
// worker and applies tq_exchange_decide — the same pure function on every
// worker, so every worker takes the same decision.  Phase 2 (after the side's
// EndOfStream): Broadcast the smaller side (the other stays local) or
// HashPartition both on the join keys (fnv1a64 mod N).  Every collective (a
// decide, a side's data movement, a distributed aggregate's exchange) runs in
// DAG order on every worker (rt->exchange_turn), as NCCL requires.
bool pair_hash_partitioned(const XPair* x) { return x->decided && x->strategy == TQ_XCHG_HASH_PARTITION; }

class DecideOp : public Op {
 public:
  DecideOp(Runtime* rt, std::string n, XPair* x) : Op(rt, std::move(n), 50, 1.0), x(x) {}
  void poll(std::vector<Task>& ts) override {
    if (!x->decide_submitted && x->est_ready[0] && x->est_ready[1] && rt->exchange_turn == x->decide_turn) {
      x->decide_submitted = true;
      Task t;
      t.op = this;
      ts.push_back(std::move(t));
    }
    if (x->decided) finished = true;
  }
  bool splittable(const Task&) const override { return false; }
  void run(Task&, cudaStream_t st) override {
    const int n = tq_comm_size(rt->comm);
    uint64_t mine[2], est0[kMaxRanks], est1[kMaxRanks], all[2 * kMaxRanks];
    {
      std::lock_guard<std::mutex> g(rt->mu);
      mine[0] = x->est[0];
      mine[1] = x->est[1];
    }
    {
      TQ_HT("engine decide allgather");
      check(tq_comm_allgather_host_u64(rt->comm, mine, all, 2, st));
    }
    for (int r = 0; r < n; ++r) {
      est0[r] = all[2 * r];
      est1[r] = all[2 * r + 1];
    }
    int side = -1;
    uint64_t t0 = 0, t1 = 0;
    int strategy = tq_exchange_decide(est0, est1, n, rt->opts.broadcast_threshold ? rt->opts.broadcast_threshold
                                                                                  : TQ_BROADCAST_THRESHOLD,
                                      &side, &t0, &t1);
    // forced strategies (strategy-equivalence tests)
    if (rt->opts.force_exchange == 1) {
      strategy = TQ_XCHG_BROADCAST;
      side = t0 <= t1 ? 0 : 1;
    } else if (rt->opts.force_exchange == 2) {
      strategy = TQ_XCHG_HASH_PARTITION;
      side = -1;
    }
    std::lock_guard<std::mutex> g(rt->mu);
    x->strategy = strategy;
    x->bcast_side = side;
    x->totals[0] = t0;
    x->totals[1] = t1;
    x->decided = true;
    rt->exchange_turn++;
    rt->decisions.push_back({name, strategy, side, t0, t1});
  }
  XPair* x;
  static constexpr int kMaxRanks = 64;
};

// Merge the input batches of one exchange side: consecutive row-group views
// of one table are one larger view (zero copy); anything else is
// concatenated.  Returns true when `out` is a new owned batch.
bool merge_inputs(Runtime* rt, std::vector<HP>& in, tq_batch& out, std::vector<tq_column>& cols, cudaStream_t st) {
  if (in.size() == 1) {
    out = in[0]->dev;
    return false;
  }
  bool contiguous = !in.empty();
  for (size_t i = 0; contiguous && i < in.size(); ++i) {
    const tq_batch& b = in[i]->dev;
    contiguous = in[i]->view && b.ncols == in[0]->dev.ncols;
    if (!contiguous || i == 0) continue;
    const tq_batch& a = in[i - 1]->dev;
    for (uint32_t c = 0; c < b.ncols && contiguous; ++c) {
      const size_t w = width_of(b.cols[c].kind);
      contiguous = b.cols[c].kind != TQ_UTF8 && (const uint8_t*)b.cols[c].values == (const uint8_t*)a.cols[c].values + a.rows * w &&
                   (a.rows % 8 == 0) && ((b.cols[c].validity == nullptr) == (a.cols[c].validity == nullptr)) &&
                   (!b.cols[c].validity || b.cols[c].validity == a.cols[c].validity + a.rows / 8);
    }
  }
  if (contiguous) {
    out = in[0]->dev;
    cols.assign(out.cols, out.cols + out.ncols);
    uint64_t rows = 0;
    for (HP& h : in) rows += h->dev.rows;
    for (auto& c : cols) c.values_bytes = rows * width_of(c.kind);
    out.rows = rows;
    out.cols = cols.data();
    out.owner = nullptr;
    return false;
  }
  std::vector<tq_batch> bs;
  for (HP& h : in) bs.push_back(h->dev);
  check(tq_concat(rt->ctx, bs.data(), (uint32_t)bs.size(), &out, st));
  return true;
}

class XSideOp : public Op {
 public:
  // pred / exprs: filter + projection fused into the exchange kernel (none:
  // the input columns as they are); keys: hash-partition keys (indices into
  // the side's output columns); lip: HashPartition drops rows whose keys
  // miss the other side's (already exchanged) join table — the partitioned
  // LIP filter; src: the scan whose progress drives phase 1
  XSideOp(Runtime* rt, std::string n, int depth, XPair* x, int side, int turn, Holder* in, class ScanOp* src,
          EB* pred, std::vector<EB> exprs, std::vector<uint32_t> keys, BuildOp* lip)
      : Op(rt, std::move(n), depth, 1.5), x(x), side(side), turn(turn), in(in), src(src), pred(pred ? *pred : EB()),
        has_pred(pred), exprs(std::move(exprs)), keys(std::move(keys)), lip(lip) {}
  bool fused() const { return has_pred || !exprs.empty(); }
  void poll(std::vector<Task>& ts) override;
  bool splittable(const Task&) const override { return false; }
  void run(Task& t, cudaStream_t st) override;
  XPair* x;
  int side, turn;
  Holder* in;
  class ScanOp* src;
  EB pred;
  bool has_pred;
  std::vector<EB> exprs;
  std::vector<uint32_t> keys;
  BuildOp* lip;
  std::vector<HP> got;
  uint64_t bytes = 0;
  double est_progress = 0;
  bool est_submitted = false, submitted = false, done = false;
  uint64_t out_capacity = 0;  // agreed row capacity of this side's fused HashPartition (0: none)
};
uint64_t side_capacity(const XSideOp* x) { return x->out_capacity; }

void XSideOp::poll(std::vector<Task>& ts) {
  while (!in->empty()) {
    HP h = in->pop();
    bytes += h->bytes;
    got.push_back(h);
  }
  // ---- phase 1: a local estimate once the driving scan
  // passed the sample fraction, or this side's input ended
  if (!x->est_ready[side] && !est_submitted && rt->exchange_turn >= x->est_turn) {
    const uint64_t total = src ? src->nbatches : 0;
    const double progress = in->closed() ? 1.0 : total ? (double)got.size() / (double)total : 0.0;
    if (progress >= 1.0 || progress >= TQ_SAMPLE_FRACTION) {
      if (fused() && !got.empty()) {
        // the rows this side will ship are pred / exprs of its input: measured
        // on the batches so far (a COUNT pass over the predicate columns)
        est_submitted = true;
        est_progress = progress;
        Task t;
        t.op = this;
        t.kind = 1;
        t.inputs = got;
        ts.push_back(std::move(t));
      } else {
        uint64_t e = 0;
        tq_exchange_phase1(bytes, progress, TQ_SAMPLE_FRACTION, &e);
        x->est[side] = e;
        x->est_ready[side] = true;
        rt->poll_changed = true;
      }
    }
  }
  // ---- phase 2: the data movement, after EndOfStream, in DAG order
  const bool lip_wait = lip && x->decided && x->strategy == TQ_XCHG_HASH_PARTITION && !lip->ready &&
                        rt->opts.exchange_impl == 0;
  if (x->decided && x->est_ready[side] && in->closed() && !submitted && rt->exchange_turn == turn && !lip_wait) {
    submitted = true;
    Task t;
    t.op = this;
    t.inputs = got;
    ts.push_back(std::move(t));
  }
  if (done) finished = true;
}

void XSideOp::run(Task& t, cudaStream_t st) {
  std::vector<tq_expr> ex;
  for (auto& e : exprs) ex.push_back(e.e());
  tq_expr pe = pred.e();
  const tq_expr* pp = has_pred ? &pe : nullptr;
  const tq_expr* ep = ex.empty() ? nullptr : ex.data();
  if (t.kind == 1) {  // phase-1 estimate of a fused side
    // measure pred / exprs on a sample of the arrived rows: the first
    // TQ_SAMPLE_FRACTION of the side's (estimated) total rows, taken as a
    // zero-copy row prefix of the arrived batches
    uint64_t arrived = 0;
    for (HP& h : t.inputs) arrived += h->dev.rows;
    const double total_rows = est_progress > 0 ? (double)arrived / est_progress : (double)arrived;
    uint64_t want = std::max<uint64_t>(1 << 16, (uint64_t)(total_rows * TQ_SAMPLE_FRACTION));
    uint64_t sampled = 0, out_bytes = 0;
    for (HP& h : t.inputs) {
      if (sampled >= want) break;
      tq_batch v = h->dev;
      std::vector<tq_column> cols(v.cols, v.cols + v.ncols);
      uint64_t take = std::min<uint64_t>(v.rows, want - sampled);
      bool prefix_ok = true;
      for (auto& c : cols) prefix_ok &= c.kind != TQ_UTF8;
      if (prefix_ok && take < v.rows) {
        if (take >= 512) take = take / 512 * 512;  // tile-aligned prefix view
        for (auto& c : cols) c.values_bytes = take * width_of(c.kind);
        v.rows = take;
        v.cols = cols.data();
      }
      uint64_t rows = 0, rb = 0;
      TQ_HT("engine side estimate");
      check(tq_pipeline_estimate(rt->ctx, &v, pp, ep, (uint32_t)ex.size(), &rows, &rb, st));
      out_bytes += rows * rb;
      sampled += v.rows;
    }
    // bytes of the arrived input, extrapolated from the sample, then phase 1
    const uint64_t arrived_bytes = sampled ? (uint64_t)((double)out_bytes * (double)arrived / (double)sampled) : 0;
    uint64_t e = 0;
    tq_exchange_phase1(arrived_bytes, est_progress, TQ_SAMPLE_FRACTION, &e);
    std::lock_guard<std::mutex> g(rt->mu);
    x->est[side] = e;
    x->est_ready[side] = true;
    return;
  }
  const bool bcast = x->strategy == TQ_XCHG_BROADCAST;
  const bool local = bcast && side != x->bcast_side;
  std::vector<tq_column> vcols;
  tq_batch merged{};
  bool owned = false;
  if (local && !fused()) {
    // the side that stays local passes its batches through untouched
    for (HP& h : t.inputs) out->push(h);
  } else {
    owned = merge_inputs(rt, t.inputs, merged, vcols, st);
    tq_batch o{};
    tq_status r = TQ_OK;
    const bool fused_impl = rt->opts.exchange_impl == 0;
    if (local) {
      r = tq_pipeline_materialize(rt->ctx, &merged, pp, ep, (uint32_t)ex.size(), &o, st);
    } else if (bcast) {
      if (fused_impl) {
        r = tq_pipeline_broadcast(rt->comm, &merged, pp, ep, (uint32_t)ex.size(), &o, st);
      } else {
        tq_batch m{};
        r = tq_pipeline_materialize(rt->ctx, &merged, pp, ep, (uint32_t)ex.size(), &m, st);
        if (r == TQ_OK) r = tq_comm_allgather(rt->comm, &m, &o, nullptr, st);
        cudaStreamSynchronize(st);
        tq_batch_free(rt->ctx, &m);
      }
    } else if (fused_impl) {
      tq_bloom* bloom = nullptr;
      if (lip) r = tq_comm_gather_table_blooms(rt->comm, lip->table, &bloom, st);
      if (r == TQ_OK)
        r = tq_pipeline_partition_exchange(rt->comm, &merged, pp, ep, (uint32_t)ex.size(), keys.data(),
                                           (uint32_t)keys.size(), bloom, &o, st);
      out_capacity = tq_comm_last_exchange_capacity(rt->comm);
      cudaStreamSynchronize(st);
      if (bloom) tq_bloom_destroy(bloom);
    } else {
      const int n = tq_comm_size(rt->comm);
      std::vector<uint64_t> offs(n + 1);
      tq_batch part{};
      r = tq_pipeline_partition(rt->ctx, &merged, pp, ep, (uint32_t)ex.size(), keys.data(), (uint32_t)keys.size(),
                                (uint32_t)n, &part, offs.data(), st);
      if (r == TQ_OK) r = tq_comm_exchange(rt->comm, &part, offs.data(), &o, nullptr, st);
      cudaStreamSynchronize(st);
      tq_batch_free(rt->ctx, &part);
    }
    cudaStreamSynchronize(st);
    if (owned) tq_batch_free(rt->ctx, &merged);
    check(r);
    stat.rows_out += o.rows;
    out->push(rt->adopt(o, false));
    for (HP& h : t.inputs)
      if (!h->view) rt->free_handle(h);
  }
  std::lock_guard<std::mutex> g(rt->mu);
  done = true;
  rt->exchange_turn++;
}

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
  std::map<Holder*, ScanOp*> scan_of;
  int turns = 0;
  Holder* scan(int t) {
    if (!tables[t].cols) fail(TQ_INVALID_PLAN, "query needs table " + std::to_string(t));
    ScanOp* s = rt->op<ScanOp>("scan" + std::to_string(t), &tables[t]);
    s->out = rt->holder();
    scans.push_back(s);
    scan_of[s->out] = s;
    return s->out;
  }
  template <class T>
  Holder* wire(T* o) {
    o->out = rt->holder();
    return o->out;
  }
  // ---- distributed plans: one exchange pair per join (its decide is a
  // collective turn), one turn per side's data movement, in DAG order
  XPair* pair(const std::string& name) {
    rt->pairs.emplace_back(new XPair());
    XPair* x = rt->pairs.back().get();
    x->decide_turn = turns++;
    x->est_turn = last_decide_turn + 1;
    last_decide_turn = x->decide_turn;
    rt->op<DecideOp>("decide_" + name, x);
    return x;
  }
  Holder* side(XPair* x, int sd, const std::string& name, int depth, Holder* in, Holder* driving_scan, EB* pred,
               std::vector<EB> exprs, std::vector<uint32_t> keys, BuildOp* lip = nullptr, XSideOp** op = nullptr) {
    auto it = scan_of.find(driving_scan);
    auto* o = rt->op<XSideOp>("xchg_" + name, depth, x, sd, turns++, in, it == scan_of.end() ? nullptr : it->second,
                              pred, std::move(exprs), std::move(keys), lip);
    if (op) *op = o;
    return wire(o);
  }
  int agg_turn() { return turns++; }
  int last_decide_turn = -1;
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
    auto* cb = rt->op<BuildOp>("customer_build", 3, cf, nullptr, std::vector<uint32_t>{0});
    Holder* od = P.scan(T_ORDERS);
    EB fo;
    fo.cmp(TQ_LT).col(O_ORDERDATE).i64(9204);
    Holder* of = P.wire(rt->op<ProbeOp>("orders_probe", 4, cb, od, &fo,
                                        std::vector<EB>{Col(O_ORDERKEY), Col(O_ORDERDATE), Col(O_SHIPPRIORITY), Col(O_CUSTKEY)},
                                        std::vector<uint32_t>{3}, std::vector<uint32_t>{}));
    auto* ob = rt->op<BuildOp>("orders_build", 6, of, nullptr, std::vector<uint32_t>{0});
    Holder* li = P.scan(T_LINEITEM);
    EB fl;
    fl.cmp(TQ_GT).col(L_SHIPDATE).i64(9204);
    // lineitem filter + projection fused into the probe (one pass, nothing materialised before the join)
    Holder* j = P.wire(rt->op<ProbeOp>("lineitem_probe", 7, ob, li, &fl, std::vector<EB>{Col(L_ORDERKEY), rev()},
                                       std::vector<uint32_t>{0}, std::vector<uint32_t>{1, 2}));
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

// Distributed plans (one worker per GPU, each over its own
// row-group subset): an exchange pair before every join (broadcast the small
// side or hash-partition both, decided at run time from the workers'
// estimates), aggregates either co-partitioned with the last join or
// pre-aggregated and exchanged on the group keys.  Results: the union over
// workers of their result batches (disjoint groups).
Holder* build_dist_plan(Plan& P, int q) {
  Runtime* rt = P.rt;
  const std::vector<uint32_t> none;
  if (q == 1 || q == 6) {
    Holder* li = P.scan(T_LINEITEM);
    EB f;
    std::vector<EB> ex;
    std::vector<uint32_t> keys;
    std::vector<tq_agg> ag;
    if (q == 6) {
      f.land().land().cmp(TQ_GE).col(L_SHIPDATE).i64(8766).cmp(TQ_LT).col(L_SHIPDATE).i64(9131)
          .land().land().cmp(TQ_GE).col(L_DISCOUNT).dec(5).cmp(TQ_LE).col(L_DISCOUNT).dec(7)
          .cmp(TQ_LT).col(L_QUANTITY).dec(2400);
      EB r;
      r.ar(TQ_MUL).col(L_EXTPRICE).col(L_DISCOUNT);
      ex = {r};
      ag = {{TQ_AGG_SUM, 0}};
    } else {
      f.cmp(TQ_LE).col(L_SHIPDATE).i64(10471);
      EB dp, ch;
      dp.ar(TQ_MUL).col(L_EXTPRICE).ar(TQ_SUB).dec(100).col(L_DISCOUNT);
      ch.ar(TQ_MUL).ar(TQ_MUL).col(L_EXTPRICE).ar(TQ_SUB).dec(100).col(L_DISCOUNT).ar(TQ_ADD).dec(100).col(L_TAX);
      ex = {Col(L_RETURNFLAG), Col(L_LINESTATUS), Col(L_QUANTITY), Col(L_EXTPRICE), Col(L_DISCOUNT), dp, ch};
      keys = {0, 1};
      ag = {{TQ_AGG_SUM, 2}, {TQ_AGG_SUM, 3}, {TQ_AGG_SUM, 5}, {TQ_AGG_SUM, 6},
            {TQ_AGG_AVG, 2}, {TQ_AGG_AVG, 3}, {TQ_AGG_AVG, 4}, {TQ_AGG_COUNT_STAR, 0}};
    }
    return P.wire(rt->op<AggOp>(q == 6 ? "q6_agg" : "q1_agg", 1, li, &f, ex, keys, ag, true, nullptr, P.agg_turn()));
  }
  if (q == 3) {
    Holder* cu = P.scan(T_CUSTOMER);
    Holder* od = P.scan(T_ORDERS);
    Holder* li = P.scan(T_LINEITEM);
    // join 1: customer_f (BUILDING) x orders on custkey — customer_f is broadcast at SF100 (24 MB)
    XPair* x1 = P.pair("customer_orders");
    EB fc;
    fc.cmp(TQ_EQ).col(2).i64(1);
    Holder* cfx = P.side(x1, 0, "customer_f", 2, cu, cu, &fc, {Col(0)}, {0});
    Holder* odx = P.side(x1, 1, "orders", 2, od, od, nullptr, {}, {O_CUSTKEY});
    auto* cb = rt->op<BuildOp>("customer_build", 3, cfx, nullptr, std::vector<uint32_t>{0}, /*semi=*/true);
    EB fo;
    fo.cmp(TQ_LT).col(O_ORDERDATE).i64(9204);
    Holder* of = P.wire(rt->op<ProbeOp>("orders_probe", 4, cb, odx, &fo,
                                        std::vector<EB>{Col(O_ORDERKEY), Col(O_ORDERDATE), Col(O_SHIPPRIORITY), Col(O_CUSTKEY)},
                                        std::vector<uint32_t>{3}, none));
    // join 2: orders_f x lineitem_f on orderkey — both hash-partitioned at SF100;
    // lineitem_f's shuffle drops rows missing the orders_f tables (partitioned LIP)
    XPair* x2 = P.pair("orders_lineitem");
    XSideOp* ofs = nullptr;
    Holder* ofx = P.side(x2, 0, "orders_f", 5, of, od, nullptr, {}, {0}, nullptr, &ofs);
    auto* ob = rt->op<BuildOp>("orders_build", 6, ofx, nullptr, std::vector<uint32_t>{0}, false, ofs);
    EB fl;
    fl.cmp(TQ_GT).col(L_SHIPDATE).i64(9204);
    Holder* lfx = P.side(x2, 1, "lineitem_f", 5, li, li, &fl, {Col(L_ORDERKEY), rev()}, {0}, ob);
    Holder* j = P.wire(rt->op<ProbeOp>("lineitem_probe", 7, ob, lfx, nullptr, std::vector<EB>{}, std::vector<uint32_t>{0},
                                       std::vector<uint32_t>{1, 2}));
    // j: [o_orderdate, o_shippriority, l_orderkey, rev]; grouped by l_orderkey: co-partitioned with join 2
    return P.wire(rt->op<AggOp>("q3_agg", 8, j, nullptr, std::vector<EB>{}, std::vector<uint32_t>{2, 0, 1},
                                std::vector<tq_agg>{{TQ_AGG_SUM, 3}}, true, x2, P.agg_turn()));
  }
  if (q == 5) {
    Holder* re = P.scan(T_REGION);
    Holder* na = P.scan(T_NATION);
    Holder* cu = P.scan(T_CUSTOMER);
    Holder* od = P.scan(T_ORDERS);
    Holder* li = P.scan(T_LINEITEM);
    Holder* su = P.scan(T_SUPPLIER);
    XPair* x1 = P.pair("region_nation");
    EB fr;
    fr.cmp(TQ_EQ).col(1).i64(2);
    Holder* rx = P.side(x1, 0, "region_f", 1, re, re, &fr, {Col(0)}, {0});
    Holder* nx = P.side(x1, 1, "nation", 1, na, na, nullptr, {}, {1});
    auto* rb = rt->op<BuildOp>("region_build", 2, rx, nullptr, std::vector<uint32_t>{0}, true);
    Holder* nf = P.wire(rt->op<ProbeOp>("nation_probe", 3, rb, nx, nullptr, std::vector<EB>{Col(0), Col(1)},
                                        std::vector<uint32_t>{1}, none));
    XPair* x2 = P.pair("nation_customer");
    Holder* nfx = P.side(x2, 0, "nation_f", 4, nf, na, nullptr, {}, {0});
    Holder* cux = P.side(x2, 1, "customer", 4, cu, cu, nullptr, {}, {1});
    auto* nb = rt->op<BuildOp>("nation_build", 5, nfx, nullptr, std::vector<uint32_t>{0}, true);
    Holder* cf = P.wire(rt->op<ProbeOp>("customer_probe", 6, nb, cux, nullptr, std::vector<EB>{Col(0), Col(1)},
                                        std::vector<uint32_t>{1}, none));
    XPair* x3 = P.pair("customer_orders");
    Holder* cfx = P.side(x3, 0, "customer_f", 7, cf, cu, nullptr, {}, {0});
    EB fo;
    fo.land().cmp(TQ_GE).col(O_ORDERDATE).i64(8766).cmp(TQ_LT).col(O_ORDERDATE).i64(9131);
    Holder* odx = P.side(x3, 1, "orders_f", 7, od, od, &fo, {Col(O_ORDERKEY), Col(O_CUSTKEY)}, {1});
    auto* cb = rt->op<BuildOp>("customer_build", 8, cfx, nullptr, std::vector<uint32_t>{0});
    Holder* of = P.wire(rt->op<ProbeOp>("orders_probe", 9, cb, odx, nullptr, std::vector<EB>{},
                                        std::vector<uint32_t>{1}, std::vector<uint32_t>{1}));
    // of: [c_nationkey, o_orderkey, o_custkey]
    XPair* x4 = P.pair("orders_lineitem");
    Holder* ofx = P.side(x4, 0, "orders_j", 10, of, od, nullptr, {}, {1});
    Holder* lix = P.side(x4, 1, "lineitem", 10, li, li, nullptr, {Col(L_ORDERKEY), Col(L_SUPPKEY), rev()}, {0});
    auto* ob = rt->op<BuildOp>("orders_build", 11, ofx, nullptr, std::vector<uint32_t>{1});
    Holder* lj = P.wire(rt->op<ProbeOp>("lineitem_probe", 12, ob, lix, nullptr, std::vector<EB>{},
                                        std::vector<uint32_t>{0}, std::vector<uint32_t>{0}));
    // lj: [c_nationkey, l_orderkey, l_suppkey, rev]
    XPair* x5 = P.pair("supplier_lineitem");
    Holder* sux = P.side(x5, 0, "supplier", 13, su, su, nullptr, {}, {0, 1});
    Holder* ljx = P.side(x5, 1, "lineitem_j", 13, lj, li, nullptr, {}, {2, 0});
    auto* sb = rt->op<BuildOp>("supplier_build", 14, sux, nullptr, std::vector<uint32_t>{0, 1});
    Holder* sj = P.wire(rt->op<ProbeOp>("supplier_probe", 15, sb, ljx, nullptr, std::vector<EB>{},
                                        std::vector<uint32_t>{2, 0}, std::vector<uint32_t>{1}));
    // sj: [s_nationkey, c_nationkey, l_orderkey, l_suppkey, rev]
    return P.wire(rt->op<AggOp>("q5_agg", 16, sj, nullptr, std::vector<EB>{}, std::vector<uint32_t>{0},
                                std::vector<tq_agg>{{TQ_AGG_SUM, 4}}, true, nullptr, P.agg_turn()));
  }
  if (q == 9) {
    Holder* pa = P.scan(T_PART);
    Holder* ps = P.scan(T_PARTSUPP);
    Holder* li = P.scan(T_LINEITEM);
    Holder* su = P.scan(T_SUPPLIER);
    Holder* od = P.scan(T_ORDERS);
    XPair* x1 = P.pair("part_partsupp");
    EB fp;
    fp.cmp(TQ_LT).col(1).i64(54);
    Holder* pax = P.side(x1, 0, "part_f", 1, pa, pa, &fp, {Col(0)}, {0});
    Holder* psx = P.side(x1, 1, "partsupp", 1, ps, ps, nullptr, {}, {0});
    auto* pb = rt->op<BuildOp>("part_build", 2, pax, nullptr, std::vector<uint32_t>{0}, true);
    Holder* psf = P.wire(rt->op<ProbeOp>("partsupp_probe", 3, pb, psx, nullptr, std::vector<EB>{},
                                         std::vector<uint32_t>{0}, none));
    // psf: [ps_partkey, ps_suppkey, ps_supplycost]
    XPair* x2 = P.pair("partsupp_lineitem");
    Holder* psfx = P.side(x2, 0, "partsupp_f", 4, psf, ps, nullptr, {}, {0, 1});
    Holder* lix = P.side(x2, 1, "lineitem", 4, li, li, nullptr,
                         {Col(L_ORDERKEY), Col(L_PARTKEY), Col(L_SUPPKEY), Col(L_QUANTITY), Col(L_EXTPRICE),
                          Col(L_DISCOUNT)},
                         {1, 2});
    auto* pst = rt->op<BuildOp>("partsupp_build", 5, psfx, nullptr, std::vector<uint32_t>{0, 1});
    Holder* lj = P.wire(rt->op<ProbeOp>("lineitem_probe", 6, pst, lix, nullptr, std::vector<EB>{},
                                        std::vector<uint32_t>{1, 2}, std::vector<uint32_t>{2}));
    // lj: [ps_supplycost, l_orderkey, l_partkey, l_suppkey, qty, ep, disc]
    XPair* x3 = P.pair("supplier_lineitem");
    Holder* sux = P.side(x3, 0, "supplier", 7, su, su, nullptr, {}, {0});
    Holder* ljx = P.side(x3, 1, "lineitem_j", 7, lj, li, nullptr, {}, {3});
    auto* sb = rt->op<BuildOp>("supplier_build", 8, sux, nullptr, std::vector<uint32_t>{0});
    Holder* sj = P.wire(rt->op<ProbeOp>("supplier_probe", 9, sb, ljx, nullptr, std::vector<EB>{},
                                        std::vector<uint32_t>{3}, std::vector<uint32_t>{1}));
    // sj: [s_nationkey, ps_supplycost, l_orderkey, l_partkey, l_suppkey, qty, ep, disc]
    XPair* x4 = P.pair("orders_lineitem");
    Holder* odx = P.side(x4, 0, "orders", 10, od, od, nullptr, {Col(O_ORDERKEY), Col(O_YEAR)}, {0});
    EB amt;
    amt.ar(TQ_SUB).ar(TQ_MUL).col(6).ar(TQ_SUB).dec(100).col(7).ar(TQ_MUL).col(1).col(5);
    Holder* sjx = P.side(x4, 1, "lineitem_s", 10, sj, li, nullptr, {Col(0), Col(2), amt}, {1});
    // sjx: [s_nationkey, l_orderkey, amt]
    auto* ob = rt->op<BuildOp>("orders_build", 11, odx, nullptr, std::vector<uint32_t>{0});
    Holder* oj = P.wire(rt->op<ProbeOp>("orders_probe", 12, ob, sjx, nullptr, std::vector<EB>{},
                                        std::vector<uint32_t>{1}, std::vector<uint32_t>{1}));
    // oj: [o_year, s_nationkey, l_orderkey, amt]
    return P.wire(rt->op<AggOp>("q9_agg", 13, oj, nullptr, std::vector<EB>{}, std::vector<uint32_t>{1, 0},
                                std::vector<tq_agg>{{TQ_AGG_SUM, 3}}, true, nullptr, P.agg_turn()));
  }
  fail(TQ_INVALID_PLAN, "query " + std::to_string(q) + " has no distributed plan");
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

namespace {
tq_status run_query(tq_ctx* c, tq_comm* comm, int query, const tq_batch* tables, tq_tcf* const* files,
                    const tq_engine_opts* o, tq_batch* result, char* metrics_json, uint64_t cap) {
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
    for (int t = 0; t < 8; ++t) host_tables |= (tables[t].cols && tables[t].mem == TQ_MEM_HOST) || files[t];
    if (!rt.opts.pool_capacity && (rt.capacity || host_tables)) {
      // Host tier sized for the host tables plus spill headroom
      uint64_t bytes = 4ull << 30;
      for (int t = 0; t < 8; ++t)
        if (!files[t] && tables[t].cols && tables[t].mem == TQ_MEM_HOST)
          bytes += batch_bytes(tables[t]) + (tables[t].rows / 512 + 1) * 8 * tables[t].ncols * 2;
        else if (files[t])
          for (uint32_t g = 0; g < tq_tcf_row_groups(files[t]); ++g)
            bytes += tq_tcf_rows(files[t], g) * 64 + (2ull << 20);  // (+ one buffer tail per column)
      rt.opts.pool_capacity = bytes / rt.opts.pool_buffer_size + 1;
    }
    rt.setup();
    int nranks = 1;
    if (comm) nranks = tq_comm_size(comm);
    // N > 1 workers: the distributed plan (a query without one fails with
    // InvalidPlan rather than joining / aggregating only this worker's shard)
    Plan P{&rt, tables};
    Holder* res = nranks > 1 ? build_dist_plan(P, query) : build_plan(P, query);
    SinkOp* sink = rt.op<SinkOp>(res);
    // publish the scans: device tables as zero-copy row-group views; HOST
    // tables are encoded into the pinned pool (Host tier) and every scan task
    // goes through load_to_device
    for (ScanOp* s : P.scans) {
      tq_tcf* file = nullptr;
      for (int t = 0; t < 8; ++t)
        if (&tables[t] == (const tq_batch*)s->src && files[t]) file = files[t];
      if (file) {
        // a TCF table: one STORAGE-tier handle per row group; the scan tasks
        // (and the Pre-loading executor ahead of them) fetch its byte ranges
        // into the pinned pool and move them to the device
        if (!rt.pool) fail(TQ_INVALID_PLAN, "TCF tables need a host pool");
        for (uint32_t g = 0; g < tq_tcf_row_groups(file); ++g) {
          HP h = std::make_shared<Handle>();
          h->tier = STORAGE;
          h->file = file;
          h->row_group = g;
          uint64_t n = 0;
          std::vector<uint32_t> cols(tq_tcf_ncols(file)), gs{g};
          for (uint32_t k = 0; k < cols.size(); ++k) cols[k] = k;
          std::vector<tq_range> rs(cols.size());
          check(tq_tcf_plan_ranges(file, cols.data(), (uint32_t)cols.size(), gs.data(), 1, rs.data(), rs.size(), &n));
          for (uint64_t i = 0; i < n; ++i) h->bytes += rs[i].length;
          {
            std::lock_guard<std::mutex> lk(rt.mu);
            h->id = ++rt.next_id;
            rt.registry.push_back(h);
          }
          s->out->push(h);
          s->nbatches++;
        }
        s->finished = true;
      } else if (s->table.mem == TQ_MEM_HOST) {
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
          s->nbatches++;
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
    rt.start_threads();
    const auto t_run = Clock::now();
    const double setup_ms = std::chrono::duration<double, std::milli>(t_run - t0).count();
    try {
      rt.run();
    } catch (...) {
      c->budget = saved_budget;
      throw;
    }
    const auto t_done = Clock::now();
    const double run_ms = std::chrono::duration<double, std::milli>(t_done - t_run).count();
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
    // (run_ms: the run phase — the result's download to the host is download_ms)
    double download_ms = std::chrono::duration<double, std::milli>(Clock::now() - t_done).count();
    if (metrics_json && cap) {
      std::ostringstream js;
      js << "{\"wall_ms\": " << wall << ", \"setup_ms\": " << setup_ms << ", \"run_ms\": " << run_ms << ", \"download_ms\": " << download_ms << ", \"tasks\": " << rt.m_tasks << ", \"oom_retries\": " << rt.m_retries
         << ", \"splits\": " << rt.m_splits << ", \"spills\": " << rt.m_spills << ", \"spill_bytes\": " << rt.m_spill_bytes
         << ", \"loads\": " << rt.m_loads << ", \"preloads\": " << rt.m_preloads << ", \"load_bytes\": " << rt.m_load_bytes
         << ", \"storage_reads\": " << rt.m_storage_reads
         << ", \"peak_device_bytes\": " << rt.m_peak << ", \"device_capacity\": " << rt.capacity
         << ", \"exchange_decisions\": [";
      for (size_t i = 0; i < rt.decisions.size(); ++i) {
        const auto& d = rt.decisions[i];
        js << (i ? ", " : "") << "{\"pair\": \"" << d.name << "\", \"strategy\": \""
           << (d.strategy == TQ_XCHG_BROADCAST ? "Broadcast" : "HashPartition") << "\", \"broadcast_side\": " << d.side
           << ", \"total0\": " << d.total0 << ", \"total1\": " << d.total1 << "}";
      }
      js << "], \"timeline\": [";
      for (size_t i = 0; i < rt.timeline.size(); ++i) {
        const auto& sp = rt.timeline[i];
        js << (i ? ", " : "") << "[\"" << sp.op << "\", " << sp.kind << ", " << sp.t0 << ", " << sp.t1 << "]";
      }
      js << "], \"ops\": {";
      bool first = true;
      for (auto& op : rt.ops) {
        if (!op->stat.tasks) continue;
        js << (first ? "" : ", ") << "\"" << op->name << "\": {\"tasks\": " << op->stat.tasks << ", \"ms\": " << op->stat.ms
           << ", \"gpu_ms\": " << op->stat.gpu_ms << ", \"call_ms\": " << op->stat.first_call_ms
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
}  // namespace

tq_status tq_engine_run_query(tq_ctx* c, tq_comm* comm, int query, const tq_batch* tables, const tq_engine_opts* o,
                              tq_batch* result, char* metrics_json, uint64_t cap) {
  tq_tcf* none[8] = {};
  return run_query(c, comm, query, tables, none, o, result, metrics_json, cap);
}

tq_status tq_engine_run_query_tcf(tq_ctx* c, tq_comm* comm, int query, const char* const* paths,
                                  const tq_engine_opts* o, tq_batch* result, char* metrics_json, uint64_t cap) {
  tq_tcf* files[8] = {};
  tq_batch tabs[8] = {};
  std::vector<std::vector<tq_column>> schemas(8);
  tq_status st = TQ_OK;
  for (int t = 0; t < 8 && st == TQ_OK; ++t) {
    if (!paths[t]) continue;
    st = tq_tcf_open(paths[t], &files[t]);
    if (st != TQ_OK) break;
    // a schema-only descriptor: the plans read the kinds; the rows come from the row groups
    schemas[t].resize(tq_tcf_ncols(files[t]));
    for (uint32_t k = 0; k < schemas[t].size(); ++k) tq_tcf_column(files[t], k, &schemas[t][k]);
    for (uint32_t g = 0; g < tq_tcf_row_groups(files[t]); ++g) tabs[t].rows += tq_tcf_rows(files[t], g);
    tabs[t].ncols = (uint32_t)schemas[t].size();
    tabs[t].mem = TQ_MEM_HOST;
    tabs[t].cols = schemas[t].data();
  }
  if (st == TQ_OK) st = run_query(c, comm, query, tabs, files, o, result, metrics_json, cap);
  for (tq_tcf* f : files) tq_tcf_close(f);
  return st;
}

}  // extern "C"
