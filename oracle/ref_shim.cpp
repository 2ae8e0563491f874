// ref_shim.cpp — CPU ORACLE support (test infrastructure, NOT product code).
//
// extern "C" wrappers around the REFERENCE's own columnar code, compiled
// together with the reference sources where they lie under
// /root/reference/proj (never copied) by oracle/build_ref.sh into
// oracle/_ref/libtierq_ref.so.  Tests use it to pin the oracle restatement
// (oracle/tq_oracle.cpp) and the GPU take/concat/slice against the
// reference's transform.cpp:21-154, common.hpp:128-158, types.cpp:146-170
// and chunked.cpp:19-124.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tierq/columnar/chunked.hpp"
#include "tierq/columnar/pool.hpp"
#include "tierq/columnar/transform.hpp"
#include "tierq/columnar/types.hpp"
#include "tierq/common.hpp"
#include "../include/tq_types.h"

using namespace tierq;
using namespace tierq::columnar;

namespace {
thread_local std::string g_err;

ColumnBatch to_ref(const tq_batch* b) {
  Schema s;
  std::vector<Column> cols;
  for (uint32_t c = 0; c < b->ncols; ++c) {
    const tq_column& t = b->cols[c];
    Field f;
    f.name = "c" + std::to_string(c);
    f.dtype = DataType{TypeKind(t.kind), t.precision, t.scale};
    s.fields.push_back(f);
    Column col;
    col.dtype = f.dtype;
    const uint8_t* v = static_cast<const uint8_t*>(t.values);
    col.values.assign(v, v + t.values_bytes);
    if (t.validity) col.validity.emplace(t.validity, t.validity + (b->rows + 7) / 8);
    if (t.kind == TQ_UTF8) col.offsets.emplace(t.offsets, t.offsets + b->rows + 1);
    cols.push_back(std::move(col));
  }
  return ColumnBatch(std::move(s), b->rows, std::move(cols));
}

void from_ref(const ColumnBatch& r, tq_batch* out) {
  out->rows = r.rows();
  out->ncols = uint32_t(r.columns().size());
  out->mem = TQ_MEM_HOST;
  out->owner = nullptr;
  out->cols = static_cast<tq_column*>(std::calloc(out->ncols ? out->ncols : 1, sizeof(tq_column)));
  for (uint32_t c = 0; c < out->ncols; ++c) {
    const Column& s = r.column(c);
    tq_column& d = out->cols[c];
    d.kind = uint8_t(s.dtype.kind);
    d.precision = s.dtype.precision;
    d.scale = s.dtype.scale;
    d.values_bytes = s.values.size();
    d.values = std::malloc(s.values.size() ? s.values.size() : 1);
    if (!s.values.empty()) std::memcpy(d.values, s.values.data(), s.values.size());
    d.validity = nullptr;
    if (s.validity) {
      d.validity = static_cast<uint8_t*>(std::malloc(s.validity->size() ? s.validity->size() : 1));
      if (!s.validity->empty()) std::memcpy(d.validity, s.validity->data(), s.validity->size());
    }
    d.offsets = nullptr;
    if (s.offsets) {
      d.offsets = static_cast<int32_t*>(std::malloc(s.offsets->size() * 4));
      std::memcpy(d.offsets, s.offsets->data(), s.offsets->size() * 4);
    }
  }
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + int(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1 + int(Errc::Internal);
  }
}
}  // namespace

extern "C" {

const char* tqr_last_error(void) { return g_err.c_str(); }

void tqr_batch_free(tq_batch* b) {
  if (!b || !b->cols) return;
  for (uint32_t c = 0; c < b->ncols; ++c) {
    std::free(b->cols[c].values);
    std::free(b->cols[c].validity);
    std::free(b->cols[c].offsets);
  }
  std::free(b->cols);
  b->cols = nullptr;
}

uint64_t tqr_fnv1a64(const uint8_t* p, uint64_t n, uint64_t seed) {
  return fnv1a64(std::span<const uint8_t>(p, n), seed);
}

// First n outputs of SplitMix64(seed).next() into out.
void tqr_splitmix(uint64_t seed, uint64_t n, uint64_t* out) {
  SplitMix64 g(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = g.next();
}
// next_below(bound) sequence.
void tqr_splitmix_below(uint64_t seed, uint64_t bound, uint64_t n, uint64_t* out) {
  SplitMix64 g(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = g.next_below(bound);
}

int tqr_validate(const tq_batch* in) {
  return guard([&] { (void)to_ref(in); });
}

int tqr_take(const tq_batch* in, const uint64_t* ids, uint64_t n, tq_batch* out) {
  return guard([&] { from_ref(take(to_ref(in), std::span<const uint64_t>(ids, n)), out); });
}

int tqr_concat(const tq_batch* ins, uint32_t n, tq_batch* out) {
  return guard([&] {
    std::vector<ColumnBatch> v;
    for (uint32_t i = 0; i < n; ++i) v.push_back(to_ref(&ins[i]));
    from_ref(concat(v), out);
  });
}

int tqr_slice(const tq_batch* in, uint64_t start, uint64_t len, tq_batch* out) {
  return guard([&] { from_ref(slice(to_ref(in), start, len), out); });
}

uint64_t tqr_batch_size_bytes(const tq_batch* in) {
  uint64_t r = 0;
  guard([&] { r = batch_size_bytes(to_ref(in)); });
  return r;
}

// rebatch: returns number of output batches and their row counts (<= cap).
int tqr_rebatch_rows(const tq_batch* in, uint64_t target, uint64_t* rows_out, uint32_t cap, uint32_t* n_out) {
  return guard([&] {
    ColumnBatch b = to_ref(in);
    auto parts = rebatch(std::span<const ColumnBatch>(&b, 1), target);
    *n_out = uint32_t(parts.size());
    for (uint32_t i = 0; i < parts.size() && i < cap; ++i) rows_out[i] = parts[i].rows();
  });
}

// encode_chunked into a fresh pool; reports buffers used, tail and the
// per-section (buffer_id, offset, length) segments, then decodes and checks
// the round trip (chunked.cpp:19-124).
int tqr_chunked_layout(const tq_batch* in, uint64_t buffer_size, uint64_t capacity, uint64_t* nbuf,
                       uint64_t* tail, uint32_t* segs, uint32_t seg_cap, uint32_t* nsegs, int* roundtrip_ok) {
  return guard([&] {
    ColumnBatch b = to_ref(in);
    FixedBufferPool pool(buffer_size, capacity);
    auto cb = encode_chunked(b, pool);
    check(cb.has_value(), Errc::PoolExhausted, "pool exhausted");
    *nbuf = cb->buffers.size();
    *tail = cb->unused_tail_bytes;
    uint32_t k = 0;
    for (const auto& sec : cb->sections)
      for (const auto& s : sec.segments) {
        if (k < seg_cap) {
          segs[3 * k] = s.buffer_id;
          segs[3 * k + 1] = s.offset;
          segs[3 * k + 2] = s.length;
        }
        ++k;
      }
    *nsegs = k;
    *roundtrip_ok = decode_chunked(*cb, pool) == b ? 1 : 0;
    release_chunked(*cb, pool);
  });
}


// ---- CPU baseline over the REFERENCE's own batch and accessors -------------
// A lineitem batch converted once into the reference's ColumnBatch and kept
// resident (the GPU's tables are resident in HBM too); the timed work is a
// fused single pass of Q1 over Column::i64_at / dec_at
// (types.cpp:66-90), one thread per row range, per-thread group accumulators
// merged at the end.  Group keys are the l_returnflag / l_linestatus codes.
void* tqr_resident_make(const tq_batch* in) {
  try {
    return new ColumnBatch(to_ref(in));
  } catch (...) {
    return nullptr;
  }
}
void tqr_resident_free(void* b) { delete static_cast<ColumnBatch*>(b); }

// out: ngroups, then per group {rf, ls, sum_qty(lo,hi), sum_ep, sum_dp, sum_ch, sum_disc, count} as u64 words
// (16 words per group); returns the seconds of the fused pass.
double tqr_q1_fused(void* batch, uint32_t nthreads, uint64_t* out, uint32_t cap_groups) {
  const ColumnBatch& b = *static_cast<ColumnBatch*>(batch);
  enum { OK, PK, SK, QTY, EP, DISC, TAX, RF, LS, SD };
  struct Acc {
    int64_t rf, ls;
    int128_t qty, ep, dp, ch, disc;
    uint64_t n;
  };
  const uint64_t rows = b.rows();
  nthreads = std::max<uint32_t>(1, nthreads);
  std::vector<std::vector<Acc>> part(nthreads);
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> ts;
  for (uint32_t t = 0; t < nthreads; ++t)
    ts.emplace_back([&, t] {
      const uint64_t r0 = rows * t / nthreads, r1 = rows * (t + 1) / nthreads;
      const Column &sd = b.column(SD), &rf = b.column(RF), &ls = b.column(LS), &qty = b.column(QTY),
                   &ep = b.column(EP), &disc = b.column(DISC), &tax = b.column(TAX);
      std::vector<Acc>& g = part[t];
      for (uint64_t r = r0; r < r1; ++r) {
        if (!(sd.i64_at(r) <= 10471)) continue;
        const int64_t k0 = rf.i64_at(r), k1 = ls.i64_at(r);
        Acc* a = nullptr;
        for (Acc& x : g)
          if (x.rf == k0 && x.ls == k1) { a = &x; break; }
        if (!a) { g.push_back(Acc{k0, k1, 0, 0, 0, 0, 0, 0}); a = &g.back(); }
        const int128_t q = qty.dec_at(r), e = ep.dec_at(r), d = disc.dec_at(r), x = tax.dec_at(r);
        const int128_t dp = e * (int128_t(100) - d);
        a->qty += q;
        a->ep += e;
        a->dp += dp;
        a->ch += dp * (int128_t(100) + x);
        a->disc += d;
        a->n += 1;
      }
    });
  for (auto& t : ts) t.join();
  std::vector<Acc> all;
  for (auto& g : part)
    for (const Acc& x : g) {
      Acc* a = nullptr;
      for (Acc& y : all)
        if (y.rf == x.rf && y.ls == x.ls) { a = &y; break; }
      if (!a) { all.push_back(x); continue; }
      a->qty += x.qty; a->ep += x.ep; a->dp += x.dp; a->ch += x.ch; a->disc += x.disc; a->n += x.n;
    }
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  out[0] = all.size();
  for (size_t i = 0; i < all.size() && i < cap_groups; ++i) {
    uint64_t* o = out + 1 + 16 * i;
    const Acc& a = all[i];
    o[0] = (uint64_t)a.rf;
    o[1] = (uint64_t)a.ls;
    const int128_t v[5] = {a.qty, a.ep, a.dp, a.ch, a.disc};
    for (int k = 0; k < 5; ++k) {
      o[2 + 2 * k] = (uint64_t)v[k];
      o[3 + 2 * k] = (uint64_t)((unsigned __int128)v[k] >> 64);
    }
    o[12] = a.n;
  }
  return sec;
}

// Host memory read bandwidth (GB/s): nthreads sum disjoint slices of a
// `bytes` buffer, best of `reps` passes.
double tqr_read_bw(uint64_t bytes, uint32_t nthreads, uint32_t reps) {
  nthreads = std::max<uint32_t>(1, nthreads);
  const uint64_t n = bytes / 8;
  std::vector<uint64_t> buf(n);
  for (uint64_t i = 0; i < n; ++i) buf[i] = i * 0x9e3779b97f4a7c15ull;
  double best = 0;
  std::vector<uint64_t> sink(nthreads * 8);
  for (uint32_t k = 0; k < reps; ++k) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ts;
    for (uint32_t t = 0; t < nthreads; ++t)
      ts.emplace_back([&, t] {
        const uint64_t a = n * t / nthreads, e = n * (t + 1) / nthreads;
        uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        uint64_t i = a;
        for (; i + 4 <= e; i += 4) { s0 += buf[i]; s1 += buf[i + 1]; s2 += buf[i + 2]; s3 += buf[i + 3]; }
        for (; i < e; ++i) s0 += buf[i];
        sink[t * 8] = s0 + s1 + s2 + s3;
      });
    for (auto& t : ts) t.join();
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    best = std::max(best, (double)(n * 8) / sec / 1e9);
  }
  return best;
}

}  // extern "C"
