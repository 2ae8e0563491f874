// boundary_test.cpp — TEST INFRASTRUCTURE (not product code): the binding of
// INTEGRATION.md §2-3 compiled against the REFERENCE's own headers and
// columnar code (oracle/build_ref.sh links it with the reference sources
// where they lie under /root/reference/proj — nothing is copied) and against
// libtq_gpu.so through include/tq_gpu.h only.
//
//   reference ColumnBatch -> HostView (zero-copy tq_batch) -> tq_batch_upload
//   -> tq_filter / tq_aggregate on the GPU -> tq_batch_download -> ColumnBatch
//
// and the result is compared with the reference's own ColumnBatch
// operator== (types.hpp:137): for filter_execute against take() of the
// passing rows (transform.cpp:90-120, the reference's materialisation), for
// aggregate_execute against the SPEC.md:609 example.  Errors cross the
// C-ABI as tq_status and come back as tierq::Error{Errc} (common.hpp:57-74).
// Exit code 0 = every check passed.  Needs a GPU (run by tests/test_boundary.py
// under -m gpu).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "tierq/columnar/transform.hpp"
#include "tierq/columnar/types.hpp"
#include "tierq/common.hpp"
#include "tq_gpu.h"

using namespace tierq;
using namespace tierq::columnar;

namespace {

// borrow a reference batch as a host tq_batch (no copy).
struct HostView {
  std::vector<tq_column> cols;
  tq_batch b{};
  explicit HostView(const ColumnBatch& cb) {
    for (const auto& c : cb.columns()) {
      tq_column t{};
      t.kind = uint8_t(c.dtype.kind);  // same ordinals as TypeKind
      t.precision = c.dtype.precision;
      t.scale = c.dtype.scale;
      t.values = const_cast<uint8_t*>(c.values.data());
      t.values_bytes = c.values.size();
      t.validity = c.validity ? const_cast<uint8_t*>(c.validity->data()) : nullptr;
      t.offsets = c.offsets ? const_cast<int32_t*>(c.offsets->data()) : nullptr;
      cols.push_back(t);
    }
    b = tq_batch{cb.rows(), uint32_t(cols.size()), TQ_MEM_HOST, cols.data(), nullptr};
  }
};

// a tq_status becomes the reference's exception.
void tq_throw(tq_status s) {
  if (s) throw_error(Errc(s - 1), tq_last_error());
}

// A downloaded host tq_batch -> reference ColumnBatch (the constructor
// validates and canonicalises, types.cpp:135-144).
ColumnBatch to_ref(const tq_batch& h, const Schema& like) {
  Schema s;
  std::vector<Column> cols;
  for (uint32_t c = 0; c < h.ncols; ++c) {
    const tq_column& t = h.cols[c];
    Field f;
    f.name = c < like.fields.size() ? like.fields[c].name : "c" + std::to_string(c);
    f.dtype = DataType{TypeKind(t.kind), t.precision, t.scale};
    s.fields.push_back(f);
    Column col;
    col.dtype = f.dtype;
    const uint8_t* v = static_cast<const uint8_t*>(t.values);
    col.values.assign(v, v + t.values_bytes);
    if (t.validity) col.validity.emplace(t.validity, t.validity + (h.rows + 7) / 8);
    cols.push_back(std::move(col));
  }
  return ColumnBatch(std::move(s), h.rows, std::move(cols));
}

// GPU operator round trip: upload, op, download, back to ColumnBatch.
template <class Op>
ColumnBatch on_gpu(tq_ctx* ctx, const ColumnBatch& in, const Schema& out_like, Op op) {
  HostView hv(in);
  tq_batch dev{}, out{}, host{};
  tq_throw(tq_batch_upload(ctx, &hv.b, &dev, nullptr));
  tq_status s = op(&dev, &out);
  tq_batch_free(ctx, &dev);
  tq_throw(s);
  tq_throw(tq_batch_download(ctx, &out, &host, nullptr));
  tq_batch_free(ctx, &out);
  ColumnBatch r = to_ref(host, out_like);
  tq_host_batch_free(&host);
  return r;
}

tq_expr_node col(uint32_t c) {
  tq_expr_node n{};
  n.tag = TQ_EX_COL;
  n.column = c;
  return n;
}
tq_expr_node lit_i64(int64_t v) {
  tq_expr_node n{};
  n.tag = TQ_EX_LIT;
  n.kind = TQ_INT64;
  n.lo = uint64_t(v);
  return n;
}
tq_expr_node cmp(int op) {
  tq_expr_node n{};
  n.tag = TQ_EX_CMP;
  n.op = uint8_t(op);
  return n;
}

int failures = 0;
void expect(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "ok  " : "FAIL", what.c_str());
  if (!ok) ++failures;
}

Schema schema_of(std::initializer_list<std::pair<std::string, DataType>> fs) {
  Schema s;
  for (auto& f : fs) s.fields.push_back(Field{f.first, f.second, true});
  return s;
}

}  // namespace

int main() {
  tq_opts o{};
  tq_ctx* ctx = nullptr;
  tq_throw(tq_ctx_create(&o, &ctx));
  const DataType i64{TypeKind::Int64, 0, 0}, dec{TypeKind::Decimal, 11, 2};

  // ---- x < 5 on [1, 7, 3, null] -> [1, 3]
  {
    std::vector<int64_t> x = {1, 7, 3, 0};
    std::vector<bool> valid = {true, true, true, false};
    ColumnBatch in(schema_of({{"x", i64}}), 4, {make_i64_column(x, &valid)});
    std::vector<tq_expr_node> p = {cmp(TQ_LT), col(0), lit_i64(5)};
    ColumnBatch got = on_gpu(ctx, in, in.schema(), [&](tq_batch* d, tq_batch* out) {
      return tq_filter(ctx, d, tq_expr{p.data(), uint32_t(p.size()), 0}, out, nullptr);
    });
    std::vector<int64_t> w = {1, 3};
    std::vector<bool> wv = {true, true};
    // the reference's take keeps the input's bitmap (transform.cpp:112-116)
    ColumnBatch want(schema_of({{"x", i64}}), 2, {make_i64_column(w, &wv)});
    expect(got == want, "filter_execute SPEC.md:565 example == reference ColumnBatch");
  }

  // ---- random batch: GPU filter == reference take() of the passing rows
  {
    const uint64_t n = 100000;
    std::vector<int64_t> k(n);
    std::vector<int128_t> v(n);
    std::vector<bool> valid(n);
    uint64_t s = 42;
    for (uint64_t i = 0; i < n; ++i) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      k[i] = int64_t((s >> 33) % 1000) - 500;
      v[i] = int128_t(int64_t(s >> 20)) * 977;
      valid[i] = (s >> 7) % 10 != 0;
    }
    ColumnBatch in(schema_of({{"k", i64}, {"v", dec}}), n, {make_i64_column(k, &valid), make_dec_column(v, 11, 2)});
    std::vector<tq_expr_node> p = {cmp(TQ_GE), col(0), lit_i64(17)};
    ColumnBatch got = on_gpu(ctx, in, in.schema(), [&](tq_batch* d, tq_batch* out) {
      return tq_filter(ctx, d, tq_expr{p.data(), uint32_t(p.size()), 0}, out, nullptr);
    });
    std::vector<uint64_t> ids;
    for (uint64_t i = 0; i < n; ++i)
      if (in.column(0).valid_at(i) && in.column(0).i64_at(i) >= 17) ids.push_back(i);
    ColumnBatch want = take(in, ids);
    expect(got == want, "filter_execute 100K rows (nulls) == reference take() of the passing rows, " +
                            std::to_string(ids.size()) + " rows");
  }

  // ---- a single group, Count(*) over n rows -> n
  {
    std::vector<int64_t> x(5, 3);
    ColumnBatch in(schema_of({{"g", i64}}), 5, {make_i64_column(x)});
    const uint32_t keys[1] = {0};
    const tq_agg aggs[1] = {{TQ_AGG_COUNT_STAR, 0}};
    Schema out_s = schema_of({{"g", i64}, {"count", i64}});
    ColumnBatch got = on_gpu(ctx, in, out_s, [&](tq_batch* d, tq_batch* out) {
      return tq_aggregate(ctx, d, keys, 1, aggs, 1, out, nullptr);
    });
    std::vector<int64_t> g = {3}, c = {5};
    ColumnBatch want(out_s, 1, {make_i64_column(g), make_i64_column(c)});
    expect(got == want, "aggregate_execute SPEC.md:609 example == reference ColumnBatch");
  }

  // ---- errors cross the C-ABI as tq_status and come back as tierq::Error{Errc}
  {
    std::vector<int64_t> x = {1, 2, 3};
    ColumnBatch in(schema_of({{"x", i64}}), 3, {make_i64_column(x)});
    std::vector<tq_expr_node> p = {cmp(TQ_LT), col(5), lit_i64(1)};  // no column 5
    bool caught = false;
    try {
      on_gpu(ctx, in, in.schema(), [&](tq_batch* d, tq_batch* out) {
        return tq_filter(ctx, d, tq_expr{p.data(), uint32_t(p.size()), 0}, out, nullptr);
      });
    } catch (const Error& e) {
      caught = e.code() == Errc::InvalidPlan;
    }
    expect(caught, "InvalidPlan status -> tierq::Error{Errc::InvalidPlan}");
  }

  tq_ctx_destroy(ctx);
  std::printf("%s\n", failures ? "boundary_test FAILED" : "boundary_test ok");
  return failures ? 1 : 0;
}
