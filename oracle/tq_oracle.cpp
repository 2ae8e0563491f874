// tq_oracle.cpp — CPU ORACLE (test infrastructure; see tq_oracle.h header).
//
// Independent restatement of the reference's hot-path semantics.  Nothing in
// the product (paper_2508_05029_b200/) links or calls this file.
//
// Reference anchors (file:line under /root/reference):
//   fnv1a64 ............ proj/include/tierq/common.hpp:128-136
//   SplitMix64 ......... proj/include/tierq/common.hpp:139-158
//   bitmap helpers ..... proj/include/tierq/columnar/types.hpp:89-100
//   canonicalize ....... proj/src/columnar/types.cpp:123-131
//   slice/concat/take .. proj/src/columnar/transform.cpp:21-120
//   Expr + null rule ... SPEC.md:541-544
//   filter/project ..... SPEC.md:560-570
//   hash_partition ..... SPEC.md:589-595, 621
//   join_execute ....... SPEC.md:596-603, 622 (inner, null keys never match)
//   aggregate_execute .. SPEC.md:604-611, 617
//   oracle rules ....... SPEC.md:697-714
#include "tq_oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <string_view>
#include <unordered_map>
#include <vector>

namespace {

using i128 = __int128;
using u128 = unsigned __int128;

thread_local std::string g_err;

struct OErr {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& m) { throw OErr{code, m}; }

// ---------------------------------------------------------------- hashing / rng
uint64_t fnv1a64(const uint8_t* p, size_t n, uint64_t h = 0xcbf29ce484222325ULL) {
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}
inline uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
// k-th output (k >= 1) of SplitMix64(seed): state advances by gamma before mixing.
inline uint64_t sm_nth(uint64_t seed, uint64_t k) { return sm_mix(seed + k * kGamma); }

// ---------------------------------------------------------------- columnar
inline size_t bm_bytes(uint64_t rows) { return (rows + 7) / 8; }
inline bool bit_get(const uint8_t* bm, uint64_t i) { return (bm[i >> 3] >> (i & 7)) & 1; }
inline void bit_set(uint8_t* bm, uint64_t i, bool v) {
  if (v)
    bm[i >> 3] |= uint8_t(1u << (i & 7));
  else
    bm[i >> 3] &= uint8_t(~(1u << (i & 7)));
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

struct OCol {
  uint8_t kind = TQ_INT64, precision = 0, scale = 0;
  std::vector<uint8_t> values;
  bool has_valid = false;
  std::vector<uint8_t> validity;
  std::vector<int32_t> offsets;
};
struct OBatch {
  uint64_t rows = 0;
  std::vector<OCol> cols;
};

// Borrowed view of one column (host memory).
struct CV {
  uint8_t kind = 0, precision = 0, scale = 0;
  const uint8_t* values = nullptr;
  uint64_t values_bytes = 0;
  const uint8_t* validity = nullptr;
  const int32_t* offsets = nullptr;
  bool valid(uint64_t r) const { return !validity || bit_get(validity, r); }
  int64_t i64(uint64_t r) const { int64_t v; std::memcpy(&v, values + r * 8, 8); return v; }
  double f64(uint64_t r) const { double v; std::memcpy(&v, values + r * 8, 8); return v; }
  i128 dec(uint64_t r) const { i128 v; std::memcpy(&v, values + r * 16, 16); return v; }
  bool b(uint64_t r) const { return values[r] != 0; }
};
struct BV {
  uint64_t rows = 0;
  std::vector<CV> cols;
};

BV view(const tq_batch* b) {
  if (!b) fail(TQ_INTERNAL, "null batch");
  if (b->mem != TQ_MEM_HOST) fail(TQ_INTERNAL, "oracle needs host batches");
  BV v;
  v.rows = b->rows;
  for (uint32_t c = 0; c < b->ncols; ++c) {
    const tq_column& s = b->cols[c];
    CV cv;
    cv.kind = s.kind; cv.precision = s.precision; cv.scale = s.scale;
    cv.values = static_cast<const uint8_t*>(s.values);
    cv.values_bytes = s.values_bytes;
    // A 0-row column never carries a bitmap (types.cpp:123-131 canonicalize).
    cv.validity = b->rows ? s.validity : nullptr;
    cv.offsets = s.offsets;
    if (s.kind > TQ_DECIMAL) fail(TQ_MALFORMED_BATCH, "bad kind");
    if (s.kind == TQ_UTF8) {
      if (!s.offsets) fail(TQ_MALFORMED_BATCH, "utf8 column missing offsets");
    } else if (s.values_bytes != b->rows * width_of(s.kind)) {
      fail(TQ_MALFORMED_BATCH, "values length mismatch");
    }
    v.cols.push_back(cv);
  }
  return v;
}
BV view(const OBatch& b) {
  BV v;
  v.rows = b.rows;
  for (const auto& c : b.cols) {
    CV cv;
    cv.kind = c.kind; cv.precision = c.precision; cv.scale = c.scale;
    cv.values = c.values.data();
    cv.values_bytes = c.values.size();
    cv.validity = c.has_valid ? c.validity.data() : nullptr;
    cv.offsets = c.kind == TQ_UTF8 ? c.offsets.data() : nullptr;
    v.cols.push_back(cv);
  }
  return v;
}

// canonicalize (types.cpp:123-131): drop 0-row bitmaps, zero padding bits.
void canonicalize(OBatch& b) {
  for (auto& c : b.cols) {
    if (!c.has_valid) continue;
    if (b.rows == 0) { c.has_valid = false; c.validity.clear(); continue; }
    uint64_t tail = b.rows % 8;
    if (tail) c.validity.back() &= uint8_t((1u << tail) - 1);
  }
}

void export_batch(OBatch&& b, tq_batch* out) {
  canonicalize(b);
  out->rows = b.rows;
  out->ncols = uint32_t(b.cols.size());
  out->mem = TQ_MEM_HOST;
  out->owner = nullptr;
  out->cols = static_cast<tq_column*>(std::calloc(b.cols.size() ? b.cols.size() : 1, sizeof(tq_column)));
  for (size_t c = 0; c < b.cols.size(); ++c) {
    OCol& s = b.cols[c];
    tq_column& d = out->cols[c];
    d.kind = s.kind; d.precision = s.precision; d.scale = s.scale;
    d.values_bytes = s.values.size();
    d.values = std::malloc(s.values.size() ? s.values.size() : 1);
    if (!s.values.empty()) std::memcpy(d.values, s.values.data(), s.values.size());
    d.validity = nullptr;
    if (s.has_valid) {
      d.validity = static_cast<uint8_t*>(std::malloc(s.validity.size() ? s.validity.size() : 1));
      if (!s.validity.empty()) std::memcpy(d.validity, s.validity.data(), s.validity.size());
    }
    d.offsets = nullptr;
    if (s.kind == TQ_UTF8) {
      d.offsets = static_cast<int32_t*>(std::malloc(s.offsets.size() * 4));
      std::memcpy(d.offsets, s.offsets.data(), s.offsets.size() * 4);
    }
  }
}

// take (transform.cpp:90-120): per-row gather; bitmap iff input had one and n>0.
OBatch take(const BV& in, const uint64_t* ids, uint64_t n) {
  OBatch out;
  out.rows = n;
  for (const CV& s : in.cols) {
    OCol c;
    c.kind = s.kind; c.precision = s.precision; c.scale = s.scale;
    if (s.kind != TQ_UTF8) {
      size_t w = width_of(s.kind);
      c.values.resize(n * w);
      for (uint64_t i = 0; i < n; ++i) std::memcpy(c.values.data() + i * w, s.values + ids[i] * w, w);
    } else {
      c.offsets.reserve(n + 1);
      c.offsets.push_back(0);
      for (uint64_t i = 0; i < n; ++i) {
        int32_t a = s.offsets[ids[i]], e = s.offsets[ids[i] + 1];
        c.values.insert(c.values.end(), s.values + a, s.values + e);
        c.offsets.push_back(int32_t(c.values.size()));
      }
    }
    if (s.validity && n > 0) {
      c.has_valid = true;
      c.validity.assign(bm_bytes(n), 0);
      for (uint64_t i = 0; i < n; ++i) bit_set(c.validity.data(), i, s.valid(ids[i]));
    }
    out.cols.push_back(std::move(c));
  }
  return out;
}

bool same_schema(const BV& a, const BV& b) {
  if (a.cols.size() != b.cols.size()) return false;
  for (size_t c = 0; c < a.cols.size(); ++c)
    if (a.cols[c].kind != b.cols[c].kind || a.cols[c].precision != b.cols[c].precision ||
        a.cols[c].scale != b.cols[c].scale)
      return false;
  return true;
}

// concat (transform.cpp:49-88): bitmap if any input has one.
OBatch concat(const std::vector<BV>& ins) {
  if (ins.empty()) fail(TQ_INTERNAL, "concat of nothing");
  uint64_t rows = 0;
  for (const auto& b : ins) {
    if (!same_schema(b, ins[0])) fail(TQ_SCHEMA_MISMATCH, "concat over differing schemas");
    rows += b.rows;
  }
  OBatch out;
  out.rows = rows;
  for (size_t c = 0; c < ins[0].cols.size(); ++c) {
    OCol col;
    col.kind = ins[0].cols[c].kind; col.precision = ins[0].cols[c].precision; col.scale = ins[0].cols[c].scale;
    bool hv = false;
    for (const auto& b : ins) hv |= b.cols[c].validity != nullptr;
    if (col.kind == TQ_UTF8) col.offsets.push_back(0);
    if (hv && rows > 0) { col.has_valid = true; col.validity.assign(bm_bytes(rows), 0); }
    uint64_t cur = 0;
    for (const auto& b : ins) {
      const CV& s = b.cols[c];
      if (col.kind == TQ_UTF8) {
        int32_t base = col.offsets.back();
        for (uint64_t i = 1; i <= b.rows; ++i) col.offsets.push_back(base + s.offsets[i]);
        col.values.insert(col.values.end(), s.values, s.values + s.offsets[b.rows]);
      } else {
        col.values.insert(col.values.end(), s.values, s.values + b.rows * width_of(col.kind));
      }
      if (col.has_valid)
        for (uint64_t i = 0; i < b.rows; ++i) bit_set(col.validity.data(), cur + i, s.valid(i));
      cur += b.rows;
    }
    out.cols.push_back(std::move(col));
  }
  return out;
}

OBatch slice(const BV& in, uint64_t start, uint64_t len) {
  if (start + len > in.rows) fail(TQ_INTERNAL, "slice out of range");
  std::vector<uint64_t> ids(len);
  for (uint64_t i = 0; i < len; ++i) ids[i] = start + i;
  return take(in, ids.data(), len);
}

// ---------------------------------------------------------------- Expr typing
enum Cls { C_I = 0, C_D = 1, C_F = 2, C_B = 3, C_S = 4 };
struct Ty {
  int cls = C_I;
  int scale = 0;
};
Ty ty_of_kind(uint8_t kind, uint8_t scale) {
  switch (kind) {
    case TQ_INT64: return {C_I, 0};
    case TQ_DECIMAL: return {C_D, scale};
    case TQ_FLOAT64: return {C_F, 0};
    case TQ_BOOL: return {C_B, 0};
    case TQ_UTF8: return {C_S, 0};
  }
  fail(TQ_INVALID_PLAN, "bad type kind");
}
bool numeric(Ty t) { return t.cls == C_I || t.cls == C_D || t.cls == C_F; }

struct ENode {
  int tag = 0, op = 0;
  Ty ty;
  int a = -1, b = -1;
  uint32_t col = 0;
  bool lit_null = false;
  i128 lit_i = 0;
  double lit_f = 0;
};
struct Prog {
  std::vector<ENode> n;
  int root = -1;
};

i128 lit_int(const tq_expr_node& e) {
  if (e.kind == TQ_DECIMAL) return (i128)(((u128)e.hi << 64) | (u128)e.lo);
  return (i128)(int64_t)e.lo;
}

int parse_node(const tq_expr& x, uint32_t& pos, const BV& in, Prog& p) {
  if (pos >= x.len) fail(TQ_INVALID_PLAN, "truncated expression");
  const tq_expr_node& e = x.nodes[pos++];
  ENode n;
  n.tag = e.tag;
  n.op = e.op;
  switch (e.tag) {
    case TQ_EX_COL:
      if (e.column >= in.cols.size()) fail(TQ_INVALID_PLAN, "column out of range");
      n.col = e.column;
      n.ty = ty_of_kind(in.cols[e.column].kind, in.cols[e.column].scale);
      break;
    case TQ_EX_LIT:
      n.ty = ty_of_kind(e.kind, e.scale);
      if (n.ty.cls == C_S) fail(TQ_INVALID_PLAN, "utf8 literals unsupported");
      n.lit_null = e.is_null != 0;
      if (n.ty.cls == C_F) std::memcpy(&n.lit_f, &e.lo, 8);
      else if (n.ty.cls == C_B) n.lit_i = e.lo != 0;
      else n.lit_i = lit_int(e);
      break;
    case TQ_EX_CMP: case TQ_EX_ARITH: case TQ_EX_AND: case TQ_EX_OR: {
      n.a = parse_node(x, pos, in, p);
      n.b = parse_node(x, pos, in, p);
      Ty ta = p.n[n.a].ty, tb = p.n[n.b].ty;
      if (e.tag == TQ_EX_ARITH) {
        if (e.op > TQ_MUL) fail(TQ_INVALID_PLAN, "bad arith op");
        if (!numeric(ta) || !numeric(tb)) fail(TQ_INVALID_PLAN, "arith on non-numeric");
        if (ta.cls == C_F || tb.cls == C_F) n.ty = {C_F, 0};
        else if (ta.cls == C_D || tb.cls == C_D)
          n.ty = {C_D, e.op == TQ_MUL ? ta.scale + tb.scale : std::max(ta.scale, tb.scale)};
        else n.ty = {C_I, 0};
        if (n.ty.cls == C_D && n.ty.scale > 38) fail(TQ_INVALID_PLAN, "decimal scale overflow");
      } else if (e.tag == TQ_EX_CMP) {
        if (e.op > TQ_GT) fail(TQ_INVALID_PLAN, "bad compare op");
        bool ok = (numeric(ta) && numeric(tb)) || (ta.cls == C_B && tb.cls == C_B) ||
                  (ta.cls == C_S && tb.cls == C_S);
        if (!ok) fail(TQ_INVALID_PLAN, "compare of incompatible types");
        n.ty = {C_B, 0};
      } else {
        if (ta.cls != C_B || tb.cls != C_B) fail(TQ_INVALID_PLAN, "logic on non-bool");
        n.ty = {C_B, 0};
      }
      break;
    }
    case TQ_EX_NOT:
      n.a = parse_node(x, pos, in, p);
      if (p.n[n.a].ty.cls != C_B) fail(TQ_INVALID_PLAN, "not on non-bool");
      n.ty = {C_B, 0};
      break;
    default:
      fail(TQ_INVALID_PLAN, "unknown expression tag");
  }
  p.n.push_back(n);
  return int(p.n.size() - 1);
}

Prog compile(const tq_expr& x, const BV& in) {
  Prog p;
  uint32_t pos = 0;
  p.root = parse_node(x, pos, in, p);
  if (pos != x.len) fail(TQ_INVALID_PLAN, "trailing expression nodes");
  return p;
}

// ---------------------------------------------------------------- Expr eval (vectorized)
const double kP10d[39] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11, 1e12,
                          1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22, 1e23, 1e24, 1e25,
                          1e26, 1e27, 1e28, 1e29, 1e30, 1e31, 1e32, 1e33, 1e34, 1e35, 1e36, 1e37, 1e38};
i128 p10i(int k) {
  i128 v = 1;
  for (int i = 0; i < k; ++i) v = (i128)((u128)v * 10u);
  return v;
}
inline i128 mulw(i128 a, i128 b) { return (i128)((u128)a * (u128)b); }
inline i128 addw(i128 a, i128 b) { return (i128)((u128)a + (u128)b); }
inline i128 subw(i128 a, i128 b) { return (i128)((u128)a - (u128)b); }
inline i128 w64(i128 x) { return (i128)(int64_t)(uint64_t)(u128)x; }
inline double to_f(i128 v, Ty t) {
  if (t.cls == C_I) return (double)(int64_t)v;
  return (double)v / kP10d[t.scale];
}

struct Vec {
  Ty ty;
  std::vector<i128> i;       // C_I / C_D / C_B (0/1)
  std::vector<double> f;     // C_F
  std::vector<uint8_t> v;    // valid
  const CV* scol = nullptr;  // C_S: column view (rows are absolute r0+k)
};

void eval(const Prog& p, int idx, const BV& in, uint64_t r0, uint64_t n, Vec& out) {
  const ENode& e = p.n[idx];
  out.ty = e.ty;
  out.v.assign(n, 1);
  switch (e.tag) {
    case TQ_EX_COL: {
      const CV& c = in.cols[e.col];
      if (e.ty.cls == C_S) { out.scol = &c; }
      else if (e.ty.cls == C_F) { out.f.resize(n); for (uint64_t k = 0; k < n; ++k) out.f[k] = c.f64(r0 + k); }
      else {
        out.i.resize(n);
        if (c.kind == TQ_INT64) for (uint64_t k = 0; k < n; ++k) out.i[k] = c.i64(r0 + k);
        else if (c.kind == TQ_DECIMAL) for (uint64_t k = 0; k < n; ++k) out.i[k] = c.dec(r0 + k);
        else for (uint64_t k = 0; k < n; ++k) out.i[k] = c.b(r0 + k) ? 1 : 0;
      }
      if (c.validity) for (uint64_t k = 0; k < n; ++k) out.v[k] = c.valid(r0 + k);
      return;
    }
    case TQ_EX_LIT:
      if (e.ty.cls == C_F) out.f.assign(n, e.lit_f);
      else out.i.assign(n, e.lit_i);
      if (e.lit_null) std::fill(out.v.begin(), out.v.end(), 0);
      return;
    case TQ_EX_NOT: {
      Vec a;
      eval(p, e.a, in, r0, n, a);
      out.i.resize(n);
      for (uint64_t k = 0; k < n; ++k) { out.i[k] = a.i[k] ? 0 : 1; out.v[k] = a.v[k]; }
      return;
    }
    default: break;
  }
  Vec a, b;
  eval(p, e.a, in, r0, n, a);
  eval(p, e.b, in, r0, n, b);
  for (uint64_t k = 0; k < n; ++k) out.v[k] = a.v[k] & b.v[k];  // any null operand -> null
  if (e.tag == TQ_EX_AND || e.tag == TQ_EX_OR) {
    out.i.resize(n);
    for (uint64_t k = 0; k < n; ++k)
      out.i[k] = e.tag == TQ_EX_AND ? (a.i[k] && b.i[k]) : (a.i[k] || b.i[k]);
    return;
  }
  if (e.tag == TQ_EX_ARITH && e.ty.cls != C_F) {
    out.i.resize(n);
    i128 fa = 1, fb = 1;
    if (e.ty.cls == C_D && e.op != TQ_MUL) { fa = p10i(e.ty.scale - a.ty.scale); fb = p10i(e.ty.scale - b.ty.scale); }
    for (uint64_t k = 0; k < n; ++k) {
      i128 x = mulw(a.i[k], fa), y = mulw(b.i[k], fb), r;
      r = e.op == TQ_ADD ? addw(x, y) : e.op == TQ_SUB ? subw(x, y) : mulw(x, y);
      out.i[k] = e.ty.cls == C_I ? w64(r) : r;
    }
    return;
  }
  if (e.tag == TQ_EX_ARITH) {  // float
    out.f.resize(n);
    for (uint64_t k = 0; k < n; ++k) {
      double x = a.ty.cls == C_F ? a.f[k] : to_f(a.i[k], a.ty);
      double y = b.ty.cls == C_F ? b.f[k] : to_f(b.i[k], b.ty);
      out.f[k] = e.op == TQ_ADD ? x + y : e.op == TQ_SUB ? x - y : x * y;
    }
    return;
  }
  // compare
  out.i.resize(n);
  auto cmp3 = [&](int c) -> bool {
    switch (e.op) {
      case TQ_LT: return c < 0;
      case TQ_LE: return c <= 0;
      case TQ_EQ: return c == 0;
      case TQ_NE: return c != 0;
      case TQ_GE: return c >= 0;
      default: return c > 0;
    }
  };
  if (a.ty.cls == C_S) {
    for (uint64_t k = 0; k < n; ++k) {
      const CV& ca = *a.scol; const CV& cb = *b.scol;
      uint64_t r = r0 + k;
      std::string_view x((const char*)ca.values + ca.offsets[r], ca.offsets[r + 1] - ca.offsets[r]);
      std::string_view y((const char*)cb.values + cb.offsets[r], cb.offsets[r + 1] - cb.offsets[r]);
      int c = x.compare(y);
      out.i[k] = cmp3(c < 0 ? -1 : c > 0 ? 1 : 0);
    }
  } else if (a.ty.cls == C_F || b.ty.cls == C_F) {
    for (uint64_t k = 0; k < n; ++k) {
      double x = a.ty.cls == C_F ? a.f[k] : to_f(a.i[k], a.ty);
      double y = b.ty.cls == C_F ? b.f[k] : to_f(b.i[k], b.ty);
      bool r;
      switch (e.op) {
        case TQ_LT: r = x < y; break;
        case TQ_LE: r = x <= y; break;
        case TQ_EQ: r = x == y; break;
        case TQ_NE: r = x != y; break;
        case TQ_GE: r = x >= y; break;
        default: r = x > y;
      }
      out.i[k] = r;
    }
  } else {
    int s = std::max(a.ty.scale, b.ty.scale);
    i128 fa = p10i(s - a.ty.scale), fb = p10i(s - b.ty.scale);
    for (uint64_t k = 0; k < n; ++k) {
      i128 x = mulw(a.i[k], fa), y = mulw(b.i[k], fb);
      out.i[k] = cmp3(x < y ? -1 : x > y ? 1 : 0);
    }
  }
}

// ---------------------------------------------------------------- threading
void parallel_chunks(uint64_t n, uint32_t nthreads, uint64_t morsel,
                     const std::function<void(uint32_t tid, uint64_t r0, uint64_t r1)>& fn) {
  if (nthreads <= 1 || n <= morsel) {
    for (uint64_t r = 0; r < n; r += morsel) fn(0, r, std::min(n, r + morsel));
    return;
  }
  std::atomic<uint64_t> next{0};
  std::vector<std::thread> ts;
  std::exception_ptr err;
  std::mutex mu;
  for (uint32_t t = 0; t < nthreads; ++t)
    ts.emplace_back([&, t] {
      try {
        for (;;) {
          uint64_t r = next.fetch_add(morsel);
          if (r >= n) break;
          fn(t, r, std::min(n, r + morsel));
        }
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        err = std::current_exception();
      }
    });
  for (auto& t : ts) t.join();
  if (err) std::rethrow_exception(err);
}

constexpr uint64_t kMorsel = 1 << 16;

// ---------------------------------------------------------------- filter / project
std::vector<uint64_t> select_rows(const Prog& p, const BV& in, uint64_t r0, uint64_t r1) {
  std::vector<uint64_t> ids;
  Vec m;
  eval(p, p.root, in, r0, r1 - r0, m);
  for (uint64_t k = 0; k < r1 - r0; ++k)
    if (m.v[k] && m.i[k]) ids.push_back(r0 + k);
  return ids;
}

OBatch filter_exec(const BV& in, const tq_expr& pred, uint32_t nthreads) {
  Prog p = compile(pred, in);
  if (p.n[p.root].ty.cls != C_B) fail(TQ_INVALID_PLAN, "predicate must be bool");
  uint64_t nm = (in.rows + kMorsel - 1) / kMorsel;
  std::vector<std::vector<uint64_t>> parts(nm);
  parallel_chunks(in.rows, nthreads, kMorsel, [&](uint32_t, uint64_t r0, uint64_t r1) {
    parts[r0 / kMorsel] = select_rows(p, in, r0, r1);
  });
  std::vector<uint64_t> ids;
  for (auto& v : parts) ids.insert(ids.end(), v.begin(), v.end());
  return take(in, ids.data(), ids.size());
}

OCol vec_to_col(const Vec& v, uint64_t n, bool want_validity) {
  OCol c;
  switch (v.ty.cls) {
    case C_I: c.kind = TQ_INT64; c.values.resize(n * 8);
      for (uint64_t k = 0; k < n; ++k) { int64_t x = (int64_t)v.i[k]; std::memcpy(&c.values[k * 8], &x, 8); }
      break;
    case C_D: c.kind = TQ_DECIMAL; c.precision = 38; c.scale = uint8_t(v.ty.scale); c.values.resize(n * 16);
      for (uint64_t k = 0; k < n; ++k) std::memcpy(&c.values[k * 16], &v.i[k], 16);
      break;
    case C_F: c.kind = TQ_FLOAT64; c.values.resize(n * 8);
      for (uint64_t k = 0; k < n; ++k) std::memcpy(&c.values[k * 8], &v.f[k], 8);
      break;
    case C_B: c.kind = TQ_BOOL; c.values.resize(n);
      for (uint64_t k = 0; k < n; ++k) c.values[k] = v.i[k] ? 1 : 0;
      break;
    default: fail(TQ_INVALID_PLAN, "projection of utf8 expression unsupported");
  }
  bool any_null = false;
  for (uint64_t k = 0; k < n; ++k) any_null |= !v.v[k];
  if ((want_validity || any_null) && n > 0) {
    c.has_valid = true;
    c.validity.assign(bm_bytes(n), 0);
    for (uint64_t k = 0; k < n; ++k) bit_set(c.validity.data(), k, v.v[k]);
  }
  return c;
}

// Does the expression subtree reference a column with a bitmap or a null literal?
bool may_be_null(const Prog& p, int idx, const BV& in) {
  const ENode& e = p.n[idx];
  if (e.tag == TQ_EX_COL) return in.cols[e.col].validity != nullptr;
  if (e.tag == TQ_EX_LIT) return e.lit_null;
  bool r = may_be_null(p, e.a, in);
  if (e.b >= 0) r = r || may_be_null(p, e.b, in);
  return r;
}

OBatch project_exec(const BV& in, const tq_expr* exprs, uint32_t nexpr, uint32_t nthreads) {
  std::vector<Prog> progs;
  for (uint32_t i = 0; i < nexpr; ++i) progs.push_back(compile(exprs[i], in));
  OBatch out;
  out.rows = in.rows;
  for (uint32_t i = 0; i < nexpr; ++i) {
    const Prog& p = progs[i];
    const ENode& root = p.n[p.root];
    // Pure column reference: copy the column (keeps Utf8 and bitmap presence).
    if (root.tag == TQ_EX_COL) {
      std::vector<uint64_t> ids;
      OCol c;
      const CV& s = in.cols[root.col];
      c.kind = s.kind; c.precision = s.precision; c.scale = s.scale;
      if (s.kind == TQ_UTF8) {
        c.offsets.assign(s.offsets, s.offsets + in.rows + 1);
        c.values.assign(s.values, s.values + s.offsets[in.rows]);
      } else {
        c.values.assign(s.values, s.values + in.rows * width_of(s.kind));
      }
      if (s.validity && in.rows) { c.has_valid = true; c.validity.assign(s.validity, s.validity + bm_bytes(in.rows)); }
      out.cols.push_back(std::move(c));
      continue;
    }
    Vec all;
    all.ty = root.ty;
    uint64_t n = in.rows;
    all.v.resize(n);
    if (root.ty.cls == C_F) all.f.resize(n); else all.i.resize(n);
    parallel_chunks(n, nthreads, kMorsel, [&](uint32_t, uint64_t r0, uint64_t r1) {
      Vec v;
      eval(p, p.root, in, r0, r1 - r0, v);
      for (uint64_t k = 0; k < r1 - r0; ++k) {
        all.v[r0 + k] = v.v[k];
        if (root.ty.cls == C_F) all.f[r0 + k] = v.f[k]; else all.i[r0 + k] = v.i[k];
      }
    });
    out.cols.push_back(vec_to_col(all, n, may_be_null(p, p.root, in)));
  }
  return out;
}

// ---------------------------------------------------------------- keys
// Key words for grouping / joining: Int64 1 word, Decimal 2, Float64 1 (bits),
// Bool 1; then one word with a null bit per key column.
struct KeySpec {
  std::vector<uint32_t> cols;
  std::vector<int> words;  // per key
  int total = 0;           // incl. null word
};
KeySpec key_spec(const BV& in, const uint32_t* keys, uint32_t nkeys) {
  KeySpec ks;
  for (uint32_t k = 0; k < nkeys; ++k) {
    if (keys[k] >= in.cols.size()) fail(TQ_INVALID_PLAN, "key column out of range");
    uint8_t kind = in.cols[keys[k]].kind;
    if (kind == TQ_UTF8) fail(TQ_INVALID_PLAN, "utf8 keys unsupported");
    ks.cols.push_back(keys[k]);
    ks.words.push_back(kind == TQ_DECIMAL ? 2 : 1);
    ks.total += ks.words.back();
  }
  ks.total += 1;
  return ks;
}
// returns true if any key is null
bool key_words(const BV& in, const KeySpec& ks, uint64_t r, uint64_t* w) {
  uint64_t nullmask = 0;
  int pos = 0;
  for (size_t k = 0; k < ks.cols.size(); ++k) {
    const CV& c = in.cols[ks.cols[k]];
    bool valid = c.valid(r);
    if (!valid) nullmask |= 1ull << k;
    if (c.kind == TQ_DECIMAL) {
      i128 v = valid ? c.dec(r) : 0;
      w[pos++] = (uint64_t)(u128)v;
      w[pos++] = (uint64_t)((u128)v >> 64);
    } else if (c.kind == TQ_BOOL) {
      w[pos++] = valid ? (c.b(r) ? 1 : 0) : 0;
    } else {
      uint64_t x = 0;
      if (valid) std::memcpy(&x, c.values + r * 8, 8);
      w[pos++] = x;
    }
  }
  w[pos] = nullmask;
  return nullmask != 0;
}
uint64_t hash_words(const uint64_t* w, int n) {
  uint64_t h = 0x12345678abcdefULL;
  for (int i = 0; i < n; ++i) h = sm_mix(h ^ (w[i] + kGamma));
  return h;
}

// Open-addressing map from key words to dense group ids.
struct GroupMap {
  int kw;
  std::vector<uint64_t> keys;  // groups * kw
  std::vector<int64_t> slots;  // -1 empty
  uint64_t mask = 0;
  uint64_t n = 0;
  explicit GroupMap(int kw_) : kw(kw_) { rehash(1024); }
  void rehash(uint64_t cap) {
    slots.assign(cap, -1);
    mask = cap - 1;
    for (uint64_t g = 0; g < n; ++g) {
      uint64_t h = hash_words(&keys[g * kw], kw) & mask;
      while (slots[h] >= 0) h = (h + 1) & mask;
      slots[h] = int64_t(g);
    }
  }
  // returns group id; inserted=true if new
  uint64_t find_or_insert(const uint64_t* w, bool& inserted) {
    uint64_t h = hash_words(w, kw) & mask;
    for (;;) {
      int64_t s = slots[h];
      if (s < 0) break;
      if (std::memcmp(&keys[uint64_t(s) * kw], w, kw * 8) == 0) { inserted = false; return uint64_t(s); }
      h = (h + 1) & mask;
    }
    inserted = true;
    uint64_t g = n++;
    keys.insert(keys.end(), w, w + kw);
    slots[h] = int64_t(g);
    if (n * 2 > slots.size()) rehash(slots.size() * 2);
    return g;
  }
};

// ---------------------------------------------------------------- aggregate
struct AggInfo {
  uint32_t fn, col;
  Ty ty;  // input type
};
struct Acc {
  i128 s = 0;       // int / decimal sum (exact mod 2^128); min/max value
  double f = 0;     // float sum / min / max
  uint64_t cnt = 0; // non-null inputs (COUNT_STAR: rows)
};

void acc_update(Acc& a, const AggInfo& ai, const CV* c, uint64_t r) {
  if (ai.fn == TQ_AGG_COUNT_STAR) { a.cnt++; return; }
  if (!c->valid(r)) return;
  if (ai.fn == TQ_AGG_COUNT) { a.cnt++; return; }
  bool first = a.cnt == 0;
  a.cnt++;
  if (ai.ty.cls == C_F) {
    double x = c->f64(r);
    if (ai.fn == TQ_AGG_SUM || ai.fn == TQ_AGG_AVG) a.f += x;
    else if (first || (ai.fn == TQ_AGG_MIN ? x < a.f : x > a.f)) a.f = x;
    return;
  }
  i128 x = c->kind == TQ_DECIMAL ? c->dec(r) : c->kind == TQ_BOOL ? (i128)(c->b(r) ? 1 : 0) : (i128)c->i64(r);
  if (ai.fn == TQ_AGG_SUM || ai.fn == TQ_AGG_AVG) a.s = addw(a.s, x);
  else if (first || (ai.fn == TQ_AGG_MIN ? x < a.s : x > a.s)) a.s = x;
}
void acc_merge(Acc& a, const Acc& b, const AggInfo& ai) {
  if (b.cnt == 0) return;
  if (ai.fn == TQ_AGG_COUNT || ai.fn == TQ_AGG_COUNT_STAR) { a.cnt += b.cnt; return; }
  if (ai.fn == TQ_AGG_SUM || ai.fn == TQ_AGG_AVG) { a.s = addw(a.s, b.s); a.f += b.f; a.cnt += b.cnt; return; }
  bool take_b = a.cnt == 0;
  if (!take_b) {
    if (ai.ty.cls == C_F) take_b = ai.fn == TQ_AGG_MIN ? b.f < a.f : b.f > a.f;
    else take_b = ai.fn == TQ_AGG_MIN ? b.s < a.s : b.s > a.s;
  }
  if (take_b) { a.s = b.s; a.f = b.f; }
  a.cnt += b.cnt;
}

struct AggState {
  KeySpec ks;
  std::vector<AggInfo> ai;
  GroupMap map;
  std::vector<Acc> acc;  // groups * naggs
  AggState(const KeySpec& k, const std::vector<AggInfo>& a) : ks(k), ai(a), map(k.total) {}
  void add_rows(const BV& in, uint64_t r0, uint64_t r1) {
    std::vector<uint64_t> w(ks.total);
    size_t na = ai.size();
    std::vector<const CV*> cols(na);
    for (size_t j = 0; j < na; ++j) cols[j] = ai[j].fn == TQ_AGG_COUNT_STAR ? nullptr : &in.cols[ai[j].col];
    for (uint64_t r = r0; r < r1; ++r) {
      key_words(in, ks, r, w.data());
      bool ins;
      uint64_t g = map.find_or_insert(w.data(), ins);
      if (ins) acc.resize(acc.size() + na);
      for (size_t j = 0; j < na; ++j) acc_update(acc[g * na + j], ai[j], cols[j], r);
    }
  }
  void merge(const AggState& o) {
    size_t na = ai.size();
    for (uint64_t g = 0; g < o.map.n; ++g) {
      bool ins;
      uint64_t h = map.find_or_insert(&o.map.keys[g * ks.total], ins);
      if (ins) acc.resize(acc.size() + na);
      for (size_t j = 0; j < na; ++j) acc_merge(acc[h * na + j], o.acc[g * na + j], ai[j]);
    }
  }
};

std::vector<AggInfo> agg_infos(const BV& in, const tq_agg* aggs, uint32_t naggs) {
  std::vector<AggInfo> v;
  for (uint32_t j = 0; j < naggs; ++j) {
    AggInfo a{aggs[j].fn, aggs[j].column, {C_I, 0}};
    if (a.fn > TQ_AGG_AVG) fail(TQ_INVALID_PLAN, "bad aggregate");
    if (a.fn != TQ_AGG_COUNT_STAR) {
      if (a.col >= in.cols.size()) fail(TQ_INVALID_PLAN, "aggregate column out of range");
      a.ty = ty_of_kind(in.cols[a.col].kind, in.cols[a.col].scale);
      if (a.ty.cls == C_S) fail(TQ_INVALID_PLAN, "utf8 aggregate unsupported");
      if ((a.fn == TQ_AGG_SUM || a.fn == TQ_AGG_AVG) && a.ty.cls == C_B)
        fail(TQ_INVALID_PLAN, "sum of bool");
    }
    v.push_back(a);
  }
  return v;
}

OBatch agg_output(const BV& in, const KeySpec& ks, const std::vector<AggInfo>& ai, uint64_t ngroups,
                  const std::vector<uint64_t>& keys, const std::vector<Acc>& acc) {
  OBatch out;
  out.rows = ngroups;
  size_t na = ai.size();
  int pos = 0;
  for (size_t k = 0; k < ks.cols.size(); ++k) {
    const CV& s = in.cols[ks.cols[k]];
    OCol c;
    c.kind = s.kind; c.precision = s.precision; c.scale = s.scale;
    size_t w = width_of(s.kind);
    c.values.resize(ngroups * w);
    bool any_null = false;
    for (uint64_t g = 0; g < ngroups; ++g) {
      const uint64_t* kw = &keys[g * ks.total];
      if (s.kind == TQ_DECIMAL) std::memcpy(&c.values[g * 16], &kw[pos], 16);
      else if (s.kind == TQ_BOOL) c.values[g] = uint8_t(kw[pos]);
      else std::memcpy(&c.values[g * 8], &kw[pos], 8);
      any_null |= (kw[ks.total - 1] >> k) & 1;
    }
    if ((s.validity || any_null) && ngroups) {
      c.has_valid = true;
      c.validity.assign(bm_bytes(ngroups), 0);
      for (uint64_t g = 0; g < ngroups; ++g)
        bit_set(c.validity.data(), g, !((keys[g * ks.total + ks.total - 1] >> k) & 1));
    }
    pos += ks.words[k];
    out.cols.push_back(std::move(c));
  }
  for (size_t j = 0; j < na; ++j) {
    const AggInfo& a = ai[j];
    OCol c;
    std::vector<uint8_t> valid(ngroups, 1);
    if (a.fn == TQ_AGG_COUNT || a.fn == TQ_AGG_COUNT_STAR) {
      c.kind = TQ_INT64;
      c.values.resize(ngroups * 8);
      for (uint64_t g = 0; g < ngroups; ++g) { int64_t x = int64_t(acc[g * na + j].cnt); std::memcpy(&c.values[g * 8], &x, 8); }
    } else if (a.fn == TQ_AGG_AVG) {
      c.kind = TQ_FLOAT64;
      c.values.resize(ngroups * 8);
      for (uint64_t g = 0; g < ngroups; ++g) {
        const Acc& x = acc[g * na + j];
        double r = 0;
        if (x.cnt == 0) valid[g] = 0;
        else if (a.ty.cls == C_F) r = x.f / double(x.cnt);
        else r = to_f(x.s, a.ty.cls == C_I ? Ty{C_D, 0} : a.ty) / double(x.cnt);
        std::memcpy(&c.values[g * 8], &r, 8);
      }
    } else {  // SUM MIN MAX: same class as input; SUM(decimal) -> Decimal(38, s)
      const CV& s = in.cols[a.col];
      c.kind = s.kind; c.precision = s.precision; c.scale = s.scale;
      if (a.fn == TQ_AGG_SUM && s.kind == TQ_DECIMAL) c.precision = 38;
      size_t w = width_of(s.kind);
      c.values.resize(ngroups * w);
      for (uint64_t g = 0; g < ngroups; ++g) {
        const Acc& x = acc[g * na + j];
        if (x.cnt == 0) valid[g] = 0;
        if (s.kind == TQ_FLOAT64) std::memcpy(&c.values[g * 8], &x.f, 8);
        else if (s.kind == TQ_DECIMAL) std::memcpy(&c.values[g * 16], &x.s, 16);
        else if (s.kind == TQ_BOOL) c.values[g] = uint8_t(x.s != 0);
        else { int64_t v = (int64_t)x.s; std::memcpy(&c.values[g * 8], &v, 8); }
      }
    }
    bool any_null = false;
    for (auto v : valid) any_null |= !v;
    if (any_null) {
      c.has_valid = true;
      c.validity.assign(bm_bytes(ngroups), 0);
      for (uint64_t g = 0; g < ngroups; ++g) bit_set(c.validity.data(), g, valid[g]);
    }
    out.cols.push_back(std::move(c));
  }
  return out;
}

OBatch aggregate_exec(const BV& in, const uint32_t* keys, uint32_t nkeys, const tq_agg* aggs, uint32_t naggs,
                      int naive, uint32_t nthreads);

// Utf8 group keys (groups are equal key VALUES, a string by its
// bytes): each Utf8 key column is interned to the row index of its string's first
// occurrence (exact byte equality; a null string stays null), the aggregate runs
// on those ids, and each output key column takes the strings back at the ids with
// take (its bitmap iff the input column had one, transform.cpp:90-120).
OBatch aggregate_utf8_keys(const BV& in, const uint32_t* keys, uint32_t nkeys, const tq_agg* aggs, uint32_t naggs,
                           int naive, uint32_t nthreads) {
  for (uint32_t j = 0; j < naggs; ++j)
    if (aggs[j].fn != TQ_AGG_COUNT_STAR && aggs[j].column < in.cols.size() &&
        in.cols[aggs[j].column].kind == TQ_UTF8)
      fail(TQ_INVALID_PLAN, "utf8 aggregate unsupported");
  BV ids_in = in;
  std::vector<std::vector<int64_t>> ids(in.cols.size());
  std::vector<uint64_t> null_row(in.cols.size(), 0);
  for (uint32_t k = 0; k < nkeys; ++k) {
    const uint32_t col = keys[k];
    if (col >= in.cols.size()) fail(TQ_INVALID_PLAN, "key column out of range");
    const CV& c = in.cols[col];
    if (c.kind != TQ_UTF8 || !ids[col].empty()) continue;
    std::unordered_map<std::string_view, int64_t> first;
    ids[col].assign(std::max<uint64_t>(1, in.rows), 0);
    for (uint64_t r = 0; r < in.rows; ++r) {
      if (!c.valid(r)) {
        null_row[col] = r;
        continue;
      }
      std::string_view sv(reinterpret_cast<const char*>(c.values) + c.offsets[r], size_t(c.offsets[r + 1] - c.offsets[r]));
      ids[col][r] = first.emplace(sv, int64_t(r)).first->second;
    }
    CV v;
    v.kind = TQ_INT64;
    v.values = reinterpret_cast<const uint8_t*>(ids[col].data());
    v.values_bytes = in.rows * 8;
    v.validity = c.validity;
    ids_in.cols[col] = v;
  }
  OBatch o = aggregate_exec(ids_in, keys, nkeys, aggs, naggs, naive, nthreads);
  for (uint32_t k = 0; k < nkeys; ++k) {
    const uint32_t col = keys[k];
    if (in.cols[col].kind != TQ_UTF8) continue;
    const OCol& kc = o.cols[k];
    std::vector<uint64_t> at(o.rows);
    for (uint64_t g = 0; g < o.rows; ++g) {
      const bool valid = !kc.has_valid || bit_get(kc.validity.data(), g);
      int64_t id = 0;
      std::memcpy(&id, &kc.values[g * 8], 8);
      at[g] = valid ? uint64_t(id) : null_row[col];
    }
    BV one;
    one.rows = in.rows;
    one.cols.push_back(in.cols[col]);
    OBatch t = take(one, at.data(), at.size());
    o.cols[k] = std::move(t.cols[0]);
  }
  return o;
}

OBatch aggregate_exec(const BV& in, const uint32_t* keys, uint32_t nkeys, const tq_agg* aggs, uint32_t naggs,
                      int naive, uint32_t nthreads) {
  for (uint32_t k = 0; k < nkeys; ++k)
    if (keys[k] < in.cols.size() && in.cols[keys[k]].kind == TQ_UTF8)
      return aggregate_utf8_keys(in, keys, nkeys, aggs, naggs, naive, nthreads);
  KeySpec ks = key_spec(in, keys, nkeys);
  std::vector<AggInfo> ai = agg_infos(in, aggs, naggs);
  if (naive) {  // SPEC.md:699 style: linear search over materialised groups
    std::vector<uint64_t> gk;
    std::vector<Acc> acc;
    std::vector<uint64_t> w(ks.total);
    uint64_t ng = 0;
    for (uint64_t r = 0; r < in.rows; ++r) {
      key_words(in, ks, r, w.data());
      uint64_t g = 0;
      for (; g < ng; ++g)
        if (std::memcmp(&gk[g * ks.total], w.data(), ks.total * 8) == 0) break;
      if (g == ng) { gk.insert(gk.end(), w.begin(), w.end()); acc.resize(acc.size() + naggs); ++ng; }
      for (uint32_t j = 0; j < naggs; ++j)
        acc_update(acc[g * naggs + j], ai[j], ai[j].fn == TQ_AGG_COUNT_STAR ? nullptr : &in.cols[ai[j].col], r);
    }
    return agg_output(in, ks, ai, ng, gk, acc);
  }
  uint32_t nt = std::max<uint32_t>(1, nthreads);
  std::vector<std::unique_ptr<AggState>> st;
  for (uint32_t t = 0; t < nt; ++t) st.emplace_back(new AggState(ks, ai));
  parallel_chunks(in.rows, nt, kMorsel, [&](uint32_t t, uint64_t r0, uint64_t r1) { st[t]->add_rows(in, r0, r1); });
  for (uint32_t t = 1; t < nt; ++t) st[0]->merge(*st[t]);
  return agg_output(in, ks, ai, st[0]->map.n, st[0]->map.keys, st[0]->acc);
}

// ---------------------------------------------------------------- join
OBatch join_pairs(const BV& build, const BV& probe, const std::vector<uint64_t>& bids,
                  const std::vector<uint64_t>& pids) {
  OBatch a = take(build, bids.data(), bids.size());
  OBatch b = take(probe, pids.data(), pids.size());
  for (auto& c : b.cols) a.cols.push_back(std::move(c));
  a.rows = bids.size();
  return a;
}

void check_join_keys(const BV& build, const BV& probe, const uint32_t* bk, const uint32_t* pk, uint32_t nk) {
  if (nk == 0) fail(TQ_INVALID_PLAN, "join without keys");
  for (uint32_t k = 0; k < nk; ++k) {
    if (bk[k] >= build.cols.size() || pk[k] >= probe.cols.size()) fail(TQ_INVALID_PLAN, "join key out of range");
    const CV& a = build.cols[bk[k]];
    const CV& b = probe.cols[pk[k]];
    if (a.kind != b.kind || (a.kind == TQ_DECIMAL && a.scale != b.scale))
      fail(TQ_INVALID_PLAN, "join key types differ");
    if (a.kind == TQ_FLOAT64) fail(TQ_INVALID_PLAN, "unsupported join key type");
  }
}

// Build side hash table: chains in build-row order.
struct JoinTable {
  KeySpec ks;
  std::vector<uint64_t> keys;  // build rows * kw
  std::vector<int64_t> head, next;
  uint64_t mask;
  JoinTable(const BV& build, const uint32_t* bk, uint32_t nk) : ks(key_spec(build, bk, nk)) {
    uint64_t cap = 1024;
    while (cap < build.rows * 2) cap <<= 1;
    mask = cap - 1;
    head.assign(cap, -1);
    next.assign(build.rows, -1);
    keys.resize(build.rows * ks.total);
    std::vector<int64_t> tail(cap, -1);
    for (uint64_t r = 0; r < build.rows; ++r) {
      if (key_words(build, ks, r, &keys[r * ks.total])) continue;  // null keys never match
      uint64_t h = hash_words(&keys[r * ks.total], ks.total) & mask;
      if (tail[h] < 0) head[h] = int64_t(r); else next[tail[h]] = int64_t(r);
      tail[h] = int64_t(r);
    }
  }
};

// matching (build row, probe row) pairs: probe rows in order, each probe row's
// matches in build-row order
void join_match(const BV& build, const BV& probe, const uint32_t* bk, const uint32_t* pk, uint32_t nk, int naive,
                uint32_t nthreads, std::vector<uint64_t>& bids, std::vector<uint64_t>& pids) {
  if (naive) {  // SPEC.md:699 nested loop
    KeySpec bks = key_spec(build, bk, nk), pks = key_spec(probe, pk, nk);
    std::vector<uint64_t> wb(bks.total), wp(pks.total);
    for (uint64_t p = 0; p < probe.rows; ++p) {
      if (key_words(probe, pks, p, wp.data())) continue;
      for (uint64_t b = 0; b < build.rows; ++b) {
        if (key_words(build, bks, b, wb.data())) continue;
        if (std::memcmp(wb.data(), wp.data(), bks.total * 8) == 0) { bids.push_back(b); pids.push_back(p); }
      }
    }
    return;
  }
  JoinTable t(build, bk, nk);
  KeySpec pks = key_spec(probe, pk, nk);
  uint64_t nm = (probe.rows + kMorsel - 1) / kMorsel;
  std::vector<std::vector<uint64_t>> vb(nm), vp(nm);
  parallel_chunks(probe.rows, nthreads, kMorsel, [&](uint32_t, uint64_t r0, uint64_t r1) {
    std::vector<uint64_t> w(pks.total);
    auto& ob = vb[r0 / kMorsel];
    auto& op = vp[r0 / kMorsel];
    for (uint64_t p = r0; p < r1; ++p) {
      if (key_words(probe, pks, p, w.data())) continue;
      uint64_t h = hash_words(w.data(), pks.total) & t.mask;
      for (int64_t b = t.head[h]; b >= 0; b = t.next[b])
        if (std::memcmp(&t.keys[uint64_t(b) * t.ks.total], w.data(), pks.total * 8) == 0) {
          ob.push_back(uint64_t(b));
          op.push_back(p);
        }
    }
  });
  for (uint64_t m = 0; m < nm; ++m) {
    bids.insert(bids.end(), vb[m].begin(), vb[m].end());
    pids.insert(pids.end(), vp[m].begin(), vp[m].end());
  }
  }

// Utf8 join keys (equal key VALUES match, a string by its
// bytes): each Utf8 key pair is matched on ids from one dictionary over both
// sides' strings (a null string stays null and never matches); the output rows
// are the original columns taken at the matched rows.
OBatch join_exec(const BV& build, const BV& probe, const uint32_t* bk, const uint32_t* pk, uint32_t nk, int naive,
                 uint32_t nthreads) {
  check_join_keys(build, probe, bk, pk, nk);
  std::vector<uint64_t> bids, pids;
  BV bl = build, pl = probe;
  std::vector<uint32_t> nbk(bk, bk + nk), npk(pk, pk + nk);
  std::vector<std::unique_ptr<std::vector<int64_t>>> store;
  auto lower = [&](const CV& c, uint64_t rows, std::unordered_map<std::string_view, int64_t>& dict) {
    store.emplace_back(new std::vector<int64_t>(std::max<uint64_t>(1, rows), 0));
    std::vector<int64_t>& ids = *store.back();
    for (uint64_t r = 0; r < rows; ++r) {
      if (!c.valid(r)) continue;
      std::string_view sv(reinterpret_cast<const char*>(c.values) + c.offsets[r], size_t(c.offsets[r + 1] - c.offsets[r]));
      ids[r] = dict.emplace(sv, int64_t(dict.size())).first->second;
    }
    CV v;
    v.kind = TQ_INT64;
    v.values = reinterpret_cast<const uint8_t*>(ids.data());
    v.values_bytes = rows * 8;
    v.validity = c.validity;
    return v;
  };
  for (uint32_t k = 0; k < nk; ++k) {
    if (build.cols[bk[k]].kind != TQ_UTF8) continue;
    std::unordered_map<std::string_view, int64_t> dict;
    bl.cols.push_back(lower(build.cols[bk[k]], build.rows, dict));
    pl.cols.push_back(lower(probe.cols[pk[k]], probe.rows, dict));
    nbk[k] = uint32_t(bl.cols.size() - 1);
    npk[k] = uint32_t(pl.cols.size() - 1);
  }
  join_match(bl, pl, nbk.data(), npk.data(), nk, naive, nthreads, bids, pids);
  return join_pairs(build, probe, bids, pids);
}

// ---------------------------------------------------------------- partition
// part(r) = fnv1a64(LE bytes of key(r), chained over key columns) mod n.
void partition_ids(const BV& in, const uint32_t* keys, uint32_t nkeys, uint32_t nparts, uint32_t* pid) {
  if (nparts == 0) fail(TQ_INVALID_PLAN, "zero partitions");
  for (uint32_t k = 0; k < nkeys; ++k)
    if (keys[k] >= in.cols.size()) fail(TQ_INVALID_PLAN, "partition key out of range");
  static const uint8_t zeros[16] = {0};
  for (uint64_t r = 0; r < in.rows; ++r) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint32_t k = 0; k < nkeys; ++k) {
      const CV& c = in.cols[keys[k]];
      bool v = c.valid(r);
      if (c.kind == TQ_UTF8) {
        if (v) h = fnv1a64(c.values + c.offsets[r], size_t(c.offsets[r + 1] - c.offsets[r]), h);
      } else {
        size_t w = width_of(c.kind);
        h = fnv1a64(v ? c.values + r * w : zeros, w, h);
      }
    }
    pid[r] = uint32_t(h % nparts);
  }
}

// ---------------------------------------------------------------- datagen
// DESIGN.md §4.  U(name, i, n) = SplitMix64(fnv1a64(name, 42)).next()^(i+1) % n.
uint64_t col_seed(const char* name) { return fnv1a64((const uint8_t*)name, std::strlen(name), 42); }
inline uint64_t U(uint64_t seed, uint64_t i, uint64_t n) { return sm_nth(seed, i + 1) % n; }

uint64_t scaled(double base, double sf, uint64_t minimum) {
  double v = std::llround(base * sf);
  return std::max<uint64_t>(minimum, uint64_t(v));
}
uint64_t n_orders(double sf) { return scaled(1500000, sf, 1); }
uint64_t n_customer(double sf) { return scaled(150000, sf, 1); }
uint64_t n_supplier(double sf) { return scaled(10000, sf, 4); }
uint64_t n_part(double sf) { return scaled(200000, sf, 1); }

const int64_t kYearStart[] = {8035, 8401, 8766, 9131, 9496, 9862, 10227, 10592};  // 1992..1999
int64_t year_of(int64_t d) {
  int y = 0;
  while (y + 1 < 8 && d >= kYearStart[y + 1]) ++y;
  return 1992 + y;
}
int64_t retail_cents(int64_t p) { return 90000 + ((p / 10) % 20001) + 100 * (p % 1000); }
int64_t ps_supp(int64_t p, int64_t j, int64_t ns) { return ((p - 1 + j * (ns / 4 + (p - 1) / ns)) % ns) + 1; }
const int64_t kNationRegion[25] = {0, 1, 1, 1, 4, 0, 3, 3, 2, 2, 4, 4, 2, 4, 0, 0, 0, 1, 2, 3, 4, 2, 3, 3, 1};

OCol mk_col(uint8_t kind, uint64_t rows, uint8_t prec = 0, uint8_t scale = 0) {
  OCol c;
  c.kind = kind; c.precision = prec; c.scale = scale;
  c.values.resize(rows * width_of(kind));
  return c;
}
inline void put64(OCol& c, uint64_t r, int64_t v) { std::memcpy(&c.values[r * 8], &v, 8); }
inline void putdec(OCol& c, uint64_t r, i128 v) { std::memcpy(&c.values[r * 16], &v, 16); }

uint64_t table_rows(int t, double sf) {
  switch (t) {
    case TQ_T_ORDERS: return n_orders(sf);
    case TQ_T_CUSTOMER: return n_customer(sf);
    case TQ_T_SUPPLIER: return n_supplier(sf);
    case TQ_T_PART: return n_part(sf);
    case TQ_T_PARTSUPP: return 4 * n_part(sf);
    case TQ_T_NATION: return 25;
    case TQ_T_REGION: return 5;
    case TQ_T_LINEITEM: {
      uint64_t no = n_orders(sf), s = col_seed("orders.o_nlines"), n = 0;
      for (uint64_t i = 0; i < no; ++i) n += 1 + U(s, i, 7);
      return n;
    }
  }
  fail(TQ_INVALID_PLAN, "unknown table");
}

// A worker's row-group subset (GPU tq_datagen_shard, datagen.cu): rows
// [n * shard / nshards, n * (shard + 1) / nshards) of the full table, values
// equal to the full table's rows; lineitem = the lines of those orders.
OBatch datagen(int t, double sf, uint32_t nthreads, uint32_t shard = 0, uint32_t nshards = 1) {
  OBatch b;
  if (nshards == 0 || shard >= nshards) fail(TQ_INVALID_PLAN, "bad shard");
  uint64_t nc = n_customer(sf), ns = n_supplier(sf), np = n_part(sf), no = n_orders(sf);
  auto lo_of = [&](uint64_t n) { return n * shard / nshards; };
  auto hi_of = [&](uint64_t n) { return n * (shard + 1) / nshards; };
  switch (t) {
    case TQ_T_ORDERS: {
      const uint64_t lo = lo_of(no), n = hi_of(no) - lo;
      b.rows = n;
      b.cols = {mk_col(TQ_INT64, n), mk_col(TQ_INT64, n), mk_col(TQ_INT64, n), mk_col(TQ_INT64, n),
                mk_col(TQ_INT64, n)};
      uint64_t s1 = col_seed("orders.o_custkey"), s2 = col_seed("orders.o_orderdate");
      parallel_chunks(n, nthreads, kMorsel, [&](uint32_t, uint64_t r0, uint64_t r1) {
        for (uint64_t r = r0; r < r1; ++r) {
          const uint64_t i = lo + r;
          int64_t od = 8035 + int64_t(U(s2, i, 2406));
          put64(b.cols[0], r, int64_t(i + 1));
          put64(b.cols[1], r, 1 + int64_t(U(s1, i, nc)));
          put64(b.cols[2], r, od);
          put64(b.cols[3], r, 0);
          put64(b.cols[4], r, year_of(od));
        }
      });
      return b;
    }
    case TQ_T_LINEITEM: {
      uint64_t sl = col_seed("orders.o_nlines"), sod = col_seed("orders.o_orderdate");
      const uint64_t olo = lo_of(no), ohi = hi_of(no);
      std::vector<uint64_t> off(no + 1, 0);
      for (uint64_t i = 0; i < no; ++i) off[i + 1] = off[i] + 1 + U(sl, i, 7);
      const uint64_t base = off[olo], nl = off[ohi] - base;
      b.rows = nl;
      for (int c = 0; c < 3; ++c) b.cols.push_back(mk_col(TQ_INT64, nl));
      for (int c = 0; c < 4; ++c) b.cols.push_back(mk_col(TQ_DECIMAL, nl, 11, 2));
      for (int c = 0; c < 3; ++c) b.cols.push_back(mk_col(TQ_INT64, nl));
      uint64_t sp = col_seed("lineitem.l_partkey"), ss = col_seed("lineitem.l_suppkey"),
               sq = col_seed("lineitem.l_quantity"), sd = col_seed("lineitem.l_discount"),
               st = col_seed("lineitem.l_tax"), srd = col_seed("lineitem.l_receiptdate"),
               srf = col_seed("lineitem.l_returnflag"), ssd = col_seed("lineitem.l_shipdate");
      parallel_chunks(ohi - olo, nthreads, 1 << 14, [&](uint32_t, uint64_t o0, uint64_t o1) {
        for (uint64_t o = olo + o0; o < olo + o1; ++o) {
          int64_t od = 8035 + int64_t(U(sod, o, 2406));
          for (uint64_t r = off[o]; r < off[o + 1]; ++r) {
            const uint64_t w = r - base;  // row within the shard
            int64_t pk = 1 + int64_t(U(sp, r, np));
            int64_t sk = ps_supp(pk, int64_t(U(ss, r, 4)), int64_t(ns));
            int64_t qty = 1 + int64_t(U(sq, r, 50));
            int64_t ship = od + 1 + int64_t(U(ssd, r, 121));
            int64_t receipt = ship + 1 + int64_t(U(srd, r, 30));
            int64_t rf = receipt <= 9298 ? (U(srf, r, 2) == 0 ? 'R' : 'A') : 'N';
            put64(b.cols[0], w, int64_t(o + 1));
            put64(b.cols[1], w, pk);
            put64(b.cols[2], w, sk);
            putdec(b.cols[3], w, (i128)qty * 100);
            putdec(b.cols[4], w, (i128)qty * retail_cents(pk));
            putdec(b.cols[5], w, (i128)U(sd, r, 11));
            putdec(b.cols[6], w, (i128)U(st, r, 9));
            put64(b.cols[7], w, rf);
            put64(b.cols[8], w, ship > 9298 ? 'O' : 'F');
            put64(b.cols[9], w, ship);
          }
        }
      });
      return b;
    }
    case TQ_T_CUSTOMER: {
      const uint64_t lo = lo_of(nc), n = hi_of(nc) - lo;
      b.rows = n;
      b.cols = {mk_col(TQ_INT64, n), mk_col(TQ_INT64, n), mk_col(TQ_INT64, n)};
      uint64_t s1 = col_seed("customer.c_nationkey"), s2 = col_seed("customer.c_mktsegment");
      for (uint64_t r = 0; r < n; ++r) {
        const uint64_t i = lo + r;
        put64(b.cols[0], r, int64_t(i + 1));
        put64(b.cols[1], r, int64_t(U(s1, i, 25)));
        put64(b.cols[2], r, int64_t(U(s2, i, 5)));
      }
      return b;
    }
    case TQ_T_SUPPLIER: {
      const uint64_t lo = lo_of(ns), n = hi_of(ns) - lo;
      b.rows = n;
      b.cols = {mk_col(TQ_INT64, n), mk_col(TQ_INT64, n)};
      uint64_t s1 = col_seed("supplier.s_nationkey");
      for (uint64_t r = 0; r < n; ++r) {
        const uint64_t i = lo + r;
        put64(b.cols[0], r, int64_t(i + 1));
        put64(b.cols[1], r, int64_t(U(s1, i, 25)));
      }
      return b;
    }
    case TQ_T_PART: {
      const uint64_t lo = lo_of(np), n = hi_of(np) - lo;
      b.rows = n;
      b.cols = {mk_col(TQ_INT64, n), mk_col(TQ_INT64, n)};
      uint64_t s1 = col_seed("part.p_color");
      for (uint64_t r = 0; r < n; ++r) {
        const uint64_t i = lo + r;
        put64(b.cols[0], r, int64_t(i + 1));
        put64(b.cols[1], r, int64_t(U(s1, i, 1000)));
      }
      return b;
    }
    case TQ_T_PARTSUPP: {
      const uint64_t lo = lo_of(4 * np), n = hi_of(4 * np) - lo;
      b.rows = n;
      b.cols = {mk_col(TQ_INT64, n), mk_col(TQ_INT64, n), mk_col(TQ_DECIMAL, n, 11, 2)};
      uint64_t s1 = col_seed("partsupp.ps_supplycost");
      for (uint64_t r = 0; r < n; ++r) {
        const uint64_t i = lo + r;
        int64_t p = int64_t(i / 4) + 1;
        put64(b.cols[0], r, p);
        put64(b.cols[1], r, ps_supp(p, int64_t(i % 4), int64_t(ns)));
        putdec(b.cols[2], r, (i128)(100 + U(s1, i, 99901)));
      }
      return b;
    }
    case TQ_T_NATION:
    case TQ_T_REGION: {
      const uint64_t total = t == TQ_T_NATION ? 25 : 5;
      const uint64_t lo = lo_of(total), n = hi_of(total) - lo;
      b.rows = n;
      b.cols = {mk_col(TQ_INT64, n), mk_col(TQ_INT64, n)};
      for (uint64_t r = 0; r < n; ++r) {
        const uint64_t i = lo + r;
        put64(b.cols[0], r, int64_t(i));
        put64(b.cols[1], r, t == TQ_T_NATION ? kNationRegion[i] : int64_t(i));
      }
      return b;
    }
  }
  fail(TQ_INVALID_PLAN, "unknown table");
}

// ---------------------------------------------------------------- query DAGs
// Small expression builder (prefix order).
struct EB {
  std::vector<tq_expr_node> n;
  EB& col(uint32_t c) { tq_expr_node x{}; x.tag = TQ_EX_COL; x.column = c; n.push_back(x); return *this; }
  EB& i64(int64_t v) { tq_expr_node x{}; x.tag = TQ_EX_LIT; x.kind = TQ_INT64; x.lo = uint64_t(v); n.push_back(x); return *this; }
  EB& dec(int64_t v, uint8_t s) {
    tq_expr_node x{}; x.tag = TQ_EX_LIT; x.kind = TQ_DECIMAL; x.scale = s;
    x.lo = uint64_t(v); x.hi = v < 0 ? ~0ull : 0; n.push_back(x); return *this;
  }
  EB& cmp(int op) { tq_expr_node x{}; x.tag = TQ_EX_CMP; x.op = uint8_t(op); n.push_back(x); return *this; }
  EB& ar(int op) { tq_expr_node x{}; x.tag = TQ_EX_ARITH; x.op = uint8_t(op); n.push_back(x); return *this; }
  EB& land() { tq_expr_node x{}; x.tag = TQ_EX_AND; n.push_back(x); return *this; }
  tq_expr e() const { return tq_expr{n.data(), uint32_t(n.size()), 0}; }
};

// lineitem columns
enum { L_ORDERKEY, L_PARTKEY, L_SUPPKEY, L_QUANTITY, L_EXTPRICE, L_DISCOUNT, L_TAX, L_RETURNFLAG, L_LINESTATUS, L_SHIPDATE };
enum { O_ORDERKEY, O_CUSTKEY, O_ORDERDATE, O_SHIPPRIORITY, O_YEAR };

OBatch proj_cols(const BV& in, std::initializer_list<uint32_t> cols, uint32_t nt) {
  std::vector<EB> bs;
  for (uint32_t c : cols) { EB b; b.col(c); bs.push_back(b); }
  std::vector<tq_expr> ex;
  for (auto& b : bs) ex.push_back(b.e());
  return project_exec(in, ex.data(), uint32_t(ex.size()), nt);
}

OBatch query(int q, const tq_batch* tables, uint32_t nt) {
  auto T = [&](int t) { return view(&tables[t]); };
  if (q == TQ_Q6) {
    BV li = T(TQ_T_LINEITEM);
    // (shipdate >= 8766 and shipdate < 9131) and ((disc >= 0.05 and disc <= 0.07) and qty < 24)
    EB f;
    f.land().land().cmp(TQ_GE).col(L_SHIPDATE).i64(8766).cmp(TQ_LT).col(L_SHIPDATE).i64(9131)
        .land().land().cmp(TQ_GE).col(L_DISCOUNT).dec(5, 2).cmp(TQ_LE).col(L_DISCOUNT).dec(7, 2)
        .cmp(TQ_LT).col(L_QUANTITY).dec(2400, 2);
    OBatch fl = filter_exec(li, f.e(), nt);
    EB rev;
    rev.ar(TQ_MUL).col(L_EXTPRICE).col(L_DISCOUNT);
    tq_expr ex = rev.e();
    OBatch pr = project_exec(view(fl), &ex, 1, nt);
    tq_agg a{TQ_AGG_SUM, 0};
    return aggregate_exec(view(pr), nullptr, 0, &a, 1, 0, nt);
  }
  if (q == TQ_Q1) {
    BV li = T(TQ_T_LINEITEM);
    EB f;
    f.cmp(TQ_LE).col(L_SHIPDATE).i64(10471);
    OBatch fl = filter_exec(li, f.e(), nt);
    // project: rf, ls, qty, ep, disc, dp = ep*(1-disc), ch = dp*(1+tax)
    EB e0, e1, e2, e3, e4, e5, e6;
    e0.col(L_RETURNFLAG); e1.col(L_LINESTATUS); e2.col(L_QUANTITY); e3.col(L_EXTPRICE); e4.col(L_DISCOUNT);
    e5.ar(TQ_MUL).col(L_EXTPRICE).ar(TQ_SUB).dec(100, 2).col(L_DISCOUNT);
    e6.ar(TQ_MUL).ar(TQ_MUL).col(L_EXTPRICE).ar(TQ_SUB).dec(100, 2).col(L_DISCOUNT).ar(TQ_ADD).dec(100, 2).col(L_TAX);
    tq_expr ex[7] = {e0.e(), e1.e(), e2.e(), e3.e(), e4.e(), e5.e(), e6.e()};
    OBatch pr = project_exec(view(fl), ex, 7, nt);
    uint32_t keys[2] = {0, 1};
    tq_agg aggs[8] = {{TQ_AGG_SUM, 2}, {TQ_AGG_SUM, 3}, {TQ_AGG_SUM, 5}, {TQ_AGG_SUM, 6},
                      {TQ_AGG_AVG, 2}, {TQ_AGG_AVG, 3}, {TQ_AGG_AVG, 4}, {TQ_AGG_COUNT_STAR, 0}};
    return aggregate_exec(view(pr), keys, 2, aggs, 8, 0, nt);
  }
  if (q == TQ_Q3) {
    BV cu = T(TQ_T_CUSTOMER), od = T(TQ_T_ORDERS), li = T(TQ_T_LINEITEM);
    EB fc; fc.cmp(TQ_EQ).col(2).i64(1);
    OBatch c1 = filter_exec(cu, fc.e(), nt);
    OBatch cf = proj_cols(view(c1), {0}, nt);  // c_custkey
    EB fo; fo.cmp(TQ_LT).col(O_ORDERDATE).i64(9204);
    OBatch o1 = filter_exec(od, fo.e(), nt);
    uint32_t bk = 0, pk = O_CUSTKEY;
    OBatch oj = join_exec(view(cf), view(o1), &bk, &pk, 1, 0, nt);  // [c_custkey, o_*]
    OBatch of = proj_cols(view(oj), {1 + O_ORDERKEY, 1 + O_ORDERDATE, 1 + O_SHIPPRIORITY}, nt);
    EB fl; fl.cmp(TQ_GT).col(L_SHIPDATE).i64(9204);
    OBatch l1 = filter_exec(li, fl.e(), nt);
    EB k0, rv;
    k0.col(L_ORDERKEY);
    rv.ar(TQ_MUL).col(L_EXTPRICE).ar(TQ_SUB).dec(100, 2).col(L_DISCOUNT);
    tq_expr ex[2] = {k0.e(), rv.e()};
    OBatch lf = project_exec(view(l1), ex, 2, nt);
    uint32_t bk2 = 0, pk2 = 0;
    OBatch j = join_exec(view(of), view(lf), &bk2, &pk2, 1, 0, nt);  // [o_orderkey, o_orderdate, o_shippriority, l_orderkey, rev]
    uint32_t keys[3] = {3, 1, 2};
    tq_agg a{TQ_AGG_SUM, 4};
    return aggregate_exec(view(j), keys, 3, &a, 1, 0, nt);
  }
  if (q == TQ_Q5) {
    BV re = T(TQ_T_REGION), na = T(TQ_T_NATION), cu = T(TQ_T_CUSTOMER), od = T(TQ_T_ORDERS),
       li = T(TQ_T_LINEITEM), su = T(TQ_T_SUPPLIER);
    EB fr; fr.cmp(TQ_EQ).col(1).i64(2);  // r_name = ASIA
    OBatch r1 = filter_exec(re, fr.e(), nt);
    uint32_t a0 = 0, a1 = 1;
    OBatch nj = join_exec(view(r1), na, &a0, &a1, 1, 0, nt);  // [r_regionkey, r_name, n_nationkey, n_regionkey]
    OBatch nf = proj_cols(view(nj), {2}, nt);                 // n_nationkey
    uint32_t b1 = 0, p1 = 1;
    OBatch cj = join_exec(view(nf), cu, &b1, &p1, 1, 0, nt);  // [n_nationkey, c_custkey, c_nationkey, c_mktsegment]
    OBatch cf = proj_cols(view(cj), {1, 2}, nt);              // c_custkey, c_nationkey
    EB fo; fo.land().cmp(TQ_GE).col(O_ORDERDATE).i64(8766).cmp(TQ_LT).col(O_ORDERDATE).i64(9131);
    OBatch o1 = filter_exec(od, fo.e(), nt);
    uint32_t b2 = 0, p2 = O_CUSTKEY;
    OBatch oj = join_exec(view(cf), view(o1), &b2, &p2, 1, 0, nt);  // [c_custkey, c_nationkey, o_*]
    OBatch of = proj_cols(view(oj), {2 + O_ORDERKEY, 1}, nt);       // o_orderkey, c_nationkey
    EB k0, k1, rv;
    k0.col(L_ORDERKEY); k1.col(L_SUPPKEY);
    rv.ar(TQ_MUL).col(L_EXTPRICE).ar(TQ_SUB).dec(100, 2).col(L_DISCOUNT);
    tq_expr ex[3] = {k0.e(), k1.e(), rv.e()};
    OBatch lf = project_exec(li, ex, 3, nt);  // l_orderkey, l_suppkey, rev
    uint32_t b3 = 0, p3 = 0;
    OBatch lj = join_exec(view(of), view(lf), &b3, &p3, 1, 0, nt);  // [o_orderkey, c_nationkey, l_orderkey, l_suppkey, rev]
    uint32_t b4[2] = {0, 1}, p4[2] = {3, 1};
    OBatch sj = join_exec(su, view(lj), b4, p4, 2, 0, nt);  // [s_suppkey, s_nationkey, ...5]
    uint32_t keys[1] = {1};
    tq_agg a{TQ_AGG_SUM, 6};
    return aggregate_exec(view(sj), keys, 1, &a, 1, 0, nt);
  }
  if (q == TQ_Q9) {
    BV pa = T(TQ_T_PART), ps = T(TQ_T_PARTSUPP), li = T(TQ_T_LINEITEM), su = T(TQ_T_SUPPLIER), od = T(TQ_T_ORDERS);
    EB fp; fp.cmp(TQ_LT).col(1).i64(54);
    OBatch p1 = filter_exec(pa, fp.e(), nt);
    OBatch pf = proj_cols(view(p1), {0}, nt);
    uint32_t b1 = 0, q1 = 0;
    OBatch psj = join_exec(view(pf), ps, &b1, &q1, 1, 0, nt);  // [p_partkey, ps_partkey, ps_suppkey, ps_supplycost]
    OBatch psf = proj_cols(view(psj), {1, 2, 3}, nt);
    OBatch lf = proj_cols(li, {L_ORDERKEY, L_PARTKEY, L_SUPPKEY, L_QUANTITY, L_EXTPRICE, L_DISCOUNT}, nt);
    uint32_t b2[2] = {0, 1}, q2[2] = {1, 2};
    OBatch lj = join_exec(view(psf), view(lf), b2, q2, 2, 0, nt);
    // [ps_partkey, ps_suppkey, ps_supplycost, l_orderkey, l_partkey, l_suppkey, l_qty, l_ep, l_disc]
    uint32_t b3 = 0, q3 = 5;
    OBatch sj = join_exec(su, view(lj), &b3, &q3, 1, 0, nt);
    // [s_suppkey, s_nationkey, ps_partkey, ps_suppkey, ps_supplycost, l_orderkey, l_partkey, l_suppkey, l_qty, l_ep, l_disc]
    OBatch of = proj_cols(od, {O_ORDERKEY, O_YEAR}, nt);
    uint32_t b4 = 0, q4 = 5;
    OBatch oj = join_exec(view(of), view(sj), &b4, &q4, 1, 0, nt);
    // [o_orderkey, o_year, s_suppkey, s_nationkey, ps_partkey, ps_suppkey, ps_supplycost, l_orderkey, l_partkey, l_suppkey, l_qty, l_ep, l_disc]
    EB n0, y0, amt;
    n0.col(3); y0.col(1);
    amt.ar(TQ_SUB).ar(TQ_MUL).col(11).ar(TQ_SUB).dec(100, 2).col(12).ar(TQ_MUL).col(6).col(10);
    tq_expr ex[3] = {n0.e(), y0.e(), amt.e()};
    OBatch pr = project_exec(view(oj), ex, 3, nt);
    uint32_t keys[2] = {0, 1};
    tq_agg a{TQ_AGG_SUM, 2};
    return aggregate_exec(view(pr), keys, 2, &a, 1, 0, nt);
  }
  fail(TQ_INVALID_PLAN, "unknown query");
}

template <typename F>
tq_status guard(F&& f) {
  try {
    f();
    return TQ_OK;
  } catch (const OErr& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TQ_INTERNAL;
  }
}

}  // namespace

extern "C" {

void tqo_batch_free(tq_batch* b) {
  if (!b || !b->cols) return;
  for (uint32_t c = 0; c < b->ncols; ++c) {
    std::free(b->cols[c].values);
    std::free(b->cols[c].validity);
    std::free(b->cols[c].offsets);
  }
  std::free(b->cols);
  b->cols = nullptr;
  b->ncols = 0;
  b->rows = 0;
}
const char* tqo_last_error(void) { return g_err.c_str(); }
uint64_t tqo_fnv1a64(const uint8_t* bytes, uint64_t n, uint64_t seed) { return fnv1a64(bytes, n, seed); }
uint64_t tqo_splitmix_nth(uint64_t seed, uint64_t k) { return sm_nth(seed, k); }

tq_status tqo_take(const tq_batch* in, const uint64_t* ids, uint64_t n, tq_batch* out) {
  return guard([&] { export_batch(take(view(in), ids, n), out); });
}
tq_status tqo_concat(const tq_batch* ins, uint32_t n, tq_batch* out) {
  return guard([&] {
    std::vector<BV> v;
    for (uint32_t i = 0; i < n; ++i) v.push_back(view(&ins[i]));
    export_batch(concat(v), out);
  });
}
tq_status tqo_slice(const tq_batch* in, uint64_t start, uint64_t len, tq_batch* out) {
  return guard([&] { export_batch(slice(view(in), start, len), out); });
}
tq_status tqo_filter(const tq_batch* in, tq_expr pred, tq_batch* out) {
  return guard([&] { export_batch(filter_exec(view(in), pred, 1), out); });
}
tq_status tqo_project(const tq_batch* in, const tq_expr* exprs, uint32_t n, tq_batch* out) {
  return guard([&] { export_batch(project_exec(view(in), exprs, n, 1), out); });
}
tq_status tqo_partition_ids(const tq_batch* in, const uint32_t* keys, uint32_t nkeys, uint32_t nparts,
                            uint32_t* pid) {
  return guard([&] { partition_ids(view(in), keys, nkeys, nparts, pid); });
}
tq_status tqo_hash_partition(const tq_batch* in, const uint32_t* keys, uint32_t nkeys, uint32_t nparts,
                             tq_batch* outs) {
  return guard([&] {
    BV v = view(in);
    std::vector<uint32_t> pid(v.rows);
    partition_ids(v, keys, nkeys, nparts, pid.data());
    std::vector<std::vector<uint64_t>> ids(nparts);
    for (uint64_t r = 0; r < v.rows; ++r) ids[pid[r]].push_back(r);
    for (uint32_t p = 0; p < nparts; ++p) export_batch(take(v, ids[p].data(), ids[p].size()), &outs[p]);
  });
}
tq_status tqo_join(const tq_batch* build, const tq_batch* probe, const uint32_t* bkeys, const uint32_t* pkeys,
                   uint32_t nkeys, int naive, tq_batch* out) {
  return guard([&] { export_batch(join_exec(view(build), view(probe), bkeys, pkeys, nkeys, naive, 1), out); });
}
tq_status tqo_aggregate(const tq_batch* in, const uint32_t* keys, uint32_t nkeys, const tq_agg* aggs,
                        uint32_t naggs, int naive, tq_batch* out) {
  return guard([&] { export_batch(aggregate_exec(view(in), keys, nkeys, aggs, naggs, naive, 1), out); });
}
uint64_t tqo_table_rows(int table, double sf) {
  uint64_t r = 0;
  guard([&] { r = table_rows(table, sf); });
  return r;
}
tq_status tqo_datagen(int table, double sf, uint32_t nthreads, tq_batch* out) {
  return guard([&] { export_batch(datagen(table, sf, nthreads), out); });
}

tq_status tqo_datagen_shard(int table, double sf, uint32_t shard, uint32_t nshards, uint32_t nthreads, tq_batch* out) {
  return guard([&] { export_batch(datagen(table, sf, nthreads, shard, nshards), out); });
}
tq_status tqo_query(int q, const tq_batch* tables, uint32_t nthreads, tq_batch* out) {
  return guard([&] { export_batch(query(q, tables, nthreads), out); });
}

}  // extern "C"
