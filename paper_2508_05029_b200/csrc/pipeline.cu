// pipeline.cu — the staged warp-tile pipeline kernels (see pipeline.h).
//
// Per CTA (persistent, grid = k x 148 SMs): thread 0 streams the referenced
// column slices of tile t+nstages into a ring of shared-memory stages with
// cp.async.bulk (TMA 1-D bulk copies, mbarrier complete_tx), while 8 warps
// run the Expr register machine over tile t (each warp owns 64 rows, 2 per
// lane) and feed the sink.  This replaces the reference's per-row
// Column::*_at loops (types.cpp:66-90) and take() (transform.cpp:90-120).
#include <cfloat>

#include "device.cuh"
#include "pipeline.h"

namespace tq {

__constant__ double c_p10[39] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11, 1e12,
                                 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22, 1e23, 1e24, 1e25,
                                 1e26, 1e27, 1e28, 1e29, 1e30, 1e31, 1e32, 1e33, 1e34, 1e35, 1e36, 1e37, 1e38};

// ------------------------------------------------------------------ per-warp context
struct WCtx {
  const PipeParams* p;
  const uint8_t* stage;  // current stage base
  const DLit* lits;      // smem copy
  uint8_t* vslot;        // [slot][v][32] x 16 B  (this warp)
  u32* vvalid;           // [slot][v]
  u32* bslot;            // [slot][v][2] (value, valid)
  u32 row0;              // tile-relative first row of this warp
  u32 nrows;             // rows in the tile
  u32 lane;
};

__device__ __forceinline__ u32 trow(const WCtx& w, int v) { return w.row0 + (u32)v * 32u + w.lane; }

__device__ __forceinline__ bool col_valid(const WCtx& w, int c, int v) {
  const StagedCol& sc = w.p->cols[c];
  if (!sc.validity) return true;
  const u32* bm = (const u32*)(w.stage + sc.voff);
  return (bm[(w.row0 >> 5) + v] >> w.lane) & 1u;
}

__device__ __forceinline__ i128 get_i(const WCtx& w, uint8_t k, uint16_t idx, int v, bool& valid) {
  switch (k) {
    case K_COL_I64: {
      valid = col_valid(w, idx, v);
      return (i128)((const long long*)(w.stage + w.p->cols[idx].off))[trow(w, v)];
    }
    case K_COL_DEC: {
      valid = col_valid(w, idx, v);
      const ulonglong2 x = ((const ulonglong2*)(w.stage + w.p->cols[idx].off))[trow(w, v)];
      return mk128(x.x, x.y);
    }
    case K_COL_BOOL: {
      valid = col_valid(w, idx, v);
      return (i128)(w.stage[w.p->cols[idx].off + trow(w, v)] != 0);
    }
    case K_TMP_I: {
      valid = (w.vvalid[idx * kV + v] >> w.lane) & 1u;
      const ulonglong2 x = ((const ulonglong2*)w.vslot)[(idx * kV + v) * 32 + w.lane];
      return mk128(x.x, x.y);
    }
    case K_TMP_B: {
      const u32* b = w.bslot + (idx * kV + v) * 2;
      valid = (b[1] >> w.lane) & 1u;
      return (i128)((b[0] >> w.lane) & 1u);
    }
    case K_LIT_I:
    case K_LIT_B: {
      const DLit& l = w.lits[idx];
      valid = l.valid != 0;
      return mk128(l.lo, l.hi);
    }
    default:
      valid = false;
      return 0;
  }
}

__device__ __forceinline__ double get_f(const WCtx& w, uint8_t k, uint16_t idx, int v, uint8_t scale, bool& valid) {
  switch (k) {
    case K_COL_F64:
      valid = col_valid(w, idx, v);
      return ((const double*)(w.stage + w.p->cols[idx].off))[trow(w, v)];
    case K_TMP_F: {
      valid = (w.vvalid[idx * kV + v] >> w.lane) & 1u;
      return ((const double*)w.vslot)[((idx * kV + v) * 32 + w.lane) * 2];
    }
    case K_LIT_F: {
      const DLit& l = w.lits[idx];
      valid = l.valid != 0;
      return l.f;
    }
    default: {
      i128 x = get_i(w, k, idx, v, valid);
      return i128_to_f64(x) / c_p10[scale];
    }
  }
}

__device__ __forceinline__ bool get_b(const WCtx& w, uint8_t k, uint16_t idx, int v, bool& valid) {
  if (k == K_TMP_B) {
    const u32* b = w.bslot + (idx * kV + v) * 2;
    valid = (b[1] >> w.lane) & 1u;
    return (b[0] >> w.lane) & 1u;
  }
  return get_i(w, k, idx, v, valid) != 0;
}

__device__ __forceinline__ void put_i(const WCtx& w, uint8_t dst, int v, i128 x, bool valid) {
  ((ulonglong2*)w.vslot)[(dst * kV + v) * 32 + w.lane] = make_ulonglong2(lo64(x), hi64(x));
  u32 m = __ballot_sync(kFull, valid);
  if (w.lane == 0) w.vvalid[dst * kV + v] = m;
}
__device__ __forceinline__ void put_f(const WCtx& w, uint8_t dst, int v, double x, bool valid) {
  ((double*)w.vslot)[((dst * kV + v) * 32 + w.lane) * 2] = x;
  u32 m = __ballot_sync(kFull, valid);
  if (w.lane == 0) w.vvalid[dst * kV + v] = m;
}
__device__ __forceinline__ void put_b(const WCtx& w, uint8_t dst, int v, bool x, bool valid) {
  u32 mv = __ballot_sync(kFull, x);
  u32 mn = __ballot_sync(kFull, valid);
  if (w.lane == 0) {
    w.bslot[(dst * kV + v) * 2] = mv;
    w.bslot[(dst * kV + v) * 2 + 1] = mn;
  }
}

__device__ __forceinline__ bool cmp_res(int c, uint8_t sub) {
  switch (sub) {
    case TQ_LT: return c < 0;
    case TQ_LE: return c <= 0;
    case TQ_EQ: return c == 0;
    case TQ_NE: return c != 0;
    case TQ_GE: return c >= 0;
    default: return c > 0;
  }
}

// Run instructions [begin, end) over this warp's rows.
__device__ void run_code(const WCtx& w, const DInstr* code, int begin, int end) {
  for (int pc = begin; pc < end; ++pc) {
    const DInstr in = code[pc];
    switch (in.op) {
      case OP_ADD_I:
      case OP_SUB_I:
      case OP_MUL_I: {
        i128 fa = in.fa != 0xff ? mk128(w.lits[in.fa].lo, w.lits[in.fa].hi) : (i128)1;
        i128 fb = in.fb != 0xff ? mk128(w.lits[in.fb].lo, w.lits[in.fb].hi) : (i128)1;
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool va, vb;
          i128 x = get_i(w, in.ak, in.a, v, va);
          i128 y = get_i(w, in.bk, in.b, v, vb);
          if (in.fa != 0xff) x = mul128(x, fa);
          if (in.fb != 0xff) y = mul128(y, fb);
          i128 r = in.op == OP_ADD_I ? add128(x, y) : in.op == OP_SUB_I ? sub128(x, y) : mul128(x, y);
          if (in.wrap) r = wrap64(r);
          put_i(w, in.dst, v, r, va && vb);
        }
        break;
      }
      case OP_ADD_F:
      case OP_SUB_F:
      case OP_MUL_F: {
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool va, vb;
          double x = get_f(w, in.ak, in.a, v, in.fa, va);
          double y = get_f(w, in.bk, in.b, v, in.fb, vb);
          double r = in.op == OP_ADD_F ? x + y : in.op == OP_SUB_F ? x - y : x * y;
          put_f(w, in.dst, v, r, va && vb);
        }
        break;
      }
      case OP_CMP_I: {
        i128 fa = in.fa != 0xff ? mk128(w.lits[in.fa].lo, w.lits[in.fa].hi) : (i128)1;
        i128 fb = in.fb != 0xff ? mk128(w.lits[in.fb].lo, w.lits[in.fb].hi) : (i128)1;
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool va, vb;
          i128 x = get_i(w, in.ak, in.a, v, va);
          i128 y = get_i(w, in.bk, in.b, v, vb);
          if (in.fa != 0xff) x = mul128(x, fa);
          if (in.fb != 0xff) y = mul128(y, fb);
          put_b(w, in.dst, v, cmp_res(x < y ? -1 : (x > y ? 1 : 0), in.sub), va && vb);
        }
        break;
      }
      case OP_CMP_F: {
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool va, vb;
          double x = get_f(w, in.ak, in.a, v, in.fa, va);
          double y = get_f(w, in.bk, in.b, v, in.fb, vb);
          bool r;
          switch (in.sub) {
            case TQ_LT: r = x < y; break;
            case TQ_LE: r = x <= y; break;
            case TQ_EQ: r = x == y; break;
            case TQ_NE: r = x != y; break;
            case TQ_GE: r = x >= y; break;
            default: r = x > y;
          }
          put_b(w, in.dst, v, r, va && vb);
        }
        break;
      }
      case OP_CMP_B: {
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool va, vb;
          int x = get_b(w, in.ak, in.a, v, va), y = get_b(w, in.bk, in.b, v, vb);
          put_b(w, in.dst, v, cmp_res(x - y, in.sub), va && vb);
        }
        break;
      }
      case OP_AND:
      case OP_OR: {
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool va, vb;
          bool x = get_b(w, in.ak, in.a, v, va), y = get_b(w, in.bk, in.b, v, vb);
          put_b(w, in.dst, v, in.op == OP_AND ? (x && y) : (x || y), va && vb);
        }
        break;
      }
      case OP_NOT: {
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool va;
          bool x = get_b(w, in.ak, in.a, v, va);
          put_b(w, in.dst, v, !x, va);
        }
        break;
      }
      default:
        break;
    }
  }
}

// Rows of this warp that exist and pass the predicate, per v.
__device__ __forceinline__ u32 pass_mask(const WCtx& w, int v) {
  bool exists = trow(w, v) < w.nrows;
  bool pass = exists;
  if (w.p->pred_kind != K_NONE) {
    bool valid;
    bool x = get_b(w, w.p->pred_kind, w.p->pred_idx, v, valid);
    pass = exists && valid && x;
  }
  return __ballot_sync(kFull, pass);
}

// ------------------------------------------------------------------ keys
// Key words of this lane's row (v); returns true if any key is null.  The
// last word (index key_words) holds one null bit per key.
__device__ __forceinline__ bool key_words(const WCtx& w, int v, u64* kw) {
  const PipeParams& p = *w.p;
  u64 nullmask = 0;
  int pos = 0;
  for (u32 k = 0; k < p.nkeys; ++k) {
    const KeyOpnd& ko = p.keys[k];
    bool valid;
    if (ko.kind == K_COL_F64 || ko.kind == K_TMP_F || ko.kind == K_LIT_F) {
      double d = get_f(w, ko.kind, ko.idx, v, 0, valid);
      kw[pos++] = valid ? (u64)__double_as_longlong(d) : 0;
    } else {
      i128 x = get_i(w, ko.kind, ko.idx, v, valid);
      if (!valid) x = 0;
      kw[pos++] = lo64(x);
      if (ko.words == 2) kw[pos++] = hi64(x);
    }
    if (!valid) nullmask |= 1ull << k;
  }
  kw[pos] = nullmask;
  return nullmask != 0;
}

// fnv1a64 over the LE bytes of the keys (reference common.hpp:128-136),
// chained across key columns; a null key hashes as zero bytes.
__device__ __forceinline__ u64 partition_hash(const WCtx& w, const u64* kw) {
  const PipeParams& p = *w.p;
  u64 h = kFnvBasis;
  int pos = 0;
  for (u32 k = 0; k < p.nkeys; ++k) {
    const KeyOpnd& ko = p.keys[k];
    if (ko.bytes == 16) {
      h = fnv_bytes(h, kw[pos], 8);
      h = fnv_bytes(h, kw[pos + 1], 8);
    } else {
      h = fnv_bytes(h, kw[pos], ko.bytes);
    }
    pos += ko.words;
  }
  return h;
}

// ------------------------------------------------------------------ join table
__device__ __forceinline__ const long long* jt_entry(const JoinTable& t, u64 slot) {
  return (const long long*)(t.entries + slot * t.stride);
}

__device__ __forceinline__ bool jt_key_eq(const JoinTable& t, const long long* e, const u64* kw) {
  for (u32 i = 0; i < t.kw; ++i)
    if ((u64)e[1 + i] != kw[i]) return false;
  return true;
}

// Number of build rows whose keys equal kw.
__device__ __forceinline__ u32 jt_count(const JoinTable& t, const u64* kw) {
  u64 mask = t.cap - 1;
  u64 s = key_hash(kw, (int)t.kw) & mask;
  u32 n = 0;
  for (;;) {
    const long long* e = jt_entry(t, s);
    long long row = e[0];
    if (row < 0) break;
    if (jt_key_eq(t, e, kw)) ++n;
    s = (s + 1) & mask;
  }
  return n;
}

// ------------------------------------------------------------------ emit helpers
__device__ __forceinline__ void store_out(const OutCol& o, u64 pos, const WCtx& w, int v, long long brow) {
  bool valid = true;
  if (o.src == OUT_BUILD) {
    const uint8_t* src = o.bvalues + (u64)brow * o.width;
    if (o.width == 16) *(ulonglong2*)(o.values + pos * 16) = *(const ulonglong2*)src;
    else if (o.width == 8) *(u64*)(o.values + pos * 8) = *(const u64*)src;
    else o.values[pos] = *src;
    if (o.bvalidity) valid = bm_get(o.bvalidity, (u64)brow);
  } else {
    switch (o.kind) {
      case K_COL_I64:
      case K_COL_F64: {
        const StagedCol& sc = w.p->cols[o.idx];
        *(u64*)(o.values + pos * 8) = ((const u64*)(w.stage + sc.off))[trow(w, v)];
        valid = col_valid(w, o.idx, v);
        break;
      }
      case K_COL_DEC: {
        const StagedCol& sc = w.p->cols[o.idx];
        *(ulonglong2*)(o.values + pos * 16) = ((const ulonglong2*)(w.stage + sc.off))[trow(w, v)];
        valid = col_valid(w, o.idx, v);
        break;
      }
      case K_COL_BOOL: {
        const StagedCol& sc = w.p->cols[o.idx];
        o.values[pos] = w.stage[sc.off + trow(w, v)];
        valid = col_valid(w, o.idx, v);
        break;
      }
      case K_TMP_F:
      case K_LIT_F: {
        double d = get_f(w, o.kind, o.idx, v, 0, valid);
        *(double*)(o.values + pos * 8) = d;
        break;
      }
      case K_TMP_B:
      case K_LIT_B: {
        bool b = get_b(w, o.kind, o.idx, v, valid);
        o.values[pos] = b ? 1 : 0;
        break;
      }
      default: {  // K_TMP_I / K_LIT_I
        i128 x = get_i(w, o.kind, o.idx, v, valid);
        if (o.width == 16) *(ulonglong2*)(o.values + pos * 16) = make_ulonglong2(lo64(x), hi64(x));
        else *(u64*)(o.values + pos * 8) = lo64(x);
      }
    }
  }
  if (o.validity && valid) bm_set_atomic(o.validity, pos);
}

// ------------------------------------------------------------------ aggregation
constexpr u32 kStEmpty = 0, kStBusy = 1, kStReady = 2;

__device__ __forceinline__ bool keys_equal(const volatile u64* a, const u64* b, u32 n) {
  for (u32 i = 0; i < n; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

// Find-or-insert `kw` (kwa words) in a state/keys open-addressing table.
// Returns slot or -1 when all `limit` probes are taken by other keys.
__device__ long long table_find_insert(u32* state, u64* keys, u64 cap, u32 kwa, const u64* kw, u64 h, u64 limit,
                                       unsigned long long* counter) {
  u64 mask = cap - 1;
  u64 s = h & mask;
  for (u64 probe = 0; probe < limit; ++probe) {
    volatile u32* st = state + s;
    u32 cur = *st;
    if (cur == kStEmpty) {
      cur = atomicCAS(state + s, kStEmpty, kStBusy);
      if (cur == kStEmpty) {
        for (u32 i = 0; i < kwa; ++i) keys[s * kwa + i] = kw[i];
        __threadfence();
        atomicExch(state + s, kStReady);
        if (counter) atomicAdd(counter, 1ull);
        return (long long)s;
      }
    }
    while (cur == kStBusy) cur = *st;
    if (keys_equal((volatile u64*)(keys + s * kwa), kw, kwa)) return (long long)s;
    s = (s + 1) & mask;
  }
  return -1;
}

// Accumulator identity values.
__device__ __forceinline__ void acc_identity(uint8_t op, u64& lo, u64& hi) {
  switch (op) {
    case ACC_MIN_I: lo = ~0ull; hi = 0x7fffffffffffffffull; break;
    case ACC_MAX_I: lo = 0; hi = 0x8000000000000000ull; break;
    case ACC_MIN_F: lo = (u64)__double_as_longlong(__longlong_as_double(0x7ff0000000000000ll)); hi = 0; break;
    case ACC_MAX_F: lo = (u64)__double_as_longlong(__longlong_as_double((long long)0xfff0000000000000ull)); hi = 0; break;
    default: lo = 0; hi = 0;
  }
}

// Apply a warp-reduced contribution into a plain (non-atomic) accumulator.
__device__ __forceinline__ void acc_apply_plain(uint8_t op, u64* a, i128 xi, double xf, u64 cnt) {
  switch (op) {
    case ACC_SUM_I: { i128 c = mk128(a[0], a[1]); c = add128(c, xi); a[0] = lo64(c); a[1] = hi64(c); break; }
    case ACC_SUM_F: { double d = __longlong_as_double((long long)a[0]); d += xf; a[0] = (u64)__double_as_longlong(d); break; }
    case ACC_CNT: a[0] += cnt; break;
    case ACC_MIN_I: { i128 c = mk128(a[0], a[1]); if (xi < c) { a[0] = lo64(xi); a[1] = hi64(xi); } break; }
    case ACC_MAX_I: { i128 c = mk128(a[0], a[1]); if (xi > c) { a[0] = lo64(xi); a[1] = hi64(xi); } break; }
    case ACC_MIN_F: { double d = __longlong_as_double((long long)a[0]); if (xf < d) a[0] = (u64)__double_as_longlong(xf); break; }
    case ACC_MAX_F: { double d = __longlong_as_double((long long)a[0]); if (xf > d) a[0] = (u64)__double_as_longlong(xf); break; }
  }
}
__device__ __forceinline__ void acc_apply_atomic(uint8_t op, u64* a, i128 xi, double xf, u64 cnt) {
  switch (op) {
    case ACC_SUM_I: if (xi != 0) atomic_add_i128(a, xi); break;
    case ACC_SUM_F: atomicAdd((double*)a, xf); break;
    case ACC_CNT: if (cnt) atomicAdd((unsigned long long*)a, (unsigned long long)cnt); break;
    case ACC_MIN_I: atomic_minmax_i128((u128*)a, xi, true); break;
    case ACC_MAX_I: atomic_minmax_i128((u128*)a, xi, false); break;
    case ACC_MIN_F: atomic_minmax_f64((double*)a, xf, true); break;
    case ACC_MAX_F: atomic_minmax_f64((double*)a, xf, false); break;
  }
}

// Warp-reduce accumulator `a` over lanes in `members` (all lanes participate).
__device__ __forceinline__ void acc_reduce(const WCtx& w, const AccSpec& as, int v, bool member, i128& xi,
                                           double& xf, u64& cnt) {
  bool valid = true;
  xi = 0;
  xf = 0;
  cnt = 0;
  switch (as.op) {
    case ACC_CNT: {
      if (as.kind != K_NONE) {
        bool vv;
        if (as.kind == K_COL_F64 || as.kind == K_TMP_F || as.kind == K_LIT_F) (void)get_f(w, as.kind, as.idx, v, 0, vv);
        else (void)get_i(w, as.kind, as.idx, v, vv);
        valid = vv;
      }
      cnt = __popc(__ballot_sync(kFull, member && valid));
      return;
    }
    case ACC_SUM_I: {
      i128 x = get_i(w, as.kind, as.idx, v, valid);
      xi = warp_sum_i128(member && valid ? x : (i128)0);
      return;
    }
    case ACC_SUM_F: {
      double x = get_f(w, as.kind, as.idx, v, as.scale, valid);
      xf = warp_sum_f64(member && valid ? x : 0.0);
      return;
    }
    case ACC_MIN_I:
    case ACC_MAX_I: {
      i128 x = get_i(w, as.kind, as.idx, v, valid);
      u64 ilo, ihi;
      acc_identity(as.op, ilo, ihi);
      if (!(member && valid)) x = mk128(ilo, ihi);
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) {
        i128 o = shfl_xor_i128(x, m);
        x = as.op == ACC_MIN_I ? (o < x ? o : x) : (o > x ? o : x);
      }
      xi = x;
      return;
    }
    default: {  // MIN_F / MAX_F
      double x = get_f(w, as.kind, as.idx, v, as.scale, valid);
      u64 ilo, ihi;
      acc_identity(as.op, ilo, ihi);
      if (!(member && valid)) x = __longlong_as_double((long long)ilo);
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) {
        double o = __shfl_xor_sync(kFull, x, m);
        x = as.op == ACC_MIN_F ? fmin(x, o) : fmax(x, o);
      }
      xf = x;
      return;
    }
  }
}

// Global-table slot for kw (insert if new); -1 on overflow.
__device__ __forceinline__ long long agg_global_slot(const PipeParams& p, const u64* kw, u32 kwa, u64 h) {
  long long s = table_find_insert(p.agg.state, p.agg.keys, p.agg.cap, kwa, kw, h, p.agg.cap < 512 ? p.agg.cap : 512,
                                  p.agg.nused);
  if (s < 0) atomicExch(p.agg.overflow, 1u);
  return s;
}

// ------------------------------------------------------------------ stage loading
__device__ __forceinline__ void issue_tile(const PipeParams& p, uint8_t* stage, uint64_t* bar, u32 tile) {
  u64 r0 = (u64)tile * kTile;
  u64 n = p.rows - r0;
  bool full = n >= (u64)kTile;
  u32 bytes = 0;
  if (full)
    for (u32 c = 0; c < p.nstaged; ++c)
      if (p.cols[c].bulk_ok) bytes += kTile * p.cols[c].width + (p.cols[c].validity ? kTile / 8 : 0);
  mbar_arrive_expect_tx(bar, bytes);
  if (!full) return;
  for (u32 c = 0; c < p.nstaged; ++c) {
    const StagedCol& sc = p.cols[c];
    if (!sc.bulk_ok) continue;
    bulk_g2s(stage + sc.off, sc.values + r0 * sc.width, kTile * sc.width, bar);
    if (sc.validity) bulk_g2s(stage + sc.voff, sc.validity + r0 / 8, kTile / 8, bar);
  }
}

// Plain cooperative loads for tail tiles and misaligned columns.
__device__ void manual_tile(const PipeParams& p, uint8_t* stage, u32 tile) {
  u64 r0 = (u64)tile * kTile;
  u64 n = min((u64)kTile, p.rows - r0);
  bool full = n == (u64)kTile;
  for (u32 c = 0; c < p.nstaged; ++c) {
    const StagedCol& sc = p.cols[c];
    if (full && sc.bulk_ok) continue;
    u64 bytes = n * sc.width;
    const uint8_t* src = sc.values + r0 * sc.width;
    for (u64 i = threadIdx.x; i < bytes; i += kThreads) stage[sc.off + i] = src[i];
    if (sc.validity) {
      u64 vb = (n + 7) / 8;
      for (u64 i = threadIdx.x; i < kTile / 8; i += kThreads)
        stage[sc.voff + i] = i < vb ? sc.validity[r0 / 8 + i] : 0;
    }
  }
}

__device__ __forceinline__ bool tile_needs_manual(const PipeParams& p, u32 tile) {
  u64 r0 = (u64)tile * kTile;
  if (p.rows - r0 < (u64)kTile) return true;
  for (u32 c = 0; c < p.nstaged; ++c)
    if (!p.cols[c].bulk_ok) return true;
  return false;
}

// ------------------------------------------------------------------ the kernel
template <int SINK>
__global__ void __launch_bounds__(kThreads) pipe_kernel(const __grid_constant__ PipeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  DInstr* s_code = (DInstr*)(smem + p.off_code);
  DLit* s_lits = (DLit*)(smem + p.off_lits);
  uint64_t* bars = (uint64_t*)(smem + p.off_bar);
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (u32 i = threadIdx.x; i < p.ncode; i += kThreads) s_code[i] = p.code[i];
  for (u32 i = threadIdx.x; i < p.nlits; i += kThreads) s_lits[i] = p.lits[i];
  if (threadIdx.x == 0) {
    for (u32 s = 0; s < p.nstages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }

  // sink shared state
  u32* s_cnt = (u32*)(smem + p.off_sink);                  // [kWarps][ndest] (COUNT/EMIT)
  unsigned long long* s_base = (unsigned long long*)(s_cnt + kWarps * kMaxDest);  // [kWarps][ndest]
  // AGG: local table
  const u32 kwa = p.key_words + 1;
  const u32 G = p.local_groups;
  u32* l_state = (u32*)(smem + p.off_sink);
  u64* l_keys = (u64*)(smem + p.off_sink + ((G * 4 + 15) & ~15u));
  u64* l_acc = l_keys + (u64)G * kwa;  // [kWarps][G][nacc][2]
  if (SINK == SINK_COUNT || SINK == SINK_EMIT) {
    for (u32 i = threadIdx.x; i < kWarps * kMaxDest; i += kThreads) s_cnt[i] = 0;
  }
  if (SINK == SINK_AGG) {
    for (u32 i = threadIdx.x; i < G; i += kThreads) l_state[i] = kStEmpty;
    for (u32 i = threadIdx.x; i < kWarps * G * p.nacc; i += kThreads) {
      u64 lo, hi;
      acc_identity(p.acc[i % p.nacc].op, lo, hi);
      l_acc[2 * i] = lo;
      l_acc[2 * i + 1] = hi;
    }
  }
  __syncthreads();

  WCtx w;
  w.p = &p;
  w.lits = s_lits;
  w.vslot = smem + p.off_vslot + (size_t)warp * p.nvslots * kV * 32 * 16;
  w.vvalid = (u32*)(smem + p.off_vvalid) + (size_t)warp * p.nvslots * kV;
  w.bslot = (u32*)(smem + p.off_bslot) + (size_t)warp * p.nbslots * kV * 2;
  w.row0 = warp * 32 * kV;
  w.lane = lane;

  const u32 first = blockIdx.x, step = gridDim.x;
  if (threadIdx.x == 0) {
    for (u32 s = 0; s < p.nstages; ++s) {
      u32 t = first + s * step;
      if (t < p.ntiles) issue_tile(p, smem + p.off_stage + s * p.stage_bytes, &bars[s], t);
    }
  }

  u32 k = 0;
  for (u32 tile = first; tile < p.ntiles; tile += step, ++k) {
    const u32 s = k % p.nstages;
    uint8_t* stage = smem + p.off_stage + s * p.stage_bytes;
    mbar_wait(&bars[s], (k / p.nstages) & 1);
    if (tile_needs_manual(p, tile)) {
      manual_tile(p, stage, tile);
      __syncthreads();
    }
    const u64 r0 = (u64)tile * kTile;
    w.stage = stage;
    w.nrows = (u32)min((u64)kTile, p.rows - r0);

    // ---- predicate, then (if any row survives) the rest of the program
    run_code(w, s_code, 0, p.npred);
    u32 pm[kV];
    u32 any = 0;
#pragma unroll
    for (int v = 0; v < kV; ++v) { pm[v] = pass_mask(w, v); any |= pm[v]; }
    if (any) run_code(w, s_code, p.npred, p.ncode);

    if (SINK == SINK_COUNT || SINK == SINK_EMIT) {
      u32 dest[kV];
      u32 mult[kV];
#pragma unroll
      for (int v = 0; v < kV; ++v) {
        bool pass = (pm[v] >> lane) & 1u;
        dest[v] = 0;
        mult[v] = pass ? 1u : 0u;
        if (any && p.dest_kind != DEST_FILTER) {
          u64 kw[kMaxKeyWords + 1];
          bool has_null = key_words(w, v, kw);
          if (p.dest_kind == DEST_PARTITION) {
            dest[v] = (u32)(partition_hash(w, kw) % p.ndest);
          } else {  // probe: null keys never match
            mult[v] = (pass && !has_null) ? jt_count(p.jt, kw) : 0u;
          }
        }
      }
      // per-warp counts per destination
      if (p.dest_kind == DEST_PROBE) {
        u32 tot = 0;
#pragma unroll
        for (int v = 0; v < kV; ++v) tot += mult[v];
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) tot += __shfl_xor_sync(kFull, tot, m);
        if (lane == 0) s_cnt[warp * kMaxDest] = tot;
      } else {
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool pass = mult[v] != 0;
          u32 peers = __match_any_sync(kFull, pass ? dest[v] : 0xffffffffu);
          if (pass && (peers & lanemask_lt()) == 0) s_cnt[warp * kMaxDest + dest[v]] += __popc(peers);
          __syncwarp();
        }
      }
      __syncthreads();
      if (SINK == SINK_COUNT) {
        for (u32 d = threadIdx.x; d < p.ndest; d += kThreads) {
          u32 t = 0;
          for (u32 ww = 0; ww < kWarps; ++ww) { t += s_cnt[ww * kMaxDest + d]; s_cnt[ww * kMaxDest + d] = 0; }
          p.tile_counts[(u64)d * p.ntiles + tile] = t;
        }
      } else {
        // warp bases = tile offset + counts of earlier warps
        for (u32 d = threadIdx.x; d < p.ndest; d += kThreads) {
          // dense 1:1 projection: no count phase, tile t starts at row t*kTile
          unsigned long long b = p.tile_offsets ? p.tile_offsets[(u64)d * p.ntiles + tile] : (u64)tile * kTile;
          for (u32 ww = 0; ww < kWarps; ++ww) {
            s_base[ww * kMaxDest + d] = b;
            b += s_cnt[ww * kMaxDest + d];
            s_cnt[ww * kMaxDest + d] = 0;
          }
        }
        __syncthreads();
        unsigned long long* wb = s_base + warp * kMaxDest;
        if (p.dest_kind == DEST_PROBE) {
#pragma unroll
          for (int v = 0; v < kV; ++v) {
            u32 m = mult[v];
            u32 incl = m;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              u32 y = __shfl_up_sync(kFull, incl, o);
              if (lane >= (u32)o) incl += y;
            }
            u32 total = __shfl_sync(kFull, incl, 31);
            unsigned long long pos = wb[0] + (incl - m);
            __syncwarp();
            if (lane == 0) wb[0] += total;
            __syncwarp();
            if (m) {
              u64 kw[kMaxKeyWords + 1];
              key_words(w, v, kw);
              const JoinTable& t = p.jt;
              u64 mask = t.cap - 1;
              u64 sl = key_hash(kw, (int)t.kw) & mask;
              for (;;) {
                const long long* e = jt_entry(t, sl);
                long long brow = e[0];
                if (brow < 0) break;
                if (jt_key_eq(t, e, kw)) {
                  for (u32 c = 0; c < p.nout; ++c) store_out(p.out[c], pos, w, v, brow);
                  ++pos;
                }
                sl = (sl + 1) & mask;
              }
            }
          }
        } else {
#pragma unroll
          for (int v = 0; v < kV; ++v) {
            bool pass = mult[v] != 0;
            u32 peers = __match_any_sync(kFull, pass ? dest[v] : 0xffffffffu);
            unsigned long long pos = 0;
            if (pass) pos = wb[dest[v]] + __popc(peers & lanemask_lt());
            __syncwarp();
            if (pass && (peers & lanemask_lt()) == 0) wb[dest[v]] += __popc(peers);
            __syncwarp();
            if (pass)
              for (u32 c = 0; c < p.nout; ++c) store_out(p.out[c], pos, w, v, -1);
          }
        }
      }
    } else if (SINK == SINK_BUILD) {
      if (any) {
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool pass = (pm[v] >> lane) & 1u;
          u64 kw[kMaxKeyWords + 1];
          bool has_null = key_words(w, v, kw);
          if (pass && !has_null) {
            const JoinTable& t = p.jt;
            u64 mask = t.cap - 1;
            u64 sl = key_hash(kw, (int)t.kw) & mask;
            long long row = (long long)(p.row_base + r0 + trow(w, v));
            for (;;) {
              long long* e = (long long*)(t.entries + sl * t.stride);
              if (atomicCAS((unsigned long long*)e, (unsigned long long)-1ll, (unsigned long long)row) ==
                  (unsigned long long)-1ll) {
                for (u32 i = 0; i < t.kw; ++i) e[1 + i] = (long long)kw[i];
                break;
              }
              sl = (sl + 1) & mask;
            }
          }
        }
      }
    } else if (SINK == SINK_AGG) {
      if (any) {
        u64* myacc = l_acc + (u64)warp * G * p.nacc * 2;
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool pass = (pm[v] >> lane) & 1u;
          u64 kw[kMaxKeyWords + 1];
          key_words(w, v, kw);
          u64 h = key_hash(kw, (int)kwa);
          // one lookup per distinct hash in the warp
          u32 hp = __match_any_sync(kFull, pass ? h : ~0ull);
          u32 leader = __ffs(hp) - 1;
          long long slot = -1;  // < G: local; >= G: G + global slot
          bool mine_leader = pass && leader == lane;
          if (mine_leader) {
            long long s = G ? table_find_insert(l_state, l_keys, G, kwa, kw, h, G, nullptr) : -1;
            if (s < 0) {
              s = agg_global_slot(p, kw, kwa, h);
              slot = s < 0 ? -2 : (long long)G + s;
            } else {
              slot = s;
            }
          }
          slot = __shfl_sync(kFull, slot, leader);
          if (pass && !mine_leader && slot != -2) {
            // verify (hash collision within the warp): compare stored keys
            const u64* sk = slot < (long long)G ? l_keys + (u64)slot * kwa : p.agg.keys + (u64)(slot - G) * kwa;
            bool eq = true;
            for (u32 i = 0; i < kwa; ++i) eq &= ((const volatile u64*)sk)[i] == kw[i];
            if (!eq) {
              long long s = G ? table_find_insert(l_state, l_keys, G, kwa, kw, h, G, nullptr) : -1;
              if (s < 0) {
                s = agg_global_slot(p, kw, kwa, h);
                slot = s < 0 ? -2 : (long long)G + s;
              } else {
                slot = s;
              }
            }
          }
          bool has = pass && slot != -2;
          u32 todo = __ballot_sync(kFull, has);
          while (todo) {
            u32 ld = __ffs(todo) - 1;
            long long gs = __shfl_sync(kFull, slot, ld);
            bool member = has && slot == gs;
            todo &= ~__ballot_sync(kFull, member);
            for (u32 a = 0; a < p.nacc; ++a) {
              i128 xi;
              double xf;
              u64 cnt;
              acc_reduce(w, p.acc[a], v, member, xi, xf, cnt);
              if (lane == ld) {
                if (gs < (long long)G) acc_apply_plain(p.acc[a].op, myacc + ((u64)gs * p.nacc + a) * 2, xi, xf, cnt);
                else acc_apply_atomic(p.acc[a].op, p.agg.acc + ((u64)(gs - G) * p.nacc + a) * 2, xi, xf, cnt);
              }
            }
          }
        }
      }
    }

    __syncthreads();  // stage s fully consumed
    if (threadIdx.x == 0) {
      u32 nt = tile + p.nstages * step;
      if (nt < p.ntiles) {
        fence_proxy_async();
        issue_tile(p, stage, &bars[s], nt);
      }
    }
  }

  if (SINK == SINK_AGG && G > 0) {
    __syncthreads();
    // merge the per-warp copies of each local group into the global table
    for (u32 g = warp; g < G; g += kWarps) {
      if (l_state[g] != kStReady) continue;
      long long gs = -1;
      if (lane == 0) {
        u64 kw[kMaxKeyWords + 1];
        for (u32 i = 0; i < kwa; ++i) kw[i] = l_keys[(u64)g * kwa + i];
        gs = agg_global_slot(p, kw, kwa, key_hash(kw, (int)kwa));
      }
      gs = __shfl_sync(kFull, gs, 0);
      if (gs < 0) continue;
      for (u32 a = lane; a < p.nacc; a += 32) {
        const AccSpec& as = p.acc[a];
        u64 lo, hi;
        acc_identity(as.op, lo, hi);
        u64 tot[2] = {lo, hi};
        for (u32 ww = 0; ww < kWarps; ++ww) {
          const u64* src = l_acc + (((u64)ww * G + g) * p.nacc + a) * 2;
          i128 xi = mk128(src[0], src[1]);
          double xf = __longlong_as_double((long long)src[0]);
          acc_apply_plain(as.op, tot, xi, xf, src[0]);
        }
        acc_apply_atomic(as.op, p.agg.acc + ((u64)gs * p.nacc + a) * 2, mk128(tot[0], tot[1]),
                         __longlong_as_double((long long)tot[0]), tot[0]);
      }
    }
  }
}

template __global__ void pipe_kernel<SINK_COUNT>(const __grid_constant__ PipeParams p);
template __global__ void pipe_kernel<SINK_EMIT>(const __grid_constant__ PipeParams p);
template __global__ void pipe_kernel<SINK_AGG>(const __grid_constant__ PipeParams p);
template __global__ void pipe_kernel<SINK_BUILD>(const __grid_constant__ PipeParams p);

// ------------------------------------------------------------------ host launch
cudaError_t launch_pipeline(int sink, const PipeParams& p, u32 smem_bytes, u32 grid, cudaStream_t st) {
  void (*fn)(PipeParams) = nullptr;
  switch (sink) {
    case SINK_COUNT: fn = pipe_kernel<SINK_COUNT>; break;
    case SINK_EMIT: fn = pipe_kernel<SINK_EMIT>; break;
    case SINK_AGG: fn = pipe_kernel<SINK_AGG>; break;
    default: fn = pipe_kernel<SINK_BUILD>; break;
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
  if (e != cudaSuccess) return e;
  fn<<<grid, kThreads, smem_bytes, st>>>(p);
  return cudaGetLastError();
}

}  // namespace tq
