// interp.cuh — the generic program policy: the Expr register machine
// (program.h) interpreted per warp over shared-memory value slots.  Compiled
// ahead of time into libtq_gpu.so; runs any program, including ones the
// NVRTC specialiser (jit.cu) declines or fails to compile.
#pragma once
#include "kernel_common.cuh"

namespace tq {

__constant__ double c_p10[39] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11, 1e12,
                                 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22, 1e23, 1e24, 1e25,
                                 1e26, 1e27, 1e28, 1e29, 1e30, 1e31, 1e32, 1e33, 1e34, 1e35, 1e36, 1e37, 1e38};

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

// ------------------------------------------------------------------ emit helpers
__device__ __forceinline__ void store_out(const OutCol& o, u64 pos, const WCtx& w, int v, long long brow, bool vbit) {
  bool valid = true;
  uint8_t* dst = o.values + w.out_delta;
  if (o.src == OUT_BUILD) {
    store_build(o, pos, brow, w.out_delta);
    return;
  } else {
    switch (o.kind) {
      case K_COL_I64:
      case K_COL_F64: {
        const StagedCol& sc = w.p->cols[o.idx];
        *(u64*)(dst + pos * 8) = ((const u64*)(w.stage + sc.off))[trow(w, v)];
        valid = col_valid(w, o.idx, v);
        break;
      }
      case K_COL_DEC: {
        const StagedCol& sc = w.p->cols[o.idx];
        *(ulonglong2*)(dst + pos * 16) = ((const ulonglong2*)(w.stage + sc.off))[trow(w, v)];
        valid = col_valid(w, o.idx, v);
        break;
      }
      case K_COL_BOOL: {
        const StagedCol& sc = w.p->cols[o.idx];
        dst[pos] = w.stage[sc.off + trow(w, v)];
        valid = col_valid(w, o.idx, v);
        break;
      }
      case K_TMP_F:
      case K_LIT_F: {
        double d = get_f(w, o.kind, o.idx, v, 0, valid);
        *(double*)(dst + pos * 8) = d;
        break;
      }
      case K_TMP_B:
      case K_LIT_B: {
        bool b = get_b(w, o.kind, o.idx, v, valid);
        dst[pos] = b ? 1 : 0;
        break;
      }
      default: {  // K_TMP_I / K_LIT_I
        i128 x = get_i(w, o.kind, o.idx, v, valid);
        if (o.width == 16) *(ulonglong2*)(dst + pos * 16) = make_ulonglong2(lo64(x), hi64(x));
        else *(u64*)(dst + pos * 8) = lo64(x);
      }
    }
  }
  if (o.validity && vbit && valid) bm_set_atomic(o.validity + w.out_delta, pos);
}


struct InterpP {
  static constexpr bool kInterp = true;
  static constexpr int kKwa = 0, kKw = 0, kNacc = 0;
  static constexpr bool kKey1x8 = false;
  __device__ __forceinline__ static u32 nacc(const PipeParams& p) { return p.nacc; }
  __device__ __forceinline__ static u32 nplanes(const PipeParams& p) { return p.nplanes; }
  __device__ __forceinline__ static uint8_t acc_op(const PipeParams& p, u32 a) { return p.acc[a].op; }
  __device__ __forceinline__ static uint8_t acc_kind(const PipeParams& p, u32 a) { return p.acc[a].kind; }
  __device__ __forceinline__ static u32 acc_plane(const PipeParams& p, u32 a) { return p.acc_plane[a]; }

  struct Raw {};  // the interpreter reads the stage directly (held until the tile ends)
  __device__ __forceinline__ static void load(const WCtx&, int, Raw&) {}
  __device__ __forceinline__ static u32 tile_begin(WCtx& w, const DInstr* code, u32* pm, const Raw*) {
    const PipeParams& p = *w.p;
    run_code(w, code, 0, p.npred);
    u32 any = 0;
#pragma unroll
    for (int v = 0; v < kV; ++v) {
      pm[v] = pass_mask(w, v);
      any |= pm[v];
    }
    if (any) run_code(w, code, p.npred, p.ncode);
    return any;
  }
  __device__ __forceinline__ static bool keys(const WCtx& w, int v, u64* kw, const Raw&) {
    return key_words(w, v, kw);
  }
  __device__ __forceinline__ static void accs(const WCtx& w, int v, RowVals& x, const Raw&) {
    const PipeParams& p = *w.p;
    for (u32 a = 0; a < p.nacc; ++a) {
      const AccSpec& as = p.acc[a];
      bool valid = true;
      x.ai[a] = 0;
      x.af[a] = 0;
      if (as.op == ACC_CNT) {
        if (as.kind != K_NONE) {
          if (as.kind == K_COL_F64 || as.kind == K_TMP_F || as.kind == K_LIT_F) (void)get_f(w, as.kind, as.idx, v, 0, valid);
          else (void)get_i(w, as.kind, as.idx, v, valid);
        }
      } else if (as.op == ACC_SUM_I || as.op == ACC_MIN_I || as.op == ACC_MAX_I) {
        x.ai[a] = get_i(w, as.kind, as.idx, v, valid);
      } else {
        x.af[a] = get_f(w, as.kind, as.idx, v, as.scale, valid);
      }
      x.av[a] = valid;
    }
  }
  __device__ __forceinline__ static void store(const WCtx& w, int v, u64 pos, long long brow, const Raw&) {
    const PipeParams& p = *w.p;
    for (u32 c = 0; c < p.nout; ++c) store_out(p.out[c], pos, w, v, brow, (w.vmask >> c) & 1u);
  }
};

}  // namespace tq
