// datagen.cu — synthetic TPC-H-style tables generated on the device
// (DESIGN.md §4).  Every value is a pure function of (column seed, row):
// U(seed, i, n) = SplitMix64(seed).next()^(i+1) % n, the counter-based form
// of reference common.hpp:139-158 (output k = mix(seed + k*gamma)), so the
// tables are bit-identical to the CPU generator in oracle/tq_oracle.cpp.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.h"
#include "device.cuh"

namespace tq {

static u64 fnv_str(const char* s, u64 h) {
  for (; *s; ++s) {
    h ^= (uint8_t)*s;
    h *= kFnvPrime;
  }
  return h;
}
static u64 col_seed(const char* name) { return fnv_str(name, 42); }

__device__ __forceinline__ u64 U(u64 seed, u64 i, u64 n) { return sm_nth(seed, i + 1) % n; }

__device__ __forceinline__ long long year_of(long long d) {
  const long long ys[8] = {8035, 8401, 8766, 9131, 9496, 9862, 10227, 10592};
  int y = 0;
  while (y + 1 < 8 && d >= ys[y + 1]) ++y;
  return 1992 + y;
}
__device__ __forceinline__ long long retail_cents(long long p) { return 90000 + ((p / 10) % 20001) + 100 * (p % 1000); }
__device__ __forceinline__ long long ps_supp(long long p, long long j, long long ns) {
  return ((p - 1 + j * (ns / 4 + (p - 1) / ns)) % ns) + 1;
}

struct Seeds {
  u64 s[12];
};

#define GRID_LOOP(i, n) for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (u64)gridDim.x * blockDim.x)

__global__ void k_orders(u64 lo, u64 n, u64 nc, Seeds S, long long* ok0, long long* ck0, long long* od0,
                         long long* sp0, long long* yr0) {
  GRID_LOOP(j, n) {
    u64 i = lo + j;
    long long *ok = ok0 - lo, *ck = ck0 - lo, *od = od0 - lo, *sp = sp0 - lo, *yr = yr0 - lo;
    long long d = 8035 + (long long)U(S.s[1], i, 2406);
    ok[i] = (long long)i + 1;
    ck[i] = 1 + (long long)U(S.s[0], i, nc);
    od[i] = d;
    sp[i] = 0;
    yr[i] = year_of(d);
  }
}

__global__ void k_nlines(u64 no, u64 seed, u32* n) {
  GRID_LOOP(i, no) n[i] = 1 + (u32)U(seed, i, 7);
}

struct LiOut {
  long long *ok, *pk, *sk, *rf, *ls, *sd;
  ulonglong2 *qty, *ep, *disc, *tax;
};

// orders [olo, olo+n); output row = global lineitem row - off[olo]
__global__ void k_lineitem(u64 olo, u64 n, const u64* off, u64 np, u64 ns, Seeds S, LiOut o0) {
  const u64 rbase = off[olo];
  LiOut o = o0;
  o.ok -= rbase; o.pk -= rbase; o.sk -= rbase; o.rf -= rbase; o.ls -= rbase; o.sd -= rbase;
  o.qty -= rbase; o.ep -= rbase; o.disc -= rbase; o.tax -= rbase;
  GRID_LOOP(j, n) {
    u64 oi = olo + j;
    long long od = 8035 + (long long)U(S.s[0], oi, 2406);
    for (u64 r = off[oi]; r < off[oi + 1]; ++r) {
      long long pk = 1 + (long long)U(S.s[1], r, np);
      long long sk = ps_supp(pk, (long long)U(S.s[2], r, 4), (long long)ns);
      long long qty = 1 + (long long)U(S.s[3], r, 50);
      long long ship = od + 1 + (long long)U(S.s[8], r, 121);
      long long receipt = ship + 1 + (long long)U(S.s[6], r, 30);
      long long rf = receipt <= 9298 ? (U(S.s[7], r, 2) == 0 ? 'R' : 'A') : 'N';
      o.ok[r] = (long long)oi + 1;
      o.pk[r] = pk;
      o.sk[r] = sk;
      o.qty[r] = make_ulonglong2((u64)(qty * 100), 0);
      o.ep[r] = make_ulonglong2((u64)(qty * retail_cents(pk)), 0);
      o.disc[r] = make_ulonglong2(U(S.s[4], r, 11), 0);
      o.tax[r] = make_ulonglong2(U(S.s[5], r, 9), 0);
      o.rf[r] = rf;
      o.ls[r] = ship > 9298 ? 'O' : 'F';
      o.sd[r] = ship;
    }
  }
}

__global__ void k_simple(int table, u64 lo, u64 n, u64 ns, Seeds S, long long* c0_, long long* c1_, void* c2_) {
  GRID_LOOP(j, n) {
    u64 i = lo + j;
    long long* c0 = c0_ - lo;
    long long* c1 = c1_ - lo;
    void* c2 = c2_ ? (void*)((uint8_t*)c2_ - lo * (table == 5 ? 16 : 8)) : nullptr;
    switch (table) {
      case 2:  // customer
        c0[i] = (long long)i + 1;
        c1[i] = (long long)U(S.s[0], i, 25);
        ((long long*)c2)[i] = (long long)U(S.s[1], i, 5);
        break;
      case 3:  // supplier
        c0[i] = (long long)i + 1;
        c1[i] = (long long)U(S.s[0], i, 25);
        break;
      case 4:  // part
        c0[i] = (long long)i + 1;
        c1[i] = (long long)U(S.s[0], i, 1000);
        break;
      case 5: {  // partsupp
        long long p = (long long)(i / 4) + 1;
        c0[i] = p;
        c1[i] = ps_supp(p, (long long)(i % 4), (long long)ns);
        ((ulonglong2*)c2)[i] = make_ulonglong2(100 + U(S.s[0], i, 99901), 0);
        break;
      }
      case 6: {  // nation
        const long long reg[25] = {0, 1, 1, 1, 4, 0, 3, 3, 2, 2, 4, 4, 2, 4, 0, 0, 0, 1, 2, 3, 4, 2, 3, 3, 1};
        c0[i] = (long long)i;
        c1[i] = reg[i];
        break;
      }
      default:  // region
        c0[i] = (long long)i;
        c1[i] = (long long)i;
    }
  }
}

static uint64_t scaled(double base, double sf, uint64_t minimum) {
  double v = (double)std::llround(base * sf);
  return std::max<uint64_t>(minimum, (uint64_t)v);
}

static tq_column colspec(uint8_t kind, uint8_t prec = 0, uint8_t scale = 0) {
  tq_column c{};
  c.kind = kind;
  c.precision = prec;
  c.scale = scale;
  return c;
}

void datagen(tq_ctx* c, int table, double sf, uint32_t shard, uint32_t nshards, tq_batch* out, cudaStream_t st) {
  if (nshards == 0 || shard >= nshards) fail(TQ_INVALID_PLAN, "bad shard");
  uint64_t nc = scaled(150000, sf, 1), ns = scaled(10000, sf, 4), np = scaled(200000, sf, 1),
           no = scaled(1500000, sf, 1);
  auto range = [&](uint64_t n, uint64_t& lo, uint64_t& hi) {
    lo = n * shard / nshards;
    hi = n * (shard + 1) / nshards;
  };
  u32 grid = (u32)c->sms * 8;
  Seeds S{};
  auto I64 = colspec(TQ_INT64);
  auto DEC = colspec(TQ_DECIMAL, 11, 2);
  auto L = [&](int i) { return (long long*)out->cols[i].values; };
  uint64_t lo, hi;
  switch (table) {
    case 0: {
      range(no, lo, hi);
      alloc_batch(c, hi - lo, {I64, I64, I64, I64, I64}, std::vector<bool>(5, false), out, st);
      S.s[0] = col_seed("orders.o_custkey");
      S.s[1] = col_seed("orders.o_orderdate");
      if (hi > lo) k_orders<<<grid, 256, 0, st>>>(lo, hi - lo, nc, S, L(0), L(1), L(2), L(3), L(4));
      counted_launch(c);
      break;
    }
    case 1: {
      range(no, lo, hi);
      u32* nl = (u32*)dalloc(c, no * 4, st);
      u64* off = (u64*)dalloc(c, (no + 1) * 8, st);
      k_nlines<<<grid, 256, 0, st>>>(no, col_seed("orders.o_nlines"), nl);
      counted_launch(c);
      extern void scan_u32_public(tq_ctx*, const u32*, u64, u64*, u64*, cudaStream_t);
      scan_u32_public(c, nl, no, off, off + no, st);
      uint64_t r01[2] = {0, 0};
      TQ_CUDA(cudaMemcpyAsync(&r01[0], off + lo, 8, cudaMemcpyDeviceToHost, st));
      TQ_CUDA(cudaMemcpyAsync(&r01[1], off + hi, 8, cudaMemcpyDeviceToHost, st));
      TQ_CUDA(cudaStreamSynchronize(st));
      uint64_t rows = r01[1] - r01[0];
      try {
        alloc_batch(c, rows, {I64, I64, I64, DEC, DEC, DEC, DEC, I64, I64, I64}, std::vector<bool>(10, false), out,
                    st);
      } catch (...) {
        dfree(c, nl, no * 4, st);
        dfree(c, off, (no + 1) * 8, st);
        throw;
      }
      S.s[0] = col_seed("orders.o_orderdate");
      S.s[1] = col_seed("lineitem.l_partkey");
      S.s[2] = col_seed("lineitem.l_suppkey");
      S.s[3] = col_seed("lineitem.l_quantity");
      S.s[4] = col_seed("lineitem.l_discount");
      S.s[5] = col_seed("lineitem.l_tax");
      S.s[6] = col_seed("lineitem.l_receiptdate");
      S.s[7] = col_seed("lineitem.l_returnflag");
      S.s[8] = col_seed("lineitem.l_shipdate");
      LiOut o;
      o.ok = L(0); o.pk = L(1); o.sk = L(2);
      o.qty = (ulonglong2*)out->cols[3].values;
      o.ep = (ulonglong2*)out->cols[4].values;
      o.disc = (ulonglong2*)out->cols[5].values;
      o.tax = (ulonglong2*)out->cols[6].values;
      o.rf = L(7); o.ls = L(8); o.sd = L(9);
      if (hi > lo) k_lineitem<<<grid, 256, 0, st>>>(lo, hi - lo, off, np, ns, S, o);
      counted_launch(c);
      dfree(c, nl, no * 4, st);
      dfree(c, off, (no + 1) * 8, st);
      break;
    }
    default: {
      uint64_t n;
      std::vector<tq_column> sch;
      switch (table) {
        case 2: n = nc; sch = {I64, I64, I64}; S.s[0] = col_seed("customer.c_nationkey"); S.s[1] = col_seed("customer.c_mktsegment"); break;
        case 3: n = ns; sch = {I64, I64}; S.s[0] = col_seed("supplier.s_nationkey"); break;
        case 4: n = np; sch = {I64, I64}; S.s[0] = col_seed("part.p_color"); break;
        case 5: n = 4 * np; sch = {I64, I64, DEC}; S.s[0] = col_seed("partsupp.ps_supplycost"); break;
        case 6: n = 25; sch = {I64, I64}; break;
        case 7: n = 5; sch = {I64, I64}; break;
        default: fail(TQ_INVALID_PLAN, "unknown table");
      }
      range(n, lo, hi);
      alloc_batch(c, hi - lo, sch, std::vector<bool>(sch.size(), false), out, st);
      if (hi > lo)
        k_simple<<<grid, 256, 0, st>>>(table, lo, hi - lo, ns, S, L(0), L(1), sch.size() > 2 ? out->cols[2].values : nullptr);
      counted_launch(c);
    }
  }
  TQ_CUDA(cudaGetLastError());
}

}  // namespace tq

extern "C" tq_status tq_datagen(tq_ctx* c, int table, double sf, tq_batch* out, void* stream) {
  return tq::guard([&] { tq::datagen(c, table, sf, 0, 1, out, tq::pick(c, stream)); });
}
extern "C" tq_status tq_datagen_shard(tq_ctx* c, int table, double sf, uint32_t shard, uint32_t nshards,
                                      tq_batch* out, void* stream) {
  return tq::guard([&] { tq::datagen(c, table, sf, shard, nshards, out, tq::pick(c, stream)); });
}
