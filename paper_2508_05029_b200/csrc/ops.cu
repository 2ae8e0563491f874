// ops.cu — host orchestration of the operators on top of
// the pipeline kernels, plus the small helper kernels: tile-count scan,
// aggregation-table init/finalize, take / concat / slice.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ctx.h"
#include "device.cuh"
#include "pipeline.h"
#include "program.h"
#include "peer.h"

struct tq_join_table {
  tq_ctx* ctx;
  tq::JoinTable jt;
  uint8_t* mem = nullptr;  // the allocation: [entries (none when semi-only) | Bloom | flags | exact bitmap]
  // semi-only table (no entries): how to build the real table if a probe finds
  // the bitmap was not exact / the keys not unique
  std::shared_ptr<void> semi_prog;  // Prog
  std::vector<uint32_t> semi_keys;
  uint64_t semi_bloom_keys = 0;
  // the agreed row count the Bloom filter was sized from (tq_join_build_sized /
  // tq_pipeline_build_ex; 0 = the table's own rows): the partitioned LIP
  // all-gather needs every rank's filter sized from the same count
  uint64_t bloom_keys = 0;
  uint64_t bytes;
  cudaStream_t stream;
  tq_batch build;                      // borrowed descriptors (cols copied)
  std::vector<uint8_t> key_cls, key_scale;
  // a semi-only table is materialised at most once, under this lock; the
  // replaced allocation may still be read by another probe's kernel on another
  // stream, so it is retired and freed with the table
  std::mutex mu;
  std::vector<std::pair<uint8_t*, uint64_t>> retired;
  // Utf8 build columns (tq_join_build): the table is built over a lowered copy
  // of the batch — Utf8 keys as the fnv1a64 of their bytes, Utf8 payloads as row
  // ids, plus a row-id column — whose buffers it owns; the probe compares the
  // key strings of every candidate pair and gathers the output strings.
  bool utf8 = false;
  std::vector<tq_column> orig_cols;  // the caller's build columns (descriptors)
  uint64_t orig_rows = 0;
  std::vector<uint8_t> key_utf8;     // per key: a Utf8 key
  std::vector<uint32_t> key_cols;    // per key: its build column
  std::vector<std::pair<void*, uint64_t>> own;
};

namespace tq {

cudaError_t launch_pipeline_prog(tq_ctx* c, int sink, const PipeParams& p, u32 smem, u32 grid, cudaStream_t st,
                                 const std::vector<DInstr>& code, const std::vector<DLit>& lits);

// ================================================================== scan
constexpr int kScanItems = 8;
// partitioned LIP filter (tq_join_build_sized / tq_comm_gather_table_blooms):
// bits per key of the most rows any rank received; 16 measured best at SF100
// N=2 (8: more false positives shipped and probed, 32+: the gathered filter
// falls out of L2)
constexpr uint64_t kLipBloomBitsPerKey = 16;
constexpr int kScanBlock = 256 * kScanItems;

__device__ __forceinline__ u64 block_excl_scan(u64 v, u64* s_warp, u64& total) {
  u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u64 incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u64 y = __shfl_up_sync(kFull, incl, o);
    if (lane >= (u32)o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    u64 x = lane < 8 ? s_warp[lane] : 0;
    u64 xi = x;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      u64 y = __shfl_up_sync(kFull, xi, o);
      if (lane >= (u32)o) xi += y;
    }
    if (lane < 8) s_warp[8 + lane] = xi - x;
    if (lane == 7) s_warp[16] = xi;
  }
  __syncthreads();
  total = s_warp[16];
  u64 r = s_warp[8 + warp] + incl - v;
  __syncthreads();
  return r;
}

// a thread's kScanItems (8) consecutive counts: two 16-B loads when whole and
// aligned (the scans of a 15M-slice partition count are bandwidth-bound)
__device__ __forceinline__ void scan_load8(const u32* in, u64 n, u64 base, u32* v) {
  static_assert(kScanItems == 8, "two uint4 per thread");
  if (base + 8 <= n && ((uintptr_t)(in + base) & 15) == 0) {
    const uint4 a = __ldg((const uint4*)(in + base)), b = __ldg((const uint4*)(in + base) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = base + i < n ? in[base + i] : 0;
  }
}

__global__ void k_scan_partials(const u32* in, u64 n, u64* partial) {
  __shared__ u64 s[24];
  u64 base = (u64)blockIdx.x * kScanBlock + threadIdx.x * kScanItems;
  u64 sum = 0;
  u32 v[kScanItems];
  scan_load8(in, n, base, v);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) sum += v[i];
  u64 tot;
  block_excl_scan(sum, s, tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void k_scan_prefix(u64* partial, u64 nb, u64* total) {
  __shared__ u64 s[24];
  u64 carry = 0;
  for (u64 b0 = 0; b0 < nb; b0 += 256) {
    u64 i = b0 + threadIdx.x;
    u64 v = i < nb ? partial[i] : 0;
    u64 tot;
    u64 ex = block_excl_scan(v, s, tot);
    if (i < nb) partial[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void k_scan_apply(const u32* in, u64 n, const u64* partial, u64* out) {
  __shared__ u64 s[24];
  u64 base = (u64)blockIdx.x * kScanBlock + threadIdx.x * kScanItems;
  u32 v[kScanItems];
  u64 sum = 0;
  scan_load8(in, n, base, v);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) sum += v[i];
  u64 tot;
  u64 run = partial[blockIdx.x] + block_excl_scan(sum, s, tot);
  if (base + 8 <= n && ((uintptr_t)(out + base) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < kScanItems; i += 2) {
      *(ulonglong2*)(out + base + i) = make_ulonglong2(run, run + v[i]);
      run += v[i] + v[i + 1];
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) {
      out[base + i] = run;
      run += v[i];
    }
}

// exclusive scan of n u32 -> u64; *total_dev = sum
static void scan_u32(tq_ctx* c, const u32* in, u64 n, u64* out, u64* total_dev, cudaStream_t st) {
  u64 nb = (n + kScanBlock - 1) / kScanBlock;
  if (nb == 0) nb = 1;
  u64* partial = (u64*)dalloc(c, nb * 8, st);
  const int ph = prof_begin(c, "scan", st);
  k_scan_partials<<<(u32)nb, 256, 0, st>>>(in, n, partial);
  k_scan_prefix<<<1, 256, 0, st>>>(partial, nb, total_dev);
  k_scan_apply<<<(u32)nb, 256, 0, st>>>(in, n, partial, out);
  prof_end(c, ph, st);
  for (int i = 0; i < 3; ++i) counted_launch(c);
  TQ_CUDA(cudaGetLastError());
  dfree(c, partial, nb * 8, st);
}

__global__ void k_set_u64_one(u64* p, u64 v) { *p = v; }
static void k_set_u64_ext(u64* p, u64 v, cudaStream_t st) {
  k_set_u64_one<<<1, 1, 0, st>>>(p, v);
}

// offsets[d*ntiles] for each dest + total -> pinned[0..ndest]
__global__ void k_dest_starts(const u64* offsets, u32 nslices, u32 ndest, const u64* total, u64* pinned) {
  u32 d = threadIdx.x;
  if (d < ndest) pinned[d] = offsets[(u64)d * nslices];
  if (d == 0) pinned[ndest] = *total;
}

// ================================================================== program setup
struct Prog {
  ProgramBuilder pb;
  bool has_pred = false;
  int pred_h = -1;
  std::vector<int> outs;  // root handles of projected columns
  explicit Prog(std::vector<ColumnDesc> s) : pb(std::move(s)) {}
};

static std::vector<ColumnDesc> schema_of(const tq_batch* in) {
  std::vector<ColumnDesc> s;
  for (uint32_t i = 0; i < in->ncols; ++i)
    s.push_back({in->cols[i].kind, in->cols[i].precision, in->cols[i].scale,
                 in->rows > 0 && in->cols[i].validity != nullptr});
  return s;
}

static void check_device_batch(const tq_batch* b) {
  if (!b || b->mem != TQ_MEM_DEVICE) fail(TQ_INTERNAL, "expected a device batch");
  for (uint32_t i = 0; i < b->ncols; ++i) {
    const tq_column& c = b->cols[i];
    if (c.kind > TQ_DECIMAL) fail(TQ_MALFORMED_BATCH, "bad column kind");
    if (c.kind != TQ_UTF8 && c.values_bytes != b->rows * width_of(c.kind))
      fail(TQ_MALFORMED_BATCH, "values length mismatch");
  }
}

// pred may be null; exprs==null && all_cols -> every input column passes through
static void compile_prog(Prog& P, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs, uint32_t nexprs,
                         bool all_cols) {
  TQ_HT("compile_prog");
  try {
    if (pred) {
      P.pred_h = P.pb.add_root(*pred);
      P.has_pred = true;
      P.pb.end_predicate();
    }
    if (exprs)
      for (uint32_t i = 0; i < nexprs; ++i) P.outs.push_back(P.pb.add_root(exprs[i]));
    else if (all_cols)
      for (uint32_t i = 0; i < in->ncols; ++i) P.outs.push_back(P.pb.add_column(i));
    P.pb.finish();
    if (P.has_pred && P.pb.root(P.pred_h).cls != C_B) fail(TQ_INVALID_PLAN, "predicate must be boolean");
  } catch (const CompileError& e) {
    fail(e.status, e.msg);
  }
}

static const void* upload_program(tq_ctx* c, const ProgramBuilder& pb, const DInstr** code, const DLit** lits) {
  std::string key;
  key.append((const char*)pb.code().data(), pb.code().size() * sizeof(DInstr));
  key.push_back('|');
  key.append((const char*)pb.lits().data(), pb.lits().size() * sizeof(DLit));
  std::lock_guard<std::mutex> g(c->mu);
  auto it = c->prog_cache.find(key);
  void* d;
  if (it != c->prog_cache.end()) {
    d = it->second;
  } else {
    size_t cb = pb.code().size() * sizeof(DInstr);
    size_t bytes = round_up(cb, 32) + pb.lits().size() * sizeof(DLit) + 32;
    TQ_CUDA(cudaMalloc(&d, bytes));
    std::vector<uint8_t> h(bytes, 0);
    std::memcpy(h.data(), pb.code().data(), cb);
    std::memcpy(h.data() + round_up(cb, 32), pb.lits().data(), pb.lits().size() * sizeof(DLit));
    TQ_CUDA(cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice));
    c->prog_cache[key] = d;
  }
  *code = (const DInstr*)d;
  *lits = (const DLit*)((uint8_t*)d + round_up(pb.code().size() * sizeof(DInstr), 32));
  return d;
}

static uint8_t out_kind_of(const Operand& o, const tq_batch* in, const ProgramBuilder& pb, uint8_t* prec,
                           uint8_t* scale) {
  *prec = 0;
  *scale = 0;
  switch (o.kind) {
    case K_COL_I64: return TQ_INT64;
    case K_COL_F64: return TQ_FLOAT64;
    case K_COL_BOOL: return TQ_BOOL;
    case K_COL_DEC: {
      const tq_column& c = in->cols[pb.staged()[o.idx]];
      *prec = c.precision;
      *scale = c.scale;
      return TQ_DECIMAL;
    }
    default: break;
  }
  switch (o.cls) {
    case C_I: return TQ_INT64;
    case C_D: *prec = 38; *scale = o.scale; return TQ_DECIMAL;
    case C_F: return TQ_FLOAT64;
    default: return TQ_BOOL;
  }
}

// Fill program + staging part of PipeParams and the smem layout.
struct Plan {
  PipeParams p;
  u32 smem = 0, grid = 0;
};

static u32 align_up(u32 x, u32 a) { return (x + a - 1) / a * a; }

static void plan_launch(tq_ctx* c, const tq_batch* in, Prog& P, Plan& L, u32 sink_bytes, cudaStream_t st) {
  TQ_HT("plan_launch");
  PipeParams& p = L.p;
  std::memset(&p, 0, sizeof(p));
  const ProgramBuilder& pb = P.pb;
  upload_program(c, pb, &p.code, &p.lits);
  p.rows = in->rows;
  p.ntiles = (u32)((in->rows + kTile - 1) / kTile);
  p.ncode = (uint16_t)pb.code().size();
  p.npred = (uint16_t)pb.n_pred_instr();
  p.nlits = (uint16_t)pb.lits().size();
  p.nvslots = (uint16_t)std::max(1, pb.value_slots());
  p.nbslots = (uint16_t)std::max(1, pb.bool_slots());
  p.pred_kind = K_NONE;
  if (P.has_pred) {
    p.pred_kind = pb.root(P.pred_h).kind;
    p.pred_idx = pb.root(P.pred_h).idx;
  }
  // staged columns and per-stage layout
  p.nstaged = (uint16_t)pb.staged().size();
  u32 off = 0;
  for (u32 i = 0; i < p.nstaged; ++i) {
    const tq_column& col = in->cols[pb.staged()[i]];
    StagedCol& sc = p.cols[i];
    sc.values = (const uint8_t*)col.values;
    sc.validity = in->rows > 0 ? col.validity : nullptr;
    sc.width = (u32)width_of(col.kind);
    sc.kind = col.kind;
    sc.bulk_ok = ((uintptr_t)col.values % 16 == 0) && (!sc.validity || (uintptr_t)sc.validity % 16 == 0);
    off = align_up(off, 128);
    sc.off = off;
    off += kTile * sc.width;
    if (sc.validity) {
      off = align_up(off, 16);
      sc.voff = off;
      off += kTile / 8;
    }
  }
  p.stage_bytes = align_up(std::max(off, 128u), 128);
  p.all_bulk = 1;
  for (u32 i = 0; i < p.nstaged; ++i) p.all_bulk &= p.cols[i].bulk_ok;
  p.load_mask = p.nstaged >= 32 ? 0xffffffffu : (1u << p.nstaged) - 1;
  // fixed regions
  u32 o = 0;
  p.off_code = o;
  o += align_up(p.ncode * sizeof(DInstr), 128);
  p.off_lits = o;
  o += align_up(std::max<u32>(1, p.nlits) * sizeof(DLit), 128);
  p.off_vslot = o;
  o += kWarps * p.nvslots * kV * 32 * 16;
  p.off_vvalid = o;
  o += align_up(kWarps * p.nvslots * kV * 4, 16);
  p.off_bslot = o;
  o += align_up(kWarps * p.nbslots * kV * 8, 16);
  p.off_sink = o;
  o += align_up(sink_bytes, 128);
  p.off_bar = o;
  o += 2 * kMaxStages * 8 + 8;  // full / empty barriers + the AGG sink's per-CTA new-group count
  o = align_up(o, 128);
  const u32 kSmemMax = 227 * 1024;
  if (o + p.stage_bytes > kSmemMax) fail(TQ_INVALID_PLAN, "batch too wide for one pipeline tile");
  u32 budget = kSmemMax - o;
  // two CTAs per SM when both fit with >= 2 stages, else one CTA with up to 4 stages
  u32 per_sm = c->ctas_per_sm;
  u32 half = 113 * 1024;
  if (per_sm == 0) per_sm = (o < half && (half - o) / p.stage_bytes >= 2) ? 2 : 1;
  u32 limit = per_sm >= 2 ? (half > o ? half - o : 0) : budget;
  static const u32 max_stages = [] {  // TQ_MAXSTAGES: experiments only
    const char* e = getenv("TQ_MAXSTAGES");
    return e ? (u32)std::max(1, std::min(atoi(e), kMaxStages)) : (u32)kMaxStages;
  }();
  u32 ns = std::min<u32>(max_stages, limit / p.stage_bytes);
  if (ns == 0) { per_sm = 1; ns = std::min<u32>(kMaxStages, budget / p.stage_bytes); }
  if (ns == 0) fail(TQ_INVALID_PLAN, "batch too wide for one pipeline tile");
  p.nstages = ns;
  {  // L2 prefetch distance (tiles beyond the ring); TQ_PF overrides
    static const int pf_env = [] {
      const char* e = getenv("TQ_PF");
      return e ? atoi(e) : -1;
    }();
    p.pf_dist = pf_env >= 0 ? (u32)pf_env : 0;  // measured slower when on (TMA queue contention)
  }
  p.off_stage = o;
  L.smem = o + ns * p.stage_bytes;
  L.grid = std::max<u32>(1, std::min<u32>(p.ntiles, (u32)c->sms * per_sm));
  (void)st;
}

static void launch(tq_ctx* c, int sink, Plan& L, const Prog& P, cudaStream_t st) {
  TQ_HT("launch(pipeline)");
  if (L.p.ntiles == 0) return;
  static const char* names[] = {"pipe_count", "pipe_emit", "pipe_agg", "pipe_build"};
  const char* nm = names[sink];
  if (sink == SINK_EMIT && L.p.dest_kind == DEST_PEER) nm = L.p.bcast ? "pipe_broadcast" : "pipe_scatter";
  else if (sink == SINK_EMIT && L.p.dest_kind == DEST_PROBE1) nm = "pipe_probe1";
  int h = prof_begin(c, nm, st);
  TQ_CUDA(launch_pipeline_prog(c, sink, L.p, L.smem, L.grid, st, P.pb.code(), P.pb.lits()));
  prof_end(c, h, st);
  counted_launch(c);
}

// COUNT pass of a two-pass FILTER / PARTITION: the generated predicate / keys
// over plain coalesced loads (count_direct_body) instead of the stage ring;
// falls back to the pipeline's COUNT sink when there is no generated code.
// TQ_COUNT_DIRECT=0: always the pipeline (A/B measurements).
static void launch_count(tq_ctx* c, Plan& L, const Prog& P, cudaStream_t st) {
  static const bool on = [] {
    const char* e = getenv("TQ_COUNT_DIRECT");
    return !(e && e[0] == '0');
  }();
  if (L.p.ntiles == 0) return;
  if (on && kV == 1 &&
      (L.p.dest_kind == DEST_FILTER || L.p.dest_kind == DEST_PARTITION || L.p.dest_kind == DEST_PROBE)) {
    TQ_HT("launch(count_direct)");
    int h = prof_begin(c, "count_direct", st);
    const int mode = L.p.dest_kind == DEST_FILTER  ? CD_FILTER
                     : L.p.dest_kind == DEST_PROBE ? CD_PROBE
                     : L.p.ndest > 32             ? CD_PART_MANY
                     : L.p.semi_bloom             ? CD_PART_FEW_LIP
                                                  : CD_PART_FEW;
    const cudaError_t e = launch_pipeline_prog(c, SINK_COUNT_DIRECT + mode, L.p, 0, (u32)c->sms * 8, st,
                                               P.pb.code(), P.pb.lits());
    prof_end(c, h, st);
    if (e == cudaSuccess) {
      counted_launch(c);
      return;
    }
    if (e != cudaErrorNotSupported) TQ_CUDA(e);
  }
  launch(c, SINK_COUNT, L, P, st);
}

static void set_keys(PipeParams& p, const ProgramBuilder& pb, const std::vector<int>& handles) {
  if (handles.size() > (size_t)kMaxKeys) fail(TQ_INVALID_PLAN, "too many keys");
  p.nkeys = (u32)handles.size();
  u32 words = 0;
  for (size_t i = 0; i < handles.size(); ++i) {
    const Operand& o = pb.root(handles[i]);
    KeyOpnd& k = p.keys[i];
    k.kind = o.kind;
    k.idx = o.idx;
    k.words = o.cls == C_D ? 2 : 1;
    k.bytes = o.cls == C_D ? 16 : o.cls == C_B ? 1 : 8;
    words += k.words;
  }
  if (words > (u32)kMaxKeyWords) fail(TQ_INVALID_PLAN, "keys too wide");
  p.key_words = words;
}

// ================================================================== materializing sinks
enum MatMode { MAT_FILTER, MAT_PARTITION, MAT_PROBE };

struct tq_bloom_impl;
struct MatArgs {
  const uint32_t* semi_words = nullptr;  // LIP Bloom filter on the partition keys
  uint64_t semi_mask = 0;
  uint64_t semi_part_words = 0;  // partitioned filter: part d at d * semi_part_words
  int mode = MAT_FILTER;
  std::vector<uint32_t> key_roots;  // indices into P.outs
  uint32_t nparts = 1;
  const tq_join_table* table = nullptr;
  std::vector<uint32_t> build_cols;
  bool prehashed = false;  // the one key is the row's partition hash (Utf8 keys)
  // asynchronous form (tq_filter_async / tq_hash_partition_async): no host sync;
  // the output is allocated at the input's row count and the part starts + total
  // (ndest + 1 values) land in this caller-owned pinned slot, valid once the
  // stream reaches the end of the call
  uint64_t* async_slot = nullptr;
};

// ---- closing the holes of DEST_PROBE1's chunked output (kernel_common.cuh,
// chunk_reserve).  Rows were written to [0, R) in kChunk-row chunks; each CTA's
// last chunk may be partly unused, so n = R - holes rows exist.  The used rows
// at positions >= n are moved into the holes below n (any bijection will do:
// join output order is unspecified), then bitmap bits >= n are cleared.
struct ChunkOut {
  uint8_t* values[kMaxOut];
  uint8_t* validity[kMaxOut];
  uint32_t width[kMaxOut];
  uint32_t ncols;
};
// plan: [0] n, [1] moves, [2] hole ranges, [3] source ranges, then
// hole start[nh], hole prefix[nh + 1], source start[ns], source prefix[ns + 1]
//
// Block-wide exclusive scan of (count, length) pairs over 1024 threads;
// returns the exclusive prefixes and leaves the block totals in *tc / *tl.
__device__ __forceinline__ void block_scan2(u32 c, u64 l, u32& ec, u64& el, u32* tc, u64* tl) {
  __shared__ u32 wc[32];
  __shared__ u64 wl[32];
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 ic = c;
  u64 il = l;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 yc = __shfl_up_sync(0xffffffffu, ic, o);
    const u64 yl = __shfl_up_sync(0xffffffffu, il, o);
    if (lane >= (u32)o) { ic += yc; il += yl; }
  }
  if (lane == 31) { wc[warp] = ic; wl[warp] = il; }
  __syncthreads();
  if (warp == 0) {
    const u32 nw = blockDim.x >> 5;
    u32 xc = lane < nw ? wc[lane] : 0;
    u64 xl = lane < nw ? wl[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 yc = __shfl_up_sync(0xffffffffu, xc, o);
      const u64 yl = __shfl_up_sync(0xffffffffu, xl, o);
      if (lane >= (u32)o) { xc += yc; xl += yl; }
    }
    if (lane < nw) { wc[lane] = xc; wl[lane] = xl; }
    if (lane == nw - 1) { *tc = xc; *tl = xl; }
  }
  __syncthreads();
  ec = ic - c + (warp ? wc[warp - 1] : 0);
  el = il - l + (warp ? wl[warp - 1] : 0);
  __syncthreads();
}

// One block; every loop is a parallel pass (a serial single-thread plan cost
// ~45 us for 296 CTAs).  Ranges are listed in CTA / chunk order.
__global__ void k_chunk_plan(const u64* tails, u32 nctas, const u64* gcursor, u64* plan) {
  extern __shared__ u64 sm_chunk[];
  u64* tb = sm_chunk;          // [nctas] last-chunk base
  u64* tu = tb + nctas;        // [nctas] used rows
  u64* uj = tu + nctas;        // [nctas + 2] used rows of the chunks at/after floor(n / kChunk)
  __shared__ unsigned long long holes_total;
  __shared__ u32 tot_c;
  __shared__ u64 tot_l;
  if (threadIdx.x == 0) holes_total = 0;
  __syncthreads();
  unsigned long long my_holes = 0;
  for (u32 i = threadIdx.x; i < nctas; i += blockDim.x) {
    tb[i] = tails[2 * i];
    tu[i] = tails[2 * i + 1];
    if (tu[i] < (u64)kChunk) my_holes += kChunk - tu[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) my_holes += __shfl_xor_sync(0xffffffffu, my_holes, o);
  if ((threadIdx.x & 31) == 0 && my_holes) atomicAdd(&holes_total, my_holes);
  __syncthreads();
  const u64 R = *gcursor, n = R - holes_total;
  const u64 j0 = n / kChunk, nj = R / kChunk - j0;
  for (u64 i = threadIdx.x; i < nj; i += blockDim.x) uj[i] = kChunk;
  __syncthreads();
  for (u32 i = threadIdx.x; i < nctas; i += blockDim.x)
    if (tu[i] < (u64)kChunk && tb[i] >= j0 * kChunk) uj[tb[i] / kChunk - j0] = tu[i];
  __syncthreads();
  u64* hs = plan + 4;
  u64* hp = hs + nctas;
  u64* ss = hp + nctas + 1;
  u64* sp = ss + nctas + 2;
  // holes: the unused tail of every partly used chunk below n
  u32 nh = 0;
  u64 tot = 0;
  for (u32 base = 0; base < nctas; base += blockDim.x) {
    const u32 i = base + threadIdx.x;
    u64 a = 0, len = 0;
    if (i < nctas && tu[i] < (u64)kChunk && tb[i] < n) {
      a = tb[i] + tu[i];
      const u64 e = min(tb[i] + (u64)kChunk, n);
      len = a < e ? e - a : 0;
    }
    u32 ec;
    u64 el;
    block_scan2(len ? 1u : 0u, len, ec, el, &tot_c, &tot_l);
    if (len) {
      hs[nh + ec] = a;
      hp[nh + ec + 1] = tot + el + len;
    }
    nh += tot_c;
    tot += tot_l;
    __syncthreads();
  }
  // sources: the used rows at/after n
  u32 ns = 0;
  u64 tot2 = 0;
  for (u64 base = 0; base < nj; base += blockDim.x) {
    const u64 j = base + threadIdx.x;
    u64 a = 0, len = 0;
    if (j < nj) {
      const u64 s0 = (j0 + j) * kChunk, e = s0 + uj[j];
      a = max(s0, n);
      len = a < e ? e - a : 0;
    }
    u32 ec;
    u64 el;
    block_scan2(len ? 1u : 0u, len, ec, el, &tot_c, &tot_l);
    if (len) {
      ss[ns + ec] = a;
      sp[ns + ec + 1] = tot2 + el + len;
    }
    ns += tot_c;
    tot2 += tot_l;
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  hp[0] = 0;
  sp[0] = 0;
  plan[0] = n;
  plan[1] = tot == tot2 ? tot : ~0ull;  // (equal by construction)
  plan[2] = nh;
  plan[3] = ns;
}

__device__ __forceinline__ u64 range_at(const u64* start, const u64* pref, u64 nr, u64 k) {
  u64 lo = 0, hi = nr;  // last range with pref <= k
  while (hi - lo > 1) {
    const u64 mid = (lo + hi) / 2;
    if (pref[mid] <= k) lo = mid;
    else hi = mid;
  }
  return start[lo] + (k - pref[lo]);
}

__global__ void k_chunk_move(const u64* plan, u32 nctas, const __grid_constant__ ChunkOut o) {
  const u64 moves = plan[1];
  if (moves == ~0ull) return;
  const u64 nh = plan[2], ns = plan[3];
  const u64* hs = plan + 4;
  const u64* hp = hs + nctas;
  const u64* ss = hp + nctas + 1;
  const u64* sp = ss + nctas + 2;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < moves; k += (u64)gridDim.x * blockDim.x) {
    const u64 dst = range_at(hs, hp, nh, k), src = range_at(ss, sp, ns, k);
    for (u32 c = 0; c < o.ncols; ++c) {
      const u32 w = o.width[c];
      if (w == 16) ((ulonglong2*)o.values[c])[dst] = ((const ulonglong2*)o.values[c])[src];
      else if (w == 8) ((u64*)o.values[c])[dst] = ((const u64*)o.values[c])[src];
      else o.values[c][dst] = o.values[c][src];
      if (o.validity[c] && bm_get(o.validity[c], src)) bm_set_atomic(o.validity[c], dst);
    }
  }
}

__global__ void k_chunk_clear_tail(const u64* plan, const __grid_constant__ ChunkOut o) {
  const u64 n = plan[0];
  const u32 c = threadIdx.x;
  if (c >= o.ncols || !o.validity[c] || (n & 7) == 0) return;
  o.validity[c][n >> 3] &= (uint8_t)((1u << (n & 7)) - 1);
}

static void run_build(tq_ctx* c, const tq_batch* in, Prog& P, const std::vector<uint32_t>& key_roots,
                      tq_join_table** out, cudaStream_t st, uint64_t bloom_keys, bool semi_only,
                      bool allow_direct = true);

// A semi-only table whose bitmap turned out not exact (or keys not unique):
// build the real hash table from the same input and program, in place.
static void semi_table_materialize(tq_ctx* c, tq_join_table* t, cudaStream_t st) {
  std::lock_guard<std::mutex> g(t->mu);
  if (t->jt.entries != nullptr) return;  // another probe materialised it first
  if (host_timing_on()) {
    uint32_t f[2] = {0, 0};
    if (t->jt.dup_dev) cudaMemcpy(&f[0], t->jt.dup_dev, 4, cudaMemcpyDeviceToHost);
    if (t->jt.exact_flag) cudaMemcpy(&f[1], t->jt.exact_flag, 4, cudaMemcpyDeviceToHost);
    fprintf(stderr, "[tq] materialise %s table: %llu rows, dup %u, not-exact %u, range %llu\n",
            t->jt.direct ? "direct" : "semi", (unsigned long long)t->build.rows, f[0], f[1],
            (unsigned long long)t->jt.exact_range);
  }
  tq_join_table* full = nullptr;
  Prog& P = *(Prog*)t->semi_prog.get();
  run_build(c, &t->build, P, t->semi_keys, &full, st, t->semi_bloom_keys, false, /*allow_direct=*/false);
  t->retired.emplace_back(t->mem, t->bytes);
  std::free(t->build.cols);
  t->jt = full->jt;
  t->mem = full->mem;
  t->bytes = full->bytes;
  t->build = full->build;
  t->semi_prog.reset();
  full->build.cols = nullptr;
  delete full;
}

static void run_materialize(tq_ctx* c, const tq_batch* in, Prog& P, const MatArgs& A, tq_batch* out,
                            uint64_t* part_offsets, cudaStream_t st) {
  Plan L;
  u32 sink_bytes = kWarps * kMaxDest * 4 + kWarps * kMaxDest * 8;
  plan_launch(c, in, P, L, sink_bytes, st);
  PipeParams& p = L.p;
  p.dest_kind = A.mode == MAT_FILTER ? DEST_FILTER : A.mode == MAT_PARTITION ? DEST_PARTITION : DEST_PROBE;
  p.ndest = A.mode == MAT_PARTITION ? A.nparts : 1;
  if (p.ndest == 0 || p.ndest > (u32)kMaxDest) fail(TQ_INVALID_PLAN, "partition count out of range (1..64)");
  std::vector<int> kh;
  for (uint32_t k : A.key_roots) {
    if (k >= P.outs.size()) fail(TQ_INVALID_PLAN, "key column out of range");
    kh.push_back(P.outs[k]);
  }
  set_keys(p, P.pb, kh);
  p.key_prehashed = A.prehashed ? 1u : 0u;
  p.semi_bloom = A.semi_words;
  p.semi_mask = A.semi_mask;
  p.semi_part_words = A.semi_part_words;
  if (A.mode == MAT_PROBE) {
    const tq_join_table* t = A.table;
    if (kh.size() != t->key_cls.size()) fail(TQ_INVALID_PLAN, "probe/build key count differs");
    for (size_t i = 0; i < kh.size(); ++i) {
      const Operand& o = P.pb.root(kh[i]);
      if (o.cls != t->key_cls[i] || (o.cls == C_D && o.scale != t->key_scale[i]))
        fail(TQ_INVALID_PLAN, "join key types differ");
    }
    p.jt = t->jt;
    p.probe_semi = A.build_cols.empty() ? 1u : 0u;
  }
  // output schema
  std::vector<tq_column> sch;
  std::vector<bool> wv;
  std::vector<OutCol> outs;
  if (A.mode == MAT_PROBE) {
    for (uint32_t bc : A.build_cols) {
      if (bc >= A.table->build.ncols) fail(TQ_INVALID_PLAN, "build column out of range");
      const tq_column& col = A.table->build.cols[bc];
      if (col.kind == TQ_UTF8) fail(TQ_INVALID_PLAN, "utf8 columns are not supported on the GPU path");
      tq_column d{};
      d.kind = col.kind; d.precision = col.precision; d.scale = col.scale;
      sch.push_back(d);
      wv.push_back(col.validity != nullptr && A.table->build.rows > 0);
      OutCol oc{};
      oc.src = OUT_BUILD;
      oc.width = (uint8_t)width_of(col.kind);
      oc.out_kind = col.kind;
      oc.bvalues = (const uint8_t*)col.values;
      oc.bvalidity = A.table->build.rows > 0 ? col.validity : nullptr;
      outs.push_back(oc);
    }
  }
  for (int h : P.outs) {
    const Operand& o = P.pb.root(h);
    tq_column d{};
    d.kind = out_kind_of(o, in, P.pb, &d.precision, &d.scale);
    sch.push_back(d);
    wv.push_back(o.maybe_null);
    OutCol oc{};
    oc.src = OUT_OPND;
    oc.kind = o.kind;
    oc.idx = o.idx;
    oc.width = (uint8_t)width_of(d.kind);
    oc.out_kind = d.kind;
    outs.push_back(oc);
  }
  if (outs.size() > (size_t)kMaxOut) fail(TQ_INVALID_PLAN, "too many output columns");

  uint64_t row_bytes = 0;
  for (auto& sc : sch) row_bytes += width_of(sc.kind);
  // single-pass probe needs a worst-case (one match per probe row) output buffer:
  // only when it is small against the Device budget left
  uint64_t cap_bytes = in->rows * row_bytes;
  uint64_t room = c->budget ? (c->budget > c->in_use.load() ? c->budget - c->in_use.load() : 0) : (64ull << 30);
  // a table without hash entries (semi-only, or direct-indexed) is probed
  // single-pass; if it is not usable the probe asks for the hash table
  const bool no_hash = A.mode == MAT_PROBE && A.table->jt.entries == nullptr;
  if (no_hash && A.table->jt.direct == nullptr && !A.build_cols.empty())
    fail(TQ_INVALID_PLAN, "semi-join build table: the probe cannot take build columns");
  const bool probe1 = A.mode == MAT_PROBE && (A.table->jt.unique || no_hash) &&
                      ((cap_bytes <= (8ull << 30) && cap_bytes * 4 <= room) || no_hash);
  if (probe1) {
    // single pass: capacity = probe rows (<= 1 match each), exact size read back
    p.dest_kind = DEST_PROBE1;
    // rows land in kChunk-row chunks: room for one partly used chunk per CTA
    const uint64_t cap_rows = in->rows + (uint64_t)L.grid * kChunk;
    alloc_batch(c, cap_rows, sch, wv, out, st);
    // cursor, dup flag, tails, plan
    const uint64_t scratch = 16 + L.grid * 16 + (10 + 4 * (uint64_t)L.grid) * 8;
    uint8_t* sb = (uint8_t*)dalloc(c, scratch, st);
    u64* cursor = (u64*)sb;
    u32* dup = (u32*)(cursor + 1);
    u64* tails = cursor + 2;
    u64* plan = tails + 2 * L.grid;
    TQ_CUDA(cudaMemsetAsync(cursor, 0, 16, st));
    p.cursor = cursor;
    p.chunk_tail = tails;
    p.dup_flag = dup;
    p.nout = (u32)outs.size();
    ChunkOut co{};
    co.ncols = p.nout;
    for (size_t i = 0; i < outs.size(); ++i) {
      outs[i].values = (uint8_t*)out->cols[i].values;
      outs[i].validity = out->cols[i].validity;
      p.out[i] = outs[i];
      co.values[i] = outs[i].values;
      co.validity[i] = outs[i].validity;
      co.width[i] = (u32)width_of(out->cols[i].kind);
    }
    launch(c, SINK_EMIT, L, P, st);
    if (p.ntiles == 0) {
      TQ_CUDA(cudaMemsetAsync(plan, 0, 8, st));
    } else {
      const int ph = prof_begin(c, "probe1_fixup", st);
      k_chunk_plan<<<1, 1024, (3 * L.grid + 2) * 8, st>>>(tails, L.grid, cursor, plan);
      k_chunk_move<<<c->sms * 2, 256, 0, st>>>(plan, L.grid, co);
      k_chunk_clear_tail<<<1, 32, 0, st>>>(plan, co);
      prof_end(c, ph, st);
      for (int k = 0; k < 3; ++k) counted_launch(c);
      TQ_CUDA(cudaGetLastError());
    }
    uint64_t n = 0;
    bool dup_keys = false, need_table = false;
    {
      TQ_CUDA(cudaMemcpyAsync(pinned_scratch(c), plan, 16, cudaMemcpyDeviceToHost, st));
      TQ_CUDA(cudaMemcpyAsync((uint8_t*)pinned_scratch(c) + 16, dup, 4, cudaMemcpyDeviceToHost, st));
      { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
      n = ((uint64_t*)pinned_scratch(c))[0];
      const uint32_t flag = ((uint32_t*)pinned_scratch(c))[4];
      dup_keys = flag == 1;
      need_table = flag == 2 || (flag == 1 && A.table->jt.entries == nullptr);
      if (!flag && p.ntiles && ((uint64_t*)pinned_scratch(c))[1] == ~0ull)
        fail(TQ_INTERNAL, "probe output chunk plan inconsistent");
    }
    dfree(c, sb, scratch, st);
    if (need_table) {
      // a semi-only build whose bitmap was not exact / keys not unique
      tq_batch_free(c, out);
      semi_table_materialize(c, const_cast<tq_join_table*>(A.table), st);
      run_materialize(c, in, P, A, out, part_offsets, st);
      return;
    }
    if (dup_keys) {
      // a probe key matched two build rows: the build side is not unique on
      // this key -> drop this pass, remember it on the table, probe two-pass
      tq_batch_free(c, out);
      const_cast<tq_join_table*>(A.table)->jt.unique = 0;  // a cached hint; every writer stores 0
      p.dest_kind = DEST_PROBE;
      p.cursor = nullptr;
      p.chunk_tail = nullptr;
      p.dup_flag = nullptr;
      goto two_pass;
    }
    out->rows = n;
    for (uint32_t i = 0; i < out->ncols; ++i) {
      out->cols[i].values_bytes = n * width_of(out->cols[i].kind);
      if (n == 0) out->cols[i].validity = nullptr;  // a 0-row column carries no bitmap
    }
    return;
  }

two_pass:
  // ---- count phase (skipped for dense 1:1 projections), per warp-slice of a tile
  const bool dense = A.mode == MAT_FILTER && !P.has_pred;
  uint64_t total = dense ? in->rows : 0;
  std::vector<uint64_t> starts(p.ndest + 1, 0);
  u32* counts = nullptr;
  u64* offsets = nullptr;
  const u64 nslices = (u64)p.ntiles * kWarps;
  u64 ncnt = (u64)p.ndest * nslices;
  if (A.async_slot) {
    if (A.mode == MAT_PROBE) fail(TQ_INVALID_PLAN, "no asynchronous probe (its output is not bounded by its input)");
    u64* dev_starts = (u64*)dalloc(c, (p.ndest + 1) * 8, st);
    if (!dense && p.ntiles > 0) {
      counts = (u32*)dalloc(c, ncnt * 4, st);
      offsets = (u64*)dalloc(c, (ncnt + 1) * 8, st);
      p.tile_counts = counts;
      std::vector<int> need = kh;
      if (P.has_pred) need.push_back(P.pred_h);
      const u32 all = p.load_mask;
      p.load_mask = P.pb.column_deps(need);
      launch_count(c, L, P, st);
      p.load_mask = all;
      scan_u32(c, counts, ncnt, offsets, offsets + ncnt, st);
      k_dest_starts<<<1, 128, 0, st>>>(offsets, (u32)nslices, p.ndest, offsets + ncnt, dev_starts);
      counted_launch(c);
      p.tile_offsets = offsets;
    } else {
      for (u32 d = 0; d <= p.ndest; ++d) k_set_u64_ext(dev_starts + d, d == 0 || !dense ? 0 : in->rows, st);
    }
    TQ_CUDA(cudaGetLastError());
    TQ_CUDA(cudaMemcpyAsync(A.async_slot, dev_starts, (p.ndest + 1) * 8, cudaMemcpyDeviceToHost, st));
    dfree(c, dev_starts, (p.ndest + 1) * 8, st);
    // every input row can pass: the output's capacity (trimmed by tq_batch_set_rows)
    try {
      alloc_batch(c, in->rows, sch, wv, out, st);
    } catch (...) {
      if (counts) dfree(c, counts, ncnt * 4, st);
      if (offsets) dfree(c, offsets, (ncnt + 1) * 8, st);
      throw;
    }
    p.nout = (u32)outs.size();
    for (size_t i = 0; i < outs.size(); ++i) {
      outs[i].values = (uint8_t*)out->cols[i].values;
      outs[i].validity = out->cols[i].validity;
      p.out[i] = outs[i];
    }
    if (in->rows > 0) launch(c, SINK_EMIT, L, P, st);
    if (counts) dfree(c, counts, ncnt * 4, st);
    if (offsets) dfree(c, offsets, (ncnt + 1) * 8, st);
    return;
  }
  if (!dense && p.ntiles > 0) {
    counts = (u32*)dalloc(c, ncnt * 4, st);
    offsets = (u64*)dalloc(c, (ncnt + 1) * 8, st);
    p.tile_counts = counts;
    {
      // the COUNT pass only needs the predicate and key columns
      std::vector<int> need = kh;
      if (P.has_pred) need.push_back(P.pred_h);
      const u32 all = p.load_mask;
      p.load_mask = P.pb.column_deps(need);
      launch_count(c, L, P, st);
      p.load_mask = all;
    }
    scan_u32(c, counts, ncnt, offsets, offsets + ncnt, st);
    {
      u64* pin = (u64*)pinned_scratch(c);
      k_dest_starts<<<1, 128, 0, st>>>(offsets, (u32)nslices, p.ndest, offsets + ncnt, pin);
      counted_launch(c);
      TQ_CUDA(cudaGetLastError());
      { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
      for (u32 d = 0; d <= p.ndest; ++d) starts[d] = pin[d];
    }
    total = starts[p.ndest];
    p.tile_offsets = offsets;
  } else if (!dense) {
    total = 0;
  } else {
    for (u32 d = 0; d <= p.ndest; ++d) starts[d] = d == 0 ? 0 : total;
  }
  if (part_offsets) {
    for (u32 d = 0; d < p.ndest; ++d) part_offsets[d] = starts[d];
    part_offsets[p.ndest] = total;
  }
  // ---- emit phase
  try {
    alloc_batch(c, total, sch, wv, out, st);
  } catch (...) {
    if (counts) dfree(c, counts, ncnt * 4, st);
    if (offsets) dfree(c, offsets, (ncnt + 1) * 8, st);
    throw;
  }
  p.nout = (u32)outs.size();
  for (size_t i = 0; i < outs.size(); ++i) {
    outs[i].values = (uint8_t*)out->cols[i].values;
    outs[i].validity = out->cols[i].validity;
    p.out[i] = outs[i];
  }
  if (total > 0) launch(c, SINK_EMIT, L, P, st);
  if (counts) dfree(c, counts, ncnt * 4, st);
  if (offsets) dfree(c, offsets, (ncnt + 1) * 8, st);
}

// ================================================================== join build

// ================================================================== fused partition + NVLink scatter
// Every rank scans its rows once; each row that passes the predicate (and the
// LIP Bloom filter) is written straight into the receive window of the rank
// its key hashes to (fnv1a64 mod n, as tq_hash_partition), through CUDA IPC
// mappings of the peers' windows over NVLink — the partitioned staging batch
// and the NCCL payload copy of partition + tq_comm_exchange disappear.
// Receivers then close the holes of the chunked layout and copy their rows out.
__global__ void k_set_u64(u64* p, u64 v) { *p = v; }

__global__ void k_tail_reset(u64* tails, u64 nslots) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < nslots; i += (u64)gridDim.x * blockDim.x) {
    tails[2 * i] = 0;
    tails[2 * i + 1] = kChunk;  // "full": no hole unless a CTA writes its tail here
  }
}

static void run_partition_exchange(tq_ctx* c, tq_comm* cm, const tq_batch* in, Prog& P,
                                   const std::vector<uint32_t>& key_roots, const uint32_t* semi_words,
                                   uint64_t semi_mask, uint64_t semi_part_words, tq_batch* out, uint64_t* rows_sent,
                                   cudaStream_t st, bool bcast = false) {
  const int n = comm_size(cm), me = comm_rank(cm);
  if (n > kMaxPeers) fail(TQ_INVALID_PLAN, "too many ranks for the fused exchange");
  Plan L;
  u32 sink_bytes = kWarps * kMaxDest * 4 + kWarps * kMaxDest * 8;
  plan_launch(c, in, P, L, sink_bytes, st);
  PipeParams& p = L.p;
  if (L.grid > (u32)kMaxTailCtas) L.grid = kMaxTailCtas;
  p.dest_kind = DEST_PEER;
  p.ndest = (u32)n;
  std::vector<int> kh;
  for (uint32_t k : key_roots) {
    if (k >= P.outs.size()) fail(TQ_INVALID_PLAN, "key column out of range");
    kh.push_back(P.outs[k]);
  }
  set_keys(p, P.pb, kh);
  p.bcast = bcast ? 1u : 0u;
  p.semi_bloom = semi_words;
  p.semi_mask = semi_mask;
  p.semi_part_words = semi_part_words;
  std::vector<tq_column> sch;
  std::vector<bool> wv;
  std::vector<OutCol> outs;
  for (int h : P.outs) {
    const Operand& o = P.pb.root(h);
    tq_column d{};
    d.kind = out_kind_of(o, in, P.pb, &d.precision, &d.scale);
    sch.push_back(d);
    wv.push_back(o.maybe_null);
    OutCol oc{};
    oc.src = OUT_OPND;
    oc.kind = o.kind;
    oc.idx = o.idx;
    oc.width = (uint8_t)width_of(d.kind);
    oc.out_kind = d.kind;
    outs.push_back(oc);
  }
  if (outs.size() > (size_t)kMaxOut) fail(TQ_INVALID_PLAN, "too many output columns");
  p.nout = (u32)outs.size();

  // window capacity (rows).  The data-region layout is a function of the
  // capacity, and the capacity a function of the window size, which every
  // rank holds identically (windows only grow collectively) -> no per-call
  // agreement on the size and no host sync before the kernel.  The first
  // exchange on a communicator agrees on a first size (all-gather of every
  // rank's guess); a receiver whose counter passed the capacity makes every
  // rank grow the window and re-run.
  // Validity: whether output k can be null is a LOCAL property (this rank's
  // input bitmaps; a 0-row input has none), so the layout reserves a bitmap
  // for every column and the ranks' masks are all-gathered before the kernel;
  // bits are written for the OR of the masks and the output carries a bitmap
  // iff any rank's part can hold a null (concat rule, transform.cpp:63-68).
  u64 vmask_local = 0;
  for (size_t k = 0; k < outs.size(); ++k)
    if (wv[k]) vmask_local |= 1ull << k;
  const u64 nslots = (u64)n * kMaxTailCtas;
  const u64 data0 = round_up(256 + nslots * 16, 256);
  auto layout_end = [&](u64 cap) {
    u64 end = data0;
    for (size_t k = 0; k < outs.size(); ++k) {
      end = round_up(end + cap * outs[k].width, 256);
      end = round_up(end + (cap + 7) / 8, 256);
    }
    return end;
  };
  // scratch: [0, n) all-gathered counts, [n] this rank's count, [n+1] rows sent,
  // [n+2] this rank's validity mask, [n+3, 2n+3) the all-gathered masks
  const u64 scratch_words = 3 * (u64)n + 8;
  u64* scratch = (u64*)dalloc(c, 8 * scratch_words, st);
  u64* sent_dev = scratch + n + 1;
  u64* vmask_in = scratch + n + 2;
  u64* vmask_all = scratch + n + 3;
  u64 cap = 0;
  if (comm_window_bytes(cm) == 0) {
    const bool filtered = P.has_pred || semi_words;
    // a receiver gets ~ (all ranks' rows) / n ~ this rank's rows when balanced
    // (a broadcast: all ranks' rows)
    u64 guess = std::max<u64>(filtered ? in->rows / 4 : in->rows * 5 / 4, 1ull << 16);
    if (bcast) guess *= (u64)n;
    TQ_CUDA(cudaMemcpyAsync(scratch + n, &guess, 8, cudaMemcpyHostToDevice, st));
    comm_allgather_u64(cm, scratch + n, scratch, 1, st);
    std::vector<u64> g(n);
    TQ_CUDA(cudaMemcpyAsync(g.data(), scratch, 8 * n, cudaMemcpyDeviceToHost, st));
    { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
    for (u64 x : g) guess = std::max(guess, x);
    cap = guess;
  } else {
    // the largest capacity whose layout fits half of the current window
    const u64 win = comm_window_bytes(cm) / 2 / 256 * 256;
    u64 per_row8 = 0;  // bits per row
    for (size_t k = 0; k < outs.size(); ++k) per_row8 += 8 * outs[k].width + 1;
    const u64 slack = data0 + 2 * 256 * (outs.size() + 1);
    cap = win > slack ? (win - slack) * 8 / std::max<u64>(1, per_row8) : 0;
    while (cap > 0 && layout_end(cap) > win) cap -= std::max<u64>(1, cap / 1024);
  }
  const u64 plan_words = 4 + 4 * nslots + 6;
  u64* plan = (u64*)dalloc(c, plan_words * 8, st);
  static bool smem_set = false;
  const u32 plan_smem = (u32)((3 * nslots + 2) * 8);
  if (!smem_set || plan_smem > 48 * 1024) {
    TQ_CUDA(cudaFuncSetAttribute(k_chunk_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    smem_set = true;
  }
  for (int attempt = 0;; ++attempt) {
    // layout of the data region (same on every rank: cap is)
    std::vector<u64> voff(outs.size()), boff(outs.size(), 0);
    u64 end = data0;
    for (size_t k = 0; k < outs.size(); ++k) {
      voff[k] = end;
      end = round_up(end + cap * outs[k].width, 256);
      boff[k] = end;
      end = round_up(end + (cap + 7) / 8, 256);
    }
    TQ_HT("pex total attempt");
    PeerView v = [&] {
      TQ_HT("pex window");
      return peer_window(cm, 2 * end, st, /*agreed=*/true);
    }();
    const int half = (int)(comm_epoch(cm) & 1);
    const u64 hoff = (u64)half * (comm_window_bytes(cm) / 2 / 256 * 256);
    uint8_t* base = v.local + hoff;
    u64* counter = (u64*)base;
    u64* tails = (u64*)(base + 256);
    TQ_CUDA(cudaMemsetAsync(sent_dev, 0, 8, st));
    // reset this half of the window (row counter, tail slots, every column's
    // bitmap); the validity-mask all-gather that follows is also the barrier
    // that orders every rank's reset before any rank scatters into it
    TQ_CUDA(cudaMemsetAsync(counter, 0, 8, st));
    k_tail_reset<<<(u32)std::min<u64>(1024, (nslots + 255) / 256), 256, 0, st>>>(tails, nslots);
    counted_launch(c);
    for (size_t k = 0; k < outs.size(); ++k) TQ_CUDA(cudaMemsetAsync(base + boff[k], 0, (cap + 7) / 8, st));
    k_set_u64<<<1, 1, 0, st>>>(vmask_in, vmask_local);
    counted_launch(c);
    {
      TQ_HT("pex barrier1");
      const int ph = prof_begin(c, "pex_barrier1", st);
      comm_allgather_u64(cm, vmask_in, vmask_all, 1, st);
      prof_end(c, ph, st);
    }
    for (int d = 0; d < n; ++d) {
      p.peer_delta[d] = (long long)(v.peer[d] - v.local);
      p.peer_counter[d] = (unsigned long long*)(v.peer[d] + hoff);
      p.peer_tails[d] = (unsigned long long*)(v.peer[d] + hoff + 256);
    }
    p.peer_cap = cap;
    p.tail_slot0 = (u32)me * kMaxTailCtas;
    p.peer_vmask = vmask_all;
    p.cursor = sent_dev;
    ChunkOut co{};
    co.ncols = p.nout;
    for (size_t k = 0; k < outs.size(); ++k) {
      outs[k].values = base + voff[k];
      outs[k].validity = base + boff[k];
      p.out[k] = outs[k];
      co.values[k] = outs[k].values;
      co.width[k] = outs[k].width;
    }
    launch(c, SINK_EMIT, L, P, st);
    {
      TQ_HT("pex barrier2");
      const int ph = prof_begin(c, "pex_barrier2", st);
      peer_barrier(cm, st);  // every rank's scatter into this window has completed
      prof_end(c, ph, st);
    }
    const int ph_plan = prof_begin(c, "pex_plan_counts", st);
    k_chunk_plan<<<1, 1024, plan_smem, st>>>(tails, (u32)nslots, counter, plan);
    counted_launch(c);
    TQ_CUDA(cudaMemcpyAsync(scratch + n, counter, 8, cudaMemcpyDeviceToDevice, st));
    comm_allgather_u64(cm, scratch + n, scratch, 1, st);
    prof_end(c, ph_plan, st);
    u64 n_rows = 0, moves = 0, rmax = 0, sent_rows = 0, vor = 0;
    {
      u64* pin = (u64*)pinned_scratch(c);
      TQ_CUDA(cudaMemcpyAsync(pin, plan, 16, cudaMemcpyDeviceToHost, st));
      TQ_CUDA(cudaMemcpyAsync(pin + 2, scratch, 8 * n, cudaMemcpyDeviceToHost, st));
      TQ_CUDA(cudaMemcpyAsync(pin + 2 + n, sent_dev, 8, cudaMemcpyDeviceToHost, st));
      TQ_CUDA(cudaMemcpyAsync(pin + 3 + n, vmask_all, 8 * n, cudaMemcpyDeviceToHost, st));
      { TQ_HT("pex sync after plan"); TQ_CUDA(cudaStreamSynchronize(st)); }
      n_rows = pin[0];
      moves = pin[1];
      for (int d = 0; d < n; ++d) rmax = std::max(rmax, pin[2 + d]);
      sent_rows = pin[2 + n];
      for (int d = 0; d < n; ++d) vor |= pin[3 + n + d];
    }
    if (rmax > cap) {  // some receiver overflowed: every rank sees the same rmax and re-runs
      if (attempt > 4) fail(TQ_INTERNAL, "fused exchange window did not converge");
      cap = rmax + rmax / 8 + (u64)kChunk * 64;
      continue;
    }
    if (moves == ~0ull) fail(TQ_INTERNAL, "fused exchange chunk plan inconsistent");
    std::vector<bool> wv_out(outs.size());
    for (size_t k = 0; k < outs.size(); ++k) {
      wv_out[k] = (vor >> k) & 1;
      co.validity[k] = wv_out[k] ? outs[k].validity : nullptr;
    }
    const int ph_fix = prof_begin(c, "pex_fix_copyout", st);
    k_chunk_move<<<c->sms * 2, 256, 0, st>>>(plan, (u32)nslots, co);
    k_chunk_clear_tail<<<1, 32, 0, st>>>(plan, co);
    counted_launch(c);
    counted_launch(c);
    TQ_CUDA(cudaGetLastError());
    alloc_batch(c, n_rows, sch, wv_out, out, st);
    for (size_t k = 0; k < outs.size(); ++k) {
      if (n_rows) TQ_CUDA(cudaMemcpyAsync(out->cols[k].values, co.values[k], n_rows * outs[k].width,
                                          cudaMemcpyDeviceToDevice, st));
      if (wv_out[k] && n_rows)
        TQ_CUDA(cudaMemcpyAsync(out->cols[k].validity, co.validity[k], (n_rows + 7) / 8, cudaMemcpyDeviceToDevice, st));
    }
    comm_epoch(cm) += 1;
    prof_end(c, ph_fix, st);
    if (rows_sent) *rows_sent = sent_rows;
    // the Bloom size of the table built on this output (tq_join_build_sized)
    // follows from it: the most rows any rank received (identical on every
    // rank), not the window capacity, which only grows over the comm's life
    comm_last_cap(cm) = std::max<u64>(rmax, 1);
    break;
  }
  dfree(c, plan, plan_words * 8, st);
  dfree(c, scratch, 8 * scratch_words, st);
}

// min / max of a plain Int64 key column (+ whether any row is null), for the
// direct aggregation's range pass when there is no predicate: 16-B loads,
// one set of atomics per block.
// out[3] != 0: the column is NOT non-decreasing (or has a null).
template <int MB>
__global__ void __launch_bounds__(256, MB) k_key_range(const long long* v, const uint8_t* valid, u64 rows, long long* out) {
  __shared__ long long s_mn[8], s_mx[8];
  __shared__ int s_null, s_unsorted;
  if (threadIdx.x == 0) s_null = s_unsorted = 0;
  __syncthreads();
  long long mn = 0x7fffffffffffffffll, mx = (long long)0x8000000000000000ull;
  bool nul = false, unsorted = false;
  const u64 pairs = rows / 2;
  const longlong2* v2 = (const longlong2*)v;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (!valid) {  // no bitmap: four independent 16-B loads in flight per thread
    const u64 lane = threadIdx.x & 31;
    // (warp-uniform trip count: the shuffles below need every lane)
    for (; i0 - lane + 31 + 3 * stride < pairs; i0 += 4 * stride) {
      longlong2 x[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) x[k] = __ldg(v2 + i0 + k * stride);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mn = min(mn, min(x[k].x, x[k].y));
        mx = max(mx, max(x[k].x, x[k].y));
        // sortedness: within the pair, and against the next pair's first value
        // (the next lane's; lane 31 loads it)
        long long nx = (long long)__shfl_down_sync(kFull, (unsigned long long)x[k].x, 1);
        const u64 pi = i0 + k * stride;
        if ((threadIdx.x & 31) == 31) nx = 2 * pi + 2 < rows ? __ldg(v + 2 * pi + 2) : x[k].y;
        unsorted |= x[k].x > x[k].y || x[k].y > nx;
      }
    }
  }
  for (u64 i = i0; i < pairs + (rows & 1); i += stride) {
    long long a, b;
    bool va = true, vb = true;
    if (i < pairs) {
      const longlong2 x = __ldg(v2 + i);
      a = x.x;
      b = x.y;
      if (valid) {
        va = bm_get(valid, 2 * i);
        vb = bm_get(valid, 2 * i + 1);
      }
    } else {  // odd tail row
      a = b = v[rows - 1];
      if (valid) va = vb = bm_get(valid, rows - 1);
    }
    if (va) { mn = min(mn, a); mx = max(mx, a); } else nul = true;
    if (vb) { mn = min(mn, b); mx = max(mx, b); } else nul = true;
    unsorted |= a > b || (2 * i + 2 < rows && b > __ldg(v + 2 * i + 2));
  }
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    mn = min(mn, (long long)__shfl_xor_sync(kFull, (unsigned long long)mn, m));
    mx = max(mx, (long long)__shfl_xor_sync(kFull, (unsigned long long)mx, m));
  }
  if (__any_sync(kFull, nul) && (threadIdx.x & 31) == 0) s_null = 1;
  if (__any_sync(kFull, unsorted) && (threadIdx.x & 31) == 0) s_unsorted = 1;
  if ((threadIdx.x & 31) == 0) {
    s_mn[threadIdx.x >> 5] = mn;
    s_mx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) {
      mn = min(mn, s_mn[w]);
      mx = max(mx, s_mx[w]);
    }
    if (mn <= mx) {
      atomicMin(out, mn);
      atomicMax(out + 1, mx);
    }
    if (s_null) atomicOr((unsigned long long*)out + 2, 1ull);
    if (s_unsorted || s_null) atomicOr((unsigned long long*)out + 3, 1ull);
  }
}

// occupancy of the range pass: 6 CTAs per SM (<= 42 registers, a 28-B spill)
// measured 0.116-0.122 ms vs 0.129-0.134 at 4 (63 registers) on SF10 orderkey
// (TQ_KR_MB: experiments only)
static void launch_key_range(tq_ctx* c, cudaStream_t st, const long long* v, const uint8_t* valid, u64 rows,
                             long long* out) {
  static const int mb = [] {
    const char* e = getenv("TQ_KR_MB");
    return e ? atoi(e) : 6;
  }();
  if (mb == 6) k_key_range<6><<<c->sms * 6, 256, 0, st>>>(v, valid, rows, out);
  else if (mb == 5) k_key_range<5><<<c->sms * 5, 256, 0, st>>>(v, valid, rows, out);
  else k_key_range<4><<<c->sms * 4, 256, 0, st>>>(v, valid, rows, out);
}

static void run_build(tq_ctx* c, const tq_batch* in, Prog& P, const std::vector<uint32_t>& key_roots,
                      tq_join_table** out, cudaStream_t st, uint64_t bloom_keys, bool semi_only, bool allow_direct) {
  Plan L;
  plan_launch(c, in, P, L, 0, st);
  PipeParams& p = L.p;
  std::vector<int> kh;
  for (uint32_t k : key_roots) {
    if (k >= P.outs.size()) fail(TQ_INVALID_PLAN, "key column out of range");
    kh.push_back(P.outs[k]);
  }
  if (kh.empty()) fail(TQ_INVALID_PLAN, "join without keys");
  set_keys(p, P.pb, kh);
  tq_join_table* t = new tq_join_table();
  t->ctx = c;
  t->stream = st;
  for (int h : kh) {
    const Operand& o = P.pb.root(h);
    if (o.cls == C_F || o.cls == C_S) {
      delete t;
      fail(TQ_INVALID_PLAN, "unsupported join key type");
    }
    t->key_cls.push_back(o.cls);
    t->key_scale.push_back(o.scale);
  }
  // load factor 0.25..0.5 (linear probing: short clusters, little warp divergence)
  uint64_t cap = 1024;
  while (cap < in->rows * 2) cap <<= 1;
  t->jt.cap = cap;
  t->jt.kw = p.key_words;
  t->jt.stride = (u32)round_up(8 * (1 + p.key_words), 16);
  // blocked Bloom filter, ~8 bits per build row: rejects non-matching probes in L2
  // (bloom_keys: size for that many keys at kLipBloomBitsPerKey instead, a row
  // count every rank agrees on, so the ranks' filters can be all-gathered as one
  // partitioned filter)
  uint64_t words = 1024;
  while (words * 32 < std::max<uint64_t>(in->rows * 8, bloom_keys * kLipBloomBitsPerKey)) words <<= 1;
  t->jt.bloom_mask = words - 1;
  // One-word keys also get an exact membership bitmap over [0, exact_range)
  // and the build's duplicate-key / exact-range flags.  A semi-only build (a
  // semi-join's build side) has no hash table at all.  Otherwise, when the
  // address space fits, the build is DIRECT-indexed: a 4-B row slot per key
  // value in [0, 32 x rows) (never initialised: the bitmap says which slots
  // were written), no hash table, no CAS — a plain store per build row, and a
  // probe reads one slot per hit.  Dense keys (TPC-H's) make both the stores
  // and the probe's reads of neighbouring keys coalesce.  Keys outside the
  // range or repeated send the first probe back to the host, which then
  // builds the hash table (as for a semi-only table).
  const bool exact = t->jt.kw == 1;
  const bool semi = semi_only && exact;
  uint64_t ewords = words;  // exact bitmap words (range 32 x ewords)
  // The bitmap / direct range [0, 32 x ewords) must cover the keys.  A plain
  // Int64 key column of a large build is measured first (k_key_range: one
  // 8-B read per row + a host sync), so e.g. a hash-partitioned orders_f —
  // 1/N of the rows, keys spread over the whole orderkey range — still gets
  // an exact bitmap and a direct table; otherwise the range is 32 x rows.
  uint64_t key_max = 0;
  bool measured = false;
  {
    const Operand& ko = P.pb.root(kh[0]);
    if (exact && ko.kind == K_COL_I64 && !P.has_pred && in->rows >= (1u << 16)) {
      const tq_column& col = in->cols[P.pb.staged()[ko.idx]];
      long long* kr = (long long*)dalloc(c, 32, st);
      const long long init[4] = {0x7fffffffffffffffll, (long long)0x8000000000000000ull, 0, 0};
      TQ_CUDA(cudaMemcpyAsync(kr, init, 32, cudaMemcpyHostToDevice, st));
      launch_key_range(c, st, (const long long*)col.values, col.validity, in->rows, kr);
      counted_launch(c);
      long long* pin = (long long*)pinned_scratch(c);
      TQ_CUDA(cudaMemcpyAsync(pin, kr, 16, cudaMemcpyDeviceToHost, st));
      { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
      dfree(c, kr, 32, st);
      if (pin[0] >= 0 && pin[0] <= pin[1]) {
        key_max = (uint64_t)pin[1];
        measured = true;
      }
    }
  }
  auto range_words = [&](uint64_t base_words) {
    uint64_t w = std::max<uint64_t>(words, base_words);
    if (measured) w = std::max<uint64_t>(w, round_up(key_max / 32 + 1, 1024));
    return w;
  };
  bool direct = false;
  if (exact && !semi && allow_direct && in->rows < (1ull << 31)) {
    static const bool no_direct = [] { const char* e = getenv("TQ_DIRECT"); return e && e[0] == '0'; }();
    const uint64_t dw = range_words(round_up(in->rows, 1024));  // range >= 32 x rows and > the largest key
    const uint64_t room = c->budget ? (c->budget > c->in_use.load() ? c->budget - c->in_use.load() : 0) : (64ull << 30);
    // the slots are address space (never initialised); cap them at 64 slots per build row
    if (!no_direct && dw * 32 * 4 <= room / 4 && dw * 32 <= std::max<uint64_t>(64 * in->rows, 1u << 20)) {
      direct = true;
      ewords = dw;
    }
  }
  if (semi) ewords = range_words(round_up(in->rows, 1024));  // bitmap only
  // a hash table keeps an exact bitmap over the measured key range too (1 bit
  // per key value; the probes then never need the Bloom filter), up to 256 bits per row
  if (exact && !semi && !direct && measured && range_words(words) * 32 <= 256 * std::max<uint64_t>(in->rows, 1024))
    ewords = range_words(words);
  const bool hashed = !semi && !direct;
  uint64_t ebytes = hashed ? cap * t->jt.stride : 0;
  const uint64_t aux = words * 4 + 16 + (exact ? ewords * 4 : 0);  // Bloom, flags, exact bitmap
  const uint64_t dbytes = direct ? ewords * 32 * 4 : 0;
  t->bytes = ebytes + aux + dbytes;
  try {
    t->mem = (uint8_t*)dalloc(c, t->bytes, st);
  } catch (...) {
    delete t;
    throw;
  }
  t->jt.entries = hashed ? t->mem : nullptr;
  t->jt.bloom = (uint32_t*)(t->mem + ebytes);
  if (hashed) TQ_CUDA(cudaMemsetAsync(t->jt.entries, 0xff, ebytes, st));
  TQ_CUDA(cudaMemsetAsync(t->jt.bloom, 0, aux, st));
  t->jt.dup_dev = t->jt.kw == 1 && (t->jt.stride == 16 || !hashed) ? (uint32_t*)(t->jt.bloom + words) : nullptr;
  t->jt.exact_flag = exact ? (uint32_t*)(t->jt.bloom + words) + 1 : nullptr;
  t->jt.exact_bits = exact ? (uint32_t*)(t->jt.bloom + words) + 4 : nullptr;
  t->jt.exact_range = exact ? ewords * 32 : 0;
  t->jt.direct = direct ? (uint32_t*)(t->mem + ebytes + aux) : nullptr;
  // a direct table's probes test the exact bitmap; its Bloom filter is only
  // built when asked for (bloom_keys: the partitioned LIP filter)
  if (direct && bloom_keys == 0) t->jt.bloom = nullptr;
  {  // TQ_BLOOM=0: experiments only (probe without the Bloom pre-check)
    static const bool no_bloom = [] { const char* e = getenv("TQ_BLOOM"); return e && e[0] == '0'; }();
    if (no_bloom) t->jt.bloom = nullptr;
  }
  t->build = *in;
  t->build.owner = nullptr;
  t->build.cols = (tq_column*)std::malloc(sizeof(tq_column) * std::max<uint32_t>(1, in->ncols));
  std::memcpy(t->build.cols, in->cols, sizeof(tq_column) * in->ncols);
  p.jt = t->jt;
  p.row_base = 0;
  // TQ_BUILD_PASSES (experiments): fill the table in slot-range passes so each
  // pass's CASes hit an L2-resident range.  Measured slower on the 512-MB
  // orders table (0.93 ms in one pass; 1.26 / 1.74 / 2.57 ms in 4 / 8 / 16):
  // every pass pays the per-tile pipeline latency over all rows, so the
  // default is one pass.
  u32 passes = 1;
  {
    static const long env_passes = [] { const char* e = getenv("TQ_BUILD_PASSES"); return e ? atol(e) : -1L; }();
    if (env_passes > 0 && hashed) passes = (u32)env_passes;
  }
  for (u32 k = 0; k < passes; ++k) {
    p.slot_lo = passes > 1 ? cap / passes * k : 0;
    p.slot_hi = passes > 1 ? cap / passes * (k + 1) : 0;
    p.build_skip_aux = k > 0;
    launch(c, SINK_BUILD, L, P, st);
  }
  if (!hashed) {
    // usable without a hash table only when the bitmap is exact and proved the
    // keys unique (atomicOr return values) — known on the device only; a probe
    // that finds otherwise flags it and the host then builds the real table
    // (semi_table_materialize) and re-runs that probe.  No host sync here.
    t->semi_prog = std::make_shared<Prog>(P);
    t->semi_keys = key_roots;
    t->semi_bloom_keys = bloom_keys;
  }
  t->bloom_keys = bloom_keys;
  // No uniqueness pass and no host sync: a probe first assumes unique build
  // keys (the PK side of a PK-FK join) and runs in one pass.  One-word keys
  // are proven unique (or not) by the build itself (jt.dup_dev); otherwise the
  // pass walks each matched cluster for a second match.  A probe that finds
  // one re-runs two-pass and marks the table (jt.unique = 0) for later probes.
  t->jt.unique = 1;
  *out = t;
}

// ================================================================== aggregation
enum AggOutKind : uint8_t {
  AO_SUM_I64 = 0, AO_SUM_DEC, AO_SUM_F, AO_CNT, AO_AVG_I, AO_AVG_F, AO_MM_I64, AO_MM_DEC, AO_MM_BOOL, AO_MM_F
};
struct AggOut {
  uint8_t kind, acc, cnt, scale;
  uint8_t* values;
  uint8_t* validity;
};
struct KeyOut {
  uint8_t kind, word, bit, _p;
  uint8_t* values;
  uint8_t* validity;
};
struct FinalParams {
  AggTable t;
  u32 kwa, nacc, nkeys, naggs;
  KeyOut keys[kMaxKeys];
  AggOut aggs[32];
  unsigned long long* counter;
  u32 direct, cnt_acc;  // direct table: occupied iff acc[cnt_acc] != 0; key = key_min + slot
  long long key_min;
  u64 null_slot;
};

__device__ __forceinline__ bool agg_slot_used(const FinalParams& f, u64 s) {
  return s < f.t.cap && (f.direct ? __ldg(direct_acc(f.t, f.cnt_acc, s)) != 0 : __ldg(f.t.state + s) == 2);
}
__device__ __forceinline__ void agg_emit_group(const FinalParams& f, u64 s, u64 row);
__device__ __forceinline__ void agg_emit_keys(const FinalParams& f, u64 s, u64 row);
__device__ __forceinline__ void agg_store_value(const FinalParams& f, const AggOut& ao, u64 row, u64 m0, u64 m1,
                                                u64 cnt);

// Compaction of the occupied slots into output rows, in slot order.  A block
// takes chunks of kFinItems x 256 contiguous slots; item i of thread t is slot
// chunk + i * 256 + t (coalesced reads), its row = the chunk's base + the
// occupied slots before it in the chunk (coalesced writes: a warp's item
// lands on consecutive rows), and the chunk's rows are reserved with ONE
// global atomic (a reservation per 256 slots put ~60K atomics on the one
// cursor for 15M groups).
constexpr u32 kFinItems = 4;
__global__ void __launch_bounds__(256) k_agg_final(const __grid_constant__ FinalParams f) {
  __shared__ u32 s_off[kFinItems][8];   // per (item, warp): rows before it in the chunk
  __shared__ u32 s_ball[kFinItems][8];  // per (item, warp): occupied lanes
  __shared__ unsigned long long s_base;
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 chunk = (u64)kFinItems * 256;
  const u64 nchunks = (f.t.cap + chunk - 1) / chunk;
  for (u64 c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const u64 s0 = c * chunk + threadIdx.x;
#pragma unroll
    for (u32 i = 0; i < kFinItems; ++i) {
      const u32 b = __ballot_sync(kFull, agg_slot_used(f, s0 + (u64)i * 256));
      if (lane == 0) {
        s_off[i][warp] = __popc(b);
        s_ball[i][warp] = b;
      }
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the kFinItems x 8 (item, warp) counts, item-major
      constexpr u32 kPer = kFinItems * 8 / 32;
      u32 v[kPer], sum = 0;
#pragma unroll
      for (u32 k = 0; k < kPer; ++k) {
        v[k] = (&s_off[0][0])[lane * kPer + k];
        sum += v[k];
      }
      u32 incl = sum;
#pragma unroll
      for (u32 o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      u32 run = incl - sum;
#pragma unroll
      for (u32 k = 0; k < kPer; ++k) {
        (&s_off[0][0])[lane * kPer + k] = run;
        run += v[k];
      }
      const u32 tot = __shfl_sync(kFull, incl, 31);
      if (lane == 0) s_base = tot ? atomicAdd(f.counter, (unsigned long long)tot) : 0;
    }
    __syncthreads();
    const u64 base = s_base;
    // (4 items unrolled: independent accumulator loads in flight; 16 unrolled
    // copies of the emit body stalled on instruction fetch)
    if (f.direct && f.naggs == 1) {
      // one aggregate over a direct table (e.g. a high-cardinality Sum): the
      // accumulator words of all kFinItems slots are loaded (predicated, no
      // branch) before any store, so their latencies overlap instead of
      // serialising item by item
      const AggOut& ao = f.aggs[0];
      const bool two = f.t.dwidth[ao.acc] >= 2;
      u64 m0[kFinItems], m1[kFinItems], cn[kFinItems];
#pragma unroll
      for (u32 i = 0; i < kFinItems; ++i) {
        const bool occ = (s_ball[i][warp] >> lane) & 1u;
        const u64 sl = occ ? s0 + (u64)i * 256 : 0;
        const u64* src = direct_acc(f.t, ao.acc, sl);
        m0[i] = occ ? __ldg(src) : 0ull;
        m1[i] = occ && two ? __ldg(src + 1) : 0ull;
        cn[i] = ao.cnt == 0xff ? 1ull : occ ? __ldg(direct_acc(f.t, ao.cnt, sl)) : 0ull;
      }
#pragma unroll
      for (u32 i = 0; i < kFinItems; ++i) {
        const u32 b = s_ball[i][warp];
        if ((b >> lane) & 1u) {
          const u64 row = base + s_off[i][warp] + __popc(b & lanemask_lt());
          agg_emit_keys(f, s0 + (u64)i * 256, row);
          agg_store_value(f, ao, row, m0[i], m1[i], cn[i]);
        }
      }
    } else {
#pragma unroll
      for (u32 i = 0; i < kFinItems; ++i) {
        const u32 b = s_ball[i][warp];
        if ((b >> lane) & 1u) agg_emit_group(f, s0 + (u64)i * 256, base + s_off[i][warp] + __popc(b & lanemask_lt()));
      }
    }
    __syncthreads();  // s_off / s_base are rewritten next chunk
  }
}

__device__ __forceinline__ void agg_emit_keys(const FinalParams& f, u64 s, u64 row) {
  u64 dk[2] = {(u64)f.key_min + s, s == f.null_slot ? 1ull : 0ull};  // direct: key word, null word
  const u64* kw = f.direct ? dk : f.t.keys + s * f.kwa;
  u64 nullw = kw[f.kwa - 1];
  for (u32 k = 0; k < f.nkeys; ++k) {
    const KeyOut& ko = f.keys[k];
    bool isnull = (nullw >> ko.bit) & 1;
    if (ko.kind == TQ_DECIMAL) {
      ((u64*)ko.values)[2 * row] = kw[ko.word];
      ((u64*)ko.values)[2 * row + 1] = kw[ko.word + 1];
    } else if (ko.kind == TQ_BOOL) {
      ko.values[row] = (uint8_t)kw[ko.word];
    } else {
      ((u64*)ko.values)[row] = kw[ko.word];
    }
    if (ko.validity && !isnull) bm_set_atomic(ko.validity, row);
  }
}

// one aggregate's output at `row` from its raw accumulator words and count
__device__ __forceinline__ void agg_store_value(const FinalParams& f, const AggOut& ao, u64 row, u64 m0, u64 m1,
                                                u64 cnt) {
  u64 m[2] = {m0, m1};
  if (f.direct && (ao.kind == AO_SUM_I64 || ao.kind == AO_SUM_DEC || ao.kind == AO_AVG_I)) {
    // direct table: integer sums are kept as {low-limb sum, high-part sum}
    const i128 v = add128((i128)(long long)m[1] * ((i128)1 << 32), (i128)m[0]);
    m[0] = lo64(v);
    m[1] = hi64(v);
  }
  {
    bool valid = cnt != 0;
    switch (ao.kind) {
      case AO_SUM_I64:
      case AO_MM_I64:
        ((u64*)ao.values)[row] = m[0];
        break;
      case AO_SUM_DEC:
      case AO_MM_DEC:
        ((u64*)ao.values)[2 * row] = m[0];
        ((u64*)ao.values)[2 * row + 1] = m[1];
        break;
      case AO_MM_BOOL:
        ao.values[row] = m[0] != 0;
        break;
      case AO_SUM_F:
      case AO_MM_F:
        ((u64*)ao.values)[row] = m[0];
        break;
      case AO_CNT:
        ((u64*)ao.values)[row] = m[0];
        valid = true;
        break;
      case AO_AVG_I: {
        double d = valid ? i128_to_f64(mk128(m[0], m[1])) / pow(10.0, (double)ao.scale) / (double)cnt : 0.0;
        ((double*)ao.values)[row] = d;
        break;
      }
      case AO_AVG_F: {
        double d = valid ? __longlong_as_double((long long)m[0]) / (double)cnt : 0.0;
        ((double*)ao.values)[row] = d;
        break;
      }
    }
    if (ao.validity && valid) bm_set_atomic(ao.validity, row);
  }
}

__device__ __forceinline__ void agg_emit_group(const FinalParams& f, u64 s, u64 row) {
  agg_emit_keys(f, s, row);
  const u64* acc = f.t.acc + s * f.nacc * 2;
  for (u32 a = 0; a < f.naggs; ++a) {
    const AggOut& ao = f.aggs[a];
    // read-only in this kernel: non-coherent loads, which the compiler may
    // issue ahead of the previous group's stores (they cannot alias)
    const u64* src = f.direct ? direct_acc(f.t, ao.acc, s) : acc + 2 * ao.acc;
    const u64 m0 = __ldg(src), m1 = (f.direct && f.t.dwidth[ao.acc] < 2) ? 0ull : __ldg(src + 1);
    const u64 cnt = ao.cnt == 0xff ? 1 : __ldg(f.direct ? direct_acc(f.t, ao.cnt, s) : acc + 2 * ao.cnt);
    agg_store_value(f, ao, row, m0, m1, cnt);
  }
}

// direct aggregation table: every slot's accumulators start at their identity
struct AccOps {
  uint8_t op[kMaxAcc];
};
__global__ void k_acc_init(AggTable t, u64 slots, u32 nacc, AccOps ops) {
  const u64 n = slots * nacc;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u32 a = (u32)(i / slots);
    u64 lo, hi;
    acc_identity(ops.op[a], lo, hi);
    u64* m = direct_acc(t, a, i % slots);
    m[0] = lo;
    if (t.dwidth[a] > 1) m[1] = hi;
  }
}

struct AggPlan {
  uint8_t kind, acc, cnt, scale;
  tq_column col;
  bool nullable;
};
struct AggSpec {
  std::vector<AccSpec> acc;   // deduplicated accumulators
  std::vector<AggPlan> ap;    // one output per aggregate, referencing acc
};

// Aggregates -> accumulators + output plans.
static AggSpec plan_aggs(const tq_batch* in, Prog& P, const tq_agg* aggs, uint32_t naggs) {
  AggSpec S;
  std::vector<AccSpec>& acc = S.acc;
  auto acc_of = [&](uint8_t op, uint8_t kind, uint16_t idx) -> uint8_t {
    for (size_t i = 0; i < acc.size(); ++i)
      if (acc[i].op == op && acc[i].kind == kind && acc[i].idx == idx) return (uint8_t)i;
    if (acc.size() >= (size_t)kMaxAcc) fail(TQ_INVALID_PLAN, "too many aggregates");
    AccSpec a{};
    a.op = op; a.kind = kind; a.idx = idx;
    acc.push_back(a);
    return (uint8_t)(acc.size() - 1);
  };
  if (naggs > 32) fail(TQ_INVALID_PLAN, "too many aggregates");
  for (uint32_t j = 0; j < naggs; ++j) {
    AggPlan a{};
    a.cnt = 0xff;
    uint32_t fn = aggs[j].fn;
    if (fn > TQ_AGG_AVG) fail(TQ_INVALID_PLAN, "bad aggregate");
    if (fn == TQ_AGG_COUNT_STAR) {
      a.kind = AO_CNT;
      a.acc = acc_of(ACC_CNT, K_NONE, 0);
      a.col.kind = TQ_INT64;
      S.ap.push_back(a);
      continue;
    }
    if (aggs[j].column >= P.outs.size()) fail(TQ_INVALID_PLAN, "aggregate column out of range");
    const Operand& o = P.pb.root(P.outs[aggs[j].column]);
    uint8_t prec, scale;
    uint8_t kind = out_kind_of(o, in, P.pb, &prec, &scale);
    uint8_t cnt_acc = o.maybe_null ? acc_of(ACC_CNT, o.kind, o.idx) : acc_of(ACC_CNT, K_NONE, 0);
    a.nullable = o.maybe_null;
    switch (fn) {
      case TQ_AGG_COUNT:
        a.kind = AO_CNT;
        a.acc = cnt_acc;
        a.col.kind = TQ_INT64;
        break;
      case TQ_AGG_SUM:
        if (o.cls == C_B) fail(TQ_INVALID_PLAN, "sum of bool");
        if (o.cls == C_F) { a.kind = AO_SUM_F; a.acc = acc_of(ACC_SUM_F, o.kind, o.idx); a.col.kind = TQ_FLOAT64; }
        else if (o.cls == C_D) {
          a.kind = AO_SUM_DEC; a.acc = acc_of(ACC_SUM_I, o.kind, o.idx);
          a.col.kind = TQ_DECIMAL; a.col.precision = 38; a.col.scale = scale;
        } else { a.kind = AO_SUM_I64; a.acc = acc_of(ACC_SUM_I, o.kind, o.idx); a.col.kind = TQ_INT64; }
        a.cnt = o.maybe_null ? cnt_acc : 0xff;
        break;
      case TQ_AGG_AVG:
        if (o.cls == C_B) fail(TQ_INVALID_PLAN, "avg of bool");
        if (o.cls == C_F) { a.kind = AO_AVG_F; a.acc = acc_of(ACC_SUM_F, o.kind, o.idx); }
        else { a.kind = AO_AVG_I; a.acc = acc_of(ACC_SUM_I, o.kind, o.idx); a.scale = o.cls == C_D ? o.scale : 0; }
        a.cnt = cnt_acc;
        a.col.kind = TQ_FLOAT64;
        break;
      default: {  // MIN / MAX
        bool mn = fn == TQ_AGG_MIN;
        if (o.cls == C_F) { a.kind = AO_MM_F; a.acc = acc_of(mn ? ACC_MIN_F : ACC_MAX_F, o.kind, o.idx); }
        else {
          a.kind = o.cls == C_D ? AO_MM_DEC : o.cls == C_B ? AO_MM_BOOL : AO_MM_I64;
          a.acc = acc_of(mn ? ACC_MIN_I : ACC_MAX_I, o.kind, o.idx);
        }
        a.col.kind = kind; a.col.precision = prec; a.col.scale = scale;
        a.cnt = o.maybe_null ? cnt_acc : 0xff;
      }
    }
    S.ap.push_back(a);
  }
  return S;
}

// One hash group-by pass over `in`.  ap == nullptr -> PARTIAL output: the key
// columns then one column per raw accumulator (int128 accumulators as
// Decimal(38,0), counts Int64, float accumulators Float64) for a later merge.
static void agg_core(tq_ctx* c, const tq_batch* in, Prog& P, const std::vector<int>& kh,
                     const std::vector<AccSpec>& acc, const std::vector<AggPlan>* ap, tq_batch* out, cudaStream_t st,
                     const std::vector<uint8_t>* raw_ops = nullptr) {
  const u32 nacc = (u32)acc.size();
  // local (per-CTA) group table: per-lane private accumulator planes (8 B;
  // MIN/MAX of int128 take two) sized to the shared memory left after two stages
  u32 kwa_guess = 1;
  for (int h : kh) kwa_guess += P.pb.root(h).cls == C_D ? 2 : 1;
  u32 nplanes = 0;
  uint8_t planes[kMaxAcc] = {};
  for (u32 i = 0; i < nacc; ++i) {
    planes[i] = (uint8_t)nplanes;
    nplanes += (acc[i].op == ACC_MIN_I || acc[i].op == ACC_MAX_I) ? 2 : 1;
  }
  auto sink_bytes = [&](u32 g) {
    return align_up(g * 4, 16) + g * kwa_guess * 8 + g * 8 + g * std::max<u32>(1, nplanes) * kThreads * 8;
  };
  u32 G = 0;
  {
    Plan probe;
    plan_launch(c, in, P, probe, 0, st);
    u32 fixed = probe.smem - probe.p.nstages * probe.p.stage_bytes;  // everything but the stages
    u32 avail = 227 * 1024 - fixed - 2 * probe.p.stage_bytes - 1024;
    G = kh.empty() ? 1 : 64;  // a global aggregate has exactly one group
    while (G > 1 && sink_bytes(G) > avail) G >>= 1;
    if (sink_bytes(G) > avail) G = 0;
  }
  Plan L;
  PipeParams& p = L.p;
  auto setup = [&](u32 g) {
    L = Plan{};
    plan_launch(c, in, P, L, g ? sink_bytes(g) : 64, st);
    set_keys(p, P.pb, kh);
    p.nacc = nacc;
    for (u32 i = 0; i < nacc; ++i) { p.acc[i] = acc[i]; p.acc_plane[i] = planes[i]; }
    p.nplanes = std::max<u32>(1, nplanes);
    p.local_groups = g;
  };
  setup(G);
  const u32 kwa = p.key_words + 1;

  // ---- DIRECT aggregation: one integer key whose values over the passing
  // rows span a dense range (e.g. group by orderkey: 15M groups at SF10).
  // A range pass (min / max of the key, only the key and predicate columns
  // are read) sizes a table of one slot per key value; no hash, no claim
  // protocol, no regrowth re-runs, and clustered keys update neighbouring
  // slots.  Only for final aggregates with a Count(*) accumulator (it marks
  // the occupied slots) and inputs large enough to pay for the range pass.
  bool direct = false, key_sorted = false;
  long long kmin = 0;
  uint64_t R = 0;
  u32 cnt_idx = 0;
  {
    static const bool no_direct = [] { const char* e = getenv("TQ_DIRECT"); return e && e[0] == '0'; }();
    bool has_cnt = false;
    for (u32 i = 0; i < nacc; ++i)
      if (acc[i].op == ACC_CNT && acc[i].kind == K_NONE) { has_cnt = true; cnt_idx = i; break; }
    if (!no_direct && ap && has_cnt && kh.size() == 1 && P.pb.root(kh[0]).cls == C_I && in->rows >= (4ull << 20)) {
      Plan Lr;
      plan_launch(c, in, P, Lr, 64, st);
      set_keys(Lr.p, P.pb, kh);
      Lr.p.dest_kind = DEST_RANGE;
      std::vector<int> need = kh;
      if (P.has_pred) need.push_back(P.pred_h);
      Lr.p.load_mask = P.pb.column_deps(need);
      long long* kr = (long long*)dalloc(c, 32, st);
      // {min, max, any null, not sorted}; the pipeline range pass (a predicate
      // or a computed key) does not check sortedness
      const long long init[4] = {0x7fffffffffffffffll, (long long)0x8000000000000000ull, 0, 1};
      TQ_CUDA(cudaMemcpyAsync(kr, init, 32, cudaMemcpyHostToDevice, st));
      Lr.p.key_range = kr;
      const Operand& ko = P.pb.root(kh[0]);
      if (!P.has_pred && ko.kind == K_COL_I64) {  // a plain key column: one streaming reduction
        const tq_column& col = in->cols[P.pb.staged()[ko.idx]];
        TQ_CUDA(cudaMemsetAsync(kr + 3, 0, 8, st));
        const int ph = prof_begin(c, "key_range", st);
        launch_key_range(c, st, (const long long*)col.values, in->rows ? col.validity : nullptr,
                                                 in->rows, kr);
        prof_end(c, ph, st);
        counted_launch(c);
        TQ_CUDA(cudaGetLastError());
      } else {
        launch(c, SINK_COUNT, Lr, P, st);
      }
      long long mn, mx;
      {
        TQ_CUDA(cudaMemcpyAsync(pinned_scratch(c), kr, 32, cudaMemcpyDeviceToHost, st));
        { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
        mn = ((long long*)pinned_scratch(c))[0];
        mx = ((long long*)pinned_scratch(c))[1];
        key_sorted = ((long long*)pinned_scratch(c))[3] == 0;
      }
      dfree(c, kr, 32, st);
      const uint64_t room = c->budget ? (c->budget > c->in_use.load() ? c->budget - c->in_use.load() : 0) : (64ull << 30);
      const uint64_t span = mx >= mn ? (uint64_t)mx - (uint64_t)mn + 1 : 0;  // 0: no non-null key
      if ((mx < mn || (span != 0 && span <= 2 * in->rows)) && (span + 1) * nacc * 16 <= room / 2 &&
          span < (1ull << 40)) {
        direct = true;
        kmin = mx >= mn ? mn : 0;
        R = span;
      }
    }
  }
  if (direct) setup(0);

  // ---- global table; grows x4 and re-runs on overflow (on_oom-style retry)
  // initial table for min(rows, 1M) groups at load <= 0.5
  uint64_t cap = 1024;
  if (!kh.empty())
    while (cap < std::min<uint64_t>(in->rows, 1ull << 20) * 2) cap <<= 1;
  {  // TQ_AGG_CAP: experiments only (initial global table slots)
    static const uint64_t cap_env = [] { const char* e = getenv("TQ_AGG_CAP"); return e ? strtoull(e, nullptr, 10) : 0ull; }();
    if (cap_env && !kh.empty()) { cap = 1024; while (cap < cap_env) cap <<= 1; }
  }
  uint64_t ngroups = 0;
  AggTable t{};
  uint64_t tbytes = 0;
  if (direct) {
    // slots [0, R) = key values kmin .., slot R = the null key
    const uint64_t cap0 = cap;  // (the hash table's first size, if this falls back)
    cap = R + 1;
    uint64_t words = 0;  // per slot, over all accumulators (counts take one word)
    for (u32 i = 0; i < nacc; ++i) {
      t.dwidth[i] = acc[i].op == ACC_CNT ? 1 : 2;
      words += t.dwidth[i];
    }
    t.dstride = (cap + 1) & ~1ull;
    tbytes = t.dstride * words * 8 + 64;
    uint8_t* base = (uint8_t*)dalloc(c, tbytes, st);
    t.state = (uint32_t*)base;  // (no state words: freed through this base)
    t.keys = nullptr;
    t.acc = (u64*)base;
    t.cap = cap;
    uint8_t* tail = base + t.dstride * words * 8;
    t.nused = (unsigned long long*)tail;
    t.overflow = (uint32_t*)(tail + 8);
    TQ_CUDA(cudaMemsetAsync(tail, 0, 16, st));
    bool minmax = false;
    AccOps ops{};
    for (u32 i = 0; i < nacc; ++i) {
      ops.op[i] = acc[i].op;
      minmax |= acc[i].op == ACC_MIN_I || acc[i].op == ACC_MAX_I || acc[i].op == ACC_MIN_F || acc[i].op == ACC_MAX_F;
    }
    t.direct = 1;
    t.sorted = key_sorted ? 1u : 0u;
    t.cnt_acc = cnt_idx;
    t.key_min = kmin;
    t.direct_slots = R;
    if (minmax) {
      k_acc_init<<<(u32)std::min<uint64_t>((cap * nacc + 255) / 256, (uint64_t)c->sms * 8), 256, 0, st>>>(t, cap,
                                                                                                       nacc, ops);
      counted_launch(c);
    } else {
      TQ_CUDA(cudaMemsetAsync(t.acc, 0, t.dstride * words * 8, st));
    }
    p.agg = t;
    launch(c, SINK_AGG, L, P, st);
    uint32_t ovf = 0;
    {
      TQ_CUDA(cudaMemcpyAsync(pinned_scratch(c), tail, 16, cudaMemcpyDeviceToHost, st));
      { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
      ovf = ((uint32_t*)pinned_scratch(c))[2];
    }
    if (ovf) {  // a run's integer sum beyond int64: re-run exactly on the hash table
      dfree(c, base, tbytes, st);
      direct = false;
      t = AggTable{};
      cap = cap0;
      setup(G);
    } else {
      // groups are counted by the finalize (its output cursor): capacity R + 1
      ngroups = cap;
    }
  }
  for (int attempt = 0; !direct; ++attempt) {
    tbytes = cap * 4 + cap * kwa * 8 + cap * std::max<u32>(1, nacc) * 16 + 64;
    uint8_t* base = (uint8_t*)dalloc(c, tbytes, st);
    t.state = (uint32_t*)base;
    t.keys = (u64*)(base + round_up(cap * 4, 16));
    t.acc = t.keys + cap * kwa;
    t.cap = cap;
    uint8_t* tail = (uint8_t*)(t.acc + cap * std::max<u32>(1, nacc) * 2);
    t.nused = (unsigned long long*)tail;
    t.overflow = (uint32_t*)(tail + 8);
    TQ_CUDA(cudaMemsetAsync(tail, 0, 16, st));
    // only the state words: a slot's accumulators are initialised by the
    // thread that claims it (AccClaimInit, kernel_common.cuh)
    TQ_CUDA(cudaMemsetAsync(t.state, 0, cap * 4, st));
    p.agg = t;
    launch(c, SINK_AGG, L, P, st);
    uint32_t ovf = 0;
    {
      TQ_CUDA(cudaMemcpyAsync(pinned_scratch(c), tail, 16, cudaMemcpyDeviceToHost, st));
      { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
      ngroups = ((uint64_t*)pinned_scratch(c))[0];
      ovf = ((uint32_t*)pinned_scratch(c))[2];
    }
    if (!ovf) break;
    dfree(c, base, tbytes, st);
    if (attempt > 12) fail(TQ_RESERVATION_EXCEEDED, "aggregation table overflow");
    // x16 while the input is much larger than the table (high-cardinality
    // group-by: fewer discarded attempts), else x4
    cap *= in->rows >= 8 * cap ? 16 : 4;
    // more than ~0.5M groups: a per-CTA table of <= 64 groups only misses and
    // its shared memory halves the resident CTAs -> global table only
    if (G && cap >= (1ull << 22)) {
      G = 0;
      setup(0);
    }
  }
  uint8_t* tbase = (uint8_t*)t.state;
  // ---- output batch
  std::vector<tq_column> sch;
  std::vector<bool> wv;
  for (int h : kh) {
    const Operand& o = P.pb.root(h);
    tq_column d{};
    d.kind = out_kind_of(o, in, P.pb, &d.precision, &d.scale);
    sch.push_back(d);
    wv.push_back(o.maybe_null);
  }
  std::vector<AggPlan> raw;
  if (!ap) {  // PARTIAL: raw accumulators
    for (u32 i = 0; i < nacc; ++i) {
      AggPlan a{};
      a.acc = (uint8_t)i;
      a.cnt = 0xff;
      // (raw_ops: the ORIGINAL accumulator ops when merging partials, whose
      // counts are summed as ints but stay Int64 partial columns)
      switch (raw_ops ? (*raw_ops)[i] : acc[i].op) {
        case ACC_SUM_I: case ACC_MIN_I: case ACC_MAX_I: a.kind = AO_SUM_DEC; a.col.kind = TQ_DECIMAL; a.col.precision = 38; break;
        case ACC_CNT: a.kind = AO_SUM_I64; a.col.kind = TQ_INT64; break;
        default: a.kind = AO_SUM_F; a.col.kind = TQ_FLOAT64;
      }
      raw.push_back(a);
    }
    ap = &raw;
  }
  for (auto& a : *ap) {
    sch.push_back(a.col);
    bool can_null = a.kind != AO_CNT && a.cnt != 0xff && a.nullable;
    wv.push_back(can_null);
  }
  try {
    alloc_batch(c, ngroups, sch, wv, out, st);
  } catch (...) {
    dfree(c, tbase, tbytes, st);
    throw;
  }
  if (ngroups > 0) {
    FinalParams f{};
    f.t = t;
    f.kwa = kwa;
    f.nacc = nacc;
    f.nkeys = (u32)kh.size();
    f.naggs = (u32)ap->size();
    u32 word = 0;
    for (u32 k = 0; k < f.nkeys; ++k) {
      KeyOut& ko = f.keys[k];
      ko.kind = out->cols[k].kind;
      ko.word = (uint8_t)word;
      ko.bit = (uint8_t)k;
      ko.values = (uint8_t*)out->cols[k].values;
      ko.validity = out->cols[k].validity;
      word += p.keys[k].words;
    }
    for (u32 a = 0; a < f.naggs; ++a) {
      const AggPlan& pl = (*ap)[a];
      AggOut& ao = f.aggs[a];
      ao.kind = pl.kind;
      ao.acc = pl.acc;
      ao.cnt = pl.kind == AO_CNT ? 0xff : pl.cnt;
      if (pl.kind == AO_AVG_I || pl.kind == AO_AVG_F) ao.cnt = pl.cnt;
      ao.scale = pl.scale;
      ao.values = (uint8_t*)out->cols[f.nkeys + a].values;
      ao.validity = out->cols[f.nkeys + a].validity;
    }
    f.direct = direct ? 1u : 0u;
    f.cnt_acc = cnt_idx;
    f.key_min = kmin;
    f.null_slot = R;
    f.counter = (unsigned long long*)(t.nused + 0);  // reuse as output cursor
    TQ_CUDA(cudaMemsetAsync(t.nused, 0, 8, st));
    u32 nb = (u32)std::min<uint64_t>((uint64_t)c->sms * 16, (cap + kFinItems * 256 - 1) / (kFinItems * 256));
    const int ph = prof_begin(c, "agg_final", st);
    k_agg_final<<<nb, 256, 0, st>>>(f);
    prof_end(c, ph, st);
    counted_launch(c);
    TQ_CUDA(cudaGetLastError());
    if (direct) {  // the output was sized for every slot: trim to the groups written
      uint64_t n = 0;
      {
        TQ_CUDA(cudaMemcpyAsync(pinned_scratch(c), t.nused, 8, cudaMemcpyDeviceToHost, st));
        { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
        n = ((uint64_t*)pinned_scratch(c))[0];
      }
      out->rows = n;
      for (uint32_t i = 0; i < out->ncols; ++i) {
        out->cols[i].values_bytes = n * width_of(out->cols[i].kind);
        if (n == 0) out->cols[i].validity = nullptr;
      }
    }
  }
  dfree(c, tbase, tbytes, st);
}

static std::vector<int> key_handles(Prog& P, const uint32_t* keys, uint32_t nkeys) {
  std::vector<int> kh;
  for (uint32_t k = 0; k < nkeys; ++k) {
    if (keys[k] >= P.outs.size()) fail(TQ_INVALID_PLAN, "key column out of range");
    kh.push_back(P.outs[keys[k]]);
  }
  return kh;
}

static void run_aggregate(tq_ctx* c, const tq_batch* in, Prog& P, const uint32_t* keys, uint32_t nkeys,
                          const tq_agg* aggs, uint32_t naggs, tq_batch* out, cudaStream_t st) {
  AggSpec S = plan_aggs(in, P, aggs, naggs);
  agg_core(c, in, P, key_handles(P, keys, nkeys), S.acc, &S.ap, out, st);
}

// aggregate_execute over fixed-width key columns (every input column projected)
void run_aggregate_plain(tq_ctx* c, const tq_batch* in, const uint32_t* keys, uint32_t nkeys, const tq_agg* aggs,
                         uint32_t naggs, tq_batch* out, cudaStream_t st) {
  Prog P(schema_of(in));
  compile_prog(P, in, nullptr, nullptr, 0, true);
  run_aggregate(c, in, P, keys, nkeys, aggs, naggs, out, st);
}

// ================================================================== take / concat / slice
// dst already points at the first destination row; validity bits land at
// dbit + i of dvalid (bitmap zeroed by the allocator).
__global__ void k_take_fixed(const uint8_t* src, const uint8_t* svalid, const u64* ids, u64 n, u32 width,
                             uint8_t* dst, uint8_t* dvalid, u64 id_base, u64 dbit) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    u64 r = ids ? ids[i] : id_base + i;
    if (width == 16) ((ulonglong2*)dst)[i] = ((const ulonglong2*)src)[r];
    else if (width == 8) ((u64*)dst)[i] = ((const u64*)src)[r];
    else if (width == 1) dst[i] = src[r];
    if (dvalid && (!svalid || bm_get(svalid, r))) bm_set_atomic(dvalid, dbit + i);
  }
}
__global__ void k_take_utf8_len(const int32_t* soff, const u64* ids, u64 n, u32* len, u64 id_base) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    u64 r = ids ? ids[i] : id_base + i;
    len[i] = (u32)(soff[r + 1] - soff[r]);
  }
}
__global__ void k_take_utf8_copy(const uint8_t* src, const int32_t* soff, const u64* ids, u64 n, const u64* doff,
                                 uint8_t* dst, int32_t* doff32, u64 id_base, int32_t out_base) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    u64 r = ids ? ids[i] : id_base + i;
    int32_t a = soff[r], e = soff[r + 1];
    u64 o = doff[i];
    for (int32_t k = a; k < e; ++k) dst[o + (k - a)] = src[k];
    doff32[i] = out_base + (int32_t)o;
    if (i == n - 1) doff32[n] = out_base + (int32_t)(o + (e - a));
  }
}

static u32 grid_for(tq_ctx* c, u64 n) { return (u32)std::max<u64>(1, std::min<u64>((n + 255) / 256, c->sms * 8)); }

// gather rows (ids on device, or the contiguous range [base, base+n)) of `in` into
// rows [dst_row, dst_row+n) of the already-allocated `out` (dst bitmaps zeroed).
static void gather_into(tq_ctx* c, const tq_batch* in, const u64* ids, u64 n, u64 base, tq_batch* out, u64 dst_row,
                        std::vector<int32_t>& utf8_cursor, cudaStream_t st) {
  if (n == 0) return;
  for (uint32_t k = 0; k < in->ncols; ++k) {
    const tq_column& s = in->cols[k];
    tq_column& d = out->cols[k];
    const uint8_t* svalid = in->rows ? s.validity : nullptr;
    if (s.kind != TQ_UTF8) {
      u32 w = (u32)width_of(s.kind);
      k_take_fixed<<<grid_for(c, n), 256, 0, st>>>((const uint8_t*)s.values, svalid, ids, n, w,
                                                    (uint8_t*)d.values + dst_row * w, d.validity, base, dst_row);
      counted_launch(c);
    } else {
      u32* len = (u32*)dalloc(c, n * 4, st);
      u64* off = (u64*)dalloc(c, (n + 1) * 8, st);
      k_take_utf8_len<<<grid_for(c, n), 256, 0, st>>>(s.offsets, ids, n, len, base);
      counted_launch(c);
      scan_u32(c, len, n, off, off + n, st);
      k_take_utf8_copy<<<grid_for(c, n), 256, 0, st>>>((const uint8_t*)s.values, s.offsets, ids, n, off,
                                                        (uint8_t*)d.values + utf8_cursor[k], d.offsets + dst_row,
                                                        base, utf8_cursor[k]);
      counted_launch(c);
      if (d.validity) {
        k_take_fixed<<<grid_for(c, n), 256, 0, st>>>(nullptr, svalid, ids, n, 0, nullptr, d.validity, base, dst_row);
        counted_launch(c);
      }
      uint64_t tot = 0;
      TQ_CUDA(cudaMemcpyAsync(&tot, off + n, 8, cudaMemcpyDeviceToHost, st));
      { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
      utf8_cursor[k] += (int32_t)tot;
      dfree(c, len, n * 4, st);
      dfree(c, off, (n + 1) * 8, st);
    }
    TQ_CUDA(cudaGetLastError());
  }
}

// utf8 bytes of rows ids / range
static u64 utf8_bytes_of(tq_ctx* c, const tq_column& s, const u64* ids, u64 n, u64 base, cudaStream_t st) {
  if (n == 0) return 0;
  if (!ids) {
    int32_t a = 0, e = 0;
    TQ_CUDA(cudaMemcpyAsync(&a, s.offsets + base, 4, cudaMemcpyDeviceToHost, st));
    TQ_CUDA(cudaMemcpyAsync(&e, s.offsets + base + n, 4, cudaMemcpyDeviceToHost, st));
    { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
    return (u64)(e - a);
  }
  u32* len = (u32*)dalloc(c, n * 4, st);
  u64* off = (u64*)dalloc(c, (n + 1) * 8, st);
  k_take_utf8_len<<<grid_for(c, n), 256, 0, st>>>(s.offsets, ids, n, len, 0);
  counted_launch(c);
  scan_u32(c, len, n, off, off + n, st);
  u64 tot = 0;
  TQ_CUDA(cudaMemcpyAsync(&tot, off + n, 8, cudaMemcpyDeviceToHost, st));
  { TQ_HT("stream sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
  dfree(c, len, n * 4, st);
  dfree(c, off, (n + 1) * 8, st);
  return tot;
}

__global__ void k_set_first_offset(int32_t* off) { off[0] = 0; }

static void take_impl(tq_ctx* c, const tq_batch* in, const u64* ids, u64 n, u64 base, tq_batch* out,
                      cudaStream_t st) {
  std::vector<tq_column> sch(in->cols, in->cols + in->ncols);
  std::vector<bool> wv;
  std::vector<uint64_t> ub;
  for (uint32_t k = 0; k < in->ncols; ++k) {
    wv.push_back(in->rows > 0 && in->cols[k].validity != nullptr);  // take: bitmap iff input had one (n>0)
    ub.push_back(in->cols[k].kind == TQ_UTF8 ? utf8_bytes_of(c, in->cols[k], ids, n, base, st) : 0);
  }
  alloc_batch(c, n, sch, wv, out, st, &ub);
  std::vector<int32_t> cur(in->ncols, 0);
  for (uint32_t k = 0; k < in->ncols; ++k)
    if (in->cols[k].kind == TQ_UTF8) {
      k_set_first_offset<<<1, 1, 0, st>>>(out->cols[k].offsets);
      counted_launch(c);
    }
  gather_into(c, in, ids, n, base, out, 0, cur, st);
}

}  // namespace tq

using namespace tq;

extern "C" {

tq_status tq_take(tq_ctx* c, const tq_batch* in, const uint64_t* ids, uint64_t n, tq_batch* out, void* stream) {
  return guard([&] {
    check_device_batch(in);
    take_impl(c, in, (const u64*)ids, n, 0, out, pick(c, stream));
  });
}

tq_status tq_slice(tq_ctx* c, const tq_batch* in, uint64_t start, uint64_t len, tq_batch* out, void* stream) {
  return guard([&] {
    check_device_batch(in);
    if (start + len > in->rows) fail(TQ_INTERNAL, "slice out of range");
    take_impl(c, in, nullptr, len, start, out, pick(c, stream));
  });
}

tq_status tq_concat(tq_ctx* c, const tq_batch* ins, uint32_t n, tq_batch* out, void* stream) {
  return guard([&] {
    if (n == 0) fail(TQ_INTERNAL, "concat of nothing");
    cudaStream_t st = pick(c, stream);
    const tq_batch& f = ins[0];
    uint64_t rows = 0;
    for (uint32_t i = 0; i < n; ++i) {
      check_device_batch(&ins[i]);
      if (ins[i].ncols != f.ncols) fail(TQ_SCHEMA_MISMATCH, "concat over differing schemas");
      for (uint32_t k = 0; k < f.ncols; ++k)
        if (ins[i].cols[k].kind != f.cols[k].kind || ins[i].cols[k].scale != f.cols[k].scale ||
            ins[i].cols[k].precision != f.cols[k].precision)
          fail(TQ_SCHEMA_MISMATCH, "concat over differing schemas");
      rows += ins[i].rows;
    }
    std::vector<tq_column> sch(f.cols, f.cols + f.ncols);
    std::vector<bool> wv(f.ncols, false);
    std::vector<uint64_t> ub(f.ncols, 0);
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t k = 0; k < f.ncols; ++k) {
        if (ins[i].rows > 0 && ins[i].cols[k].validity) wv[k] = true;  // bitmap if any input has one
        if (f.cols[k].kind == TQ_UTF8) ub[k] += utf8_bytes_of(c, ins[i].cols[k], nullptr, ins[i].rows, 0, st);
      }
    alloc_batch(c, rows, sch, wv, out, st, &ub);
    std::vector<int32_t> cur(f.ncols, 0);
    for (uint32_t k = 0; k < f.ncols; ++k)
      if (f.cols[k].kind == TQ_UTF8) {
        k_set_first_offset<<<1, 1, 0, st>>>(out->cols[k].offsets);
        counted_launch(c);
      }
    uint64_t at = 0;
    for (uint32_t i = 0; i < n; ++i) {
      gather_into(c, &ins[i], nullptr, ins[i].rows, 0, out, at, cur, st);
      at += ins[i].rows;
    }
  });
}

// rebatch cut points (transform.cpp:133-150): one thread walks the prefix
// sums of the per-row cost, each cut a binary search for the first row where
// the bytes since the last cut reach the target.
__global__ void k_rebatch_cuts(const u64* pref, u64 rows, u64 target, u64* cuts, u32 cap, u32* ncuts) {
  u64 start = 0;
  u32 n = 0;
  while (start < rows && n < cap) {
    // first r >= start with pref[r + 1] - pref[start] >= target
    u64 lo = start, hi = rows;  // answer in [start, rows)
    while (lo < hi) {
      const u64 mid = (lo + hi) / 2;
      if (pref[mid + 1] - pref[start] >= target) hi = mid;
      else lo = mid + 1;
    }
    if (lo + 1 >= rows) break;  // the rest is the last batch
    cuts[n++] = lo + 1;
    start = lo + 1;
  }
  *ncuts = n;
}

__global__ void k_row_cost(const int32_t* const* offs, u32 nutf8, u64 rows, u32 fixed, u32* cost) {
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (u64)gridDim.x * blockDim.x) {
    u32 c = fixed;
    for (u32 k = 0; k < nutf8; ++k) c += (u32)(offs[k][r + 1] - offs[k][r]);
    cost[r] = c;
  }
}

tq_status tq_rebatch(tq_ctx* c, const tq_batch* ins, uint32_t n, uint64_t target, tq_batch** outs, uint32_t* nout,
                     void* stream) {
  return guard([&] {
    if (target == 0) fail(TQ_INTERNAL, "rebatch target must be positive");
    *outs = nullptr;
    *nout = 0;
    if (n == 0) return;
    cudaStream_t st = pick(c, stream);
    tq_batch all{};
    bool owned = false;
    if (n == 1) {
      check_device_batch(&ins[0]);
      all = ins[0];
    } else {
      tq_status r = tq_concat(c, ins, n, &all, st);
      if (r != TQ_OK) fail(r, g_err);
      owned = true;
    }
    // batch_size_bytes (types.cpp:166-170) and the fixed per-row estimate
    uint64_t total = 0, fixed = 0;
    std::vector<const int32_t*> utf8;
    for (uint32_t k = 0; k < all.ncols; ++k) {
      const tq_column& col = all.cols[k];
      total += col.values_bytes;
      if (col.validity && all.rows) total += (all.rows + 7) / 8;
      if (col.kind == TQ_UTF8) {
        total += (all.rows + 1) * 4;
        utf8.push_back(col.offsets);
      }
      fixed += width_of(col.kind) + 1;
    }
    std::vector<uint64_t> cuts;
    if (all.rows > 0 && total > target * 2) {
      if (utf8.empty()) {
        // every row costs `fixed`: cut every ceil(target / fixed) rows
        const uint64_t k = (target + fixed - 1) / fixed;
        for (uint64_t r = k; r < all.rows; r += k) cuts.push_back(r);
      } else {
        const uint64_t rows = all.rows;
        u32* cost = (u32*)dalloc(c, rows * 4, st);
        u64* pref = (u64*)dalloc(c, (rows + 1) * 8, st);
        const int32_t** d_offs = (const int32_t**)dalloc(c, utf8.size() * 8, st);
        TQ_CUDA(cudaMemcpyAsync(d_offs, utf8.data(), utf8.size() * 8, cudaMemcpyHostToDevice, st));
        k_row_cost<<<grid_for(c, rows), 256, 0, st>>>(d_offs, (u32)utf8.size(), rows, (u32)fixed, cost);
        counted_launch(c);
        // exclusive scan into pref[0..rows), total at pref[rows]: pref[r+1] - pref[s] = bytes of rows s..r
        scan_u32(c, cost, rows, pref, pref + rows, st);
        const uint32_t cap = (uint32_t)std::min<uint64_t>(rows, total / std::max<uint64_t>(1, target / 2) + 4);
        u64* d_cuts = (u64*)dalloc(c, cap * 8ull + 8, st);
        u32* d_n = (u32*)(d_cuts + cap);
        k_rebatch_cuts<<<1, 1, 0, st>>>(pref, rows, target, d_cuts, cap, d_n);
        counted_launch(c);
        uint32_t nc = 0;
        TQ_CUDA(cudaMemcpyAsync(&nc, d_n, 4, cudaMemcpyDeviceToHost, st));
        TQ_CUDA(cudaStreamSynchronize(st));
        cuts.resize(nc);
        if (nc) TQ_CUDA(cudaMemcpy(cuts.data(), d_cuts, nc * 8ull, cudaMemcpyDeviceToHost));
        dfree(c, d_cuts, cap * 8ull + 8, st);
        dfree(c, d_offs, utf8.size() * 8, st);
        dfree(c, pref, (rows + 1) * 8, st);
        dfree(c, cost, rows * 4, st);
      }
    }
    std::vector<tq_batch> parts;
    if (cuts.empty()) {
      if (owned) {
        parts.push_back(all);
        owned = false;
      } else {
        tq_batch cp{};
        take_impl(c, &all, nullptr, all.rows, 0, &cp, st);  // the reference returns a copy
        parts.push_back(cp);
      }
    } else {
      uint64_t start = 0;
      cuts.push_back(all.rows);
      for (uint64_t e : cuts) {
        tq_batch part{};
        take_impl(c, &all, nullptr, e - start, start, &part, st);
        parts.push_back(part);
        start = e;
      }
    }
    if (owned) tq_batch_free(c, &all);
    *outs = (tq_batch*)std::malloc(sizeof(tq_batch) * parts.size());
    std::memcpy(*outs, parts.data(), sizeof(tq_batch) * parts.size());
    *nout = (uint32_t)parts.size();
  });
}

}  // extern "C"

// ================================================================== Utf8 columns on the pipeline path
// The pipeline kernels move fixed-width values.  A Utf8 column rides through
// filter / project / partition as the ROW ID of its row (an appended iota
// column the program copies instead), and the strings are gathered by those
// ids afterwards with the reference's take (transform.cpp:90-120: bitmap iff
// the input had one).  Utf8 partition keys: a pre-pass computes the row's
// partition hash — fnv1a64 chained over the key columns' bytes, the string's
// bytes for Utf8 (a null string adds none, a null fixed-width key its width in
// zero bytes) — and the kernel partitions on it as is (key_prehashed).
// Utf8 group keys (aggregate_execute) and join keys / payloads (join_execute):
// aggregate_utf8_keys / join_probe_utf8 below.  Utf8 in predicates and
// arithmetic: InvalidPlan.
namespace tq {

__global__ void k_iota(u64* v, u64 n) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) v[i] = i;
}

struct HashKeyCol {
  const uint8_t* values;
  const int32_t* offsets;  // Utf8
  const uint8_t* validity;
  uint32_t width;          // fixed width (0 = Utf8)
};
struct HashKeys {
  HashKeyCol k[kMaxKeys];
  u32 n;
};
__global__ void k_partition_hash(const __grid_constant__ HashKeys K, u64 rows, u64* out) {
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (u64)gridDim.x * blockDim.x) {
    u64 h = kFnvBasis;
    for (u32 k = 0; k < K.n; ++k) {
      const HashKeyCol& c = K.k[k];
      const bool valid = !c.validity || bm_get(c.validity, r);
      if (c.width == 0) {
        if (!valid) continue;
        for (int32_t i = c.offsets[r]; i < c.offsets[r + 1]; ++i) h = (h ^ c.values[i]) * kFnvPrime;
      } else {
        for (u32 i = 0; i < c.width; ++i) h = (h ^ (valid ? c.values[r * c.width + i] : 0)) * kFnvPrime;
      }
    }
    out[r] = h;
  }
}

struct Utf8Lower {
  bool active = false;
  tq_batch aug{};                // the input + iota (row id) column [+ partition hash column]
  std::vector<tq_column> cols;
  uint32_t rowid = 0, hash = 0;  // column indices in aug
  void* iota = nullptr;
  void* hmem = nullptr;
  uint64_t bytes = 0;
  tq_ctx* c = nullptr;
  cudaStream_t st = nullptr;
  ~Utf8Lower() {
    if (iota) dfree(c, iota, bytes, st);
    if (hmem) dfree(c, hmem, bytes, st);
  }
};

bool has_utf8(const tq_batch* in) {
  for (uint32_t i = 0; i < in->ncols; ++i)
    if (in->cols[i].kind == TQ_UTF8) return true;
  return false;
}

// aug = in + an Int64 row-id column (+ the partition hash of `hash_keys`)
void utf8_lower(tq_ctx* c, const tq_batch* in, Utf8Lower& U, cudaStream_t st, const uint32_t* hash_keys = nullptr,
                uint32_t nhash = 0) {
  U.active = true;
  U.c = c;
  U.st = st;
  U.bytes = std::max<uint64_t>(8, in->rows * 8);
  U.cols.assign(in->cols, in->cols + in->ncols);
  U.iota = dalloc(c, U.bytes, st);
  k_iota<<<grid_for(c, in->rows), 256, 0, st>>>((u64*)U.iota, in->rows);
  counted_launch(c);
  tq_column id{};
  id.kind = TQ_INT64;
  id.values = U.iota;
  id.values_bytes = in->rows * 8;
  U.rowid = (uint32_t)U.cols.size();
  U.cols.push_back(id);
  if (nhash) {
    if (nhash > (uint32_t)kMaxKeys) fail(TQ_INVALID_PLAN, "too many keys");
    HashKeys K{};
    K.n = nhash;
    for (uint32_t k = 0; k < nhash; ++k) {
      if (hash_keys[k] >= in->ncols) fail(TQ_INVALID_PLAN, "key column out of range");
      const tq_column& col = in->cols[hash_keys[k]];
      if (col.kind == TQ_FLOAT64) fail(TQ_INVALID_PLAN, "unsupported partition key type");
      K.k[k] = HashKeyCol{(const uint8_t*)col.values, col.offsets, in->rows ? col.validity : nullptr,
                          col.kind == TQ_UTF8 ? 0u : (uint32_t)width_of(col.kind)};
    }
    U.hmem = dalloc(c, U.bytes, st);
    k_partition_hash<<<grid_for(c, in->rows), 256, 0, st>>>(K, in->rows, (u64*)U.hmem);
    counted_launch(c);
    tq_column hc{};
    hc.kind = TQ_INT64;
    hc.values = U.hmem;
    hc.values_bytes = in->rows * 8;
    U.hash = (uint32_t)U.cols.size();
    U.cols.push_back(hc);
  }
  TQ_CUDA(cudaGetLastError());
  U.aug = *in;
  U.aug.ncols = (uint32_t)U.cols.size();
  U.aug.cols = U.cols.data();
  U.aug.owner = nullptr;
}

// The expressions the kernel evaluates: a pure Utf8 column reference becomes
// the row-id column (src[j] = that Utf8 input column), anything else is kept.
struct LoweredExprs {
  std::vector<std::vector<tq_expr_node>> nodes;
  std::vector<tq_expr> ex;
  std::vector<int> src;  // per output: the Utf8 input column to gather, or -1
};
void lower_exprs(const tq_batch* in, const Utf8Lower& U, const tq_expr* exprs, uint32_t n, LoweredExprs& L) {
  const uint32_t cnt = exprs ? n : in->ncols;
  L.nodes.resize(cnt);
  for (uint32_t j = 0; j < cnt; ++j) {
    tq_expr_node col{};
    col.tag = TQ_EX_COL;
    if (!exprs) {
      col.column = in->cols[j].kind == TQ_UTF8 ? U.rowid : j;
      L.nodes[j] = {col};
      L.src.push_back(in->cols[j].kind == TQ_UTF8 ? (int)j : -1);
    } else {
      const tq_expr& e = exprs[j];
      const bool utf8_col = e.len == 1 && e.nodes[0].tag == TQ_EX_COL && e.nodes[0].column < in->ncols &&
                            in->cols[e.nodes[0].column].kind == TQ_UTF8;
      if (utf8_col) {
        col.column = U.rowid;
        L.nodes[j] = {col};
        L.src.push_back((int)e.nodes[0].column);
      } else {
        L.nodes[j].assign(e.nodes, e.nodes + e.len);
        L.src.push_back(-1);
      }
    }
  }
  for (auto& v : L.nodes) L.ex.push_back(tq_expr{v.data(), (uint32_t)v.size(), 0});
}

// Replace every row-id output column j (src[j] >= 0) by the strings of input
// column src[j] gathered at those ids; drop the outputs >= keep.
void utf8_raise(tq_ctx* c, const tq_batch* in, const std::vector<int>& src, uint32_t keep, tq_batch* out,
                cudaStream_t st) {
  Owner* own = (Owner*)out->owner;
  auto release = [&](void* p) {
    for (size_t b = 0; b < own->bufs.size(); ++b)
      if (own->bufs[b].first == p) {
        dfree(c, p, own->bufs[b].second, st);
        own->bufs.erase(own->bufs.begin() + b);
        return;
      }
  };
  for (uint32_t j = 0; j < out->ncols && j < src.size(); ++j) {
    if (src[j] < 0) continue;
    tq_batch one{in->rows, 1, TQ_MEM_DEVICE, &in->cols[src[j]], nullptr};
    tq_batch g{};
    take_impl(c, &one, (const u64*)out->cols[j].values, out->rows, 0, &g, st);
    release(out->cols[j].values);
    if (out->cols[j].validity) release(out->cols[j].validity);
    out->cols[j] = g.cols[0];
    Owner* go = (Owner*)g.owner;
    for (auto& b : go->bufs) own->bufs.push_back(b);
    delete go;
    std::free(g.cols);
  }
  for (uint32_t j = keep; j < out->ncols; ++j) {
    release(out->cols[j].values);
    if (out->cols[j].validity) release(out->cols[j].validity);
  }
  out->ncols = std::min(out->ncols, keep);
}

// ---- Utf8 group keys (aggregate_execute: a group is one key
// VALUE, a string by its bytes).  The kernels group fixed-width words, so each
// Utf8 key column is replaced by the fnv1a64 of its bytes (a null string stays
// null) and every group also takes MIN(row id), a representative row whose
// string becomes the output key (take, transform.cpp:90-120).  Grouping by the
// hash equals grouping by the string iff no two different strings share a hash:
// that is CHECKED, not assumed — one row per hash (MIN(row id) by hash) is
// joined back to every row and the bytes are compared; a collision fails the
// operator (Internal) instead of merging two groups.

// flag = 1 if the strings at rows a[i] and b[i] differ, for any i
__global__ void k_utf8_pairs_differ(const uint8_t* bytes, const int32_t* off, const long long* a,
                                    const long long* b, u64 n, u32* flag) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const long long x = a[i], y = b[i];
    if (x == y) continue;
    const int32_t x0 = off[x], xl = off[x + 1] - x0, y0 = off[y], yl = off[y + 1] - y0;
    bool diff = xl != yl;
    for (int32_t j = 0; !diff && j < xl; ++j) diff = bytes[x0 + j] != bytes[y0 + j];
    if (diff) atomicOr(flag, 1u);
  }
}

static void status_check(tq_status s) {
  if (s != TQ_OK) fail(s, tq_last_error());
}

struct DevBufs {  // scratch buffers freed on every exit path
  tq_ctx* c;
  cudaStream_t st;
  std::vector<std::pair<void*, uint64_t>> v;
  void* get(uint64_t bytes) {
    v.push_back({dalloc(c, bytes, st), bytes});
    return v.back().first;
  }
  ~DevBufs() {
    for (auto& b : v) dfree(c, b.first, b.second, st);
  }
};

// every non-null row's string equals the string of the first row with its hash
static void check_utf8_hash_unique(tq_ctx* c, const tq_batch* in, const tq_batch* aug, uint32_t col, uint32_t rid,
                                   cudaStream_t st, DevBufs& B) {
  tq_batch reps{};  // [hash, MIN(row id)] per distinct hash
  const tq_agg mn{TQ_AGG_MIN, rid};
  run_aggregate_plain(c, aug, &col, 1, &mn, 1, &reps, st);
  tq_join_table* jt = nullptr;
  tq_batch pairs{};
  const uint32_t k0 = 0;
  try {
    status_check(tq_join_build(c, &reps, &k0, 1, &jt, st));
    tq_column pc[2] = {aug->cols[col], aug->cols[rid]};
    tq_batch probe{aug->rows, 2, TQ_MEM_DEVICE, pc, nullptr};
    status_check(tq_join_probe(c, jt, &probe, &k0, 1, &pairs, st));  // [hash, rep, hash, row id]
    u32* flag = (u32*)B.get(4);
    TQ_CUDA(cudaMemsetAsync(flag, 0, 4, st));
    if (pairs.rows) {
      const tq_column& s = in->cols[col];
      k_utf8_pairs_differ<<<grid_for(c, pairs.rows), 256, 0, st>>>(
          (const uint8_t*)s.values, s.offsets, (const long long*)pairs.cols[1].values,
          (const long long*)pairs.cols[3].values, pairs.rows, flag);
      counted_launch(c);
      TQ_CUDA(cudaGetLastError());
    }
    u32* pin = (u32*)pinned_scratch(c);
    TQ_CUDA(cudaMemcpyAsync(pin, flag, 4, cudaMemcpyDeviceToHost, st));
    TQ_CUDA(cudaStreamSynchronize(st));
    if (pin[0]) fail(TQ_INTERNAL, "utf8 group key: two different strings share a 64-bit hash (aggregate refused)");
  } catch (...) {
    if (pairs.cols) tq_batch_free(c, &pairs);
    if (jt) tq_join_table_destroy(c, jt);
    tq_batch_free(c, &reps);
    throw;
  }
  tq_batch_free(c, &pairs);
  tq_join_table_destroy(c, jt);
  tq_batch_free(c, &reps);
}

void aggregate_utf8_keys(tq_ctx* c, const tq_batch* in, const uint32_t* keys, uint32_t nkeys, const tq_agg* aggs,
                         uint32_t naggs, tq_batch* out, cudaStream_t st) {
  for (uint32_t a = 0; a < naggs; ++a)
    if (aggs[a].fn != TQ_AGG_COUNT_STAR && aggs[a].column < in->ncols && in->cols[aggs[a].column].kind == TQ_UTF8)
      fail(TQ_INVALID_PLAN, "utf8 aggregate unsupported");
  const uint64_t rows = in->rows, bytes = std::max<uint64_t>(8, rows * 8);
  DevBufs B{c, st, {}};
  u64* rid = (u64*)B.get(bytes);
  k_iota<<<grid_for(c, rows), 256, 0, st>>>(rid, rows);
  counted_launch(c);
  tq_column rc{};
  rc.kind = TQ_INT64;
  rc.values = rid;
  rc.values_bytes = rows * 8;
  std::vector<tq_column> cols(in->cols, in->cols + in->ncols);
  std::vector<uint32_t> hashed;
  std::vector<int> src(nkeys + naggs, -1);  // output key column j -> its Utf8 input column
  for (uint32_t k = 0; k < nkeys; ++k) {
    const uint32_t col = keys[k];
    if (col >= in->ncols) fail(TQ_INVALID_PLAN, "key column out of range");
    if (in->cols[col].kind != TQ_UTF8) continue;
    src[k] = (int)col;
    if (std::find(hashed.begin(), hashed.end(), col) != hashed.end()) continue;
    HashKeys K{};
    K.n = 1;
    K.k[0] = HashKeyCol{(const uint8_t*)in->cols[col].values, in->cols[col].offsets,
                        rows ? in->cols[col].validity : nullptr, 0u};
    u64* h = (u64*)B.get(bytes);
    k_partition_hash<<<grid_for(c, rows), 256, 0, st>>>(K, rows, h);
    counted_launch(c);
    tq_column hc{};
    hc.kind = TQ_INT64;
    hc.values = h;
    hc.values_bytes = rows * 8;
    hc.validity = rows ? in->cols[col].validity : nullptr;
    cols[col] = hc;
    hashed.push_back(col);
  }
  for (auto& col : cols)  // Utf8 columns no key or aggregate reads: fixed-width stand-ins
    if (col.kind == TQ_UTF8) col = rc;
  TQ_CUDA(cudaGetLastError());
  const uint32_t ridc = (uint32_t)cols.size();
  cols.push_back(rc);
  tq_batch aug = *in;
  aug.ncols = (uint32_t)cols.size();
  aug.cols = cols.data();
  aug.owner = nullptr;
  for (uint32_t col : hashed) check_utf8_hash_unique(c, in, &aug, col, ridc, st, B);
  std::vector<tq_agg> ag(aggs, aggs + naggs);
  ag.push_back(tq_agg{TQ_AGG_MIN, ridc});
  run_aggregate_plain(c, &aug, keys, nkeys, ag.data(), (uint32_t)ag.size(), out, st);
  // the representative row ids into the Utf8 key columns, then gather their strings
  const tq_column& rep = out->cols[out->ncols - 1];
  for (uint32_t k = 0; k < nkeys; ++k)
    if (src[k] >= 0 && out->rows)
      TQ_CUDA(cudaMemcpyAsync(out->cols[k].values, rep.values, out->rows * 8, cudaMemcpyDeviceToDevice, st));
  src.resize(out->ncols, -1);
  utf8_raise(c, in, src, out->ncols - 1, out, st);
}

// ---- Utf8 join keys and payloads (join_execute).  Both sides
// are lowered like the aggregate's keys (Utf8 keys -> fnv1a64 of the bytes, Utf8
// payloads -> row ids, + a row-id column); the hash join produces candidate
// pairs, every pair whose key strings differ (a hash collision) is dropped — so
// the result is exact — and the output strings are gathered by row id.
struct Utf8Side {
  std::vector<tq_column> cols;
  tq_batch b{};
  uint32_t rid = 0;
  std::vector<std::pair<void*, uint64_t>> bufs;
};
static void utf8_lower_side(tq_ctx* c, const tq_batch* in, const uint32_t* keys, uint32_t nkeys, Utf8Side& S,
                            cudaStream_t st) {
  const uint64_t rows = in->rows, bytes = std::max<uint64_t>(8, rows * 8);
  u64* rid = (u64*)dalloc(c, bytes, st);
  S.bufs.push_back({rid, bytes});
  k_iota<<<grid_for(c, rows), 256, 0, st>>>(rid, rows);
  counted_launch(c);
  tq_column rc{};
  rc.kind = TQ_INT64;
  rc.values = rid;
  rc.values_bytes = rows * 8;
  S.cols.assign(in->cols, in->cols + in->ncols);
  std::vector<bool> is_key(in->ncols, false);
  for (uint32_t k = 0; k < nkeys; ++k) {
    if (keys[k] >= in->ncols) fail(TQ_INVALID_PLAN, "join key out of range");
    is_key[keys[k]] = true;
  }
  for (uint32_t i = 0; i < in->ncols; ++i) {
    if (in->cols[i].kind != TQ_UTF8) continue;
    if (!is_key[i]) {
      S.cols[i] = rc;
      continue;
    }
    HashKeys K{};
    K.n = 1;
    K.k[0] = HashKeyCol{(const uint8_t*)in->cols[i].values, in->cols[i].offsets, rows ? in->cols[i].validity : nullptr,
                        0u};
    u64* h = (u64*)dalloc(c, bytes, st);
    S.bufs.push_back({h, bytes});
    k_partition_hash<<<grid_for(c, rows), 256, 0, st>>>(K, rows, h);
    counted_launch(c);
    tq_column hc{};
    hc.kind = TQ_INT64;
    hc.values = h;
    hc.values_bytes = rows * 8;
    hc.validity = rows ? in->cols[i].validity : nullptr;
    S.cols[i] = hc;
  }
  TQ_CUDA(cudaGetLastError());
  S.rid = (uint32_t)S.cols.size();
  S.cols.push_back(rc);
  S.b = *in;
  S.b.ncols = (uint32_t)S.cols.size();
  S.b.cols = S.cols.data();
  S.b.owner = nullptr;
}

// keep[i] = 0 if the key strings of output row i differ (build row a[i], probe row b[i])
__global__ void k_utf8_pair_keep(const uint8_t* bb, const int32_t* bo, const uint8_t* pb, const int32_t* po,
                                 const long long* a, const long long* b, u64 n, uint8_t* keep, u32* any_drop) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const long long x = a[i], y = b[i];
    const int32_t x0 = bo[x], xl = bo[x + 1] - x0, y0 = po[y], yl = po[y + 1] - y0;
    bool diff = xl != yl;
    for (int32_t j = 0; !diff && j < xl; ++j) diff = bb[x0 + j] != pb[y0 + j];
    if (diff) {
      keep[i] = 0;
      atomicOr(any_drop, 1u);
    }
  }
}

// drop output columns (their buffers released), keeping the others in order
static void drop_columns(tq_ctx* c, tq_batch* out, const std::vector<bool>& drop, cudaStream_t st) {
  Owner* own = (Owner*)out->owner;
  auto release = [&](void* p) {
    for (size_t b = 0; b < own->bufs.size(); ++b)
      if (own->bufs[b].first == p) {
        dfree(c, p, own->bufs[b].second, st);
        own->bufs.erase(own->bufs.begin() + b);
        return;
      }
  };
  uint32_t w = 0;
  for (uint32_t j = 0; j < out->ncols; ++j) {
    if (j < drop.size() && drop[j]) {
      release(out->cols[j].values);
      if (out->cols[j].validity) release(out->cols[j].validity);
      continue;
    }
    out->cols[w++] = out->cols[j];
  }
  out->ncols = w;
}

void join_probe_utf8(tq_ctx* c, const tq_join_table* t, const tq_batch* probe, const uint32_t* keys, uint32_t nkeys,
                     tq_batch* out, cudaStream_t st);

}  // namespace tq

// ================================================================== operator entry points
namespace {
using namespace tq;

std::vector<uint32_t> iota_u32(uint32_t n) {
  std::vector<uint32_t> v(n);
  for (uint32_t i = 0; i < n; ++i) v[i] = i;
  return v;
}

// keys given as INPUT column indices: project every input column so that
// projected column i == input column i.
void compile_all(Prog& P, const tq_batch* in, const tq_expr* pred) { compile_prog(P, in, pred, nullptr, 0, true); }
}  // namespace

extern "C" {

// Filter / project / partition over a batch that holds Utf8 columns (see
// "Utf8 columns on the pipeline path").  part_keys: hash-partition keys given
// as INPUT column indices (hash_partition) or output indices (nullptr: none).
void materialize_utf8(tq_ctx* c, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs, uint32_t nexprs,
                      const uint32_t* keys, uint32_t nkeys, bool keys_are_inputs, uint32_t nparts, tq_batch* out,
                      uint64_t* part_offsets, cudaStream_t st) {
  // partition keys that are (or project) a Utf8 column are hashed by the pre-pass
  bool utf8_key = false;
  std::vector<uint32_t> in_keys;
  for (uint32_t k = 0; k < nkeys; ++k) {
    uint32_t col = keys[k];
    if (!keys_are_inputs) {
      if (!exprs) {
        col = keys[k];
      } else {
        if (keys[k] >= nexprs) fail(TQ_INVALID_PLAN, "key column out of range");
        const tq_expr& e = exprs[keys[k]];
        if (!(e.len == 1 && e.nodes[0].tag == TQ_EX_COL)) {
          // a computed key: fixed width by construction, no pre-pass unless another key needs it
          in_keys.push_back(~0u);
          continue;
        }
        col = e.nodes[0].column;
      }
    }
    if (col >= in->ncols) fail(TQ_INVALID_PLAN, "key column out of range");
    utf8_key |= in->cols[col].kind == TQ_UTF8;
    in_keys.push_back(col);
  }
  if (utf8_key)
    for (uint32_t k : in_keys)
      if (k == ~0u) fail(TQ_INVALID_PLAN, "a computed key next to a Utf8 key is not supported");
  Utf8Lower U;
  utf8_lower(c, in, U, st, utf8_key ? in_keys.data() : nullptr, utf8_key ? (uint32_t)in_keys.size() : 0);
  LoweredExprs L;
  lower_exprs(in, U, exprs, nexprs, L);
  const uint32_t nout = (uint32_t)L.ex.size();
  std::vector<uint32_t> kr;
  if (nkeys && utf8_key) {  // partition on the precomputed hash: an extra output, dropped after
    tq_expr_node h{};
    h.tag = TQ_EX_COL;
    h.column = U.hash;
    L.nodes.push_back({h});
    L.ex.push_back(tq_expr{L.nodes.back().data(), 1, 0});
    kr.push_back(nout);
  } else {
    for (uint32_t k = 0; k < nkeys; ++k) kr.push_back(keys[k]);
  }
  // (the kernel sees the batch with the row-id / hash columns; its program
  // never references a Utf8 column — a predicate or expression that does fails)
  for (size_t j = 0; j < L.nodes.size(); ++j) L.ex[j].nodes = L.nodes[j].data();
  Prog P(schema_of(&U.aug));
  compile_prog(P, &U.aug, pred, L.ex.data(), (uint32_t)L.ex.size(), false);
  MatArgs A;
  if (nkeys) {
    A.mode = MAT_PARTITION;
    A.key_roots = kr;
    A.nparts = nparts;
  }
  A.prehashed = nkeys && utf8_key;
  run_materialize(c, &U.aug, P, A, out, part_offsets, st);
  utf8_raise(c, in, L.src, nout, out, st);
}

tq_status tq_filter(tq_ctx* c, const tq_batch* in, tq_expr pred, tq_batch* out, void* stream) {
  return guard([&] {
    check_device_batch(in);
    if (has_utf8(in)) return materialize_utf8(c, in, &pred, nullptr, 0, nullptr, 0, false, 1, out, nullptr, pick(c, stream));
    Prog P(schema_of(in));
    compile_all(P, in, &pred);
    MatArgs A;
    run_materialize(c, in, P, A, out, nullptr, pick(c, stream));
  });
}

tq_status tq_project(tq_ctx* c, const tq_batch* in, const tq_expr* exprs, uint32_t n, tq_batch* out, void* stream) {
  return guard([&] {
    check_device_batch(in);
    if (has_utf8(in)) return materialize_utf8(c, in, nullptr, exprs, n, nullptr, 0, false, 1, out, nullptr, pick(c, stream));
    Prog P(schema_of(in));
    compile_prog(P, in, nullptr, exprs, n, false);
    MatArgs A;
    run_materialize(c, in, P, A, out, nullptr, pick(c, stream));
  });
}

tq_status tq_pipeline_materialize(tq_ctx* c, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                                  uint32_t nexprs, tq_batch* out, void* stream) {
  return guard([&] {
    check_device_batch(in);
    if (has_utf8(in))
      return materialize_utf8(c, in, pred, exprs, nexprs, nullptr, 0, false, 1, out, nullptr, pick(c, stream));
    Prog P(schema_of(in));
    compile_prog(P, in, pred, exprs, nexprs, exprs == nullptr);
    MatArgs A;
    run_materialize(c, in, P, A, out, nullptr, pick(c, stream));
  });
}

tq_status tq_hash_partition(tq_ctx* c, const tq_batch* in, const uint32_t* keys, uint32_t nkeys, uint32_t nparts,
                            tq_batch* out, uint64_t* part_offsets, void* stream) {
  return guard([&] {
    check_device_batch(in);
    if (has_utf8(in))
      return materialize_utf8(c, in, nullptr, nullptr, 0, keys, nkeys, true, nparts, out, part_offsets,
                              pick(c, stream));
    Prog P(schema_of(in));
    compile_all(P, in, nullptr);
    MatArgs A;
    A.mode = MAT_PARTITION;
    A.key_roots.assign(keys, keys + nkeys);
    A.nparts = nparts;
    run_materialize(c, in, P, A, out, part_offsets, pick(c, stream));
  });
}

tq_status tq_filter_async(tq_ctx* c, const tq_batch* in, tq_expr pred, tq_batch* out, uint64_t* slot,
                          void* stream) {
  return guard([&] {
    check_device_batch(in);
    if (!slot) fail(TQ_INVALID_PLAN, "asynchronous filter without a count slot");
    if (has_utf8(in)) fail(TQ_INVALID_PLAN, "no asynchronous form for Utf8 columns (their gather needs the count)");
    Prog P(schema_of(in));
    compile_all(P, in, &pred);
    MatArgs A;
    A.async_slot = slot;
    run_materialize(c, in, P, A, out, nullptr, pick(c, stream));
  });
}

tq_status tq_hash_partition_async(tq_ctx* c, const tq_batch* in, const uint32_t* keys, uint32_t nkeys,
                                  uint32_t nparts, tq_batch* out, uint64_t* slot, void* stream) {
  return guard([&] {
    check_device_batch(in);
    if (!slot) fail(TQ_INVALID_PLAN, "asynchronous partition without a count slot");
    if (has_utf8(in)) fail(TQ_INVALID_PLAN, "no asynchronous form for Utf8 columns (their gather needs the count)");
    Prog P(schema_of(in));
    compile_all(P, in, nullptr);
    MatArgs A;
    A.mode = MAT_PARTITION;
    A.key_roots.assign(keys, keys + nkeys);
    A.nparts = nparts;
    A.async_slot = slot;
    run_materialize(c, in, P, A, out, nullptr, pick(c, stream));
  });
}

void tq_batch_set_rows(tq_batch* b, uint64_t rows) {
  if (!b || rows > b->rows) return;
  b->rows = rows;
  for (uint32_t i = 0; i < b->ncols; ++i)
    if (b->cols[i].kind != TQ_UTF8) b->cols[i].values_bytes = rows * width_of(b->cols[i].kind);
}

tq_status tq_pipeline_partition(tq_ctx* c, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                                uint32_t nexprs, const uint32_t* keys, uint32_t nkeys, uint32_t nparts,
                                tq_batch* out, uint64_t* part_offsets, void* stream) {
  return guard([&] {
    check_device_batch(in);
    if (has_utf8(in))
      return materialize_utf8(c, in, pred, exprs, nexprs, keys, nkeys, false, nparts, out, part_offsets,
                              pick(c, stream));
    Prog P(schema_of(in));
    compile_prog(P, in, pred, exprs, nexprs, exprs == nullptr);
    MatArgs A;
    A.mode = MAT_PARTITION;
    A.key_roots.assign(keys, keys + nkeys);
    A.nparts = nparts;
    run_materialize(c, in, P, A, out, part_offsets, pick(c, stream));
  });
}

tq_status tq_join_build(tq_ctx* c, const tq_batch* build, const uint32_t* keys, uint32_t nkeys, tq_join_table** out,
                        void* stream) {
  return tq_join_build_sized(c, build, keys, nkeys, 0, out, stream);
}

tq_status tq_join_build_semi(tq_ctx* c, const tq_batch* build, const uint32_t* keys, uint32_t nkeys,
                             tq_join_table** out, void* stream) {
  return tq_pipeline_build_semi(c, build, nullptr, keys, nkeys, out, stream);
}

tq_status tq_join_build_sized(tq_ctx* c, const tq_batch* build, const uint32_t* keys, uint32_t nkeys,
                              uint64_t bloom_keys, tq_join_table** out, void* stream) {
  return guard([&] {
    check_device_batch(build);
    if (has_utf8(build)) {  // Utf8 keys / payloads: a table over the lowered batch
      cudaStream_t st = pick(c, stream);
      Utf8Side S;
      try {
        utf8_lower_side(c, build, keys, nkeys, S, st);
      } catch (...) {
        for (auto& b : S.bufs) dfree(c, b.first, b.second, st);
        throw;
      }
      tq_status r = tq_join_build_sized(c, &S.b, keys, nkeys, bloom_keys, out, stream);
      if (r != TQ_OK) {
        for (auto& b : S.bufs) dfree(c, b.first, b.second, st);
        fail(r, tq_last_error());
      }
      tq_join_table* t = *out;
      t->utf8 = true;
      t->orig_cols.assign(build->cols, build->cols + build->ncols);
      t->orig_rows = build->rows;
      for (uint32_t k = 0; k < nkeys; ++k) {
        t->key_utf8.push_back(build->cols[keys[k]].kind == TQ_UTF8 ? 1 : 0);
        t->key_cols.push_back(keys[k]);
      }
      t->own = std::move(S.bufs);
      return;
    }
    Prog P(schema_of(build));
    std::vector<tq_expr_node> nodes(nkeys);
    std::vector<tq_expr> ex(nkeys);
    for (uint32_t k = 0; k < nkeys; ++k) {
      nodes[k] = tq_expr_node{};
      nodes[k].tag = TQ_EX_COL;
      nodes[k].column = keys[k];
      ex[k] = tq_expr{&nodes[k], 1, 0};
    }
    compile_prog(P, build, nullptr, ex.data(), nkeys, false);
    run_build(c, build, P, iota_u32(nkeys), out, pick(c, stream), bloom_keys, false);
  });
}

static tq_status pipeline_build_impl(tq_ctx* c, const tq_batch* in, const tq_expr* pred, const uint32_t* keys,
                                     uint32_t nkeys, tq_join_table** out, void* stream, bool semi,
                                     uint64_t bloom_keys = 0) {
  return guard([&] {
    check_device_batch(in);
    Prog P(schema_of(in));
    std::vector<tq_expr_node> nodes(nkeys);
    std::vector<tq_expr> ex(nkeys);
    for (uint32_t k = 0; k < nkeys; ++k) {
      nodes[k] = tq_expr_node{};
      nodes[k].tag = TQ_EX_COL;
      nodes[k].column = keys[k];
      ex[k] = tq_expr{&nodes[k], 1, 0};
    }
    compile_prog(P, in, pred, ex.data(), nkeys, false);
    run_build(c, in, P, iota_u32(nkeys), out, pick(c, stream), bloom_keys, semi);
  });
}

tq_status tq_pipeline_build_ex(tq_ctx* c, const tq_batch* in, const tq_expr* pred, const uint32_t* keys,
                               uint32_t nkeys, uint64_t bloom_keys, int semi, tq_join_table** out, void* stream) {
  return pipeline_build_impl(c, in, pred, keys, nkeys, out, stream, semi != 0, bloom_keys);
}

tq_status tq_pipeline_estimate(tq_ctx* c, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                               uint32_t nexprs, uint64_t* out_rows, uint64_t* out_row_bytes, void* stream) {
  return guard([&] {
    check_device_batch(in);
    cudaStream_t st = pick(c, stream);
    Prog P(schema_of(in));
    compile_prog(P, in, pred, exprs, nexprs, exprs == nullptr);
    uint64_t w = 0;
    for (int h : P.outs) {
      uint8_t prec, scale;
      w += width_of(out_kind_of(P.pb.root(h), in, P.pb, &prec, &scale));
    }
    if (out_row_bytes) *out_row_bytes = w;
    uint64_t rows = in->rows;
    if (P.has_pred && in->rows > 0) {
      // the COUNT pass of a filter over the predicate columns only
      Plan L;
      plan_launch(c, in, P, L, kWarps * kMaxDest * 4 + kWarps * kMaxDest * 8, st);
      PipeParams& p = L.p;
      p.dest_kind = DEST_FILTER;
      p.ndest = 1;
      const u64 ncnt = (u64)p.ntiles * kWarps;
      u32* counts = (u32*)dalloc(c, ncnt * 4, st);
      u64* offsets = (u64*)dalloc(c, (ncnt + 1) * 8, st);
      p.tile_counts = counts;
      p.load_mask = P.pb.column_deps({P.pred_h});
      launch_count(c, L, P, st);
      scan_u32(c, counts, ncnt, offsets, offsets + ncnt, st);
      {
        TQ_CUDA(cudaMemcpyAsync(pinned_scratch(c), offsets + ncnt, 8, cudaMemcpyDeviceToHost, st));
        { TQ_HT("estimate sync"); TQ_CUDA(cudaStreamSynchronize(st)); }
        rows = ((uint64_t*)pinned_scratch(c))[0];
      }
      dfree(c, counts, ncnt * 4, st);
      dfree(c, offsets, (ncnt + 1) * 8, st);
    }
    if (out_rows) *out_rows = rows;
  });
}

tq_status tq_pipeline_build(tq_ctx* c, const tq_batch* in, const tq_expr* pred, const uint32_t* keys, uint32_t nkeys,
                            tq_join_table** out, void* stream) {
  return pipeline_build_impl(c, in, pred, keys, nkeys, out, stream, false);
}

tq_status tq_pipeline_build_semi(tq_ctx* c, const tq_batch* in, const tq_expr* pred, const uint32_t* keys,
                                 uint32_t nkeys, tq_join_table** out, void* stream) {
  return pipeline_build_impl(c, in, pred, keys, nkeys, out, stream, true);
}

tq_status tq_join_probe(tq_ctx* c, const tq_join_table* t, const tq_batch* probe, const uint32_t* keys,
                        uint32_t nkeys, tq_batch* out, void* stream) {
  return guard([&] {
    check_device_batch(probe);
    if (t->utf8 || has_utf8(probe)) {
      join_probe_utf8(c, t, probe, keys, nkeys, out, pick(c, stream));
      return;
    }
    Prog P(schema_of(probe));
    compile_all(P, probe, nullptr);
    MatArgs A;
    A.mode = MAT_PROBE;
    A.key_roots.assign(keys, keys + nkeys);
    A.table = t;
    A.build_cols = iota_u32(t->build.ncols);
    run_materialize(c, probe, P, A, out, nullptr, pick(c, stream));
  });
}

tq_status tq_pipeline_probe(tq_ctx* c, const tq_join_table* t, const tq_batch* in, const tq_expr* pred,
                            const tq_expr* exprs, uint32_t nexprs, const uint32_t* keys, uint32_t nkeys,
                            const uint32_t* build_cols, uint32_t nbuild_cols, tq_batch* out, void* stream) {
  return guard([&] {
    check_device_batch(in);
    Prog P(schema_of(in));
    compile_prog(P, in, pred, exprs, nexprs, exprs == nullptr);
    MatArgs A;
    A.mode = MAT_PROBE;
    A.key_roots.assign(keys, keys + nkeys);
    A.table = t;
    if (build_cols) A.build_cols.assign(build_cols, build_cols + nbuild_cols);
    else A.build_cols = iota_u32(t->build.ncols);
    run_materialize(c, in, P, A, out, nullptr, pick(c, stream));
  });
}

void tq_join_table_destroy(tq_ctx* c, tq_join_table* t) {
  if (!t) return;
  (void)c;
  dfree(t->ctx, t->mem, t->bytes, t->ctx->stream);  // see tq_batch_free
  for (auto& r : t->retired) dfree(t->ctx, r.first, r.second, t->ctx->stream);
  for (auto& b : t->own) dfree(t->ctx, b.first, b.second, t->ctx->stream);
  std::free(t->build.cols);
  delete t;
}

tq_status tq_aggregate(tq_ctx* c, const tq_batch* in, const uint32_t* keys, uint32_t nkeys, const tq_agg* aggs,
                       uint32_t naggs, tq_batch* out, void* stream) {
  return guard([&] {
    check_device_batch(in);
    for (uint32_t k = 0; k < nkeys; ++k)
      if (keys[k] < in->ncols && in->cols[keys[k]].kind == TQ_UTF8) {
        aggregate_utf8_keys(c, in, keys, nkeys, aggs, naggs, out, pick(c, stream));
        return;
      }
    run_aggregate_plain(c, in, keys, nkeys, aggs, naggs, out, pick(c, stream));
  });
}

tq_status tq_pipeline_aggregate(tq_ctx* c, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                                uint32_t nexprs, const uint32_t* keys, uint32_t nkeys, const tq_agg* aggs,
                                uint32_t naggs, tq_batch* out, void* stream) {
  return guard([&] {
    TQ_HT("tq_pipeline_aggregate");
    check_device_batch(in);
    Prog P(schema_of(in));
    compile_prog(P, in, pred, exprs, nexprs, exprs == nullptr);
    run_aggregate(c, in, P, keys, nkeys, aggs, naggs, out, pick(c, stream));
  });
}

}  // extern "C"

namespace tq {
void scan_u32_public(tq_ctx* c, const u32* in, u64 n, u64* out, u64* total_dev, cudaStream_t st) {
  scan_u32(c, in, n, out, total_dev, st);
}
}  // namespace tq

// ================================================================== streaming aggregation state
// tq_agg_update aggregates each batch into a PARTIAL (keys + raw accumulators);
// tq_agg_finalize merges the partials (sums of sums / counts, min of mins, ...)
// and produces the SPEC.md:604-611 outputs.  Exact: int128 sums are
// associative, so the result does not depend on how rows were batched.
struct tq_agg_state {
  tq_ctx* ctx = nullptr;
  bool has_pred = false, has_exprs = false;
  std::vector<tq_expr_node> pred;
  std::vector<std::vector<tq_expr_node>> exprs;
  std::vector<uint32_t> keys;
  std::vector<tq_agg> aggs;
  bool planned = false;
  std::vector<tq::AggPlan> ap;
  std::vector<uint8_t> acc_ops;
  std::vector<tq_batch> partials;
};

namespace {
tq_expr as_expr(const std::vector<tq_expr_node>& v) { return tq_expr{v.data(), (uint32_t)v.size(), 0}; }
}  // namespace

extern "C" {

tq_status tq_agg_create(tq_ctx* c, const tq_expr* pred, const tq_expr* exprs, uint32_t nexprs, const uint32_t* keys,
                        uint32_t nkeys, const tq_agg* aggs, uint32_t naggs, tq_agg_state** out) {
  return guard([&] {
    tq_agg_state* s = new tq_agg_state();
    s->ctx = c;
    if (pred) {
      s->has_pred = true;
      s->pred.assign(pred->nodes, pred->nodes + pred->len);
    }
    if (exprs) {
      s->has_exprs = true;
      for (uint32_t i = 0; i < nexprs; ++i) s->exprs.emplace_back(exprs[i].nodes, exprs[i].nodes + exprs[i].len);
    }
    s->keys.assign(keys, keys + nkeys);
    s->aggs.assign(aggs, aggs + naggs);
    *out = s;
  });
}

tq_status tq_agg_update(tq_agg_state* s, const tq_batch* in, void* stream) {
  return guard([&] {
    check_device_batch(in);
    tq_ctx* c = s->ctx;
    cudaStream_t st = pick(c, stream);
    Prog P(schema_of(in));
    tq_expr pe = as_expr(s->pred);
    std::vector<tq_expr> ex;
    for (auto& e : s->exprs) ex.push_back(as_expr(e));
    compile_prog(P, in, s->has_pred ? &pe : nullptr, s->has_exprs ? ex.data() : nullptr, (uint32_t)ex.size(),
                 !s->has_exprs);
    AggSpec S = plan_aggs(in, P, s->aggs.data(), (uint32_t)s->aggs.size());
    if (!s->planned) {
      s->ap = S.ap;
      for (auto& a : S.acc) s->acc_ops.push_back(a.op);
      s->planned = true;
    } else if (S.acc.size() != s->acc_ops.size()) {
      fail(TQ_SCHEMA_MISMATCH, "aggregate input schema changed between batches");
    }
    // an empty batch adds nothing, except that the state's first partial
    // (0 rows) carries the partial schema (finalize / take_partial of a
    // worker whose input was empty)
    if (in->rows == 0 && !s->partials.empty()) return;
    tq_batch part{};
    agg_core(c, in, P, key_handles(P, s->keys.data(), (uint32_t)s->keys.size()), S.acc, nullptr, &part, st);
    s->partials.push_back(part);
  });
}

tq_status tq_agg_take_partial(tq_agg_state* s, tq_batch* out, void* stream) {
  return guard([&] {
    tq_ctx* c = s->ctx;
    cudaStream_t st = pick(c, stream);
    if (!s->planned) fail(TQ_INVALID_PLAN, "aggregate state has seen no batch (no schema)");
    const uint32_t nk = (uint32_t)s->keys.size();
    if (s->partials.empty()) fail(TQ_INTERNAL, "no partial to take (every update appends one)");
    tq_batch merged{};
    const tq_batch* src = &s->partials[0];
    if (s->partials.size() > 1) {
      tq_status r = tq_concat(c, s->partials.data(), (uint32_t)s->partials.size(), &merged, st);
      if (r != TQ_OK) fail(r, g_err);
      src = &merged;
    }
    // merge the partials into one partial (sum of sums, min of mins, ...)
    Prog P(schema_of(src));
    compile_prog(P, src, nullptr, nullptr, 0, true);
    std::vector<int> kh;
    for (uint32_t k = 0; k < nk; ++k) kh.push_back(P.outs[k]);
    std::vector<AccSpec> macc;
    for (size_t i = 0; i < s->acc_ops.size(); ++i) {
      const Operand& o = P.pb.root(P.outs[nk + i]);
      AccSpec a{};
      a.op = s->acc_ops[i] == ACC_CNT ? (uint8_t)ACC_SUM_I : s->acc_ops[i];
      a.kind = o.kind;
      a.idx = o.idx;
      macc.push_back(a);
    }
    try {
      agg_core(c, src, P, kh, macc, nullptr, out, st, &s->acc_ops);
    } catch (...) {
      if (src == &merged) tq_batch_free(c, &merged);
      throw;
    }
    if (src == &merged) tq_batch_free(c, &merged);
    // a merged count partial is an int128 sum: keep the partial schema (Int64 counts)
    for (size_t i = 0; i < s->acc_ops.size(); ++i)
      if (s->acc_ops[i] == ACC_CNT && out->cols[nk + i].kind != TQ_INT64) fail(TQ_INTERNAL, "partial count schema");
    for (auto& b : s->partials) tq_batch_free(c, &b);
    s->partials.clear();
  });
}

tq_status tq_agg_add_partial(tq_agg_state* s, const tq_batch* partial, void* stream) {
  return guard([&] {
    check_device_batch(partial);
    tq_ctx* c = s->ctx;
    if (!s->planned) fail(TQ_INVALID_PLAN, "aggregate state has seen no batch (no schema)");
    if (partial->ncols != s->keys.size() + s->acc_ops.size()) fail(TQ_SCHEMA_MISMATCH, "partial aggregate schema");
    tq_batch copy{};
    tq_status r = tq_slice(c, partial, 0, partial->rows, &copy, stream);
    if (r != TQ_OK) fail(r, g_err);
    s->partials.push_back(copy);
  });
}

tq_status tq_agg_finalize(tq_agg_state* s, tq_batch* out, void* stream) {
  return guard([&] {
    tq_ctx* c = s->ctx;
    cudaStream_t st = pick(c, stream);
    const uint32_t nk = (uint32_t)s->keys.size();
    if (s->partials.empty()) {
      // empty input -> empty output
      alloc_batch(c, 0, {}, {}, out, st);
      return;
    }
    tq_batch merged{};
    const tq_batch* src = &s->partials[0];
    if (s->partials.size() > 1) {
      tq_status r = tq_concat(c, s->partials.data(), (uint32_t)s->partials.size(), &merged, st);
      if (r != TQ_OK) fail(r, g_err);
      src = &merged;
    }
    Prog P(schema_of(src));
    compile_prog(P, src, nullptr, nullptr, 0, true);
    std::vector<int> kh;
    for (uint32_t k = 0; k < nk; ++k) kh.push_back(P.outs[k]);
    std::vector<AccSpec> macc;
    for (size_t i = 0; i < s->acc_ops.size(); ++i) {
      const Operand& o = P.pb.root(P.outs[nk + i]);
      AccSpec a{};
      a.op = s->acc_ops[i] == ACC_CNT ? (uint8_t)ACC_SUM_I : s->acc_ops[i];
      a.kind = o.kind;
      a.idx = o.idx;
      macc.push_back(a);
    }
    try {
      agg_core(c, src, P, kh, macc, &s->ap, out, st);
    } catch (...) {
      if (src == &merged) tq_batch_free(c, &merged);
      throw;
    }
    if (src == &merged) tq_batch_free(c, &merged);
  });
}

void tq_agg_destroy(tq_agg_state* s) {
  if (!s) return;
  for (auto& b : s->partials) tq_batch_free(s->ctx, &b);
  delete s;
}

}  // extern "C"


// ================================================================== LIP Bloom filters
struct tq_bloom {
  tq_ctx* ctx;
  uint32_t* words;
  uint64_t nwords;  // power of two (per part)
  uint32_t parts = 1;  // > 1: part d = rank d's table filter, words [d * nwords, (d + 1) * nwords)
  uint32_t kw;
  std::vector<uint8_t> key_cls, key_scale;
};

namespace {
__global__ void k_bloom_or(uint32_t* dst, const uint32_t* all, uint64_t nwords, int n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (int r = 0; r < n; ++r) v |= all[(uint64_t)r * nwords + i];
    dst[i] = v;
  }
}
}  // namespace

extern "C" {

tq_status tq_bloom_build(tq_ctx* c, const tq_batch* in, const uint32_t* keys, uint32_t nkeys, uint64_t expected_keys,
                         tq_bloom** out, void* stream) {
  return guard([&] {
    check_device_batch(in);
    cudaStream_t st = pick(c, stream);
    Prog P(schema_of(in));
    std::vector<tq_expr_node> nodes(nkeys);
    std::vector<tq_expr> ex(nkeys);
    for (uint32_t k = 0; k < nkeys; ++k) {
      nodes[k] = tq_expr_node{};
      nodes[k].tag = TQ_EX_COL;
      nodes[k].column = keys[k];
      ex[k] = tq_expr{&nodes[k], 1, 0};
    }
    compile_prog(P, in, nullptr, ex.data(), nkeys, false);
    Plan L;
    plan_launch(c, in, P, L, 0, st);
    PipeParams& p = L.p;
    std::vector<int> kh(P.outs.begin(), P.outs.end());
    if (kh.empty()) fail(TQ_INVALID_PLAN, "bloom filter without keys");
    set_keys(p, P.pb, kh);
    tq_bloom* b = new tq_bloom();
    b->ctx = c;
    b->kw = p.key_words;
    for (int h : kh) {
      b->key_cls.push_back(P.pb.root(h).cls);
      b->key_scale.push_back(P.pb.root(h).scale);
    }
    uint64_t words = 1024;
    while (words * 32 < std::max<uint64_t>(expected_keys, in->rows) * 10) words <<= 1;  // ~10 bits per key
    b->nwords = words;
    b->words = (uint32_t*)dalloc(c, words * 4, st);
    TQ_CUDA(cudaMemsetAsync(b->words, 0, words * 4, st));
    p.jt = JoinTable{};
    p.jt.entries = nullptr;  // Bloom-only build
    p.jt.kw = p.key_words;
    p.jt.cap = 1;
    p.jt.bloom = b->words;
    p.jt.bloom_mask = words - 1;
    launch(c, SINK_BUILD, L, P, st);
    *out = b;
  });
}

void tq_bloom_destroy(tq_bloom* b) {
  if (!b) return;
  dfree(b->ctx, b->words, b->nwords * 4 * b->parts, b->ctx->stream);
  delete b;
}

uint64_t tq_bloom_words(const tq_bloom* b) { return b->nwords; }
uint32_t* tq_bloom_data(tq_bloom* b) { return b->words; }

tq_status tq_bloom_or_gathered(tq_bloom* b, const uint32_t* gathered, int nranks, void* stream) {
  return guard([&] {
    cudaStream_t st = pick(b->ctx, stream);
    k_bloom_or<<<(u32)std::min<uint64_t>(4096, (b->nwords + 255) / 256), 256, 0, st>>>(b->words, gathered, b->nwords,
                                                                                      nranks);
    counted_launch(b->ctx);
    TQ_CUDA(cudaGetLastError());
  });
}

tq_status tq_pipeline_partition_semi(tq_ctx* c, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                                     uint32_t nexprs, const uint32_t* keys, uint32_t nkeys, uint32_t nparts,
                                     const tq_bloom* semi, tq_batch* out, uint64_t* part_offsets, void* stream) {
  return guard([&] {
    check_device_batch(in);
    Prog P(schema_of(in));
    compile_prog(P, in, pred, exprs, nexprs, exprs == nullptr);
    MatArgs A;
    A.mode = MAT_PARTITION;
    A.key_roots.assign(keys, keys + nkeys);
    A.nparts = nparts;
    if (semi) {
      if (semi->key_cls.size() != nkeys) fail(TQ_INVALID_PLAN, "semi-join key count differs");
      for (uint32_t k = 0; k < nkeys; ++k) {
        if (keys[k] >= P.outs.size()) fail(TQ_INVALID_PLAN, "key column out of range");
        const Operand& o = P.pb.root(P.outs[keys[k]]);
        if (o.cls != semi->key_cls[k] || (o.cls == C_D && o.scale != semi->key_scale[k]))
          fail(TQ_INVALID_PLAN, "semi-join key types differ");
      }
      if (semi->parts > 1 && semi->parts != nparts) fail(TQ_INVALID_PLAN, "partitioned semi filter: parts differ");
      A.semi_words = semi->words;
      A.semi_mask = semi->nwords - 1;
      A.semi_part_words = semi->parts > 1 ? semi->nwords : 0;
    }
    run_materialize(c, in, P, A, out, part_offsets, pick(c, stream));
  });
}

tq_status tq_comm_gather_table_blooms(tq_comm* comm, const tq_join_table* t, tq_bloom** out, void* stream) {
  return guard([&] {
    tq_ctx* c = comm_ctx(comm);
    cudaStream_t st = pick(c, stream);
    const int n = comm_size(comm);
    if (!t->jt.bloom) fail(TQ_INVALID_PLAN, "join table has no Bloom filter");
    const uint64_t per = t->jt.bloom_mask + 1;  // words; >= 1024, so a whole number of u64
    tq_bloom* b = new tq_bloom();
    b->ctx = c;
    b->kw = t->jt.kw;
    b->key_cls = t->key_cls;
    b->key_scale = t->key_scale;
    b->nwords = per;
    b->parts = (uint32_t)n;
    // Precondition (collective): every rank built its table with the same
    // agreed bloom_keys (e.g. tq_comm_last_exchange_capacity right after the
    // exchange that delivered the build side), so every filter has the same
    // word count.  Checked locally against the table's own agreed count before
    // the collective (no size all-gather, no host sync).
    uint64_t expect = 1024;
    while (expect * 32 < t->bloom_keys * kLipBloomBitsPerKey) expect <<= 1;
    if (t->bloom_keys == 0 || per != expect) {
      delete b;
      fail(TQ_INVALID_PLAN, "table Bloom filter not sized from an agreed row count (tq_join_build_sized)");
    }
    b->words = (uint32_t*)dalloc(c, per * 4 * n, st);
    const int ph = prof_begin(c, "nccl_gather_blooms", st);
    comm_allgather_u64(comm, (const unsigned long long*)t->jt.bloom, (unsigned long long*)b->words, per / 2, st);
    prof_end(c, ph, st);
    comm_add_sent(comm, per * 4 * (n - 1));
    *out = b;
  });
}

uint64_t tq_comm_last_exchange_capacity(tq_comm* comm) { return comm_last_cap(comm); }

tq_status tq_pipeline_broadcast(tq_comm* comm, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                                uint32_t nexprs, tq_batch* out, void* stream) {
  return guard([&] {
    tq_ctx* c = comm_ctx(comm);
    check_device_batch(in);
    if (has_utf8(in)) {  // fixed-width windows: Utf8 columns take the NCCL all-gather (every rank: same schema)
      tq_batch m{};
      tq_status r = tq_pipeline_materialize(c, in, pred, exprs, nexprs, &m, stream);
      if (r != TQ_OK) fail(r, tq_last_error());
      r = tq_comm_allgather(comm, &m, out, nullptr, stream);
      tq_batch_free(c, &m);
      if (r != TQ_OK) fail(r, tq_last_error());
      return;
    }
    Prog P(schema_of(in));
    compile_prog(P, in, pred, exprs, nexprs, exprs == nullptr);
    uint64_t sent_rows = 0;
    run_partition_exchange(c, comm, in, P, {}, nullptr, 0, 0, out, &sent_rows, pick(c, stream), /*bcast=*/true);
    uint64_t row_bytes = 0;
    for (uint32_t k = 0; k < out->ncols; ++k) row_bytes += width_of(out->cols[k].kind);
    comm_add_sent(comm, sent_rows * row_bytes);  // rows stored into other ranks' windows
  });
}

tq_status tq_pipeline_partition_exchange(tq_comm* comm, const tq_batch* in, const tq_expr* pred,
                                         const tq_expr* exprs, uint32_t nexprs, const uint32_t* keys, uint32_t nkeys,
                                         const tq_bloom* semi, tq_batch* out, void* stream) {
  return guard([&] {
    tq_ctx* c = comm_ctx(comm);
    check_device_batch(in);
    if (has_utf8(in)) {
      // the receive window is fixed-width: Utf8 columns take the NCCL exchange
      // (a schema property, so every rank takes this same path)
      if (semi) fail(TQ_INVALID_PLAN, "no LIP filter on a partition exchange with utf8 columns");
      const int n = comm_size(comm);
      std::vector<uint64_t> offs(n + 1);
      tq_batch part{};
      tq_status r = tq_pipeline_partition(c, in, pred, exprs, nexprs, keys, nkeys, (uint32_t)n, &part, offs.data(),
                                          stream);
      if (r != TQ_OK) fail(r, tq_last_error());
      r = tq_comm_exchange(comm, &part, offs.data(), out, nullptr, stream);
      tq_batch_free(c, &part);
      if (r != TQ_OK) fail(r, tq_last_error());
      // the agreed row count for a following tq_join_build_sized: the most rows any rank received
      std::vector<uint64_t> got(n);
      const uint64_t mine = out->rows;
      r = tq_comm_allgather_host_u64(comm, &mine, got.data(), 1, stream);
      if (r != TQ_OK) fail(r, tq_last_error());
      comm_last_cap(comm) = std::max<uint64_t>(1, *std::max_element(got.begin(), got.end()));
      return;
    }
    Prog P(schema_of(in));
    compile_prog(P, in, pred, exprs, nexprs, exprs == nullptr);
    std::vector<uint32_t> kr(keys, keys + nkeys);
    const uint32_t* sw = nullptr;
    uint64_t sm = 0, spw = 0;
    if (semi) {
      if (semi->key_cls.size() != nkeys) fail(TQ_INVALID_PLAN, "semi-join key count differs");
      for (uint32_t k = 0; k < nkeys; ++k) {
        if (keys[k] >= P.outs.size()) fail(TQ_INVALID_PLAN, "key column out of range");
        const Operand& o = P.pb.root(P.outs[keys[k]]);
        if (o.cls != semi->key_cls[k] || (o.cls == C_D && o.scale != semi->key_scale[k]))
          fail(TQ_INVALID_PLAN, "semi-join key types differ");
      }
      if (semi->parts > 1 && semi->parts != (uint32_t)comm_size(comm))
        fail(TQ_INVALID_PLAN, "partitioned semi filter: parts differ from the ranks");
      sw = semi->words;
      sm = semi->nwords - 1;
      spw = semi->parts > 1 ? semi->nwords : 0;
    }
    uint64_t sent_rows = 0;
    run_partition_exchange(c, comm, in, P, kr, sw, sm, spw, out, &sent_rows, pick(c, stream));
    uint64_t row_bytes = 0;
    for (uint32_t k = 0; k < out->ncols; ++k) row_bytes += width_of(out->cols[k].kind);
    comm_add_sent(comm, sent_rows * row_bytes);
  });
}

}  // extern "C"

namespace tq {
// join_execute probe with Utf8 keys / payloads on either side (see Utf8Side)
void join_probe_utf8(tq_ctx* c, const tq_join_table* t, const tq_batch* probe, const uint32_t* keys, uint32_t nkeys,
                     tq_batch* out, cudaStream_t st) {
  if (nkeys != t->key_cols.size() && t->utf8) fail(TQ_INVALID_PLAN, "join key count differs from the build's");
  for (uint32_t k = 0; k < nkeys; ++k) {
    if (keys[k] >= probe->ncols) fail(TQ_INVALID_PLAN, "join key out of range");
    const bool pu = probe->cols[keys[k]].kind == TQ_UTF8, bu = t->utf8 && t->key_utf8[k];
    if (pu != bu) fail(TQ_INVALID_PLAN, "join key types differ");
  }
  Utf8Side S;
  struct Free {
    tq_ctx* c;
    cudaStream_t st;
    Utf8Side& S;
    ~Free() {
      for (auto& b : S.bufs) dfree(c, b.first, b.second, st);
    }
  } fr{c, st, S};
  utf8_lower_side(c, probe, keys, nkeys, S, st);
  const tq_batch& tb = t->build;  // lowered build (its last column the build row id when t->utf8)
  const uint32_t nb = tb.ncols, np = S.b.ncols;
  // the build columns of the output: the lowered build's (incl. its row ids)
  {
    Prog P(schema_of(&S.b));
    compile_prog(P, &S.b, nullptr, nullptr, 0, true);
    MatArgs A;
    A.mode = MAT_PROBE;
    A.key_roots.assign(keys, keys + nkeys);
    A.table = t;
    A.build_cols = iota_u32(nb);
    run_materialize(c, &S.b, P, A, out, nullptr, st);
  }
  // out: [lowered build (nb) | lowered probe (np)]; row ids at nb - 1 (if t->utf8) and nb + np - 1
  const uint32_t brid = t->utf8 ? nb - 1 : UINT32_MAX, prid = nb + np - 1;
  // exactness: drop the pairs whose Utf8 key strings differ (fnv1a64 collisions)
  bool any_utf8_key = false;
  for (uint32_t k = 0; k < nkeys; ++k) any_utf8_key |= probe->cols[keys[k]].kind == TQ_UTF8;
  if (any_utf8_key && out->rows) {
    const uint64_t n = out->rows;
    uint8_t* keep = (uint8_t*)dalloc(c, std::max<uint64_t>(8, n), st);
    u32* drop = (u32*)dalloc(c, 8, st);
    TQ_CUDA(cudaMemsetAsync(keep, 1, n, st));
    TQ_CUDA(cudaMemsetAsync(drop, 0, 4, st));
    for (uint32_t k = 0; k < nkeys; ++k) {
      if (probe->cols[keys[k]].kind != TQ_UTF8) continue;
      const tq_column& bc = t->orig_cols[t->key_cols[k]];
      const tq_column& pc = probe->cols[keys[k]];
      k_utf8_pair_keep<<<grid_for(c, n), 256, 0, st>>>(
          (const uint8_t*)bc.values, bc.offsets, (const uint8_t*)pc.values, pc.offsets,
          (const long long*)out->cols[brid].values, (const long long*)out->cols[prid].values, n, keep, drop);
      counted_launch(c);
    }
    TQ_CUDA(cudaGetLastError());
    u32* pin = (u32*)pinned_scratch(c);
    TQ_CUDA(cudaMemcpyAsync(pin, drop, 4, cudaMemcpyDeviceToHost, st));
    TQ_CUDA(cudaStreamSynchronize(st));
    const bool dropped = pin[0] != 0;
    if (dropped) {
      std::vector<tq_column> cols(out->cols, out->cols + out->ncols);
      tq_column kc{};
      kc.kind = TQ_BOOL;
      kc.values = keep;
      kc.values_bytes = n;
      cols.push_back(kc);
      tq_batch with{n, (uint32_t)cols.size(), TQ_MEM_DEVICE, cols.data(), nullptr};
      tq_expr_node pn{};
      pn.tag = TQ_EX_COL;
      pn.column = (uint32_t)cols.size() - 1;
      tq_batch f{};
      const tq_status r = tq_filter(c, &with, tq_expr{&pn, 1, 0}, &f, st);
      if (r == TQ_OK) {
        tq_batch_free(c, out);
        *out = f;
        std::vector<bool> d(out->ncols, false);
        d[out->ncols - 1] = true;  // the keep column
        drop_columns(c, out, d, st);
      }
      dfree(c, keep, std::max<uint64_t>(8, n), st);
      dfree(c, drop, 8, st);
      if (r != TQ_OK) fail(r, tq_last_error());
    } else {
      dfree(c, keep, std::max<uint64_t>(8, n), st);
      dfree(c, drop, 8, st);
    }
  }
  // the output strings: a Utf8 column's output holds its side's row ids (a Utf8
  // payload's stand-in is the row-id column; a Utf8 key's hash is replaced by them)
  std::vector<bool> d(out->ncols, false);
  auto gather = [&](uint32_t j, const tq_column& src, uint64_t src_rows, uint32_t rid_col, bool was_key) {
    if (was_key && out->rows)
      TQ_CUDA(cudaMemcpyAsync(out->cols[j].values, out->cols[rid_col].values, out->rows * 8, cudaMemcpyDeviceToDevice,
                              st));
    tq_batch one{src_rows, 1, TQ_MEM_DEVICE, const_cast<tq_column*>(&src), nullptr};
    std::vector<int> sv(out->ncols, -1);
    sv[j] = 0;
    utf8_raise(c, &one, sv, out->ncols, out, st);
  };
  if (t->utf8) {
    std::vector<bool> bkey(t->orig_cols.size(), false);
    for (uint32_t k = 0; k < nkeys; ++k) bkey[t->key_cols[k]] = true;
    for (uint32_t j = 0; j < t->orig_cols.size(); ++j)
      if (t->orig_cols[j].kind == TQ_UTF8) gather(j, t->orig_cols[j], t->orig_rows, brid, bkey[j]);
    d[brid] = true;
  }
  {
    std::vector<bool> pkey(probe->ncols, false);
    for (uint32_t k = 0; k < nkeys; ++k) pkey[keys[k]] = true;
    for (uint32_t j = 0; j < probe->ncols; ++j)
      if (probe->cols[j].kind == TQ_UTF8) gather(nb + j, probe->cols[j], probe->rows, prid, pkey[j]);
  }
  d[prid] = true;
  drop_columns(c, out, d, st);
}
}  // namespace tq
