// kernel_common.cuh — the staged warp-tile pipeline kernel skeleton, written
// once against a program policy `P` and instantiated twice:
//   * InterpP (interp.cuh, compiled into libtq_gpu.so): the generic Expr
//     register machine interpreted per warp;
//   * a generated policy (jit.cu): the same typed program lowered to
//     straight-line CUDA and compiled at run time by NVRTC for sm_100a.
//
// Per CTA (persistent grid): thread 0 streams the referenced column slices of
// tile t+nstages into a ring of shared-memory stages with cp.async.bulk (TMA
// 1-D bulk copies, mbarrier complete_tx) while 8 warps process tile t (each
// warp owns 64 rows, 2 per lane) and feed the sink:
//   COUNT / EMIT : stable destination scatter (filter, hash_partition,
//                  join probe) with warp ballots / match_any ranks;
//   AGG          : per-lane private accumulators in smem for the CTA's first
//                  groups, a global open-addressing table beyond that;
//   BUILD        : open-addressing join-table insert (atomicCAS on the row).
// This replaces the reference's per-row Column::*_at loops
// (types.cpp:66-90) and take() (transform.cpp:90-120).
#pragma once
#include "device.cuh"
#include "pipeline.h"

namespace tq {

// ------------------------------------------------------------------ per-warp context
struct WCtx {
  const PipeParams* p;
  const uint8_t* stage;  // current stage base
  const DLit* lits;      // smem copy
  uint8_t* vslot;        // interpreter: [slot][v][32] x 16 B  (this warp)
  u32* vvalid;           // interpreter: [slot][v]
  u32* bslot;            // interpreter: [slot][v][2] (value, valid)
  u32 row0;              // tile-relative first row of this warp
  u32 nrows;             // rows in the tile
  u32 lane;
  long long out_delta;   // added to output addresses (DEST_PEER: the destination rank's window)
  u32 vmask;             // output c writes validity bits iff bit c (DEST_PEER: the ranks' agreed mask)
};

__device__ __forceinline__ u32 trow(const WCtx& w, int v) { return w.row0 + (u32)v * 32u + w.lane; }

// Inputs a sink reads for one row (only the used entries survive in JIT code).
struct RowVals {
  u64 kw[kMaxKeyWords + 1];  // key words + null word
  i128 ai[kMaxAcc];
  double af[kMaxAcc];
  bool av[kMaxAcc];
};

// ------------------------------------------------------------------ join table
__device__ __forceinline__ const long long* jt_entry(const JoinTable& t, u64 slot) {
  return (const long long*)(t.entries + slot * t.stride);
}

// 128-bit compare-and-swap of a 16-B table entry {row, key} (sm_90+):
// returns the entry's previous contents
__device__ __forceinline__ void cas128(long long* addr, u64 cmp_lo, u64 cmp_hi, u64 new_lo, u64 new_hi, u64& old_lo,
                                      u64& old_hi) {
  asm volatile(
      "{\n .reg .b128 d, c, n;\n mov.b128 c, {%2, %3};\n mov.b128 n, {%4, %5};\n"
      " atom.global.cas.b128 d, [%6], c, n;\n mov.b128 {%0, %1}, d;\n}"
      : "=l"(old_lo), "=l"(old_hi)
      : "l"(cmp_lo), "l"(cmp_hi), "l"(new_lo), "l"(new_hi), "l"(addr)
      : "memory");
}

template <int KW>
__device__ __forceinline__ bool jt_key_eq(const JoinTable& t, const long long* e, const u64* kw) {
  const u32 n = KW > 0 ? (u32)KW : t.kw;
#pragma unroll
  for (u32 i = 0; i < (KW > 0 ? (u32)KW : (u32)kMaxKeyWords); ++i) {
    if (i >= n) break;
    if ((u64)e[1 + i] != kw[i]) return false;
  }
  return true;
}

// Home slot of a key: the mixed key hash.  (Keeping blocks of 16 consecutive
// one-word keys in consecutive slots was measured: 2.4x slower builds — the
// 128-bit CASes of a warp serialise on the same lines and colliding blocks
// form long probe runs.)
template <int KW>
__device__ __forceinline__ u64 jt_home(const JoinTable& t, const u64* kw, u64 h) {
  (void)kw;
  return h & (t.cap - 1);
}

// Number of build rows whose keys equal kw.
template <int KW>
__device__ __forceinline__ u32 jt_count(const JoinTable& t, const u64* kw) {
  const u64 mask = t.cap - 1;
  u64 s = jt_home<KW>(t, kw, key_hash(kw, KW > 0 ? KW : (int)t.kw));
  u32 n = 0;
  for (;;) {
    const long long* e = jt_entry(t, s);
    if (e[0] < 0) break;
    if (jt_key_eq<KW>(t, e, kw)) ++n;
    s = (s + 1) & mask;
  }
  return n;
}

// ------------------------------------------------------------------ aggregation tables
constexpr u32 kStEmpty = 0, kStBusy = 1, kStReady = 2;

// 32-bit multiplicative hash for the small per-CTA group tables (full keys
// are compared on every hit, so only the spread matters here).
__device__ __forceinline__ u32 local_hash(const u64* kw, int n) {
  u32 x = 0;
#pragma unroll
  for (int i = 0; i < kMaxKeyWords + 1; ++i) {
    if (i >= n) break;
    x = (x ^ (u32)kw[i] ^ (u32)(kw[i] >> 32)) * 0x9E3779B1u;
  }
  return x;
}

// |v| <= 2^46: 2^16 such values sum to within int64 (per-lane plane bound)
// (non-zero bits of (v + 2^46) above bit 46, OR-able across values)
__device__ __forceinline__ u64 plane_excess(i128 v) {
  const u128 t = (u128)v + ((u128)1 << 46);
  return (u64)(t >> 64) | ((u64)t >> 47);
}
__device__ __forceinline__ bool fits_plane(i128 v) { return plane_excess(v) == 0; }

// Find-or-insert in the per-CTA (shared-memory) group table.  A ready slot's
// state holds the key's 32-bit hash with bit 1 set (never Empty/Busy), so a
// probe past a different group costs one shared load; keys are compared only
// when the tags agree.  Returns the slot or -1 when the table is full.
template <int KWA>
__device__ __forceinline__ long long local_find_insert(u32* state, u64* keys, u32 cap, u32 kwa_rt, const u64* kw,
                                                       u32 h) {
  const u32 kwa = KWA > 0 ? (u32)KWA : kwa_rt;
  const u32 tag = h | 2u;
  const u32 mask = cap - 1;
  u32 s = (h >> 16) & mask;  // top bits of the multiplicative hash
  for (u32 probe = 0; probe < cap; ++probe) {
    // acquire: a published tag orders the key loads below after it
    u32 cur = ld_acquire_cta_shared(state + s);
    if (cur == kStEmpty) {
      cur = atomicCAS(state + s, kStEmpty, kStBusy);
      if (cur == kStEmpty) {
        for (u32 i = 0; i < kwa; ++i) keys[s * kwa + i] = kw[i];
        __threadfence_block();
        atomicExch(state + s, tag);
        return (long long)s;
      }
      if (cur != kStBusy) cur = ld_acquire_cta_shared(state + s);  // the CAS saw a published tag
    }
    while (cur == kStBusy) cur = ld_acquire_cta_shared(state + s);
    if (cur == tag) {
      const volatile u64* k = keys + s * kwa;
      bool eq = true;
#pragma unroll
      for (u32 i = 0; i < (KWA > 0 ? (u32)KWA : (u32)(kMaxKeyWords + 1)); ++i) {
        if (i >= kwa) break;
        eq &= k[i] == kw[i];
      }
      if (eq) return (long long)s;
    }
    s = (s + 1) & mask;
  }
  return -1;
}

// Find-or-insert `kw` (kwa words) in a state/keys open-addressing table.
// Returns slot or -1 when `limit` probes found neither the key nor a free slot.
struct NoClaimInit {
  __device__ __forceinline__ void operator()(u64) const {}
};

// `init(slot)` runs once, by the claiming thread, before the slot is published
// (lazy per-slot initialisation: the table needs only its state words zeroed).
template <int KWA, class Init = NoClaimInit>
__device__ __forceinline__ long long table_find_insert(u32* state, u64* keys, u64 cap, u32 kwa_rt, const u64* kw,
                                                       u64 h, u64 limit, unsigned long long* counter,
                                                       const Init& init = Init()) {
  const u32 kwa = KWA > 0 ? (u32)KWA : kwa_rt;
  const u64 mask = cap - 1;
  u64 s = h & mask;
  for (u64 probe = 0; probe < limit; ++probe) {
    // every state read that can observe Ready is an acquire, so the key
    // loads below are ordered after the publication they observed (a plain
    // load seeing Ready could otherwise compare stale key words and insert
    // the group twice)
    u32 cur = ld_acquire_gpu(state + s);
    if (cur == kStEmpty) {
      cur = atomicCAS(state + s, kStEmpty, kStBusy);
      if (cur == kStEmpty) {
        for (u32 i = 0; i < kwa; ++i) keys[s * kwa + i] = kw[i];
        init(s);
        // publish: the key / accumulator stores are visible before the state
        __threadfence();
        atomicExch(state + s, kStReady);
        if (counter) atomicAdd(counter, 1ull);
        return (long long)s;
      }
      if (cur != kStBusy) cur = ld_acquire_gpu(state + s);  // the (relaxed) CAS saw Ready
    }
    while (cur == kStBusy) cur = ld_acquire_gpu(state + s);
    const volatile u64* k = keys + s * kwa;
    bool eq = true;
#pragma unroll
    for (u32 i = 0; i < (KWA > 0 ? (u32)KWA : (u32)(kMaxKeyWords + 1)); ++i) {
      if (i >= kwa) break;
      eq &= k[i] == kw[i];
    }
    if (eq) return (long long)s;
    s = (s + 1) & mask;
  }
  return -1;
}


__device__ __forceinline__ i128 shfl_up_i128(i128 v, u32 o) {
  const u64 lo = __shfl_up_sync(kFull, lo64(v), o);
  const u64 hi = __shfl_up_sync(kFull, hi64(v), o);
  return mk128(lo, hi);
}
// a float min / max run result differs from the identity (bit pattern)
__device__ __forceinline__ bool valid_any_f(double v, u64 identity_bits) {
  return (u64)__double_as_longlong(v) != identity_bits;
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

// a claimed global slot starts from the accumulators' identities
struct AccClaimInit {
  const PipeParams& p;
  __device__ __forceinline__ void operator()(u64 s) const {
    for (u32 a = 0; a < p.nacc; ++a) {
      u64 lo, hi;
      acc_identity(p.acc[a].op, lo, hi);
      p.agg.acc[(s * p.nacc + a) * 2] = lo;
      p.agg.acc[(s * p.nacc + a) * 2 + 1] = hi;
    }
  }
};

template <int KWA>
__device__ __forceinline__ long long agg_global_slot(const PipeParams& p, const u64* kw, u32 kwa, u64 h,
                                                    unsigned long long* cta_groups) {
  // new groups are counted per CTA in shared memory (one global atomic per
  // CTA at the end, not one per group); a probe run of kAggProbeLimit slots
  // flags overflow (the host grows the table x4 and re-runs)
  constexpr u64 kAggProbeLimit = 128;
  // after an overflow this launch's result is discarded (the host re-runs
  // with a larger table): stop walking the full table
  if (*(volatile u32*)p.agg.overflow) return -1;
  long long s = table_find_insert<KWA>(p.agg.state, p.agg.keys, p.agg.cap, kwa, kw, h,
                                       p.agg.cap < kAggProbeLimit ? p.agg.cap : kAggProbeLimit, cta_groups,
                                       AccClaimInit{p});
  if (s < 0 && *(volatile u32*)p.agg.overflow == 0) atomicExch(p.agg.overflow, 1u);
  return s;
}

// part = fnv1a64(LE bytes of the keys) mod n (reference common.hpp:128-136),
// chained across key columns; a null key hashes as zero bytes.  Power-of-two
// n only needs the low 32 bits of the hash (32-bit multiplies).
__device__ __forceinline__ u32 partition_of(const PipeParams& p, const u64* kw) {
  int pos = 0;
  if ((p.ndest & (p.ndest - 1)) == 0) {
    u32 h = (u32)kFnvBasis;
    for (u32 k = 0; k < p.nkeys; ++k) {
      const KeyOpnd& ko = p.keys[k];
      if (ko.bytes == 16) {
        h = fnv32_bytes(h, kw[pos], 8);
        h = fnv32_bytes(h, kw[pos + 1], 8);
      } else {
        h = fnv32_bytes(h, kw[pos], ko.bytes);
      }
      pos += ko.words;
    }
    return h & (p.ndest - 1);
  }
  u64 h = kFnvBasis;
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
  return (u32)(h % p.ndest);
}

// partition_of specialised for generated programs whose key is one 8-byte
// value (the common case): the FNV loop unrolls with constant shifts and kw
// stays in registers (the generic form loops over runtime key widths).
template <class P>
__device__ __forceinline__ u32 partition_of_p(const PipeParams& p, const u64* kw) {
  if (p.key_prehashed) return (u32)(kw[0] % p.ndest);
  if constexpr (P::kKey1x8) {
    if ((p.ndest & (p.ndest - 1)) == 0) return fnv32_bytes((u32)kFnvBasis, kw[0], 8) & (p.ndest - 1);
    return (u32)(fnv_bytes(kFnvBasis, kw[0], 8) % p.ndest);
  }
  return partition_of(p, kw);
}

// The single build row matching kw (unique-key tables), or -1.
// First build row matching kw (-1: none).  With `walk` the rest of the
// cluster is walked too, and a second match sets dup (non-unique build keys).
__device__ __forceinline__ bool jt_exact_hit(const JoinTable& t, u64 key) {
  if (key >= t.exact_range) return false;
  return (__ldg(t.exact_bits + (key >> 5)) >> (key & 31)) & 1u;
}

// exact: the build's membership bitmap is exact (jt.exact_flag == 0), so it
// replaces the Bloom pre-check (no false positives).
template <int KW>
__device__ __forceinline__ long long jt_probe_first(const JoinTable& t, const u64* kw, bool walk, bool& dup,
                                                   bool exact = false) {
  const u64 h = key_hash(kw, KW > 0 ? KW : (int)t.kw);
  if (exact) {
    if (!jt_exact_hit(t, kw[0])) return -1;
  } else if (t.bloom) {
    const u32 b = bloom_bits(h);
    if ((__ldg(t.bloom + bloom_word(h, t.bloom_mask)) & b) != b) return -1;
  }
  const u64 mask = t.cap - 1;
  long long found = -1;
  for (u64 s = jt_home<KW>(t, kw, h);; s = (s + 1) & mask) {
    const long long* e = jt_entry(t, s);
    const long long row = e[0];
    if (row < 0) return found;
    if (jt_key_eq<KW>(t, e, kw)) {
      if (!walk) return row;
      if (found >= 0) {
        dup = true;
        return found;
      }
      found = row;
    }
  }
}

// Build rows matching kw, after the (L2-resident) Bloom filter check.
template <int KW>
__device__ __forceinline__ u32 jt_probe_count(const JoinTable& t, const u64* kw, bool exact = false) {
  const u64 h = key_hash(kw, KW > 0 ? KW : (int)t.kw);
  if (exact) {
    if (!jt_exact_hit(t, kw[0])) return 0;
  } else if (t.bloom) {
    const u32 b = bloom_bits(h);
    if ((__ldg(t.bloom + bloom_word(h, t.bloom_mask)) & b) != b) return 0;
  }
  const u64 mask = t.cap - 1;
  u64 s = jt_home<KW>(t, kw, h);
  u32 n = 0;
  for (;;) {
    const long long* e = jt_entry(t, s);
    if (e[0] < 0) break;
    if (jt_key_eq<KW>(t, e, kw)) ++n;
    s = (s + 1) & mask;
  }
  return n;
}

// ------------------------------------------------------------------ stage loading
// Warm L2 with a future full tile of this CTA: more bytes in flight than the
// shared-memory ring holds, so the ring's bulk copies mostly hit L2.
__device__ __forceinline__ void prefetch_tile(const PipeParams& p, u32 tile) {
  if (tile >= p.ntiles || p.rows - (u64)tile * kTile < (u64)kTile) return;
  const u64 r0 = (u64)tile * kTile;
  for (u32 c = 0; c < p.nstaged; ++c) {
    const StagedCol& sc = p.cols[c];
    if (!sc.bulk_ok || !((p.load_mask >> c) & 1)) continue;
    bulk_prefetch_l2(sc.values + r0 * sc.width, kTile * sc.width);
    if (sc.validity) bulk_prefetch_l2(sc.validity + r0 / 8, kTile / 8);
  }
}

// Plain loads (by the producer warp) for tail tiles and misaligned columns.
__device__ __forceinline__ void manual_tile(const PipeParams& p, uint8_t* stage, u32 tile, u32 lane) {
  u64 r0 = (u64)tile * kTile;
  u64 n = min((u64)kTile, p.rows - r0);
  bool full = n == (u64)kTile;
  for (u32 c = 0; c < p.nstaged; ++c) {
    const StagedCol& sc = p.cols[c];
    if ((full && sc.bulk_ok) || !((p.load_mask >> c) & 1)) continue;
    u64 bytes = n * sc.width;
    const uint8_t* src = sc.values + r0 * sc.width;
    for (u64 i = lane; i < bytes; i += 32) stage[sc.off + i] = src[i];
    if (sc.validity) {
      u64 vb = (n + 7) / 8;
      for (u64 i = lane; i < kTile / 8; i += 32) stage[sc.voff + i] = i < vb ? sc.validity[r0 / 8 + i] : 0;
    }
  }
}

// One bulk copy of the producer warp: a staged column's values or validity
// slice of a full tile.  Lane j owns copies j and j + 32, so a tile's copies
// issue in parallel with no per-tile parameter walking (the producer shares
// its scheduler with busy consumer warps; its per-tile latency gates the ring).
struct BulkCopy {
  const uint8_t* src;  // tile t starts at src + t * bytes
  u32 bytes, dst;      // bytes per tile, offset within a stage
  bool on;
};
__device__ __forceinline__ BulkCopy bulk_copy_of(const PipeParams& p, u32 j) {
  BulkCopy b{nullptr, 0, 0, false};
  const u32 c = j >> 1;
  if (c >= p.nstaged) return b;
  const StagedCol& sc = p.cols[c];
  if (!sc.bulk_ok || !((p.load_mask >> c) & 1)) return b;
  if (j & 1) {
    if (!sc.validity) return b;
    b = BulkCopy{sc.validity, (u32)(kTile / 8), sc.voff, true};
  } else {
    b = BulkCopy{sc.values, (u32)kTile * sc.width, sc.off, true};
  }
  return b;
}

// Producer warp: keeps `nstages` tiles in flight.  Stage s is refilled once
// every consumer warp has arrived on empty[s].
__device__ __forceinline__ void produce(const PipeParams& p, uint8_t* smem, uint64_t* full, uint64_t* empty,
                                        u32 lane) {
  const BulkCopy c0 = bulk_copy_of(p, lane), c1 = bulk_copy_of(p, lane + 32);
  const u64 pol = l2_policy_evict_first();  // column tiles are read once
  u32 tile_bytes = (c0.on ? c0.bytes : 0) + (c1.on ? c1.bytes : 0);
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) tile_bytes += __shfl_xor_sync(kFull, tile_bytes, m);
  u32 k = 0, s = 0, ph = 0;
  if (lane == 0)
    for (u32 j = p.nstages; j < p.nstages + p.pf_dist; ++j) prefetch_tile(p, blockIdx.x + j * gridDim.x);
  for (u32 tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++k) {
    if (p.pf_dist && lane == 0) prefetch_tile(p, tile + (p.nstages + p.pf_dist) * gridDim.x);
    if (k >= p.nstages) mbar_wait(&empty[s], ph ^ 1u);
    uint8_t* stage = smem + p.off_stage + s * p.stage_bytes;
    const bool full_tile = p.rows - (u64)tile * kTile >= (u64)kTile;
    if (!p.all_bulk || !full_tile) {
      manual_tile(p, stage, tile, lane);
      __syncwarp();
    }
    if (lane == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&full[s], full_tile ? tile_bytes : 0);
    }
    __syncwarp();
    if (full_tile) {
      if (c0.on) bulk_g2s_hint(stage + c0.dst, c0.src + (u64)tile * c0.bytes, c0.bytes, &full[s], pol);
      if (c1.on) bulk_g2s_hint(stage + c1.dst, c1.src + (u64)tile * c1.bytes, c1.bytes, &full[s], pol);
    }
    if (++s == p.nstages) { s = 0; ph ^= 1u; }
  }
}

// ---- DEST_PROBE1 output slots: a CTA hands out rows of its current kChunk-row
// chunk through one 32-bit shared word {generation:21 | used:11}; the warp
// whose reservation crosses the chunk end allocates the next chunk with one
// global atomic (so the global cursor sees ~rows/kChunk atomics, not one per
// warp and tile).  Each CTA's last chunk may stay partly unused: the holes are
// closed after the kernel (k_chunk_plan / k_chunk_move, ops.cu).
struct ChunkCursor {
  u32 word;
  u32 _pad;
  unsigned long long base[16];  // chunk start by generation (mod 16)
};
constexpr u32 kChunkUsedBits = 11;  // used <= kChunk + kThreads < 2^11
static_assert(kChunk + kThreads < (1 << kChunkUsedBits), "chunk word layout");

// Reserve m (1..32) slots for the calling lane-0: [a, a+k1) in the current
// chunk, the rest [b, b + m - k1) in a newly allocated one.
template <bool kSystem = false>
__device__ __forceinline__ void chunk_reserve(ChunkCursor* cc, u32 m, unsigned long long* gcursor, u64& a, u32& k1,
                                              u64& b) {
  for (;;) {
    const u32 old = atomicAdd(&cc->word, m);
    const u32 gen = old >> kChunkUsedBits, off = old & ((1u << kChunkUsedBits) - 1);
    if (off + m <= (u32)kChunk) {
      a = cc->base[gen & 15] + off;
      k1 = m;
      b = 0;
      return;
    }
    if (off <= (u32)kChunk) {  // this reservation crosses the chunk end
      k1 = (u32)kChunk - off;
      a = cc->base[gen & 15] + off;
      b = kSystem ? atomicAdd_system(gcursor, (unsigned long long)kChunk) : atomicAdd(gcursor, (unsigned long long)kChunk);
      ((volatile unsigned long long*)cc->base)[(gen + 1) & 15] = b;
      __threadfence_block();
      atomicExch(&cc->word, ((gen + 1) << kChunkUsedBits) | (m - k1));
      return;
    }
    while ((((volatile u32*)&cc->word)[0] >> kChunkUsedBits) == gen) {
    }
  }
}

// named barrier over the consumer warps only
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory"); }

// ------------------------------------------------------------------ COUNT without the stage ring
// The COUNT pass of a two-pass FILTER / PARTITION reads only the predicate and
// key columns (often one 8-B column).  Through the TMA stage ring that is 4 KB
// per 512-row tile and the per-tile barrier / issue overhead, not HBM, bounds it
// (~1.7 TB/s).  Here every warp reads its 32-row slices straight from global
// memory (coalesced, U slices in flight per warp), runs the same generated
// predicate / keys / LIP check on registers (P::load_g, generated policies
// only) and writes the same per-slice counts the pipeline's COUNT sink writes
// (slice = row / 32, counts[d * nslices + slice]), so the EMIT pass is unchanged.
// One mode per generated kernel (the host picks it: SINK_COUNT_DIRECT + mode,
// part of the JIT cache key): no per-slice branches on the destination kind,
// the LIP filter or the destination count's class.
template <class P, int MODE>
__device__ __forceinline__ void count_direct_loop(const PipeParams& p) {
#ifndef TQ_CD_U
#define TQ_CD_U 4
#endif
  constexpr int U = TQ_CD_U;  // slices in flight per warp; their counts leave as 16-B stores per destination
  static_assert(U % 4 == 0 && kWarps % U == 0, "nslices must be a multiple of U, U of 4");
  __shared__ u32 s_wc[8][kMaxDest];  // CD_PART_MANY: per-warp counters (blockDim 256)
  const u32 lane = threadIdx.x & 31;
  u32* wc = s_wc[threadIdx.x >> 5];
  if (MODE == CD_PART_MANY) {
    for (u32 d = lane; d < kMaxDest; d += 32) wc[d] = 0;
    __syncwarp();
  }
  const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
  const u64 nslices = (u64)p.ntiles * kWarps;  // padded like the pipeline's: empty slices count 0
  const u32 ndest = p.ndest;
  const u32 dbits = ndest > 1 ? 32u - (u32)__clz((int)(ndest - 1)) : 0u;
  WCtx w;
  w.p = &p;
  w.stage = nullptr;
  w.lits = p.lits;
  w.vslot = nullptr;
  w.vvalid = nullptr;
  w.bslot = nullptr;
  w.row0 = 0;
  w.lane = lane;
  w.out_delta = 0;
  w.vmask = kFull;
  // CD_PROBE: the build's exact membership bitmap replaces the Bloom pre-check
  const bool exact = MODE == CD_PROBE && p.jt.exact_flag && *p.jt.exact_flag == 0;
  for (u64 s0 = gw * U; s0 < nslices; s0 += nw * U) {
    typename P::Raw raw[U];
    // rows past the end re-read the last row (no branch around the loads, so
    // the ballots below need no divergence handling); tile_begin masks them
#pragma unroll
    for (int u = 0; u < U; ++u) P::load_g(w, min((u64)((s0 + u) * 32 + lane), (u64)(p.rows - 1)), raw[u]);
    u32 cnt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const u64 r0 = (s0 + u) * 32;
      w.nrows = r0 < p.rows ? (u32)min((u64)32, p.rows - r0) : 0u;
      u32 pm = 0;
      P::tile_begin(w, nullptr, &pm, &raw[u]);
      if (MODE == CD_FILTER) {
        cnt[u] = (u32)__popc(pm);
        continue;
      }
      bool pass = (pm >> lane) & 1u;
      if (MODE == CD_PROBE) {  // output rows = matches per probe row (null keys never match)
        u32 mult = 0;
        if (pass) {
          u64 kw[kMaxKeyWords + 1];
          if (!P::keys(w, 0, kw, raw[u])) mult = jt_probe_count<P::kKw>(p.jt, kw, exact);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mult += __shfl_xor_sync(kFull, mult, o);
        cnt[u] = mult;
        continue;
      }
      // every lane hashes its row (no divergent branch); non-passing lanes are masked below
      u64 kw[kMaxKeyWords + 1];
      const bool has_null = P::keys(w, 0, kw, raw[u]);
      const u32 dest = partition_of_p<P>(p, kw);
      if (MODE == CD_PART_FEW_LIP && pass) {  // LIP, as the pipeline's COUNT sink
        const u64 hb = key_hash(kw, P::kKw > 0 ? P::kKw : (int)p.key_words);
        const u32 bb = bloom_bits(hb);
        const uint32_t* sb = p.semi_bloom + (u64)dest * p.semi_part_words;
        if (has_null || (__ldg(sb + bloom_word(hb, p.semi_mask)) & bb) != bb) pass = false;
      }
      if (MODE != CD_PART_MANY) {
        // lane d's rows = passing rows whose destination bits equal d's: one
        // ballot per destination bit (log2 ndest <= 5), one popc
        // (ballots outside any branch: no divergence-safe collective code)
        u32 m = __ballot_sync(kFull, pass);
#pragma unroll
        for (u32 b = 0; b < 5; ++b) {
          const u32 bb = __ballot_sync(kFull, (dest >> b) & 1u);
          m &= b >= dbits ? ~0u : ((lane >> b) & 1u) ? bb : ~bb;
        }
        cnt[u] = (u32)__popc(m);
      } else {
        const u32 peers = __match_any_sync(kFull, pass ? dest : 0xffffffffu);
        if (pass && (peers & lanemask_lt()) == 0) wc[dest] += (u32)__popc(peers);
        __syncwarp();
        for (u32 d = lane; d < ndest; d += 32) {
          p.tile_counts[(u64)d * nslices + s0 + u] = wc[d];
          wc[d] = 0;
        }
        __syncwarp();
      }
    }
    if (MODE != CD_PART_MANY) {
      const u32 nd = MODE == CD_FILTER || MODE == CD_PROBE ? 1u : ndest;
      if (lane < nd) {
#pragma unroll
        for (int j = 0; j < U; j += 4)
          *(uint4*)(p.tile_counts + (u64)lane * nslices + s0 + j) =
              make_uint4(cnt[j], cnt[j + 1], cnt[j + 2], cnt[j + 3]);
      }
    }
  }
}

// ------------------------------------------------------------------ the kernel body
template <int SINK, class P>
__device__ __forceinline__ void pipe_body(const PipeParams& p) {
  extern __shared__ __align__(128) uint8_t smem[];
  DInstr* s_code = (DInstr*)(smem + p.off_code);
  DLit* s_lits = (DLit*)(smem + p.off_lits);
  uint64_t* full = (uint64_t*)(smem + p.off_bar);
  uint64_t* empty = full + kMaxStages;
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int KWA = P::kKwa;  // > 0 when known at compile time

  // single-pass probe of a table whose build saw a key twice (jt.dup_dev,
  // exact for one-word keys): flag it at once — the host runs the two-pass
  // probe — instead of scanning the input for the first duplicate match.
  // (Uniform over the grid; every CTA leaves a "no hole" tail for the fix-up.)
  // (A table without hash entries — semi-only or direct — whose bitmap is not
  // exact is flagged the same way: the host builds the hash table.)
  if (SINK == SINK_EMIT && p.dest_kind == DEST_PROBE1 &&
      ((p.jt.dup_dev && *(volatile u32*)p.jt.dup_dev) ||
       (!p.jt.entries && p.jt.exact_flag && *(volatile u32*)p.jt.exact_flag))) {
    if (threadIdx.x == 0) {
      p.chunk_tail[2 * blockIdx.x] = 0;
      p.chunk_tail[2 * blockIdx.x + 1] = kChunk;
      // (a semi-only build has no table to probe two-pass: ask for the table)
      if (blockIdx.x == 0) *(volatile u32*)p.dup_flag = p.jt.entries ? 1u : 2u;
    }
    return;
  }

  if (P::kInterp) {
    for (u32 i = threadIdx.x; i < p.ncode; i += kBlock) s_code[i] = p.code[i];
    for (u32 i = threadIdx.x; i < p.nlits; i += kBlock) s_lits[i] = p.lits[i];
  }
  // AGG: new global groups of this CTA (in the padding after the barriers)
  unsigned long long* s_groups = (unsigned long long*)(smem + p.off_bar + 2 * kMaxStages * 8);
  if (threadIdx.x == 0) {
    for (u32 s = 0; s < p.nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
    *s_groups = 0;
  }

  // sink shared state
  u32* s_cnt = (u32*)(smem + p.off_sink);                                          // [kWarps][kMaxDest]
  unsigned long long* s_base = (unsigned long long*)(s_cnt + kWarps * kMaxDest);  // [kWarps][kMaxDest]
  const u32 kwa = KWA > 0 ? (u32)KWA : p.key_words + 1;
  const u32 G = p.local_groups;
  // rows one lane can add to one accumulator plane in this launch
  const bool bounded = ((p.ntiles + gridDim.x - 1) / gridDim.x) * (u32)kV <= (1u << 16);
  const u32 nacc = P::nacc(p);
  const u32 nplanes = P::nplanes(p);
  // AGG smem: [state G u32][keys G*kwa u64][gslot G i64][planes G*nplanes*kThreads u64]
  u32* l_state = (u32*)(smem + p.off_sink);
  u64* l_keys = (u64*)(smem + p.off_sink + ((G * 4 + 15) & ~15u));
  long long* l_gslot = (long long*)(l_keys + (u64)G * kwa);
  u64* l_planes = (u64*)(l_gslot + G);
  if (SINK == SINK_COUNT || SINK == SINK_EMIT) {
    for (u32 i = threadIdx.x; i < kWarps * kMaxDest; i += kThreads) s_cnt[i] = 0;
  }
  ChunkCursor* s_chunk = (ChunkCursor*)s_base;  // DEST_PROBE1 only (s_base unused there)
  if (SINK == SINK_EMIT && threadIdx.x == 0) s_chunk->word = (u32)kChunk;  // generation 0, full: first use allocates
  if (SINK == SINK_EMIT && p.dest_kind == DEST_PEER && threadIdx.x < p.ndest) s_chunk[threadIdx.x].word = (u32)kChunk;
  if (SINK == SINK_AGG && threadIdx.x < kThreads) {
    for (u32 i = threadIdx.x; i < G; i += kThreads) l_state[i] = kStEmpty;
#pragma unroll
    for (u32 a = 0; a < (P::kNacc > 0 ? (u32)P::kNacc : (u32)kMaxAcc); ++a) {
      if (a >= nacc) break;
      const uint8_t op = P::acc_op(p, a);
      u64 lo, hi;
      acc_identity(op, lo, hi);
      const u32 np = (op == ACC_MIN_I || op == ACC_MAX_I) ? 2 : 1;
      for (u32 g = 0; g < G; ++g)
        for (u32 q = 0; q < np; ++q)
          l_planes[((u64)g * nplanes + P::acc_plane(p, a) + q) * kThreads + threadIdx.x] = q ? hi : lo;
    }
  }
  __syncthreads();
  if (warp == kWarps) {  // producer warp
    produce(p, smem, full, empty, lane);
    return;
  }

  WCtx w;
  w.p = &p;
  w.lits = P::kInterp ? s_lits : p.lits;
  w.vslot = smem + p.off_vslot + (size_t)warp * p.nvslots * kV * 32 * 16;
  w.vvalid = (u32*)(smem + p.off_vvalid) + (size_t)warp * p.nvslots * kV;
  w.bslot = (u32*)(smem + p.off_bslot) + (size_t)warp * p.nbslots * kV * 2;
  w.row0 = warp * 32 * kV;
  w.lane = lane;
  w.out_delta = 0;
  w.vmask = 0xffffffffu;
  if (SINK == SINK_EMIT && p.dest_kind == DEST_PEER && p.peer_vmask) {
    // a column has a bitmap on the receivers iff any rank's input can be null
    // there (concat rule, transform.cpp:63-68): OR of the all-gathered masks
    u64 m = 0;
    for (u32 r = 0; r < p.ndest; ++r) m |= __ldg(p.peer_vmask + r);
    w.vmask = (u32)m;
  }

  const u32 first = blockIdx.x, step = gridDim.x;
  u32 s = 0, ph = 0;
  // single-pass probe: walk clusters for a duplicate match only when the build
  // did not prove its keys unique
  bool walk_dups = true;
  if (SINK == SINK_EMIT && p.dest_kind == DEST_PROBE1 && p.jt.dup_dev) walk_dups = *p.jt.dup_dev != 0;
  // probes: the build's exact membership bitmap replaces the Bloom check; a
  // semi-join (no build columns) over proven-unique keys then skips the table
  bool exact = false, semi_skip = false, direct = false;
  if ((SINK == SINK_EMIT || SINK == SINK_COUNT) && (p.dest_kind == DEST_PROBE1 || p.dest_kind == DEST_PROBE) &&
      p.jt.exact_flag) {
    exact = *p.jt.exact_flag == 0;
    semi_skip = exact && p.probe_semi && p.dest_kind == DEST_PROBE1 && !walk_dups;
    // direct-indexed table: exact bitmap + unique keys -> one 4-B slot read per hit
    direct = !semi_skip && exact && p.dest_kind == DEST_PROBE1 && !walk_dups && p.jt.direct != nullptr;
  }
  // a build without a hash table (semi-only or direct) that turned out not
  // exact / not unique: flag it (the host builds the table and re-runs this
  // probe), touch nothing
  const bool no_table =
      SINK == SINK_EMIT && p.dest_kind == DEST_PROBE1 && p.jt.entries == nullptr && !semi_skip && !direct;
  if (no_table && threadIdx.x == 0) *(volatile u32*)p.dup_flag = 2;
  // two-pass partition EMIT: this warp's scanned slice offsets (one per
  // destination) are fetched before waiting on the stage, so their latency
  // overlaps it (hash_partition 1.234 -> 1.169 ms SF10; a filter measured slower)
  const bool slice_emit = SINK == SINK_EMIT && p.tile_offsets && p.dest_kind == DEST_PARTITION;
  // DEST_RANGE: this lane's running min / max of the first key word
  long long r_min = 0x7fffffffffffffffll, r_max = (long long)0x8000000000000000ull;
  bool r_null = false;
  for (u32 tile = first; tile < p.ntiles; tile += step) {
    unsigned long long pre_base = 0;
    if (slice_emit && lane < p.ndest)
      pre_base = __ldg(p.tile_offsets + (u64)lane * ((u64)p.ntiles * kWarps) + (u64)tile * kWarps + warp);
    uint8_t* stage = smem + p.off_stage + s * p.stage_bytes;
    mbar_wait(&full[s], ph);
    const u64 r0 = (u64)tile * kTile;
    w.stage = stage;
    w.nrows = (u32)min((u64)kTile, p.rows - r0);

    // ---- generated programs copy the row's staged columns into registers
    // and hand the stage back at once (the next tile's copy overlaps all of
    // this tile's work); the interpreter reads the stage until the tile ends
    typename P::Raw raw[kV];
    if (!P::kInterp) {
#pragma unroll
      for (int v = 0; v < kV; ++v) P::load(w, v, raw[v]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ---- predicate per row, then the rest of the program
    u32 pm[kV];
    u32 any = P::tile_begin(w, s_code, pm, raw);

    if (SINK == SINK_EMIT && p.dest_kind == DEST_PEER) {
      // fused partition + NVLink scatter: every passing row goes straight into
      // its destination rank's receive window (peer memory via CUDA IPC)
#pragma unroll
      for (int v = 0; v < kV; ++v) {
        bool pass = (pm[v] >> lane) & 1u;
        u32 dest = 0;
        if (p.bcast) {
          // broadcast (a join's build side to every rank): each passing row
          // goes to every destination window
          const u32 grp = __ballot_sync(kFull, pass);
          if (grp) {
            for (u32 d = 0; d < p.ndest; ++d) {
              u64 a = 0, b = 0;
              u32 k1 = 0;
              if (lane == 0) {
                chunk_reserve<true>(s_chunk + d, (u32)__popc(grp), p.peer_counter[d], a, k1, b);
                s_cnt[warp * kMaxDest + d] += (u32)__popc(grp);
              }
              a = __shfl_sync(kFull, a, 0);
              b = __shfl_sync(kFull, b, 0);
              k1 = __shfl_sync(kFull, k1, 0);
              if (pass) {
                const u32 rank = __popc(grp & lanemask_lt());
                const u64 pos = rank < k1 ? a + rank : b + (rank - k1);
                if (pos < p.peer_cap) {
                  w.out_delta = p.peer_delta[d];
                  P::store(w, v, pos, -1, raw[v]);
                  w.out_delta = 0;
                }
              }
            }
          }
          continue;
        }
        if (pass) {
          u64 kw[kMaxKeyWords + 1];
          const bool has_null = P::keys(w, v, kw, raw[v]);
          dest = partition_of_p<P>(p, kw);
          if (p.semi_bloom) {  // LIP: keys absent from the build side's Bloom filter cannot join
            const u64 hb = key_hash(kw, P::kKw > 0 ? P::kKw : (int)p.key_words);
            const u32 bb = bloom_bits(hb);
            const uint32_t* sb = p.semi_bloom + (u64)dest * p.semi_part_words;
            if (has_null || (__ldg(sb + bloom_word(hb, p.semi_mask)) & bb) != bb) pass = false;
          }
        }
        u32 todo = __ballot_sync(kFull, pass);
        while (todo) {
          const u32 leader = __ffs(todo) - 1;
          const u32 d = __shfl_sync(kFull, dest, leader);
          const u32 grp = __ballot_sync(kFull, pass && dest == d);
          todo &= ~grp;
          u64 a = 0, b = 0;
          u32 k1 = 0;
          if (lane == leader) {
            chunk_reserve<true>(s_chunk + d, (u32)__popc(grp), p.peer_counter[d], a, k1, b);
            s_cnt[warp * kMaxDest + d] += (u32)__popc(grp);  // rows per destination (NVLink accounting)
          }
          a = __shfl_sync(kFull, a, leader);
          b = __shfl_sync(kFull, b, leader);
          k1 = __shfl_sync(kFull, k1, leader);
          if (pass && dest == d) {
            const u32 rank = __popc(grp & lanemask_lt());
            const u64 pos = rank < k1 ? a + rank : b + (rank - k1);
            if (pos < p.peer_cap) {  // beyond: counted, not written (the host grows the window and re-runs)
              w.out_delta = p.peer_delta[d];
              P::store(w, v, pos, -1, raw[v]);
              w.out_delta = 0;
            }
          }
        }
      }
    } else if (SINK == SINK_COUNT && p.dest_kind == DEST_RANGE) {
#pragma unroll
      for (int v = 0; v < kV; ++v) {
        if (!((pm[v] >> lane) & 1u)) continue;
        u64 kw[kMaxKeyWords + 1];
        if (P::keys(w, v, kw, raw[v])) {
          r_null = true;
        } else {
          r_min = min(r_min, (long long)kw[0]);
          r_max = max(r_max, (long long)kw[0]);
        }
      }
    } else if ((SINK == SINK_COUNT || SINK == SINK_EMIT) && p.dest_kind == DEST_PROBE1) {
      // single pass: unique build keys -> at most one match per probe row
#pragma unroll
      for (int v = 0; v < kV; ++v) {
        bool pass = (pm[v] >> lane) & 1u;
        long long brow = -1;
        if (pass) {
          u64 kw[kMaxKeyWords + 1];
          bool dup = false;
          if (!P::keys(w, v, kw, raw[v])) {
            if (semi_skip) brow = jt_exact_hit(p.jt, kw[0]) ? 0 : -1;  // no build column is read
            else if (direct) brow = jt_exact_hit(p.jt, kw[0]) ? (long long)__ldg(p.jt.direct + kw[0]) : -1;
            else if (!no_table) brow = jt_probe_first<P::kKw>(p.jt, kw, walk_dups, dup, exact);
          }
          if (dup && *(volatile u32*)p.dup_flag == 0) *(volatile u32*)p.dup_flag = 1;
        }
        const u32 mm = __ballot_sync(kFull, brow >= 0);
        if (mm) {
          u64 a = 0, b = 0;
          u32 k1 = 0;
          if (lane == 0) chunk_reserve(s_chunk, (u32)__popc(mm), p.cursor, a, k1, b);
          a = __shfl_sync(kFull, a, 0);
          b = __shfl_sync(kFull, b, 0);
          k1 = __shfl_sync(kFull, k1, 0);
          const u32 rank = __popc(mm & lanemask_lt());
          if (brow >= 0) P::store(w, v, rank < k1 ? a + rank : b + (rank - k1), brow, raw[v]);
        }
      }
    } else if (SINK == SINK_COUNT || SINK == SINK_EMIT) {
      // two passes, stable: COUNT writes per-warp-slice counts, EMIT scatters
      // from the scanned per-warp-slice offsets; no cross-warp synchronisation
      const u64 slice = (u64)tile * kWarps + warp;
      const u64 nslices = (u64)p.ntiles * kWarps;
      u32 dest[kV];
      u32 mult[kV];
#pragma unroll
      for (int v = 0; v < kV; ++v) {
        bool pass = (pm[v] >> lane) & 1u;
        dest[v] = 0;
        mult[v] = pass ? 1u : 0u;
        if (pass && p.dest_kind != DEST_FILTER) {
          u64 kw[kMaxKeyWords + 1];
          bool has_null = P::keys(w, v, kw, raw[v]);
          if (p.dest_kind == DEST_PARTITION) dest[v] = partition_of_p<P>(p, kw);
          if (p.dest_kind == DEST_PARTITION && p.semi_bloom) {
            // Lookahead Information Passing: a key absent from the (global or
            // destination part's) build-side Bloom filter cannot join -> never shipped
            const u64 hb = key_hash(kw, P::kKw > 0 ? P::kKw : (int)p.key_words);
            const u32 bb = bloom_bits(hb);
            const uint32_t* sb = p.semi_bloom + (u64)dest[v] * p.semi_part_words;
            if (has_null || (__ldg(sb + bloom_word(hb, p.semi_mask)) & bb) != bb) mult[v] = 0;
          }
          if (p.dest_kind != DEST_PARTITION)
            mult[v] = has_null ? 0u : jt_probe_count<P::kKw>(p.jt, kw, exact);  // null keys never match
        }
      }
      u32* wc = s_cnt + warp * kMaxDest;  // this warp's per-destination counters
      if (SINK == SINK_COUNT) {
        if (p.dest_kind == DEST_PROBE) {
          u32 tot = 0;
#pragma unroll
          for (int v = 0; v < kV; ++v) tot += mult[v];
#pragma unroll
          for (int m = 16; m > 0; m >>= 1) tot += __shfl_xor_sync(kFull, tot, m);
          if (lane == 0) p.tile_counts[slice] = tot;
        } else {
#pragma unroll
          for (int v = 0; v < kV; ++v) {
            bool pass = mult[v] != 0;
            u32 peers = __match_any_sync(kFull, pass ? dest[v] : 0xffffffffu);
            if (pass && (peers & lanemask_lt()) == 0) wc[dest[v]] += __popc(peers);
            __syncwarp();
          }
          for (u32 d = lane; d < p.ndest; d += 32) {
            p.tile_counts[(u64)d * nslices + slice] = wc[d];
            wc[d] = 0;
          }
          __syncwarp();
        }
      } else {
        unsigned long long* wb = s_base + warp * kMaxDest;
        for (u32 d = lane; d < p.ndest; d += 32)
          wb[d] = !p.tile_offsets          ? (u64)tile * kTile + w.row0
                  : slice_emit && d < 32 ? pre_base
                                         : p.tile_offsets[(u64)d * nslices + slice];
        __syncwarp();
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
              P::keys(w, v, kw, raw[v]);
              const JoinTable& t = p.jt;
              const u64 mask = t.cap - 1;
              u64 sl = jt_home<P::kKw>(t, kw, key_hash(kw, P::kKw > 0 ? P::kKw : (int)t.kw));
              for (;;) {
                const long long* e = jt_entry(t, sl);
                long long brow = e[0];
                if (brow < 0) break;
                if (jt_key_eq<P::kKw>(t, e, kw)) {
                  P::store(w, v, pos, brow, raw[v]);
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
            if (pass) P::store(w, v, pos, -1, raw[v]);
          }
        }
      }
    } else if (SINK == SINK_BUILD) {
      // read keys into registers, release the stage, then insert
      u64 kws[kV][kMaxKeyWords + 1];
      bool ok[kV];
#pragma unroll
      for (int v = 0; v < kV; ++v) {
        ok[v] = ((pm[v] >> lane) & 1u) && !P::keys(w, v, kws[v], raw[v]);  // null keys never match
      }
      if (p.jt.exact_bits && !p.build_skip_aux) {
        // exact membership bits: lanes whose keys share a bitmap word (dense,
        // often consecutive keys) merge their bits, one atomic per word
        const u64 range = p.jt.exact_range;
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          const bool in = ok[v] && kws[v][0] < range;
          const u64 word = in ? (kws[v][0] >> 5) : ~0ull;
          const u32 peers = __match_any_sync(kFull, word);
          const u32 bits = __reduce_or_sync(peers, in ? 1u << (kws[v][0] & 31) : 0u);
          if (in && (peers & lanemask_lt()) == 0) {
            const u32 old = atomicOr(p.jt.exact_bits + word, bits);
            // a bit already set, or two lanes on one bit: a key inserted twice
            if (((old & bits) != 0 || __popc(bits) < __popc(peers)) && p.jt.dup_dev &&
                *(volatile u32*)p.jt.dup_dev == 0)
              *(volatile u32*)p.jt.dup_dev = 1;
          }
          if (ok[v] && !in && *(volatile u32*)p.jt.exact_flag == 0) *(volatile u32*)p.jt.exact_flag = 1;
          // direct-indexed table: the row lands in its key's slot (dense keys:
          // neighbouring lanes store to neighbouring slots)
          if (in && p.jt.direct) p.jt.direct[kws[v][0]] = (u32)(p.row_base + r0 + trow(w, v));
        }
      }
#pragma unroll
      for (int v = 0; v < kV; ++v) {
        if (!ok[v]) continue;
        const u64* kw = kws[v];
        const JoinTable& t = p.jt;
        const u64 mask = t.cap - 1;
        const u64 hb = key_hash(kw, P::kKw > 0 ? P::kKw : (int)t.kw);
        u64 sl = jt_home<P::kKw>(t, kw, hb);
        long long row = (long long)(p.row_base + r0 + trow(w, v));
        if (t.bloom && !p.build_skip_aux) atomicOr(t.bloom + bloom_word(hb, t.bloom_mask), bloom_bits(hb));
        if (!t.entries) continue;  // Bloom-only build (LIP filter)
        // slot-range pass of a partitioned build: only keys whose home slot is
        // in [slot_lo, slot_hi) are inserted by this launch (that range of the
        // table stays L2-resident while it fills)
        if (p.slot_hi && (sl < p.slot_lo || sl >= p.slot_hi)) continue;
        if ((P::kKw == 1 || (P::kKw == 0 && t.kw == 1)) && t.dup_dev) {
          // {row, key} claimed in one 128-bit CAS against the empty pattern
          // (all ones): an equal key already present is seen atomically
          bool dup = false;
          for (;;) {
            long long* e = (long long*)(t.entries + sl * t.stride);
            u64 olo, ohi;
            cas128(e, ~0ull, ~0ull, (u64)row, kw[0], olo, ohi);
            if (olo == ~0ull && ohi == ~0ull) break;
            dup |= ohi == kw[0];
            sl = (sl + 1) & mask;
          }
          if (dup && *(volatile u32*)t.dup_dev == 0) *(volatile u32*)t.dup_dev = 1;
          if (p.cursor) atomicAdd(p.cursor, 1ull);
          continue;
        }
        for (;;) {
          long long* e = (long long*)(t.entries + sl * t.stride);
          if (atomicCAS((unsigned long long*)e, (unsigned long long)-1ll, (unsigned long long)row) ==
              (unsigned long long)-1ll) {
            if (p.cursor) atomicAdd(p.cursor, 1ull);
#pragma unroll
            for (u32 i = 0; i < (P::kKw > 0 ? (u32)P::kKw : (u32)kMaxKeyWords); ++i) {
              if (i >= t.kw) break;
              e[1 + i] = (long long)kw[i];
            }
            break;
          }
          sl = (sl + 1) & mask;
        }
      }
    } else if (SINK == SINK_AGG) {
      // read every input of the row into registers, release the stage, then
      // do the hash-table / accumulator work (keeps more tiles in flight)
      RowVals xs[kV];
#pragma unroll
      for (int v = 0; v < kV; ++v) {  // for every row: no divergent merge of the values
        P::keys(w, v, xs[v].kw, raw[v]);
        P::accs(w, v, xs[v], raw[v]);
      }
      if (p.agg.direct) {
        // DIRECT: slot = key - key_min.  Lanes holding the same slot in a
        // contiguous run (sorted / clustered keys) are reduced with a
        // segmented warp scan first; the run's last lane applies it with one
        // atomic per accumulator (one global atomic per run, not per row).
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          const bool pass = (pm[v] >> lane) & 1u;
          RowVals& x = xs[v];
          const u32 act = __ballot_sync(kFull, pass);
          if (!act) continue;
          u64 slot = ~0ull;
          if (pass) slot = x.kw[kwa - 1] ? p.agg.direct_slots : x.kw[0] - (u64)p.agg.key_min;
          const u64 prev = __shfl_up_sync(kFull, slot, 1);
          const bool head = pass && (lane == 0 || prev != slot || !((act >> (lane - 1)) & 1u));
          const u32 heads = __ballot_sync(kFull, head);
          const u32 start = 31 - __clz(heads & (lanemask_lt() | (1u << lane)) | 1u);  // my run's first lane
          const bool tail = pass && (lane == 31 || ((heads >> (lane + 1)) & 1u) || !((act >> (lane + 1)) & 1u));
          // sorted key column: a run whose key differs from the warp's first and
          // last row's key holds every row of that key (the rows before / after
          // this warp's 32 consecutive rows cannot have it) -> plain stores
          bool excl = false;
          if (p.agg.sorted) {
            const u64 rslot = trow(w, v) < w.nrows ? x.kw[0] - (u64)p.agg.key_min : ~1ull;
            const u64 first = __shfl_sync(kFull, rslot, 0), last = __shfl_sync(kFull, rslot, 31);
            excl = slot != first && slot != last;
          }
#pragma unroll
          for (u32 a = 0; a < (P::kNacc > 0 ? (u32)P::kNacc : (u32)kMaxAcc); ++a) {
            if (a >= nacc) break;
            const uint8_t op = P::acc_op(p, a);
            const bool valid = pass && x.av[a];
            u64* acc = tail ? direct_acc(p.agg, a, slot) : nullptr;
            if (op == ACC_CNT) {
              u32 sv;
              if (P::acc_kind(p, a) == K_NONE) {
                sv = lane - start + 1;  // Count(*): every row of the run counts
              } else {
                sv = valid ? 1u : 0u;  // a run is <= 32 rows
#pragma unroll
                for (u32 o = 1; o < 32; o <<= 1) {
                  const u32 y = __shfl_up_sync(kFull, sv, o);
                  if (lane >= start + o) sv += y;
                }
              }
              if (tail) {
                if (excl) acc[0] = sv;
                else atomicAdd((unsigned long long*)acc, (unsigned long long)sv);  // RED: no return
              }
            } else if (op == ACC_SUM_I) {
              // 64-bit scan when every lane's value is within +-2^58 (32 of
              // them cannot overflow), else the int128 scan
              const i128 xv = valid ? x.ai[a] : (i128)0;
              const bool narrow = __all_sync(kFull, (((u128)xv + ((u128)1 << 58)) >> 59) == 0);
              i128 sv;
              if (narrow) {
                long long v64 = (long long)lo64(xv);
#pragma unroll
                for (u32 o = 1; o < 32; o <<= 1) {
                  const long long y = (long long)__shfl_up_sync(kFull, (unsigned long long)v64, o);
                  if (lane >= start + o) v64 += y;
                }
                sv = (i128)v64;
              } else {
                sv = xv;
#pragma unroll
                for (u32 o = 1; o < 32; o <<= 1) {
                  const i128 y = shfl_up_i128(sv, o);
                  if (lane >= start + o) sv = add128(sv, y);
                }
              }
              if (tail && sv != 0) {
                // limb form {sum of low 32-bit limbs, sum of signed high parts}:
                // two fire-and-forget REDs (an int128 add with carry needs the
                // old value back: one dependent ATOM round trip per run).
                // Exact while every run's sum fits int64 (else the host
                // re-runs this aggregate on the hash table)
                if (fits64(sv)) {
                  const long long v = (long long)lo64(sv);
                  if (excl) {
                    *(ulonglong2*)acc = make_ulonglong2((unsigned long long)(v & 0xffffffffll), (unsigned long long)(v >> 32));
                  } else {
                    atomicAdd((unsigned long long*)acc, (unsigned long long)(v & 0xffffffffll));
                    atomicAdd((unsigned long long*)acc + 1, (unsigned long long)(v >> 32));
                  }
                } else if (*(volatile u32*)p.agg.overflow == 0) {
                  atomicExch(p.agg.overflow, 1u);
                }
              }
            } else if (op == ACC_SUM_F) {
              double sv = valid ? x.af[a] : 0.0;
#pragma unroll
              for (u32 o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(kFull, sv, o);
                if (lane >= start + o) sv += y;
              }
              if (tail) atomicAdd((double*)acc, sv);
            } else if (op == ACC_MIN_I || op == ACC_MAX_I) {
              u64 lo, hi;
              acc_identity(op, lo, hi);
              i128 sv = valid ? x.ai[a] : mk128(lo, hi);
#pragma unroll
              for (u32 o = 1; o < 32; o <<= 1) {
                const i128 y = shfl_up_i128(sv, o);
                if (lane >= start + o) sv = (op == ACC_MIN_I) ? (y < sv ? y : sv) : (y > sv ? y : sv);
              }
              if (tail && sv != mk128(lo, hi)) atomic_minmax_i128((u128*)acc, sv, op == ACC_MIN_I);
            } else {
              u64 lo, hi;
              acc_identity(op, lo, hi);
              double sv = valid ? x.af[a] : __longlong_as_double((long long)lo);
#pragma unroll
              for (u32 o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(kFull, sv, o);
                if (lane >= start + o) sv = (op == ACC_MIN_F) ? fmin(sv, y) : fmax(sv, y);
              }
              if (tail && valid_any_f(sv, lo)) atomic_minmax_f64((double*)acc, sv, op == ACC_MIN_F);
            }
          }
        }
      } else if (any) {
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          bool pass = (pm[v] >> lane) & 1u;
          if (!pass) continue;
          RowVals& x = xs[v];
          // cheap 32-bit hash for the CTA-local table; the global table's
          // key_hash is only computed on the (rare) paths that reach it
          long long ls = G ? local_find_insert<KWA>(l_state, l_keys, G, kwa, x.kw, local_hash(x.kw, (int)kwa)) : -1;
          // bounded planes: when every integer input of the row is within
          // +-2^46, plain 64-bit adds cannot overflow a plane (<= 2^16 rows per lane)
          u64 excess = 0;
#pragma unroll
          for (u32 a = 0; a < (P::kNacc > 0 ? (u32)P::kNacc : (u32)kMaxAcc); ++a) {
            if (a >= nacc) break;
            if (P::acc_op(p, a) == ACC_SUM_I && x.av[a]) excess |= plane_excess(x.ai[a]);
          }
          const bool fast = bounded && excess == 0;
          if (ls >= 0 && fast) {
            u64* pl0 = l_planes + (u64)ls * nplanes * kThreads + threadIdx.x;
#pragma unroll
            for (u32 a = 0; a < (P::kNacc > 0 ? (u32)P::kNacc : (u32)kMaxAcc); ++a) {
              if (a >= nacc) break;
              const uint8_t op = P::acc_op(p, a);
              if (!x.av[a]) continue;
              u64* pl = pl0 + (u64)P::acc_plane(p, a) * kThreads;
              switch (op) {
                case ACC_CNT: pl[0] += 1; break;
                case ACC_SUM_I: pl[0] += lo64(x.ai[a]); break;
                case ACC_SUM_F:
                  pl[0] = (u64)__double_as_longlong(__longlong_as_double((long long)pl[0]) + x.af[a]);
                  break;
                case ACC_MIN_I:
                case ACC_MAX_I: {
                  i128 c = mk128(pl[0], pl[kThreads]);
                  if (op == ACC_MIN_I ? x.ai[a] < c : x.ai[a] > c) {
                    pl[0] = lo64(x.ai[a]);
                    pl[kThreads] = hi64(x.ai[a]);
                  }
                  break;
                }
                default: {
                  double c = __longlong_as_double((long long)pl[0]);
                  if (op == ACC_MIN_F ? x.af[a] < c : x.af[a] > c) pl[0] = (u64)__double_as_longlong(x.af[a]);
                }
              }
            }
          } else if (ls >= 0) {
            // per-lane private accumulation (no atomics, no cross-lane traffic)
#pragma unroll
            for (u32 a = 0; a < (P::kNacc > 0 ? (u32)P::kNacc : (u32)kMaxAcc); ++a) {
              if (a >= nacc) break;
              const uint8_t op = P::acc_op(p, a);
              if (!x.av[a]) continue;
              u64* pl = l_planes + ((u64)ls * nplanes + P::acc_plane(p, a)) * kThreads + threadIdx.x;
              switch (op) {
                case ACC_CNT: pl[0] += 1; break;
                case ACC_SUM_I: {
                  const i128 xi = x.ai[a];
                  if (bounded) {  // keep the plane bound: large inputs go to the global table exactly
                    if (fits_plane(xi)) {
                      pl[0] += lo64(xi);
                    } else {
                      long long gs = agg_global_slot<KWA>(p, x.kw, kwa, key_hash(x.kw, (int)kwa), s_groups);
                      if (gs >= 0) atomic_add_i128(p.agg.acc + ((u64)gs * nacc + a) * 2, xi);
                    }
                    break;
                  }
                  long long cur = (long long)pl[0];
                  if (fits64(xi)) {
                    long long y = (long long)lo64(xi);
                    long long r = (long long)((u64)cur + (u64)y);
                    if (((cur ^ r) & (y ^ r)) >= 0) {
                      pl[0] = (u64)r;
                      break;
                    }
                  }
                  // escape: the exact int128 partial goes straight to the global table
                  long long gs = agg_global_slot<KWA>(p, x.kw, kwa, key_hash(x.kw, (int)kwa), s_groups);
                  if (gs >= 0) atomic_add_i128(p.agg.acc + ((u64)gs * nacc + a) * 2, add128((i128)cur, xi));
                  pl[0] = 0;
                  break;
                }
                case ACC_SUM_F:
                  pl[0] = (u64)__double_as_longlong(__longlong_as_double((long long)pl[0]) + x.af[a]);
                  break;
                case ACC_MIN_I:
                case ACC_MAX_I: {
                  i128 c = mk128(pl[0], pl[kThreads]);
                  if (op == ACC_MIN_I ? x.ai[a] < c : x.ai[a] > c) {
                    pl[0] = lo64(x.ai[a]);
                    pl[kThreads] = hi64(x.ai[a]);
                  }
                  break;
                }
                default: {
                  double c = __longlong_as_double((long long)pl[0]);
                  if (op == ACC_MIN_F ? x.af[a] < c : x.af[a] > c) pl[0] = (u64)__double_as_longlong(x.af[a]);
                }
              }
            }
          } else {
            // local table full: this group lives only in the global table
            long long gs = agg_global_slot<KWA>(p, x.kw, kwa, key_hash(x.kw, (int)kwa), s_groups);
            if (gs < 0) continue;
#pragma unroll
            for (u32 a = 0; a < (P::kNacc > 0 ? (u32)P::kNacc : (u32)kMaxAcc); ++a) {
              if (a >= nacc) break;
              if (!x.av[a]) continue;
              acc_apply_atomic(P::acc_op(p, a), p.agg.acc + ((u64)gs * nacc + a) * 2, x.ai[a], x.af[a], 1);
            }
          }
        }
      }
    }

    // stage s consumed by this warp (generated programs released it above)
    if (P::kInterp) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (++s == p.nstages) { s = 0; ph ^= 1u; }
  }

  if (SINK == SINK_COUNT && p.dest_kind == DEST_RANGE) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
      r_min = min(r_min, (long long)__shfl_xor_sync(kFull, (unsigned long long)r_min, m));
      r_max = max(r_max, (long long)__shfl_xor_sync(kFull, (unsigned long long)r_max, m));
    }
    const bool any_null = __any_sync(kFull, r_null);
    if (lane == 0) {  // one set of atomics per warp and launch
      if (r_min <= r_max) {
        atomicMin(p.key_range, r_min);
        atomicMax(p.key_range + 1, r_max);
      }
      if (any_null) atomicOr((unsigned long long*)p.key_range + 2, 1ull);
    }
  }
  if (SINK == SINK_EMIT && p.dest_kind == DEST_PEER) {
    consumers_sync();
    if (threadIdx.x < p.ndest) {
      const u32 d = threadIdx.x;
      const u32 word = s_chunk[d].word;
      const u32 used = min(word & ((1u << kChunkUsedBits) - 1), (u32)kChunk);
      unsigned long long* t = p.peer_tails[d] + 2ull * (p.tail_slot0 + blockIdx.x);
      t[0] = s_chunk[d].base[(word >> kChunkUsedBits) & 15];
      t[1] = used;
      // rows this CTA stored into other ranks' windows
      unsigned long long rows = 0;
      for (u32 wi = 0; wi < (u32)kWarps; ++wi) rows += s_cnt[wi * kMaxDest + d];
      if (rows && d != p.tail_slot0 / kMaxTailCtas && p.cursor) atomicAdd(p.cursor, rows);
    }
  }
  if (SINK == SINK_EMIT && p.dest_kind == DEST_PROBE1) {
    consumers_sync();
    if (threadIdx.x == 0) {
      const u32 word = s_chunk->word;
      const u32 used = min(word & ((1u << kChunkUsedBits) - 1), (u32)kChunk);
      p.chunk_tail[2 * blockIdx.x] = s_chunk->base[(word >> kChunkUsedBits) & 15];
      p.chunk_tail[2 * blockIdx.x + 1] = used;  // kChunk: no hole (also a CTA that never emitted)
    }
  }
  if (SINK == SINK_AGG && G > 0) {
    consumers_sync();
    // 1) global slot of every local group
    for (u32 g = warp; g < G; g += kWarps) {
      if (lane == 0) {
        long long gs = -1;
        if (l_state[g] > kStBusy) {  // ready (holds the key's tag)
          u64 kw[kMaxKeyWords + 1];
          for (u32 i = 0; i < kwa; ++i) kw[i] = l_keys[(u64)g * kwa + i];
          gs = agg_global_slot<KWA>(p, kw, kwa, key_hash(kw, (int)kwa), s_groups);
        }
        l_gslot[g] = gs;
      }
    }
    consumers_sync();
    // 2) reduce the per-lane planes of each (group, accumulator) and apply once
    for (u32 q = warp; q < G * nacc; q += kWarps) {
      const u32 g = q / nacc, a = q % nacc;
      const long long gs = l_gslot[g];
      if (gs < 0) continue;
      const uint8_t op = P::acc_op(p, a);
      const u64* pl = l_planes + ((u64)g * nplanes + P::acc_plane(p, a)) * kThreads;
      i128 xi = 0;
      double xf = 0;
      u64 cnt = 0;
      switch (op) {
        case ACC_CNT:
          for (u32 t = lane; t < kThreads; t += 32) cnt += pl[t];
          for (int m = 16; m > 0; m >>= 1) cnt += __shfl_xor_sync(kFull, cnt, m);
          break;
        case ACC_SUM_I:
          for (u32 t = lane; t < kThreads; t += 32) xi = add128(xi, (i128)(long long)pl[t]);
          xi = warp_sum_i128(xi);
          break;
        case ACC_SUM_F:
          for (u32 t = lane; t < kThreads; t += 32) xf += __longlong_as_double((long long)pl[t]);
          xf = warp_sum_f64(xf);
          break;
        case ACC_MIN_I:
        case ACC_MAX_I: {
          bool mn = op == ACC_MIN_I;
          u64 lo, hi;
          acc_identity(op, lo, hi);
          xi = mk128(lo, hi);
          for (u32 t = lane; t < kThreads; t += 32) {
            i128 y = mk128(pl[t], pl[kThreads + t]);
            xi = mn ? (y < xi ? y : xi) : (y > xi ? y : xi);
          }
          for (int m = 16; m > 0; m >>= 1) {
            i128 o = shfl_xor_i128(xi, m);
            xi = mn ? (o < xi ? o : xi) : (o > xi ? o : xi);
          }
          break;
        }
        default: {
          bool mn = op == ACC_MIN_F;
          xf = __longlong_as_double((long long)pl[lane]);
          for (u32 t = lane + 32; t < kThreads; t += 32) {
            double y = __longlong_as_double((long long)pl[t]);
            xf = mn ? fmin(xf, y) : fmax(xf, y);
          }
          for (int m = 16; m > 0; m >>= 1) {
            double o = __shfl_xor_sync(kFull, xf, m);
            xf = mn ? fmin(xf, o) : fmax(xf, o);
          }
        }
      }
      if (lane == 0) acc_apply_atomic(op, p.agg.acc + ((u64)gs * nacc + a) * 2, xi, xf, cnt);
    }
  }
  if (SINK == SINK_AGG) {
    consumers_sync();
    if (threadIdx.x == 0 && *s_groups) atomicAdd(p.agg.nused, *s_groups);
  }
}

// ------------------------------------------------------------------ output stores
__device__ __forceinline__ void set_valid(const OutCol& o, u64 pos, bool valid, long long delta = 0) {
  if (o.validity && valid) bm_set_atomic(o.validity + delta, pos);
}

// Copy a build-side value (probe output) by build row id.
__device__ __forceinline__ void store_build(const OutCol& o, u64 pos, long long brow, long long delta = 0) {
  const uint8_t* src = o.bvalues + (u64)brow * o.width;
  uint8_t* dst = o.values + delta;
  if (o.width == 16) *(ulonglong2*)(dst + pos * 16) = *(const ulonglong2*)src;
  else if (o.width == 8) *(u64*)(dst + pos * 8) = *(const u64*)src;
  else dst[pos] = *src;
  set_valid(o, pos, !o.bvalidity || bm_get(o.bvalidity, (u64)brow), delta);
}

}  // namespace tq
