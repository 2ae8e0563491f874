// pipeline.h — launch parameters of the staged tile pipeline kernels
// (pipeline.cu).  One kernel family covers the per-batch operators of
// SPEC.md:560-611:
//
//   source   : the batch, tile by tile, TMA bulk-copied into shared memory
//   program  : the Expr register machine (program.h): predicate, projections,
//              keys, aggregate inputs
//   sink     : COUNT  per-tile output counts for a destination function
//              EMIT   stable scatter of rows to their destinations
//                     (filter = 1 destination, hash_partition = n, join probe
//                      = k matches per row)
//              AGG    warp-aggregated hash group-by into a global table
//              BUILD  join build: open-addressing insert of (key, row)
#pragma once
#include "program_types.h"
#include "tq_types.h"

namespace tq {

#ifndef TQ_KWARPS
#define TQ_KWARPS 16
#endif
#ifndef TQ_KV
#define TQ_KV 1
#endif
constexpr int kWarps = TQ_KWARPS;         // consumer warps per CTA
constexpr int kThreads = kWarps * 32;     // consumer threads
constexpr int kBlock = kThreads + 32;     // + one producer (TMA) warp
constexpr int kV = TQ_KV;                 // rows per lane per tile
constexpr int kTile = kThreads * kV;      // rows per tile (512)
constexpr int kMaxKeys = 4;
constexpr int kMaxKeyWords = 8;         // + 1 null word
constexpr int kMaxOut = 24;
constexpr int kMaxAcc = 16;
constexpr int kMaxDest = 64;
constexpr int kMaxStages = 6;
constexpr int kChunk = 512;  // DEST_PROBE1 output rows a CTA reserves per global atomic

enum SinkKind { SINK_COUNT = 0, SINK_EMIT = 1, SINK_AGG = 2, SINK_BUILD = 3,
                SINK_COUNT_DIRECT = 4 };  // + CdMode: COUNT without the stage ring (generated code only)
// count_direct_loop modes
enum CdMode { CD_FILTER = 0, CD_PART_FEW = 1, CD_PART_FEW_LIP = 2, CD_PART_MANY = 3, CD_PROBE = 4 };
// FILTER/PARTITION/PROBE: two passes (COUNT then EMIT), stable order.
// PROBE1: single EMIT pass for unique build keys (<= 1 match per row);
//         output rows are reserved with a warp-aggregated atomic cursor.
// RANGE (with SINK_COUNT): min / max of the first key word over passing rows
//         (+ whether a key is null) -> key_range[0..2]; sizes direct aggregation.
enum DestKind { DEST_FILTER = 0, DEST_PARTITION = 1, DEST_PROBE = 2, DEST_PROBE1 = 3, DEST_PEER = 4, DEST_RANGE = 5 };
constexpr int kMaxPeers = 16;       // DEST_PEER: ranks of one communicator
constexpr int kMaxTailCtas = 512;   // DEST_PEER: per-source-rank tail slots in a receive window

struct StagedCol {
  const uint8_t* values;
  const uint8_t* validity;  // nullptr = all valid
  uint32_t width;           // 1, 8, 16
  uint32_t off;             // smem offset of values within a stage
  uint32_t voff;            // smem offset of validity within a stage
  uint8_t bulk_ok;          // base 16-B aligned -> TMA bulk copies
  uint8_t kind;
  uint8_t _pad[2];
};

struct KeyOpnd {
  uint8_t kind;     // operand kind (program.h)
  uint8_t words;    // 1 or 2 key words
  uint8_t bytes;    // partition-hash bytes: 8, 16 or 1
  uint8_t _pad;
  uint16_t idx;
  uint16_t _pad2;
};

// Join hash table: `cap` entries of `stride` bytes: int64 row (-1 empty)
// followed by `kw` key words.
struct JoinTable {
  uint8_t* entries;
  uint64_t cap;     // power of two
  uint32_t stride;  // bytes
  uint32_t kw;
  uint32_t* bloom;  // blocked Bloom filter over the build keys (nullptr = none)
  uint32_t unique;  // host hint: probe single-pass first (cleared when a probe found a duplicate)
  // device flag written by the build: 0 = build keys proven unique (16-B
  // entries are claimed with one 128-bit CAS of {row, key}, so an equal key is
  // seen atomically), 1 = a key was inserted twice; nullptr = not tracked
  // (wider keys): single-pass probes then walk each cluster to check
  uint32_t* dup_dev;
  uint64_t bloom_mask;  // words - 1 (power of two)
  // exact membership bitmap for one-word keys in [0, exact_range):
  // bit k set <=> key k was inserted.  exact_flag (device): 0 = every key was
  // in range (the bitmap is exact), 1 = not; nullptr = not built
  uint32_t* exact_bits;
  uint32_t* exact_flag;
  uint64_t exact_range;  // a multiple of 32
  // direct-indexed table (one-word keys, no hash entries): direct[k] = the
  // build row of key k, valid iff bit k of exact_bits is set (never
  // initialised: the bitmap says which slots were written).  Usable when the
  // bitmap is exact and the keys proved unique (dup_dev); otherwise a probe
  // asks the host for the hash table.  nullptr = not built
  uint32_t* direct;
};

enum OutSrc : uint8_t { OUT_OPND = 0, OUT_BUILD = 1 };
struct OutCol {
  uint8_t src;       // OUT_OPND / OUT_BUILD
  uint8_t kind;      // operand kind for OUT_OPND
  uint8_t width;     // output width (1, 8, 16)
  uint8_t out_kind;  // TQ_* of the output column
  uint16_t idx;      // operand index
  uint16_t _pad;
  uint8_t* values;
  uint8_t* validity;  // nullptr = output has no bitmap
  const uint8_t* bvalues;    // OUT_BUILD source
  const uint8_t* bvalidity;  // OUT_BUILD source validity
};

enum AccOp : uint8_t { ACC_SUM_I = 0, ACC_SUM_F, ACC_CNT, ACC_MIN_I, ACC_MAX_I, ACC_MIN_F, ACC_MAX_F };
struct AccSpec {
  uint8_t op;
  uint8_t kind;  // operand kind (K_NONE for COUNT(*))
  uint16_t idx;
  uint8_t scale; // F conversion scale for I operands of SUM_F/MIN_F/MAX_F (unused today)
  uint8_t _pad[3];
};

#ifdef __CUDACC__
// Identity of an accumulator (16 B: lo, hi words).
__host__ __device__ __forceinline__ void acc_identity(uint8_t op, unsigned long long& lo, unsigned long long& hi) {
  switch (op) {
    case ACC_MIN_I: lo = ~0ull; hi = 0x7fffffffffffffffull; break;
    case ACC_MAX_I: lo = 0; hi = 0x8000000000000000ull; break;
    case ACC_MIN_F: lo = 0x7ff0000000000000ull; hi = 0; break;
    case ACC_MAX_F: lo = 0xfff0000000000000ull; hi = 0; break;
    default: lo = 0; hi = 0;
  }
}
#endif

// Global aggregation hash table.
struct AggTable {
  uint32_t* state;   // 0 empty, 1 writing, 2 ready
  unsigned long long* keys;  // cap * kwa
  unsigned long long* acc;   // cap * nacc * 2 words (16 B per accumulator)
  uint64_t cap;      // power of two
  unsigned long long* nused;
  uint32_t* overflow;
  // DIRECT aggregation (one integer key with a dense value range [key_min,
  // key_min + direct_slots)): the accumulators of key k live in slot
  // k - key_min (slot direct_slots = the null key); no state / key words; a
  // group exists iff its Count(*) accumulator (index cnt_acc) is non-zero
  uint32_t direct;
  uint32_t cnt_acc;
  long long key_min;
  uint64_t direct_slots;
  // direct layout: one array per accumulator (structure of arrays), slot
  // width dwidth[a] words (1 = a count, 2 = a 16-B sum / min / max), each
  // array dstride >= direct_slots + 1 slots long (even: 16-B arrays stay
  // 16-B aligned for the int128 min / max CAS)
  uint8_t dwidth[kMaxAcc];
  uint64_t dstride;
  // the key column is non-decreasing (the range pass checked it): a run of
  // one key strictly inside a warp's 32 consecutive rows holds EVERY row of
  // that key, so its slot is written with plain stores instead of atomics
  uint32_t sorted;
};

#ifdef __CUDACC__
__host__ __device__ __forceinline__ unsigned long long* direct_acc(const AggTable& t, uint32_t a, uint64_t slot) {
  uint64_t off = 0;
  for (uint32_t b = 0; b < a; ++b) off += t.dwidth[b];
  return t.acc + off * t.dstride + slot * t.dwidth[a];
}
#endif

struct PipeParams {
  uint64_t rows;
  uint64_t row_base;  // added to tile-relative row ids (BUILD row ids)
  uint32_t ntiles;
  uint32_t nstages;
  uint32_t stage_bytes;
  uint32_t all_bulk;  // every staged column is TMA-eligible (16-B aligned)
  uint32_t load_mask; // staged columns this launch reads (a COUNT pass needs only
                      // the predicate/key columns; the others are never loaded)
  uint32_t pf_dist;   // L2 prefetch distance in tiles of this CTA (0 = off)
  // shared-memory layout (bytes from dynamic smem base)
  uint32_t off_code, off_lits, off_stage, off_bar, off_vslot, off_vvalid, off_bslot, off_sink;
  // program
  const DInstr* code;
  const DLit* lits;
  uint16_t ncode, npred, nlits, nstaged;
  uint16_t nvslots, nbslots;
  uint8_t pred_kind;
  uint8_t _p0;
  uint16_t pred_idx;
  StagedCol cols[kMaxStaged];
  // keys
  uint32_t nkeys, key_words;
  KeyOpnd keys[kMaxKeys];
  // destinations
  uint32_t dest_kind, ndest;
  uint32_t* tile_counts;          // [ndest][ntiles * kWarps] (per warp-slice of a tile)
  const unsigned long long* tile_offsets;  // [ndest][ntiles * kWarps] absolute output rows
  unsigned long long* cursor;     // DEST_PROBE1 chunk cursor (rows, kChunk units); BUILD inserted-row count
  unsigned long long* chunk_tail; // DEST_PROBE1: per CTA {base, used} of its last output chunk
  // DEST_PEER (fused partition + NVLink scatter): destination d's receive
  // window is this rank's window + peer_delta[d] (CUDA IPC mapping); rows are
  // reserved in kChunk-row chunks from the receiver's counter and each CTA
  // leaves its last chunk {base, used} in the receiver's tail slots.
  long long peer_delta[kMaxPeers];
  unsigned long long* peer_counter[kMaxPeers];
  unsigned long long* peer_tails[kMaxPeers];
  uint64_t peer_cap;     // rows of every receive window
  uint32_t bcast;        // DEST_PEER: every row to every rank (no keys)
  uint32_t tail_slot0;   // this rank's first tail slot (rank * kMaxTailCtas)
  // [ndest] every rank's local output-nullability mask (all-gathered before
  // the kernel): validity bits are written for the OR of the masks
  const unsigned long long* peer_vmask;
  JoinTable jt;
  // LIP semi-join filter on the key words (dest PARTITION): rows whose keys
  // miss this Bloom filter are dropped before they are partitioned / shipped
  const uint32_t* semi_bloom;
  uint64_t semi_mask;
  // partitioned semi filter: part d's Bloom words start at d * semi_part_words
  // (each rank's build-side table Bloom, all-gathered); 0 = one global filter
  uint64_t semi_part_words;
  // emit
  uint32_t nout;
  OutCol out[kMaxOut];
  // aggregate
  uint32_t nacc;
  uint32_t local_groups;  // per-CTA smem table slots (power of two, 0 = none)
  uint32_t nplanes;       // 8-byte per-lane accumulator planes per local group
  uint8_t acc_plane[kMaxAcc];
  AccSpec acc[kMaxAcc];
  AggTable agg;
  // DEST_PROBE1: set when a probe key matches a second build row (the build
  // keys are not unique; the single-pass output is discarded)
  uint32_t* dup_flag;
  // DEST_PROBE1 with no build columns (a semi-join): with an exact bitmap and
  // proven-unique build keys the table itself is never read
  uint32_t probe_semi;
  // BUILD, partitioned into slot ranges (tables much larger than L2): this
  // launch inserts only home slots in [slot_lo, slot_hi) (slot_hi = 0: all);
  // build_skip_aux: the Bloom / exact bits were set by an earlier range pass
  uint64_t slot_lo, slot_hi;
  uint32_t build_skip_aux;
  // DEST_RANGE output: {min, max, any null} of the first key word
  long long* key_range;
  // the one key is the row's partition hash already (fnv1a64 chained over
  // key columns that include Utf8, computed by a pre-pass): part = key mod n
  uint32_t key_prehashed;
};

}  // namespace tq
