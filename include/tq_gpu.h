/*
 * tq_gpu.h — the drop-in C-ABI of libtq_gpu.so (B200 / sm_100a).
 *
 * Plain C: pointers, sizes, status codes.  No exceptions cross it; status
 * 0 = OK, else 1 + tierq::Errc ordinal (tq_types.h).  Every entry point
 * replaces an operator or tier move the reference specifies; each line cites
 * the reference interface it stands in for.  `stream` is a cudaStream_t
 * (NULL = the context's own stream).  Calls that produce data-dependent
 * output sizes (filter, partition, probe, aggregate) read the size back and
 * block until the output batch is allocated; the data itself is written
 * asynchronously on `stream`.
 */
#ifndef TQ_GPU_H
#define TQ_GPU_H

#include "tq_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tq_ctx tq_ctx;
typedef struct tq_join_table tq_join_table;

typedef struct tq_opts {
  int device;                    /* CUDA device ordinal */
  uint32_t ctas_per_sm;          /* persistent grid = ctas_per_sm x SMs (0 = auto) */
  uint64_t device_budget_bytes;  /* Device-tier capacity for the ledger (0 = unlimited);
                                    SPEC.md:259-276 reserve/alloc_within */
  uint64_t pool_reserve_bytes;   /* map this much device memory into the context's pool up front
                                    (kept mapped: later allocations reuse it instead of mapping new
                                    physical memory, ~25 ms per GB, mid-query); 0 = grow on demand */
} tq_opts;

/* ---- context / errors (reference common.hpp:57-74 Error, Errc) --------- */
tq_status tq_ctx_create(const tq_opts* opts, tq_ctx** out);
void tq_ctx_destroy(tq_ctx* ctx);
const char* tq_last_error(void);                 /* thread-local message of the last failure */
const char* tq_errc_name(tq_status status);      /* common.cpp:19-41 errc_name */
tq_status tq_sync(tq_ctx* ctx, void* stream);
uint64_t tq_device_bytes_in_use(tq_ctx* ctx);    /* ledger: allocated Device-tier bytes */
uint64_t tq_device_bytes_reserved(tq_ctx* ctx);  /* device memory the context's pool holds (>= in use) */
uint32_t tq_kernel_launches(tq_ctx* ctx);        /* kernels this context has launched */
void* tq_ctx_stream(tq_ctx* ctx);                /* the context's own cudaStream_t */
/* CUDA-event timing of every pipeline kernel launch (on its launching stream);
 * tq_profile_report writes "kernel count total_ms" lines and resets. */
void tq_profile_enable(tq_ctx* ctx, int on);
uint64_t tq_profile_report(tq_ctx* ctx, char* buf, uint64_t cap);
/* Pipeline kernels are specialised per program with NVRTC (sm_100a) unless
 * disabled here or by TQ_JIT=0; tq_jit_report writes compile/cache stats. */
void tq_ctx_set_jit(tq_ctx* ctx, int on);
uint64_t tq_jit_report(tq_ctx* ctx, char* buf, uint64_t cap);
/* Host-side phase timings accumulated since the last call when the process
 * runs with TQ_HOST_TIMING=1 (one line per phase); returns the length. */
uint64_t tq_host_timing_report(char* buf, uint64_t cap);
/* page-locked, portable host memory (the Host tier of SPEC.md:236-239) */
tq_status tq_pinned_alloc(uint64_t bytes, void** out);
void tq_pinned_free(void* p);

/* ---- batches (reference types.hpp:125-143 ColumnBatch; types.cpp:146-170) --- */
/* Allocate an uninitialised device batch with the schema of `like`
 * (kind/precision/scale; a column gets a bitmap iff like->cols[i].validity != NULL). */
tq_status tq_batch_alloc(tq_ctx* ctx, const tq_batch* like, uint64_t rows, tq_batch* out, void* stream);
/* Host -> device copy into a new device batch (pinned or pageable host memory). */
tq_status tq_batch_upload(tq_ctx* ctx, const tq_batch* host, tq_batch* out, void* stream);
/* Device -> host copy into malloc'ed buffers (free with tq_host_batch_free). Synchronous. */
tq_status tq_batch_download(tq_ctx* ctx, const tq_batch* dev, tq_batch* out, void* stream);
void tq_batch_free(tq_ctx* ctx, tq_batch* b);
void tq_host_batch_free(tq_batch* b);

/* ---- columnar substrate (reference transform.cpp) ---------------------- */
/* take: transform.cpp:90-120.  ids: DEVICE array of n row ids. */
tq_status tq_take(tq_ctx* ctx, const tq_batch* in, const uint64_t* ids, uint64_t n, tq_batch* out,
                  void* stream);
/* concat: transform.cpp:49-88 (bitmap iff any input has one). */
tq_status tq_concat(tq_ctx* ctx, const tq_batch* ins, uint32_t n, tq_batch* out, void* stream);
/* slice: transform.cpp:21-47. */
tq_status tq_slice(tq_ctx* ctx, const tq_batch* in, uint64_t start, uint64_t len, tq_batch* out,
                   void* stream);
/* rebatch (reference transform.cpp:122-154): the concatenation of `ins`
 * re-cut so every output but the last holds >= target_bytes by the
 * reference's per-row estimate (sum of fixed widths + 1 per column, + the Utf8
 * payload), i.e. lands in [target / 2, 2 * target]; one batch when the total
 * (batch_size_bytes) is <= 2 * target.  *outs is malloc'ed (free with free()),
 * each batch with tq_batch_free. */
tq_status tq_rebatch(tq_ctx* ctx, const tq_batch* ins, uint32_t n, uint64_t target_bytes, tq_batch** outs,
                     uint32_t* nout, void* stream);

/* ---- operators ---------------------------------------- */
/* filter_execute: rows where pred is true; schema unchanged. */
tq_status tq_filter(tq_ctx* ctx, const tq_batch* in, tq_expr pred, tq_batch* out, void* stream);
/* project_execute: one output column per expr. */
tq_status tq_project(tq_ctx* ctx, const tq_batch* in, const tq_expr* exprs, uint32_t nexprs, tq_batch* out,
                     void* stream);
/* hash_partition: part(r) = fnv1a64(keys(r)) mod nparts
 * (common.hpp:128-136).  `out` holds the parts contiguously in part order
 * (stable within a part); part p is rows [part_offsets[p], part_offsets[p+1])
 * (host array of nparts+1). */
tq_status tq_hash_partition(tq_ctx* ctx, const tq_batch* in, const uint32_t* keys, uint32_t nkeys,
                            uint32_t nparts, tq_batch* out, uint64_t* part_offsets, void* stream);
/* Asynchronous filter / hash partition (a data-dependent count is
 * returned through a pinned host slot, valid once the stream reaches the end of
 * the call — no host sync inside).  `out` is allocated at the input's row count
 * (every row can pass) and carries that capacity as its row count until the
 * caller, after the stream event, trims it with tq_batch_set_rows(out,
 * slot[nparts]).  slot: caller-owned pinned memory (tq_pinned_alloc) of 2
 * (filter: 0, rows) or nparts + 1 (partition: part starts, then the total)
 * uint64 values — the part_offsets of the synchronous forms.  Batches with Utf8
 * columns: TQ_INVALID_PLAN (their gather needs the count on the host). */
tq_status tq_filter_async(tq_ctx* ctx, const tq_batch* in, tq_expr pred, tq_batch* out, uint64_t* slot,
                          void* stream);
tq_status tq_hash_partition_async(tq_ctx* ctx, const tq_batch* in, const uint32_t* keys, uint32_t nkeys,
                                  uint32_t nparts, tq_batch* out, uint64_t* slot, void* stream);
/* logical trim of a batch to its first `rows` rows (rows <= b->rows; buffers kept) */
void tq_batch_set_rows(tq_batch* b, uint64_t rows);
/* join_execute build side: open-addressing table over the
 * build batch (which must stay alive until the table is destroyed). */
tq_status tq_join_build(tq_ctx* ctx, const tq_batch* build, const uint32_t* keys, uint32_t nkeys,
                        tq_join_table** out, void* stream);
/* tq_join_build with the table's Bloom filter sized from bloom_keys (>= build
 * rows) at 16 bits per key: ranks that pass the same bloom_keys (the most rows
 * any rank received in the fused exchange that delivered the build side,
 * tq_comm_last_exchange_capacity) get equal-size filters, which
 * tq_comm_gather_table_blooms (tq_exchange.h) can all-gather. */
tq_status tq_join_build_sized(tq_ctx* ctx, const tq_batch* build, const uint32_t* keys, uint32_t nkeys,
                              uint64_t bloom_keys, tq_join_table** out, void* stream);
/* Build side of a SEMI-join (the probe takes no build columns, e.g. the
 * customer side of Q3): one-word keys go into an exact membership bitmap over
 * [0, 32 x words); when every key was in range and no key repeated (checked
 * from the atomicOr return values), no hash table is built at all and probes
 * test one bit per row.  Otherwise this falls back to tq_join_build.  Probes
 * of a semi-only table must pass no build columns (TQ_INVALID_PLAN). */
tq_status tq_join_build_semi(tq_ctx* ctx, const tq_batch* build, const uint32_t* keys, uint32_t nkeys,
                             tq_join_table** out, void* stream);
tq_status tq_pipeline_build_semi(tq_ctx* ctx, const tq_batch* in, const tq_expr* pred, const uint32_t* keys,
                                 uint32_t nkeys, tq_join_table** out, void* stream);
/* tq_pipeline_build / _semi with the table's Bloom filter sized for
 * bloom_keys (>= rows; 0 = rows), a row count every worker agrees on, so the
 * workers' filters can be all-gathered as one partitioned LIP filter. */
tq_status tq_pipeline_build_ex(tq_ctx* ctx, const tq_batch* in, const tq_expr* pred, const uint32_t* keys,
                               uint32_t nkeys, uint64_t bloom_keys, int semi, tq_join_table** out, void* stream);
/* Size estimate of pred / exprs over `in` without materialising it: one
 * COUNT pass over the predicate columns -> *out_rows, and the output row
 * width of exprs -> *out_row_bytes (exprs NULL: every input column).  Feeds
 * exchange_phase1 for an exchange side whose filter / projection is fused
 * into the exchange kernel. */
tq_status tq_pipeline_estimate(tq_ctx* ctx, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                               uint32_t nexprs, uint64_t* out_rows, uint64_t* out_row_bytes, void* stream);
/* join_execute probe side: inner equi-join, null keys never match; output =
 * build columns then probe columns. */
tq_status tq_join_probe(tq_ctx* ctx, const tq_join_table* table, const tq_batch* probe, const uint32_t* keys,
                        uint32_t nkeys, tq_batch* out, void* stream);
void tq_join_table_destroy(tq_ctx* ctx, tq_join_table* t);
/* aggregate_execute: keys then one column per aggregate. */
tq_status tq_aggregate(tq_ctx* ctx, const tq_batch* in, const uint32_t* keys, uint32_t nkeys, const tq_agg* aggs,
                       uint32_t naggs, tq_batch* out, void* stream);

/* Streaming aggregation state (agg_update / agg_finalize of SURVEY §8b):
 * every batch is aggregated on the GPU into partial accumulators; finalize
 * merges them and emits the aggregate_execute outputs.  Operator state is
 * serialised by the caller. */
typedef struct tq_agg_state tq_agg_state;
tq_status tq_agg_create(tq_ctx* ctx, const tq_expr* pred, const tq_expr* exprs, uint32_t nexprs, const uint32_t* keys,
                        uint32_t nkeys, const tq_agg* aggs, uint32_t naggs, tq_agg_state** out);
tq_status tq_agg_update(tq_agg_state* state, const tq_batch* in, void* stream);
/* Two-phase use across workers (local pre-aggregation, exchange
 * of the partials on the group keys, merge): take_partial merges the
 * accumulated partials into ONE partial batch (keys, then one raw accumulator
 * per column) and clears them; add_partial appends a partial batch (e.g.
 * received from other workers, possibly 0 rows) to be merged by finalize. */
tq_status tq_agg_take_partial(tq_agg_state* state, tq_batch* out, void* stream);
tq_status tq_agg_add_partial(tq_agg_state* state, const tq_batch* partial, void* stream);
tq_status tq_agg_finalize(tq_agg_state* state, tq_batch* out, void* stream);
void tq_agg_destroy(tq_agg_state* state);

/* ---- fused pipelines: Filter -> Project -> sink in one pass over the batch
 * (the per-batch operator chain of one compute task).
 * pred may be NULL; keys/aggs index the PROJECTED columns. ------------- */
tq_status tq_pipeline_materialize(tq_ctx* ctx, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                                  uint32_t nexprs, tq_batch* out, void* stream);
tq_status tq_pipeline_aggregate(tq_ctx* ctx, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                                uint32_t nexprs, const uint32_t* keys, uint32_t nkeys, const tq_agg* aggs,
                                uint32_t naggs, tq_batch* out, void* stream);
tq_status tq_pipeline_partition(tq_ctx* ctx, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                                uint32_t nexprs, const uint32_t* keys, uint32_t nkeys, uint32_t nparts,
                                tq_batch* out, uint64_t* part_offsets, void* stream);
/* probe output = build columns listed in build_cols (NULL = all build
 * columns; a non-NULL array with nbuild_cols = 0 = none), then projected probe columns */
tq_status tq_pipeline_probe(tq_ctx* ctx, const tq_join_table* table, const tq_batch* in, const tq_expr* pred,
                            const tq_expr* exprs, uint32_t nexprs, const uint32_t* keys, uint32_t nkeys,
                            const uint32_t* build_cols, uint32_t nbuild_cols, tq_batch* out, void* stream);
tq_status tq_pipeline_build(tq_ctx* ctx, const tq_batch* in, const tq_expr* pred, const uint32_t* keys,
                            uint32_t nkeys, tq_join_table** out, void* stream);

/* ---- Lookahead Information Passing: a Bloom filter over
 * build-side keys (~10 bits/key, blocked), applied to the probe side BEFORE
 * it is hash-partitioned and shuffled, so rows that cannot join never cross
 * NVLink.  Results are unchanged (a semi-join reduction).  Union across
 * workers: tq_comm_bloom_union (tq_exchange.h). */
typedef struct tq_bloom tq_bloom;
tq_status tq_bloom_build(tq_ctx* ctx, const tq_batch* in, const uint32_t* keys, uint32_t nkeys, uint64_t expected_keys,
                         tq_bloom** out, void* stream);
void tq_bloom_destroy(tq_bloom* b);
uint64_t tq_bloom_words(const tq_bloom* b);
uint32_t* tq_bloom_data(tq_bloom* b);
/* OR nranks gathered copies (nranks x words, device) into b */
tq_status tq_bloom_or_gathered(tq_bloom* b, const uint32_t* gathered, int nranks, void* stream);
tq_status tq_pipeline_partition_semi(tq_ctx* ctx, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                                     uint32_t nexprs, const uint32_t* keys, uint32_t nkeys, uint32_t nparts,
                                     const tq_bloom* semi, tq_batch* out, uint64_t* part_offsets, void* stream);

/* ---- synthetic TPC-H-style tables generated on the device,
 * bit-identical to the CPU generator (counter-based SplitMix64,
 * common.hpp:139-158).  table: 0 orders, 1 lineitem, 2 customer,
 * 3 supplier, 4 part, 5 partsupp, 6 nation, 7 region. */
tq_status tq_datagen(tq_ctx* ctx, int table, double sf, tq_batch* out, void* stream);
/* The row-group subset of worker `shard` of `nshards` (SPEC.md:661-667
 * assign_files): orders/lineitem split by order ranges (a lineitem shard holds
 * exactly the lines of its orders), other tables by contiguous row ranges.
 * Values equal the corresponding rows of the full table. */
tq_status tq_datagen_shard(tq_ctx* ctx, int table, double sf, uint32_t shard, uint32_t nshards, tq_batch* out,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TQ_GPU_H */
