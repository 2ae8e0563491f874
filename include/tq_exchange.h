/*
 * tq_exchange.h — the worker-to-worker shuffle of libtq_gpu.so: NCCL over
 * NVLink/NVSwitch, one process (one tq_ctx) per GPU.
 *
 * Replaces the reference's Network Executor data path (SPEC.md:475-534:
 * enqueue_send / send_loop / recv_loop over TCP frames) for the two
 * AdaptiveExchange strategies of SPEC.md:580-595:
 *   HashPartition -> tq_hash_partition / tq_pipeline_partition, then
 *                    tq_comm_exchange (grouped ncclSend/ncclRecv all-to-allv);
 *   Broadcast     -> tq_comm_allgather (every rank receives every rank's rows).
 * Received parts are concatenated in source-rank order (reference concat
 * semantics, transform.cpp:49-88: a bitmap if any part has one).
 */
#ifndef TQ_EXCHANGE_H
#define TQ_EXCHANGE_H

#include "tq_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tq_comm tq_comm;

/* 128-byte NCCL unique id, created on rank 0 and shared out of band. */
tq_status tq_comm_unique_id(uint8_t* id128);
tq_status tq_comm_init(tq_ctx* ctx, int rank, int nranks, const uint8_t* id128, tq_comm** out);
void tq_comm_destroy(tq_comm* comm);

/* All-to-allv: rows [part_offsets[p], part_offsets[p+1]) of `partitioned` go to
 * rank p.  `out` = concatenation of the parts received from ranks 0..n-1;
 * recv_offsets (host, n+1) gets their boundaries.  Blocks until the receive
 * sizes are known; the transfer itself is asynchronous on `stream`. */
tq_status tq_comm_exchange(tq_comm* comm, const tq_batch* partitioned, const uint64_t* part_offsets, tq_batch* out,
                           uint64_t* recv_offsets, void* stream);
/* Broadcast join side: every rank receives all ranks' rows (rank order). */
tq_status tq_comm_allgather(tq_comm* comm, const tq_batch* in, tq_batch* out, uint64_t* recv_offsets, void* stream);
/* OR a Bloom filter across all ranks (allgather + OR), for LIP before a shuffle. */
tq_status tq_comm_bloom_union(tq_comm* comm, tq_bloom* bloom, void* stream);
/* Fused hash-partition + shuffle over NVLink peer memory (replaces
 * tq_pipeline_partition[_semi] + tq_comm_exchange, SPEC.md:589-595 + 475-534):
 * evaluate pred / exprs over `in` (as tq_pipeline_partition), drop rows whose
 * keys miss `semi` (LIP; may be NULL), and write every remaining row straight
 * into the receive window of rank fnv1a64(keys) mod n — CUDA IPC mappings of
 * the peers' windows, no partitioned staging batch, no NCCL payload copy.
 * `out` = the rows all ranks sent to this one, in unspecified order.
 * Collective: every rank calls it, in the same order as its other collectives. */
tq_status tq_pipeline_partition_exchange(tq_comm* comm, const tq_batch* in, const tq_expr* pred,
                                         const tq_expr* exprs, uint32_t nexprs, const uint32_t* keys, uint32_t nkeys,
                                         const tq_bloom* semi, tq_batch* out, void* stream);
/* Fused filter / project + broadcast over NVLink peer memory (replaces
 * tq_pipeline_materialize + tq_comm_allgather for a broadcast join side,
 * SPEC.md:580-588 exchange_decide -> Broadcast): every row that passes `pred`
 * is written into every rank's receive window.  `out` = all ranks' rows, in
 * unspecified order.  Collective. */
tq_status tq_pipeline_broadcast(tq_comm* comm, const tq_batch* in, const tq_expr* pred, const tq_expr* exprs,
                                uint32_t nexprs, tq_batch* out, void* stream);
/* Partitioned LIP filter (PAPER.md:394 Lookahead Information Passing, after
 * the build side's shuffle): all-gather every rank's join-table Bloom filter
 * (equal sizes: every rank built its table with tq_join_build_sized and the
 * same agreed bloom_keys; checked against the table's own count before the
 * collective, TQ_INVALID_PLAN otherwise) into one filter whose part d is rank
 * d's.  Passed as `semi` to tq_pipeline_partition_exchange, a row is checked
 * only against the part of the rank it is sent to.  Collective. */
tq_status tq_comm_gather_table_blooms(tq_comm* comm, const tq_join_table* table, tq_bloom** out, void* stream);
/* The most rows any rank received in the last tq_pipeline_partition_exchange
 * (>= 1): identical on every rank, so a Bloom filter sized from it has the same
 * word count everywhere (tq_join_build_sized -> tq_comm_gather_table_blooms). */
uint64_t tq_comm_last_exchange_capacity(tq_comm* comm);
/* Bytes this communicator has sent to other ranks (NVLink traffic). */
uint64_t tq_comm_bytes_sent(tq_comm* comm);
int tq_comm_size(tq_comm* comm);
int tq_comm_rank(tq_comm* comm);
/* All-gather `count` u64 per rank through the communicator (host buffers:
 * in[count] -> out[nranks * count], rank order).  Collective; blocks. */
tq_status tq_comm_allgather_host_u64(tq_comm* comm, const uint64_t* in, uint64_t* out, uint64_t count, void* stream);

/* ---- AdaptiveExchange control: pure functions, the same
 * code on every worker (the engine's exchange pairs and the Python mirror,
 * paper_2508_05029_b200/exchange.py). */
#define TQ_SAMPLE_FRACTION 0.05
#define TQ_BROADCAST_THRESHOLD (16ull << 20)    /* 16 MiB per worker */
/* exchange_phase1: once scan progress >= sample_fraction (or the scan is
 * complete: progress >= 1) returns 1 with *estimate = bytes_so_far /
 * progress (0 for an empty finished input); 0 = not yet. */
int tq_exchange_phase1(uint64_t bytes_so_far, double progress, double sample_fraction, uint64_t* estimate);
enum { TQ_XCHG_HASH_PARTITION = 0, TQ_XCHG_BROADCAST = 1 };
/* exchange_decide: est0 / est1 = every worker's estimate of side 0 / 1 (n
 * each).  Broadcast of the smaller side (*broadcast_side, ties -> side 0)
 * if min(totals) <= threshold * n, else HashPartition both.  Deterministic. */
int tq_exchange_decide(const uint64_t* est0, const uint64_t* est1, int n, uint64_t threshold, int* broadcast_side,
                       uint64_t* total0, uint64_t* total1);

#ifdef __cplusplus
}
#endif
#endif /* TQ_EXCHANGE_H */
