/*
 * tq_oracle.h — CPU ORACLE (test infrastructure, NOT product code).
 *
 * A plain C++ restatement of the reference's hot-path semantics:
 *   - columnar substrate: take / concat / slice (reference
 *     proj/src/columnar/transform.cpp:21-120), fnv1a64 and SplitMix64
 *     (proj/include/tierq/common.hpp:128-158);
 *   - the operators that exist only as SPEC text: filter_execute
 *     (SPEC.md:560-566), project_execute (:567-570), hash_partition
 *     (:589-595), join_execute (:596-603), aggregate_execute (:604-611) with
 *     the Expr/null rules of SPEC.md:541-544 and the decisions recorded in
 *     DESIGN.md §3;
 *   - the synthetic TPC-H-style generator;
 *   - the five query DAGs of SURVEY Appendix D.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path
 * (libtq_gpu.so) never links or calls it.
 *
 * Parity pinning: the substrate is pinned against the reference itself
 * (oracle/_ref, built from /root/reference sources) and the SPEC inline
 * examples; the operators have no reference implementation, so
 * their parity is pinned only by SPEC examples + independent micro-oracles
 * (naive nested-loop join / row-loop evaluators in tests/).
 */
#ifndef TQ_ORACLE_H
#define TQ_ORACLE_H

#include "../include/tq_types.h"

#ifdef __cplusplus
extern "C" {
#endif

/* All output batches are malloc'ed host batches; free with tqo_batch_free. */
void tqo_batch_free(tq_batch* b);
const char* tqo_last_error(void);

uint64_t tqo_fnv1a64(const uint8_t* bytes, uint64_t n, uint64_t seed);
uint64_t tqo_splitmix_nth(uint64_t seed, uint64_t k); /* k-th next(), k >= 1 */

/* columnar substrate (transform.cpp semantics) */
tq_status tqo_take(const tq_batch* in, const uint64_t* ids, uint64_t n, tq_batch* out);
tq_status tqo_concat(const tq_batch* ins, uint32_t n, tq_batch* out);
tq_status tqo_slice(const tq_batch* in, uint64_t start, uint64_t len, tq_batch* out);

/* operators; naive=1 selects the SPEC oracle algorithms (nested loop join,
 * linear-scan grouping) used to cross-check the hash versions. */
tq_status tqo_filter(const tq_batch* in, tq_expr pred, tq_batch* out);
tq_status tqo_project(const tq_batch* in, const tq_expr* exprs, uint32_t n, tq_batch* out);
tq_status tqo_hash_partition(const tq_batch* in, const uint32_t* keys, uint32_t nkeys,
                             uint32_t nparts, tq_batch* outs);
tq_status tqo_partition_ids(const tq_batch* in, const uint32_t* keys, uint32_t nkeys,
                            uint32_t nparts, uint32_t* pid_out);
tq_status tqo_join(const tq_batch* build, const tq_batch* probe, const uint32_t* bkeys,
                   const uint32_t* pkeys, uint32_t nkeys, int naive, tq_batch* out);
tq_status tqo_aggregate(const tq_batch* in, const uint32_t* keys, uint32_t nkeys,
                        const tq_agg* aggs, uint32_t naggs, int naive, tq_batch* out);

/* synthetic TPC-H-style tables */
enum {
  TQ_T_ORDERS = 0, TQ_T_LINEITEM = 1, TQ_T_CUSTOMER = 2, TQ_T_SUPPLIER = 3,
  TQ_T_PART = 4, TQ_T_PARTSUPP = 5, TQ_T_NATION = 6, TQ_T_REGION = 7
};
uint64_t tqo_table_rows(int table, double sf);
tq_status tqo_datagen(int table, double sf, uint32_t nthreads, tq_batch* out);
// A worker's row-group subset, equal to the GPU's tq_datagen_shard (datagen.cu).
tq_status tqo_datagen_shard(int table, double sf, uint32_t shard, uint32_t nshards, uint32_t nthreads, tq_batch* out);

/* whole queries.  tables[] is indexed by TQ_T_*; only the
 * tables the query reads must be set.  nthreads=1 → single-threaded oracle;
 * nthreads>1 → the multi-threaded hash-based CPU baseline (same results). */
enum { TQ_Q1 = 1, TQ_Q3 = 3, TQ_Q5 = 5, TQ_Q6 = 6, TQ_Q9 = 9 };
tq_status tqo_query(int q, const tq_batch* tables, uint32_t nthreads, tq_batch* out);

#ifdef __cplusplus
}
#endif
#endif
