/*
 * tq_engine.h — the worker runtime of libtq_gpu.so: the reference's
 * Operator / BatchHolder / executor model (SPEC.md
 * memtier 231-335, sched 337-419, preload 421-473, engine 634-695) driving
 * the GPU operators of tq_gpu.h on one GPU.
 *
 *   BatchHolder      queue of BatchHandles; push never fails — when the
 *                    Device tier passes its high watermark, unpinned handles
 *                    are spilled to the pinned Host pool
 *   Memory Executor  spill (Device->Host) / load_to_device (Host->Device) of
 *                    chunked batches, one cudaMemcpyAsync per segment on its
 *                    own copy stream; victim selection protects the inputs of
 *                    the compute queue's top-K tasks
 *   Pre-loading      promotes Host-resident inputs of queued tasks to Device
 *                    on a side stream ahead of execution
 *   Compute Executor N threads, one CUDA stream each; priority queue
 *                    (starvation boost, input tier, plan depth, seq); run_task
 *                    = reserve -> load -> execute -> deposit -> stats ->
 *                    release; ReservationExceeded -> on_oom: double the
 *                    estimate and retry, else split, else
 *                    OutOfMemoryUnsplittable
 * Query DAGs for the benchmark shapes are built in C++.
 */
#ifndef TQ_ENGINE_H
#define TQ_ENGINE_H

#include "tq_exchange.h"
#include "tq_memexec.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tq_engine_opts {
  uint32_t compute_threads;     /* SPEC.md:407 default 4 */
  uint32_t preload;             /* 1 = run the Pre-loading executor */
  uint64_t batch_rows;          /* scan task size in rows */
  uint64_t device_budget;       /* Device tier capacity in bytes (0 = context budget / unlimited) */
  uint64_t pool_buffer_size;    /* Host pool buffer size (1 MiB) */
  uint64_t pool_capacity;       /* Host pool buffers */
  double high_watermark;        /* 0.90 */
  double low_watermark;         /* 0.70 */
  uint32_t protect_top_k;       /* 8 */
  uint32_t tables_on_host;      /* 1 = scan inputs start in the Host tier (config 5) */
  uint32_t task_batches;        /* input batches per Filter/Project/Probe task (default 1); a task with
                                   more than one is splittable by on_oom */
  /* test-only fault injection: the first inject_oom_count tasks of the operator
   * named inject_oom_op fail with ReservationExceeded before executing.
   * mode 1: the estimate then doubles as usual; mode 2: the estimate is first
   * raised to the Device capacity (the doubled one cannot fit: split / abort). */
  uint32_t inject_oom_mode;
  uint32_t inject_oom_count;
  char inject_oom_op[32];
  /* distributed plans (comm with > 1 rank): */
  uint32_t force_exchange;       /* 0 = exchange_decide; 1 = force Broadcast; 2 = force HashPartition */
  uint32_t exchange_impl;        /* 0 = fused partition / broadcast over NVLink peer memory; 1 = NCCL */
  uint64_t broadcast_threshold;  /* per worker, 0 = TQ_BROADCAST_THRESHOLD (16 MiB) */
} tq_engine_opts;

/* Input tables: tables[t] (t = 0 orders, 1 lineitem, 2 customer, 3 supplier,
 * 4 part, 5 partsupp, 6 nation, 7 region) are DEVICE batches; unused entries
 * may be zero.  With tables_on_host the engine first moves each scan batch to
 * the pinned Host pool so every scan task goes through load_to_device.
 * comm may be NULL (single worker); with a communicator of N > 1 ranks the
 * query runs as one worker of its distributed plan: an AdaptiveExchange pair
 * per join (estimates after 5% of the scan, all-gathered,
 * tq_exchange_decide -> Broadcast the small side or HashPartition both, over
 * the fused NVLink exchange), aggregates co-partitioned or pre-aggregated and
 * exchanged on the group keys; every worker returns its share of the result
 * (the union over workers is the query result; disjoint groups).  The result is a HOST
 * batch (free with tq_host_batch_free); metrics_json (may be NULL) receives
 * a JSON object of executor metrics. */
tq_status tq_engine_run_query(tq_ctx* ctx, tq_comm* comm, int query, const tq_batch* tables,
                              const tq_engine_opts* opts, tq_batch* result, char* metrics_json, uint64_t cap);

/* on_oom: the estimate doubles (*new_estimate); a task
 * whose doubled estimate fits the Device capacity (0 = unbounded) is retried,
 * else a splittable task (> 1 input batch) is split into two halves, else the
 * query aborts with OutOfMemoryUnsplittable. */
enum { TQ_OOM_RETRY = 0, TQ_OOM_SPLIT = 1, TQ_OOM_ABORT = 2 };
int tq_on_oom_decide(uint64_t estimate, uint64_t capacity, int splittable, uint64_t* new_estimate);

/* The same query over TCF files (include/tq_storage.h): paths[t] is table t's
 * file or NULL.  Every row group is a STORAGE-tier handle;
 * the scan tasks — and the Pre-loading executor ahead of them — read its
 * column ranges straight into the pinned Host pool (byte-range preload,
 * SPEC.md:444-452) and move them to the device (tq_load). */
tq_status tq_engine_run_query_tcf(tq_ctx* ctx, tq_comm* comm, int query, const char* const* paths,
                                  const tq_engine_opts* opts, tq_batch* result, char* metrics_json, uint64_t cap);

/* max(ema_peak, ema_ratio*input) * safety, or multiplier *
 * input without history; never below input_bytes. */
uint64_t tq_estimate_reservation(uint64_t samples, double ema_peak, double ema_ratio, uint64_t input_bytes,
                                 double default_multiplier, double safety);

#ifdef __cplusplus
}
#endif
#endif /* TQ_ENGINE_H */
