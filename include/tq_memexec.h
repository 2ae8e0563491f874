/*
 * tq_memexec.h — the Host memory tier and Device<->Host batch movement of
 * libtq_gpu.so (the Memory Executor's data path).
 *
 *   tq_pool      FixedBufferPool (reference pool.hpp:29-56, pool.cpp:21-68):
 *                one page-locked portable arena (cudaHostAlloc) of `capacity`
 *                buffers of `buffer_size` bytes; all-or-nothing acquire that
 *                hands out low ids first; release with double-free check.
 *   tq_chunked   ChunkedBatch (reference chunked.hpp:22-53): per column the
 *                values / validity / offsets sections laid end to end across
 *                pool buffers (a section may span buffers; only the last
 *                buffer has an unused tail) — byte-identical layout to
 *                encode_chunked (chunked.cpp:19-56).
 *   tq_spill     Device -> Host: one cudaMemcpyAsync per segment (section x
 *                buffer) from the device batch into pool buffers.
 *   tq_load      Host -> Device (load_to_device): one
 *                cudaMemcpyAsync per segment into a new device batch; the
 *                section lengths are validated first (CorruptLayout, as
 *                decode_chunked, chunked.cpp:76-118).
 * Copies run on the caller's stream (the Memory / Pre-loading executors use
 * dedicated side streams so tier moves overlap compute).
 */
#ifndef TQ_MEMEXEC_H
#define TQ_MEMEXEC_H

#include "tq_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tq_pool tq_pool;
typedef struct tq_chunked tq_chunked;

tq_status tq_pool_create(uint64_t buffer_size, uint64_t capacity, tq_pool** out);
void tq_pool_destroy(tq_pool* pool);
uint64_t tq_pool_free_count(tq_pool* pool);
uint64_t tq_pool_buffer_size(tq_pool* pool);
/* all-or-nothing: TQ_POOL_EXHAUSTED leaves the pool unchanged */
tq_status tq_pool_acquire(tq_pool* pool, uint64_t n, uint32_t* ids);
tq_status tq_pool_release(tq_pool* pool, const uint32_t* ids, uint64_t n);
uint8_t* tq_pool_buffer(tq_pool* pool, uint32_t id);

/* host batch <-> pool (encode_chunked / decode_chunked on the CPU side) */
tq_status tq_chunked_encode(tq_pool* pool, const tq_batch* host, tq_chunked** out);
tq_status tq_chunked_decode(const tq_chunked* cb, tq_batch* out_host);
/* device batch <-> pool */
tq_status tq_spill(tq_ctx* ctx, tq_pool* pool, const tq_batch* dev, tq_chunked** out, void* stream);
tq_status tq_load(tq_ctx* ctx, const tq_chunked* cb, tq_batch* out_dev, void* stream);
/* layout introspection: buffers used, unused tail, total section bytes; segs
 * gets (buffer_id, offset, length) triples in layout order; returns #segments */
uint32_t tq_chunked_layout(const tq_chunked* cb, uint64_t* nbuf, uint64_t* tail, uint64_t* total, uint32_t* segs,
                           uint32_t seg_cap);
uint64_t tq_chunked_rows(const tq_chunked* cb);
/* releases the buffers back to the pool (release_chunked, chunked.cpp:120-124) */
void tq_chunked_release(tq_chunked* cb);

#ifdef __cplusplus
}
#endif
#endif /* TQ_MEMEXEC_H */
