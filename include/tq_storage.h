/*
 * tq_storage.h — the scan side of the hot path: the TCF
 * columnar file and its byte-range preload into the pinned
 * Host pool, from which the row group goes to the GPU with one
 * cudaMemcpyAsync per segment (tq_load, the Memory executor's load_to_device).
 *
 *   layout (little-endian, SPEC.md External Interfaces):
 *     "TCF1" | row groups | footer | footer_len u32 | "TCF1"
 *   a row group stores each column's sections back to back — values, validity
 *   (if the column has a bitmap), Utf8 offsets — in column order (the batch
 *   section order of types.cpp:146-164, so a fetched column range IS its
 *   chunked-batch sections).  footer: u32 ncols, per column {u8 kind, u8
 *   precision, u8 scale, u16 name_len, name}, u32 nrow_groups, per row group
 *   {u64 rows, per column {u64 offset, u64 values_len, u64 validity_len,
 *   u64 offsets_len}}.
 *
 *   write_tcf        tq_tcf_write (row groups of ~row_group_bytes, rows a
 *                    multiple of 8 except the last so bitmaps split on bytes)
 *   read_footer      tq_tcf_open: exactly two reads (trailing 8 bytes, footer)
 *   plan_ranges      tq_tcf_plan_ranges: one range per (row group, column)
 *   coalesce_ranges  tq_coalesce_ranges (max_gap, max_merged)
 *   fetch_ranges +   tq_tcf_fetch: the needed columns' byte ranges of a row
 *   decode           group read (up to max_connections concurrent preads)
 *                    straight into pool buffers as a chunked batch — the Host
 *                    tier object tq_load moves to the device.  Ranges that
 *                    touch are read as one (gaps are never read into the pool:
 *                    a chunked batch holds only the needed sections).
 */
#ifndef TQ_STORAGE_H
#define TQ_STORAGE_H

#include "tq_memexec.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tq_tcf tq_tcf;
typedef struct tq_range {
  uint64_t offset, length;
} tq_range;

/* table: a HOST batch; names[ncols] may be NULL (c0, c1, ...). */
tq_status tq_tcf_write(const char* path, const tq_batch* table, const char* const* names, uint64_t row_group_bytes);
tq_status tq_tcf_open(const char* path, tq_tcf** out);
void tq_tcf_close(tq_tcf* f);
uint32_t tq_tcf_ncols(const tq_tcf* f);
uint32_t tq_tcf_row_groups(const tq_tcf* f);
uint64_t tq_tcf_rows(const tq_tcf* f, uint32_t row_group);
/* kind / precision / scale of column c into *col (pointers untouched); its name, or NULL */
const char* tq_tcf_column(const tq_tcf* f, uint32_t c, tq_column* col);
/* datasource reads issued so far (read_footer issues exactly 2) */
uint64_t tq_tcf_reads(const tq_tcf* f);
/* one range per (row group, needed column), sorted by offset; *n = count (<= cap written) */
tq_status tq_tcf_plan_ranges(const tq_tcf* f, const uint32_t* cols, uint32_t ncols, const uint32_t* row_groups,
                             uint32_t nrg, tq_range* out, uint64_t cap, uint64_t* n);
/* merge sorted disjoint ranges whose gap <= max_gap while the merged length <= max_merged; returns the count */
uint64_t tq_coalesce_ranges(const tq_range* in, uint64_t n, uint64_t max_gap, uint64_t max_merged, tq_range* out);
/* fetch the needed columns of a row group into `pool` as a chunked batch (columns in `cols` order) */
tq_status tq_tcf_fetch(tq_tcf* f, tq_pool* pool, uint32_t row_group, const uint32_t* cols, uint32_t ncols,
                       uint32_t max_connections, tq_chunked** out);

#ifdef __cplusplus
}
#endif
#endif /* TQ_STORAGE_H */
