/*
 * tq_types.h — plain-data layout shared by the C-ABI (tq_gpu.h) and the CPU
 * oracle (oracle/tq_oracle.h).  No functions, no torch, no C++ types.
 *
 * A batch is section-for-section the reference's ColumnBatch
 * (reference proj/include/tierq/columnar/types.hpp:104-143, batch_sections
 * in proj/src/columnar/types.cpp:146-164): per column one values section
 * (fixed width LE, or Utf8 bytes), an optional LSB-first validity bitmap of
 * ceil(rows/8) bytes (NULL = all valid), and for Utf8 an int32 offsets
 * section of rows+1 entries.
 */
#ifndef TQ_TYPES_H
#define TQ_TYPES_H

#ifndef __CUDACC_RTC__
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: 0 = OK, otherwise 1 + the ordinal of tierq::Errc
 * (reference proj/include/tierq/common.hpp:34-53), so the host wrappers can
 * re-raise the reference's own error vocabulary. */
typedef int tq_status;
enum {
  TQ_OK = 0,
  TQ_POOL_EXHAUSTED = 1,
  TQ_CORRUPT_LAYOUT = 2,
  TQ_MALFORMED_BATCH = 3,
  TQ_SCHEMA_MISMATCH = 4,
  TQ_NOT_TCF = 5,
  TQ_CORRUPT_FOOTER = 6,
  TQ_UNKNOWN_COLUMN = 7,
  TQ_CORRUPT_ROW_GROUP = 8,
  TQ_IO_ERROR = 9,
  TQ_RESERVATION_IMPOSSIBLE = 10,
  TQ_RESERVATION_EXCEEDED = 11,
  TQ_NO_ELIGIBLE_VICTIMS = 12,
  TQ_OUT_OF_MEMORY_UNSPLITTABLE = 13,
  TQ_CORRUPT_FRAME = 14,
  TQ_PEER_DISCONNECTED = 15,
  TQ_INVALID_PLAN = 16,
  TQ_WORKER_FAILURE = 17,
  TQ_INTERNAL = 18
};

/* TypeKind, reference types.hpp:26-32 (same ordinals). */
enum {
  TQ_INT64 = 0,
  TQ_FLOAT64 = 1,
  TQ_BOOL = 2,
  TQ_UTF8 = 3,
  TQ_DECIMAL = 4
};

typedef struct tq_column {
  uint8_t kind;       /* TQ_INT64 ... TQ_DECIMAL */
  uint8_t precision;  /* Decimal only (metadata) */
  uint8_t scale;      /* Decimal only */
  uint8_t _pad[5];
  void* values;       /* rows*width bytes (Utf8: offsets[rows] bytes) */
  uint64_t values_bytes;
  uint8_t* validity;  /* NULL = all valid; else ceil(rows/8) bytes LSB-first */
  int32_t* offsets;   /* Utf8 only: rows+1 entries */
} tq_column;

/* Where a batch's buffers live. */
enum { TQ_MEM_HOST = 0, TQ_MEM_DEVICE = 1 };

typedef struct tq_batch {
  uint64_t rows;
  uint32_t ncols;
  uint32_t mem;       /* TQ_MEM_HOST / TQ_MEM_DEVICE */
  tq_column* cols;    /* host array of ncols descriptors */
  void* owner;        /* allocator bookkeeping of the producing library; NULL if borrowed */
} tq_batch;

/* ---- Expr, serialized in prefix order ----------------- */
enum {
  TQ_EX_COL = 0,   /* ColumnRef(column) */
  TQ_EX_LIT = 1,   /* Literal(kind, scale, is_null, lo/hi) */
  TQ_EX_CMP = 2,   /* Compare(op) a b */
  TQ_EX_ARITH = 3, /* Arith(op) a b */
  TQ_EX_AND = 4,
  TQ_EX_OR = 5,
  TQ_EX_NOT = 6
};
enum { TQ_LT = 0, TQ_LE = 1, TQ_EQ = 2, TQ_NE = 3, TQ_GE = 4, TQ_GT = 5 };
enum { TQ_ADD = 0, TQ_SUB = 1, TQ_MUL = 2 };

typedef struct tq_expr_node {
  uint8_t tag;        /* TQ_EX_* */
  uint8_t op;         /* compare / arith op */
  uint8_t kind;       /* literal type kind */
  uint8_t scale;      /* literal decimal scale */
  uint8_t is_null;    /* literal is NULL */
  uint8_t _pad[3];
  uint32_t column;    /* ColumnRef index */
  uint32_t _pad2;
  uint64_t lo;        /* literal payload: int64 / low word of int128 / f64 bits / bool */
  uint64_t hi;        /* high word of a decimal int128 literal */
} tq_expr_node;       /* 32 bytes */

typedef struct tq_expr {
  const tq_expr_node* nodes;
  uint32_t len;
  uint32_t _pad;
} tq_expr;

/* ---- aggregates --------------------------------------- */
enum {
  TQ_AGG_SUM = 0,
  TQ_AGG_COUNT = 1,      /* non-null count of column */
  TQ_AGG_COUNT_STAR = 2, /* row count; column ignored */
  TQ_AGG_MIN = 3,
  TQ_AGG_MAX = 4,
  TQ_AGG_AVG = 5         /* Float64 = Sum / Count, nulls skipped */
};

typedef struct tq_agg {
  uint32_t fn;
  uint32_t column;
} tq_agg;

#ifdef __cplusplus
}
#endif
#endif /* TQ_TYPES_H */
