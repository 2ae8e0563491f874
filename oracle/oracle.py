"""ctypes loader for the CPU ORACLE (test infrastructure, NOT product code).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module.  It wraps:
  - liboracle.so      — the restatement (oracle/tq_oracle.cpp)
  - _ref/libtierq_ref.so — the reference's own columnar code (built from
    /root/reference sources by oracle/build_ref.sh; optional)
"""
from __future__ import annotations

import ctypes as C
import os
import sys
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2508_05029_b200.columnar import HostBatch, TqAggC, TqBatchC, TqError, TqExprC  # noqa: E402
from paper_2508_05029_b200.expr import Expr  # noqa: E402

T_ORDERS, T_LINEITEM, T_CUSTOMER, T_SUPPLIER, T_PART, T_PARTSUPP, T_NATION, T_REGION = range(8)
TABLE_NAMES = ["orders", "lineitem", "customer", "supplier", "part", "partsupp", "nation", "region"]
QUERY_TABLES = {
    1: [T_LINEITEM], 6: [T_LINEITEM], 3: [T_CUSTOMER, T_ORDERS, T_LINEITEM],
    5: [T_REGION, T_NATION, T_CUSTOMER, T_ORDERS, T_LINEITEM, T_SUPPLIER],
    9: [T_PART, T_PARTSUPP, T_LINEITEM, T_SUPPLIER, T_ORDERS],
}

_lib = None
_ref = None


def build() -> None:
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        P = C.POINTER
        L.tqo_last_error.restype = C.c_char_p
        L.tqo_fnv1a64.restype = C.c_uint64
        L.tqo_fnv1a64.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64]
        L.tqo_splitmix_nth.restype = C.c_uint64
        L.tqo_splitmix_nth.argtypes = [C.c_uint64, C.c_uint64]
        L.tqo_take.argtypes = [P(TqBatchC), P(C.c_uint64), C.c_uint64, P(TqBatchC)]
        L.tqo_concat.argtypes = [P(TqBatchC), C.c_uint32, P(TqBatchC)]
        L.tqo_slice.argtypes = [P(TqBatchC), C.c_uint64, C.c_uint64, P(TqBatchC)]
        L.tqo_filter.argtypes = [P(TqBatchC), TqExprC, P(TqBatchC)]
        L.tqo_project.argtypes = [P(TqBatchC), P(TqExprC), C.c_uint32, P(TqBatchC)]
        L.tqo_hash_partition.argtypes = [P(TqBatchC), P(C.c_uint32), C.c_uint32, C.c_uint32, P(TqBatchC)]
        L.tqo_partition_ids.argtypes = [P(TqBatchC), P(C.c_uint32), C.c_uint32, C.c_uint32, P(C.c_uint32)]
        L.tqo_join.argtypes = [P(TqBatchC), P(TqBatchC), P(C.c_uint32), P(C.c_uint32), C.c_uint32, C.c_int,
                               P(TqBatchC)]
        L.tqo_aggregate.argtypes = [P(TqBatchC), P(C.c_uint32), C.c_uint32, P(TqAggC), C.c_uint32, C.c_int,
                                    P(TqBatchC)]
        L.tqo_table_rows.restype = C.c_uint64
        L.tqo_table_rows.argtypes = [C.c_int, C.c_double]
        L.tqo_datagen.argtypes = [C.c_int, C.c_double, C.c_uint32, P(TqBatchC)]
        L.tqo_datagen_shard.argtypes = [C.c_int, C.c_double, C.c_uint32, C.c_uint32, C.c_uint32, P(TqBatchC)]
        L.tqo_query.argtypes = [C.c_int, P(TqBatchC), C.c_uint32, P(TqBatchC)]
        L.tqo_batch_free.argtypes = [P(TqBatchC)]
        _lib = L
    return _lib


def ref():
    """The reference's own columnar library, or None if it was never built."""
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libtierq_ref.so")
        if not os.path.exists(path):
            return None
        L = C.CDLL(path)
        P = C.POINTER
        L.tqr_last_error.restype = C.c_char_p
        L.tqr_fnv1a64.restype = C.c_uint64
        L.tqr_fnv1a64.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64]
        L.tqr_splitmix.argtypes = [C.c_uint64, C.c_uint64, P(C.c_uint64)]
        L.tqr_splitmix_below.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, P(C.c_uint64)]
        L.tqr_validate.argtypes = [P(TqBatchC)]
        L.tqr_take.argtypes = [P(TqBatchC), P(C.c_uint64), C.c_uint64, P(TqBatchC)]
        L.tqr_concat.argtypes = [P(TqBatchC), C.c_uint32, P(TqBatchC)]
        L.tqr_slice.argtypes = [P(TqBatchC), C.c_uint64, C.c_uint64, P(TqBatchC)]
        L.tqr_batch_size_bytes.restype = C.c_uint64
        L.tqr_batch_size_bytes.argtypes = [P(TqBatchC)]
        L.tqr_rebatch_rows.argtypes = [P(TqBatchC), C.c_uint64, P(C.c_uint64), C.c_uint32, P(C.c_uint32)]
        L.tqr_chunked_layout.argtypes = [P(TqBatchC), C.c_uint64, C.c_uint64, P(C.c_uint64), P(C.c_uint64),
                                         P(C.c_uint32), C.c_uint32, P(C.c_uint32), P(C.c_int)]
        L.tqr_batch_free.argtypes = [P(TqBatchC)]
        L.tqr_resident_make.restype = C.c_void_p
        L.tqr_resident_make.argtypes = [P(TqBatchC)]
        L.tqr_resident_free.argtypes = [C.c_void_p]
        L.tqr_q1_fused.restype = C.c_double
        L.tqr_q1_fused.argtypes = [C.c_void_p, C.c_uint32, P(C.c_uint64), C.c_uint32]
        L.tqr_read_bw.restype = C.c_double
        L.tqr_read_bw.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        _ref = L
    return _ref


def _check(st: int, L, which="tqo"):
    if st != 0:
        msg = (L.tqo_last_error() if which == "tqo" else L.tqr_last_error()) or b""
        raise TqError(st, msg.decode())


def _out(L, st, out: TqBatchC, which="tqo") -> HostBatch:
    _check(st, L, which)
    try:
        return HostBatch.from_c(out)
    finally:
        (L.tqo_batch_free if which == "tqo" else L.tqr_batch_free)(C.byref(out))


def _u32(xs: Sequence[int]):
    return (C.c_uint32 * max(1, len(xs)))(*xs)


# ---------------------------------------------------------------- oracle ops
def fnv1a64(data: bytes, seed: int = 0xCBF29CE484222325) -> int:
    return lib().tqo_fnv1a64(data, len(data), seed)


def splitmix_nth(seed: int, k: int) -> int:
    return lib().tqo_splitmix_nth(seed, k)


def take(b: HostBatch, ids: Sequence[int]) -> HostBatch:
    L, out = lib(), TqBatchC()
    arr = (C.c_uint64 * max(1, len(ids)))(*ids)
    bc = b.to_c()
    return _out(L, L.tqo_take(C.byref(bc), arr, len(ids), C.byref(out)), out)


def concat(bs: Sequence[HostBatch]) -> HostBatch:
    L, out = lib(), TqBatchC()
    cs = [b.to_c() for b in bs]
    arr = (TqBatchC * len(cs))(*cs)
    return _out(L, L.tqo_concat(arr, len(cs), C.byref(out)), out)


def slice_(b: HostBatch, start: int, n: int) -> HostBatch:
    L, out = lib(), TqBatchC()
    bc = b.to_c()
    return _out(L, L.tqo_slice(C.byref(bc), start, n, C.byref(out)), out)


def filter_execute(b: HostBatch, pred: Expr) -> HostBatch:
    L, out = lib(), TqBatchC()
    s = pred.serialize()
    bc = b.to_c()
    return _out(L, L.tqo_filter(C.byref(bc), s.c(), C.byref(out)), out)


def project_execute(b: HostBatch, exprs: Sequence[Expr]) -> HostBatch:
    L, out = lib(), TqBatchC()
    ss = [e.serialize() for e in exprs]
    arr = (TqExprC * max(1, len(ss)))(*[s.c() for s in ss])
    bc = b.to_c()
    return _out(L, L.tqo_project(C.byref(bc), arr, len(ss), C.byref(out)), out)


def partition_ids(b: HostBatch, keys: Sequence[int], nparts: int):
    import numpy as np
    L = lib()
    pid = np.zeros(max(1, b.rows), dtype=np.uint32)
    bc = b.to_c()
    _check(L.tqo_partition_ids(C.byref(bc), _u32(keys), len(keys), nparts,
                               pid.ctypes.data_as(C.POINTER(C.c_uint32))), L)
    return pid[:b.rows]


def hash_partition(b: HostBatch, keys: Sequence[int], nparts: int) -> List[HostBatch]:
    L = lib()
    outs = (TqBatchC * nparts)()
    bc = b.to_c()
    _check(L.tqo_hash_partition(C.byref(bc), _u32(keys), len(keys), nparts, outs), L)
    res = []
    for i in range(nparts):
        res.append(HostBatch.from_c(outs[i]))
        L.tqo_batch_free(C.byref(outs[i]))
    return res


def join_execute(build: HostBatch, probe: HostBatch, bkeys, pkeys, naive=False) -> HostBatch:
    L, out = lib(), TqBatchC()
    bb, pb = build.to_c(), probe.to_c()
    return _out(L, L.tqo_join(C.byref(bb), C.byref(pb), _u32(bkeys), _u32(pkeys), len(bkeys), int(naive),
                              C.byref(out)), out)


def aggregate_execute(b: HostBatch, keys, aggs, naive=False) -> HostBatch:
    """aggs: list of (fn, column)."""
    L, out = lib(), TqBatchC()
    arr = (TqAggC * max(1, len(aggs)))(*[TqAggC(f, c) for f, c in aggs])
    bc = b.to_c()
    return _out(L, L.tqo_aggregate(C.byref(bc), _u32(keys), len(keys), arr, len(aggs), int(naive),
                                   C.byref(out)), out)


def table_rows(t: int, sf: float) -> int:
    return lib().tqo_table_rows(t, sf)


def datagen(t: int, sf: float, nthreads: int = 8, shard: int = 0, nshards: int = 1) -> HostBatch:
    L, out = lib(), TqBatchC()
    if nshards > 1:
        return _out(L, L.tqo_datagen_shard(t, sf, shard, nshards, nthreads, C.byref(out)), out)
    return _out(L, L.tqo_datagen(t, sf, nthreads, C.byref(out)), out)


def query(q: int, tables: dict, nthreads: int = 1) -> HostBatch:
    """tables: {T_*: HostBatch}."""
    L, out = lib(), TqBatchC()
    arr = (TqBatchC * 8)()
    keep = []
    for t, hb in tables.items():
        c = hb.to_c()
        keep.append(c)
        arr[t] = c
    return _out(L, L.tqo_query(q, arr, nthreads, C.byref(out)), out)


# ---------------------------------------------------------------- reference substrate
def ref_take(b: HostBatch, ids) -> HostBatch:
    L, out = ref(), TqBatchC()
    arr = (C.c_uint64 * max(1, len(ids)))(*ids)
    bc = b.to_c()
    return _out(L, L.tqr_take(C.byref(bc), arr, len(ids), C.byref(out)), out, "tqr")


def ref_concat(bs) -> HostBatch:
    L, out = ref(), TqBatchC()
    cs = [b.to_c() for b in bs]
    arr = (TqBatchC * len(cs))(*cs)
    return _out(L, L.tqr_concat(arr, len(cs), C.byref(out)), out, "tqr")


def ref_batch_size_bytes(b: HostBatch) -> int:
    """The REFERENCE's batch_size_bytes (types.cpp:166-170)."""
    bc = b.to_c()
    return int(ref().tqr_batch_size_bytes(C.byref(bc)))


def ref_rebatch_rows(b: HostBatch, target: int) -> List[int]:
    """Row counts of the REFERENCE's rebatch (transform.cpp:122-154) of one batch."""
    L = ref()
    bc = b.to_c()
    cap = max(16, b.rows + 1)
    rows = (C.c_uint64 * cap)()
    n = C.c_uint32()
    _check(L.tqr_rebatch_rows(C.byref(bc), target, rows, cap, C.byref(n)), L, "tqr")
    return [int(rows[i]) for i in range(n.value)]


def ref_slice(b: HostBatch, start, n) -> HostBatch:
    L, out = ref(), TqBatchC()
    bc = b.to_c()
    return _out(L, L.tqr_slice(C.byref(bc), start, n, C.byref(out)), out, "tqr")


class RefResident:
    """A lineitem batch held as the REFERENCE's own ColumnBatch (converted once,
    kept resident like the GPU's HBM tables) for the CPU baseline."""

    def __init__(self, lineitem: HostBatch):
        L = ref()
        self._keep = lineitem.to_c()
        self.h = L.tqr_resident_make(C.byref(self._keep))
        if not self.h:
            raise RuntimeError("tqr_resident_make failed")

    def q1_fused(self, nthreads: int):
        """Q1 as one fused pass over Column::i64_at / dec_at (types.cpp:66-90),
        nthreads row ranges.  -> (HostBatch like query(1), seconds)."""
        L = ref()
        out = (C.c_uint64 * (1 + 16 * 64))()
        sec = L.tqr_q1_fused(self.h, nthreads, out, 64)
        n = int(out[0])

        def i128(lo, hi):
            v = (int(hi) << 64) | int(lo)
            return v - (1 << 128) if v >> 127 else v
        rows = []
        for g in range(n):
            o = out[1 + 16 * g: 1 + 16 * (g + 1)]
            q, e, dp, ch, d = (i128(o[2 + 2 * k], o[3 + 2 * k]) for k in range(5))
            cnt = int(o[12])
            avg = lambda v, sc: float(v) / (10.0 ** sc) / cnt
            rows.append((int(np.int64(np.uint64(o[0]))), int(np.int64(np.uint64(o[1]))), q, e, dp, ch,
                         avg(q, 2), avg(e, 2), avg(d, 2), cnt))
        b = HostBatch(n)
        cols = list(zip(*rows)) if rows else [[]] * 10
        b.cols = [HostBatch.col_i64(list(cols[0])), HostBatch.col_i64(list(cols[1])),
                  HostBatch.col_dec(list(cols[2]), 38, 2), HostBatch.col_dec(list(cols[3]), 38, 2),
                  HostBatch.col_dec(list(cols[4]), 38, 4), HostBatch.col_dec(list(cols[5]), 38, 6),
                  HostBatch.col_f64(list(cols[6])), HostBatch.col_f64(list(cols[7])), HostBatch.col_f64(list(cols[8])),
                  HostBatch.col_i64(list(cols[9]))]
        return b, sec

    def close(self):
        if self.h:
            ref().tqr_resident_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def host_read_bw(bytes_: int = 1 << 30, nthreads: int = 1, reps: int = 3) -> float:
    """Host memory read bandwidth (GB/s) with nthreads."""
    return ref().tqr_read_bw(bytes_, nthreads, reps)
