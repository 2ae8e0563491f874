"""ctypes mirror of the reference operator interface over libtq_gpu.so.

Names and argument meaning follow SPEC.md:560-611 (filter_execute,
project_execute, hash_partition, join_execute, aggregate_execute) and the
columnar substrate (take / concat / slice, transform.cpp).  Every call goes
through the C-ABI of include/tq_gpu.h into sm_100a kernels; there is no CPU
fallback: if the native library is missing the import of `lib()` raises.
Errors come back as TqError carrying the reference's Errc name.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import weakref
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .columnar import (MEM_DEVICE, HostBatch, TqAggC, TqBatchC, TqColumnC, TqError, TqExprC)
from .expr import Expr

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TQ_LIB") or os.path.join(HERE, "libtq_gpu.so")  # TQ_LIB: build-variant experiments
_lib = None
# Contexts still open at interpreter exit are closed by an atexit hook while
# the CUDA runtime is alive; frees that run later (finalizers) become no-ops.
_LIVE = weakref.WeakSet()
_SHUTDOWN = False


@atexit.register
def _close_all():
    global _SHUTDOWN
    _SHUTDOWN = True
    for ctx in list(_LIVE):
        try:
            ctx.close()
        except Exception:
            pass


class TqEngineOptsC(C.Structure):
    _fields_ = [("compute_threads", C.c_uint32), ("preload", C.c_uint32), ("batch_rows", C.c_uint64),
                ("device_budget", C.c_uint64), ("pool_buffer_size", C.c_uint64), ("pool_capacity", C.c_uint64),
                ("high_watermark", C.c_double), ("low_watermark", C.c_double), ("protect_top_k", C.c_uint32),
                ("tables_on_host", C.c_uint32), ("task_batches", C.c_uint32), ("inject_oom_mode", C.c_uint32),
                ("inject_oom_count", C.c_uint32), ("inject_oom_op", C.c_char * 32), ("force_exchange", C.c_uint32),
                ("exchange_impl", C.c_uint32), ("broadcast_threshold", C.c_uint64)]


class TqOptsC(C.Structure):
    _fields_ = [("device", C.c_int), ("ctas_per_sm", C.c_uint32), ("device_budget_bytes", C.c_uint64),
                ("pool_reserve_bytes", C.c_uint64)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (make -C paper_2508_05029_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        P, V = C.POINTER, C.c_void_p
        B = P(TqBatchC)
        L.tq_last_error.restype = C.c_char_p
        L.tq_errc_name.restype = C.c_char_p
        L.tq_ctx_create.argtypes = [P(TqOptsC), P(V)]
        L.tq_ctx_destroy.argtypes = [V]
        L.tq_sync.argtypes = [V, V]
        L.tq_device_bytes_in_use.restype = C.c_uint64
        L.tq_device_bytes_in_use.argtypes = [V]
        L.tq_kernel_launches.restype = C.c_uint32
        L.tq_kernel_launches.argtypes = [V]
        L.tq_batch_alloc.argtypes = [V, B, C.c_uint64, B, V]
        L.tq_batch_upload.argtypes = [V, B, B, V]
        L.tq_batch_download.argtypes = [V, B, B, V]
        L.tq_batch_free.argtypes = [V, B]
        L.tq_host_batch_free.argtypes = [B]
        L.tq_take.argtypes = [V, B, V, C.c_uint64, B, V]
        L.tq_concat.argtypes = [V, B, C.c_uint32, B, V]
        L.tq_slice.argtypes = [V, B, C.c_uint64, C.c_uint64, B, V]
        L.tq_rebatch.argtypes = [V, B, C.c_uint32, C.c_uint64, P(P(TqBatchC)), P(C.c_uint32), V]
        L.tq_filter.argtypes = [V, B, TqExprC, B, V]
        L.tq_project.argtypes = [V, B, P(TqExprC), C.c_uint32, B, V]
        U32 = P(C.c_uint32)
        L.tq_hash_partition.argtypes = [V, B, U32, C.c_uint32, C.c_uint32, B, P(C.c_uint64), V]
        L.tq_filter_async.argtypes = [V, B, TqExprC, B, V, V]
        L.tq_hash_partition_async.argtypes = [V, B, U32, C.c_uint32, C.c_uint32, B, V, V]
        L.tq_batch_set_rows.argtypes = [B, C.c_uint64]
        L.tq_batch_set_rows.restype = None
        L.tq_join_build.argtypes = [V, B, U32, C.c_uint32, P(V), V]
        L.tq_join_build_sized.argtypes = [V, B, U32, C.c_uint32, C.c_uint64, P(V), V]
        L.tq_join_probe.argtypes = [V, V, B, U32, C.c_uint32, B, V]
        L.tq_join_table_destroy.argtypes = [V, V]
        L.tq_aggregate.argtypes = [V, B, U32, C.c_uint32, P(TqAggC), C.c_uint32, B, V]
        E = P(TqExprC)
        L.tq_pipeline_materialize.argtypes = [V, B, E, E, C.c_uint32, B, V]
        L.tq_pipeline_aggregate.argtypes = [V, B, E, E, C.c_uint32, U32, C.c_uint32, P(TqAggC), C.c_uint32, B, V]
        L.tq_pipeline_partition.argtypes = [V, B, E, E, C.c_uint32, U32, C.c_uint32, C.c_uint32, B,
                                            P(C.c_uint64), V]
        L.tq_pipeline_probe.argtypes = [V, V, B, E, E, C.c_uint32, U32, C.c_uint32, U32, C.c_uint32, B, V]
        L.tq_pipeline_build.argtypes = [V, B, E, U32, C.c_uint32, P(V), V]
        L.tq_pipeline_build_semi.argtypes = [V, B, E, U32, C.c_uint32, P(V), V]
        L.tq_join_build_semi.argtypes = [V, B, U32, C.c_uint32, P(V), V]
        L.tq_datagen.argtypes = [V, C.c_int, C.c_double, B, V]
        L.tq_datagen_shard.argtypes = [V, C.c_int, C.c_double, C.c_uint32, C.c_uint32, B, V]
        L.tq_ctx_stream.restype = V
        L.tq_ctx_stream.argtypes = [V]
        L.tq_profile_enable.argtypes = [V, C.c_int]
        L.tq_profile_report.restype = C.c_uint64
        L.tq_profile_report.argtypes = [V, C.c_char_p, C.c_uint64]
        L.tq_pinned_alloc.argtypes = [C.c_uint64, P(V)]
        L.tq_pinned_free.argtypes = [V]
        L.tq_ctx_set_jit.argtypes = [V, C.c_int]
        L.tq_comm_unique_id.argtypes = [C.c_char_p]
        L.tq_comm_init.argtypes = [V, C.c_int, C.c_int, C.c_char_p, P(V)]
        L.tq_comm_destroy.argtypes = [V]
        L.tq_comm_exchange.argtypes = [V, B, P(C.c_uint64), B, P(C.c_uint64), V]
        L.tq_comm_allgather.argtypes = [V, B, B, P(C.c_uint64), V]
        L.tq_comm_bytes_sent.restype = C.c_uint64
        L.tq_comm_bytes_sent.argtypes = [V]
        L.tq_comm_size.argtypes = [V]
        L.tq_comm_rank.argtypes = [V]
        # memory tier (include/tq_memexec.h)
        L.tq_pool_create.argtypes = [C.c_uint64, C.c_uint64, P(V)]
        L.tq_pool_destroy.argtypes = [V]
        L.tq_pool_free_count.restype = C.c_uint64
        L.tq_pool_free_count.argtypes = [V]
        L.tq_pool_buffer_size.restype = C.c_uint64
        L.tq_pool_buffer_size.argtypes = [V]
        L.tq_pool_acquire.argtypes = [V, C.c_uint64, P(C.c_uint32)]
        L.tq_pool_release.argtypes = [V, P(C.c_uint32), C.c_uint64]
        L.tq_pool_buffer.restype = C.c_void_p
        L.tq_pool_buffer.argtypes = [V, C.c_uint32]
        L.tq_chunked_encode.argtypes = [V, B, P(V)]
        L.tq_chunked_decode.argtypes = [V, B]
        L.tq_spill.argtypes = [V, V, B, P(V), V]
        L.tq_load.argtypes = [V, V, B, V]
        L.tq_chunked_layout.restype = C.c_uint32
        L.tq_chunked_layout.argtypes = [V, P(C.c_uint64), P(C.c_uint64), P(C.c_uint64), P(C.c_uint32), C.c_uint32]
        L.tq_chunked_rows.restype = C.c_uint64
        L.tq_chunked_rows.argtypes = [V]
        L.tq_chunked_release.argtypes = [V]
        # engine (include/tq_engine.h)
        L.tq_engine_run_query.argtypes = [V, V, C.c_int, P(TqBatchC), P(TqEngineOptsC), B, C.c_char_p, C.c_uint64]
        L.tq_engine_run_query_tcf.argtypes = [V, V, C.c_int, P(C.c_char_p), P(TqEngineOptsC), B, C.c_char_p,
                                              C.c_uint64]
        L.tq_agg_create.argtypes = [V, E, E, C.c_uint32, U32, C.c_uint32, P(TqAggC), C.c_uint32, P(V)]
        L.tq_agg_update.argtypes = [V, B, V]
        L.tq_agg_finalize.argtypes = [V, B, V]
        L.tq_agg_destroy.argtypes = [V]
        L.tq_bloom_build.argtypes = [V, B, U32, C.c_uint32, C.c_uint64, P(V), V]
        L.tq_bloom_destroy.argtypes = [V]
        L.tq_pipeline_partition_semi.argtypes = [V, B, E, E, C.c_uint32, U32, C.c_uint32, C.c_uint32, V, B,
                                                 P(C.c_uint64), V]
        L.tq_pipeline_partition_exchange.argtypes = [V, B, E, E, C.c_uint32, U32, C.c_uint32, V, B, V]
        L.tq_comm_bloom_union.argtypes = [V, V, V]
        L.tq_comm_gather_table_blooms.argtypes = [V, V, P(V), V]
        L.tq_pipeline_broadcast.argtypes = [V, B, E, E, C.c_uint32, B, V]
        L.tq_comm_last_exchange_capacity.restype = C.c_uint64
        L.tq_comm_last_exchange_capacity.argtypes = [V]
        L.tq_tcf_write.argtypes = [C.c_char_p, B, P(C.c_char_p), C.c_uint64]
        L.tq_tcf_open.argtypes = [C.c_char_p, P(V)]
        L.tq_tcf_close.argtypes = [V]
        for fn in ("tq_tcf_ncols", "tq_tcf_row_groups"):
            getattr(L, fn).restype = C.c_uint32
            getattr(L, fn).argtypes = [V]
        L.tq_tcf_rows.restype = C.c_uint64
        L.tq_tcf_rows.argtypes = [V, C.c_uint32]
        L.tq_tcf_reads.restype = C.c_uint64
        L.tq_tcf_reads.argtypes = [V]
        L.tq_tcf_column.restype = C.c_char_p
        L.tq_tcf_column.argtypes = [V, C.c_uint32, P(TqColumnC)]
        L.tq_tcf_plan_ranges.argtypes = [V, P(C.c_uint32), C.c_uint32, P(C.c_uint32), C.c_uint32, P(C.c_uint64),
                                         C.c_uint64, P(C.c_uint64)]
        L.tq_coalesce_ranges.restype = C.c_uint64
        L.tq_coalesce_ranges.argtypes = [P(C.c_uint64), C.c_uint64, C.c_uint64, C.c_uint64, P(C.c_uint64)]
        L.tq_tcf_fetch.argtypes = [V, V, C.c_uint32, P(C.c_uint32), C.c_uint32, C.c_uint32, P(V)]
        L.tq_on_oom_decide.restype = C.c_int
        L.tq_on_oom_decide.argtypes = [C.c_uint64, C.c_uint64, C.c_int, P(C.c_uint64)]
        L.tq_estimate_reservation.restype = C.c_uint64
        L.tq_estimate_reservation.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_uint64, C.c_double, C.c_double]
        L.tq_jit_report.restype = C.c_uint64
        L.tq_jit_report.argtypes = [V, C.c_char_p, C.c_uint64]
        L.tq_host_timing_report.restype = C.c_uint64
        L.tq_host_timing_report.argtypes = [C.c_char_p, C.c_uint64]
        _lib = L
    return _lib


def _u32(xs: Sequence[int]):
    return (C.c_uint32 * max(1, len(xs)))(*xs)


_SER = {}  # id(expr or list) -> (object, prepared ctypes args): repeated plans skip re-serialisation


def _exprs(exprs: Optional[Sequence[Expr]]):
    if exprs is None:
        return None, 0, []
    hit = _SER.get(id(exprs))
    if hit is not None and hit[0] is exprs:
        return hit[1]
    ss = [e.serialize() for e in exprs]
    arr = (TqExprC * max(1, len(ss)))(*[s.c() for s in ss])
    res = (arr, len(ss), ss)
    if isinstance(exprs, tuple) or len(_SER) < 4096:
        _SER[id(exprs)] = (exprs, res)
    return res


def _pred(pred: Optional[Expr]):
    if pred is None:
        return None, None
    hit = _SER.get(id(pred))
    if hit is not None and hit[0] is pred:
        return hit[1]
    s = pred.serialize()
    c = s.c()
    res = (C.pointer(c), (s, c))
    if len(_SER) < 4096:
        _SER[id(pred)] = (pred, res)
    return res


class PinnedU64:
    """Caller-owned pinned host slot of n uint64 values (tq_pinned_alloc): the
    count slot of the asynchronous operators."""

    def __init__(self, n: int):
        self.ptr = C.c_void_p()
        Context._check(lib().tq_pinned_alloc(8 * max(1, n), C.byref(self.ptr)))
        self.n = n

    def __getitem__(self, i: int) -> int:
        return int(C.cast(self.ptr, C.POINTER(C.c_uint64))[i])

    def values(self) -> List[int]:
        return [self[i] for i in range(self.n)]

    def free(self):
        if self.ptr:
            lib().tq_pinned_free(self.ptr)
            self.ptr = C.c_void_p()


class DeviceBatch:
    """A device-resident batch owned by a Context (freed on close/GC).
    Views (`select`) borrow the parent's buffers and are never freed."""

    def __init__(self, ctx: "Context", c: TqBatchC, parent: "DeviceBatch" = None):
        self.ctx = ctx
        self.c = c
        self.parent = parent

    def select(self, cols: Sequence[int]) -> "DeviceBatch":
        """Column-subset view (scan projection pushdown); no copy."""
        arr = (TqColumnC * max(1, len(cols)))(*[self.c.cols[i] for i in cols])
        v = TqBatchC(self.c.rows, len(cols), MEM_DEVICE, C.cast(arr, C.POINTER(TqColumnC)), None)
        d = DeviceBatch(self.ctx, v, parent=self)
        d._arr = arr
        return d

    @property
    def rows(self) -> int:
        return int(self.c.rows)

    @property
    def ncols(self) -> int:
        return int(self.c.ncols)

    def to_host(self) -> HostBatch:
        return self.ctx.download(self)

    def set_rows(self, rows: int):
        """Trim to the first `rows` rows (an asynchronous operator's count)."""
        lib().tq_batch_set_rows(C.byref(self.c), rows)

    def free(self):
        if self.parent is not None:
            self.c = None
            return
        if self.c is not None and self.ctx.handle and not _SHUTDOWN:
            lib().tq_batch_free(self.ctx.handle, C.byref(self.c))
            self.c = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class JoinTable:
    def __init__(self, ctx: "Context", handle, build: DeviceBatch):
        self.ctx, self.handle, self.build = ctx, handle, build  # keeps the build batch alive

    def free(self):
        if self.handle and self.ctx.handle and not _SHUTDOWN:
            lib().tq_join_table_destroy(self.ctx.handle, self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Context:
    """One tq context per GPU (tq_ctx_create)."""

    def __init__(self, device: int = 0, device_budget_bytes: int = 0, ctas_per_sm: int = 0, pool_reserve_bytes: int = 0):
        L = lib()
        h = C.c_void_p()
        opts = TqOptsC(device, ctas_per_sm, device_budget_bytes, pool_reserve_bytes)
        self._check(L.tq_ctx_create(C.byref(opts), C.byref(h)))
        self.handle = h
        _LIVE.add(self)

    @staticmethod
    def _check(st: int):
        if st != 0:
            L = lib()
            raise TqError(st, (L.tq_last_error() or b"").decode())

    def close(self):
        if self.handle:
            lib().tq_ctx_destroy(self.handle)
            self.handle = None

    def sync(self, stream=None):
        self._check(lib().tq_sync(self.handle, stream))

    def bytes_in_use(self) -> int:
        return lib().tq_device_bytes_in_use(self.handle)

    def kernel_launches(self) -> int:
        return lib().tq_kernel_launches(self.handle)

    # ---- movement ----------------------------------------------------------
    def upload(self, hb: HostBatch, stream=None) -> DeviceBatch:
        hc = hb.to_c()
        out = TqBatchC()
        self._check(lib().tq_batch_upload(self.handle, C.byref(hc), C.byref(out), stream))
        self.sync(stream)
        return DeviceBatch(self, out)

    def download(self, db: DeviceBatch, stream=None) -> HostBatch:
        out = TqBatchC()
        self._check(lib().tq_batch_download(self.handle, C.byref(db.c), C.byref(out), stream))
        try:
            return HostBatch.from_c(out)
        finally:
            lib().tq_host_batch_free(C.byref(out))

    def _wrap(self, st, out):
        self._check(st)
        return DeviceBatch(self, out)

    def datagen(self, table: int, sf: float, stream=None, shard: int = 0, nshards: int = 1) -> DeviceBatch:
        out = TqBatchC()
        return self._wrap(lib().tq_datagen_shard(self.handle, table, sf, shard, nshards, C.byref(out), stream), out)

    def set_jit(self, on: bool):
        """NVRTC-specialised pipeline kernels (default) vs the AOT interpreter."""
        lib().tq_ctx_set_jit(self.handle, 1 if on else 0)

    def jit_report(self) -> dict:
        buf = C.create_string_buffer(4096)
        lib().tq_jit_report(self.handle, buf, len(buf))
        out = {}
        for line in buf.value.decode().splitlines():
            k, _, v = line.partition(" ")
            out[k] = v
        return out

    def stream(self):
        return lib().tq_ctx_stream(self.handle)

    def profile(self, on: bool):
        lib().tq_profile_enable(self.handle, 1 if on else 0)

    def profile_report(self) -> dict:
        """{kernel: (launches, total_ms)} of CUDA-event-timed pipeline kernels."""
        buf = C.create_string_buffer(1 << 16)
        lib().tq_profile_report(self.handle, buf, len(buf))
        out = {}
        for line in buf.value.decode().splitlines():
            name, n, ms = line.split()
            out[name] = (int(n), float(ms))
        return out

    # ---- substrate ---------------------------------------------------------
    def take(self, b: DeviceBatch, ids: Sequence[int], stream=None) -> DeviceBatch:
        n = len(ids)
        dids = self.upload(HostBatch(max(n, 1), [HostBatch.col_i64(list(ids) if n else [0])]), stream)
        out = TqBatchC()
        r = self._wrap(lib().tq_take(self.handle, C.byref(b.c), C.c_void_p(dids.c.cols[0].values), n,
                                     C.byref(out), stream), out)
        self.sync(stream)
        dids.free()
        return r

    def concat(self, bs: Sequence[DeviceBatch], stream=None) -> DeviceBatch:
        arr = (TqBatchC * len(bs))(*[b.c for b in bs])
        out = TqBatchC()
        return self._wrap(lib().tq_concat(self.handle, arr, len(bs), C.byref(out), stream), out)

    def slice(self, b: DeviceBatch, start: int, n: int, stream=None) -> DeviceBatch:
        out = TqBatchC()
        return self._wrap(lib().tq_slice(self.handle, C.byref(b.c), start, n, C.byref(out), stream), out)

    def rebatch(self, bs: Sequence[DeviceBatch], target_bytes: int, stream=None) -> List[DeviceBatch]:
        """reference rebatch (transform.cpp:122-154) on the GPU."""
        arr = (TqBatchC * max(1, len(bs)))(*[b.c for b in bs])
        outs = C.POINTER(TqBatchC)()
        n = C.c_uint32()
        self._check(lib().tq_rebatch(self.handle, arr, len(bs), target_bytes, C.byref(outs), C.byref(n), stream))
        res = []
        for i in range(n.value):
            c = TqBatchC()
            C.memmove(C.byref(c), C.byref(outs[i]), C.sizeof(TqBatchC))
            res.append(DeviceBatch(self, c))
        if n.value:
            libc = C.CDLL(None)
            libc.free.argtypes = [C.c_void_p]
            libc.free(C.cast(outs, C.c_void_p))
        return res

    # ---- operators --------------------------------------
    def filter_execute(self, b: DeviceBatch, pred: Expr, stream=None) -> DeviceBatch:
        s = pred.serialize()
        out = TqBatchC()
        return self._wrap(lib().tq_filter(self.handle, C.byref(b.c), s.c(), C.byref(out), stream), out)

    # ---- asynchronous forms: the count arrives in a pinned slot ----
    def filter_async(self, b: DeviceBatch, pred: Expr, slot: "PinnedU64", stream=None) -> DeviceBatch:
        """No host sync: returns a batch with the input's row count as capacity;
        after the stream reaches this point, slot[1] is the row count — trim with
        DeviceBatch.set_rows(slot[1])."""
        s = pred.serialize()
        out = TqBatchC()
        return self._wrap(lib().tq_filter_async(self.handle, C.byref(b.c), s.c(), C.byref(out), slot.ptr, stream),
                          out)

    def hash_partition_async(self, b: DeviceBatch, keys: Sequence[int], nparts: int, slot: "PinnedU64",
                             stream=None) -> DeviceBatch:
        """slot[0..nparts]: part starts then the total, valid after the stream event."""
        out = TqBatchC()
        return self._wrap(lib().tq_hash_partition_async(self.handle, C.byref(b.c), _u32(keys), len(keys), nparts,
                                                        C.byref(out), slot.ptr, stream), out)

    def project_execute(self, b: DeviceBatch, exprs: Sequence[Expr], stream=None) -> DeviceBatch:
        arr, n, _keep = _exprs(exprs)
        out = TqBatchC()
        return self._wrap(lib().tq_project(self.handle, C.byref(b.c), arr, n, C.byref(out), stream), out)

    def hash_partition(self, b: DeviceBatch, keys: Sequence[int], nparts: int,
                       stream=None) -> Tuple[DeviceBatch, List[int]]:
        offs = (C.c_uint64 * (nparts + 1))()
        out = TqBatchC()
        r = self._wrap(lib().tq_hash_partition(self.handle, C.byref(b.c), _u32(keys), len(keys), nparts,
                                               C.byref(out), offs, stream), out)
        return r, list(offs)

    def join_build(self, build: DeviceBatch, keys: Sequence[int], stream=None, bloom_keys: int = 0,
                   semi: bool = False) -> JoinTable:
        """bloom_keys > 0: size the table's Bloom filter for that many keys
        (tq_join_build_sized; equal sizes across ranks for gather_table_blooms).
        semi=True: build side of a semi-join (tq_join_build_semi)."""
        h = C.c_void_p()
        if semi:
            self._check(lib().tq_join_build_semi(self.handle, C.byref(build.c), _u32(keys), len(keys), C.byref(h),
                                                 stream))
        elif bloom_keys:
            self._check(lib().tq_join_build_sized(self.handle, C.byref(build.c), _u32(keys), len(keys), bloom_keys,
                                                  C.byref(h), stream))
        else:
            self._check(lib().tq_join_build(self.handle, C.byref(build.c), _u32(keys), len(keys), C.byref(h), stream))
        return JoinTable(self, h, build)

    def join_probe(self, t: JoinTable, probe: DeviceBatch, keys: Sequence[int], stream=None) -> DeviceBatch:
        out = TqBatchC()
        return self._wrap(lib().tq_join_probe(self.handle, t.handle, C.byref(probe.c), _u32(keys), len(keys),
                                              C.byref(out), stream), out)

    def join_execute(self, build: DeviceBatch, probe: DeviceBatch, bkeys: Sequence[int], pkeys: Sequence[int],
                     stream=None) -> DeviceBatch:
        t = self.join_build(build, bkeys, stream)
        try:
            return self.join_probe(t, probe, pkeys, stream)
        finally:
            self.sync(stream)
            t.free()

    def aggregate_execute(self, b: DeviceBatch, keys: Sequence[int], aggs: Sequence[Tuple[int, int]],
                          stream=None) -> DeviceBatch:
        arr = (TqAggC * max(1, len(aggs)))(*[TqAggC(f, c) for f, c in aggs])
        out = TqBatchC()
        return self._wrap(lib().tq_aggregate(self.handle, C.byref(b.c), _u32(keys), len(keys), arr, len(aggs),
                                             C.byref(out), stream), out)

    # ---- fused pipelines ---------------------------------------------------
    def pipeline_materialize(self, b: DeviceBatch, pred: Optional[Expr], exprs: Optional[Sequence[Expr]],
                             stream=None) -> DeviceBatch:
        pp, _k1 = _pred(pred)
        arr, n, _k2 = _exprs(exprs)
        out = TqBatchC()
        return self._wrap(lib().tq_pipeline_materialize(self.handle, C.byref(b.c), pp, arr, n, C.byref(out),
                                                        stream), out)

    def pipeline_aggregate(self, b: DeviceBatch, pred: Optional[Expr], exprs: Optional[Sequence[Expr]],
                           keys: Sequence[int], aggs: Sequence[Tuple[int, int]], stream=None) -> DeviceBatch:
        pp, _k1 = _pred(pred)
        arr, n, _k2 = _exprs(exprs)
        ag = (TqAggC * max(1, len(aggs)))(*[TqAggC(f, c) for f, c in aggs])
        out = TqBatchC()
        return self._wrap(lib().tq_pipeline_aggregate(self.handle, C.byref(b.c), pp, arr, n, _u32(keys), len(keys),
                                                      ag, len(aggs), C.byref(out), stream), out)

    def agg_stream(self, batches: Sequence[DeviceBatch], pred: Optional[Expr], exprs: Optional[Sequence[Expr]],
                   keys: Sequence[int], aggs: Sequence[Tuple[int, int]], stream=None) -> DeviceBatch:
        """Streaming aggregation state: tq_agg_create / update per batch / finalize."""
        pp, _k1 = _pred(pred)
        arr, n, _k2 = _exprs(exprs)
        ag = (TqAggC * max(1, len(aggs)))(*[TqAggC(f, c) for f, c in aggs])
        h = C.c_void_p()
        self._check(lib().tq_agg_create(self.handle, pp, arr, n, _u32(keys), len(keys), ag, len(aggs), C.byref(h)))
        try:
            for b in batches:
                self._check(lib().tq_agg_update(h, C.byref(b.c), stream))
            out = TqBatchC()
            self._check(lib().tq_agg_finalize(h, C.byref(out), stream))
            return DeviceBatch(self, out)
        finally:
            lib().tq_agg_destroy(h)

    def pipeline_partition(self, b: DeviceBatch, pred, exprs, keys: Sequence[int], nparts: int, stream=None):
        pp, _k1 = _pred(pred)
        arr, n, _k2 = _exprs(exprs)
        offs = (C.c_uint64 * (nparts + 1))()
        out = TqBatchC()
        r = self._wrap(lib().tq_pipeline_partition(self.handle, C.byref(b.c), pp, arr, n, _u32(keys), len(keys),
                                                   nparts, C.byref(out), offs, stream), out)
        return r, list(offs)

    def bloom_build(self, b: DeviceBatch, keys: Sequence[int], expected_keys: int = 0, stream=None) -> "Bloom":
        """LIP Bloom filter over the key columns of a build side."""
        h = C.c_void_p()
        self._check(lib().tq_bloom_build(self.handle, C.byref(b.c), _u32(keys), len(keys), expected_keys, C.byref(h),
                                         stream))
        return Bloom(self, h)

    def pipeline_partition_semi(self, b: DeviceBatch, pred, exprs, keys: Sequence[int], nparts: int, semi: "Bloom",
                                stream=None):
        pp, _k1 = _pred(pred)
        arr, n, _k2 = _exprs(exprs)
        offs = (C.c_uint64 * (nparts + 1))()
        out = TqBatchC()
        r = self._wrap(lib().tq_pipeline_partition_semi(self.handle, C.byref(b.c), pp, arr, n, _u32(keys), len(keys),
                                                        nparts, semi.handle if semi else None, C.byref(out), offs,
                                                        stream), out)
        return r, list(offs)

    def pipeline_build(self, b: DeviceBatch, pred, keys: Sequence[int], stream=None, semi: bool = False) -> JoinTable:
        """semi=True: build side of a semi-join (tq_pipeline_build_semi) — probes
        take no build columns; dense unique keys need no hash table."""
        pp, _k1 = _pred(pred)
        h = C.c_void_p()
        fn = lib().tq_pipeline_build_semi if semi else lib().tq_pipeline_build
        self._check(fn(self.handle, C.byref(b.c), pp, _u32(keys), len(keys), C.byref(h), stream))
        return JoinTable(self, h, b)

    def pipeline_probe(self, t: JoinTable, b: DeviceBatch, pred, exprs, keys: Sequence[int],
                       build_cols: Optional[Sequence[int]] = None, stream=None) -> DeviceBatch:
        pp, _k1 = _pred(pred)
        arr, n, _k2 = _exprs(exprs)
        bc = _u32(build_cols) if build_cols is not None else None
        nb = len(build_cols) if build_cols is not None else 0
        out = TqBatchC()
        return self._wrap(lib().tq_pipeline_probe(self.handle, t.handle, C.byref(b.c), pp, arr, n, _u32(keys),
                                                  len(keys), bc, nb, C.byref(out), stream), out)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Bloom:
    def __init__(self, ctx, h):
        self.ctx, self.handle = ctx, h

    def free(self):
        if self.handle and not _SHUTDOWN:
            lib().tq_bloom_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Comm:
    """NCCL communicator over one Context per GPU (include/tq_exchange.h)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        Context._check(lib().tq_comm_unique_id(buf))
        return buf.raw

    def __init__(self, ctx: Context, rank: int, nranks: int, uid: bytes):
        self.ctx, self.rank, self.n = ctx, rank, nranks
        h = C.c_void_p()
        Context._check(lib().tq_comm_init(ctx.handle, rank, nranks, uid, C.byref(h)))
        self.handle = h

    def exchange(self, b: DeviceBatch, part_offsets: Sequence[int], stream=None) -> Tuple[DeviceBatch, List[int]]:
        po = (C.c_uint64 * (self.n + 1))(*part_offsets)
        ro = (C.c_uint64 * (self.n + 1))()
        out = TqBatchC()
        Context._check(lib().tq_comm_exchange(self.handle, C.byref(b.c), po, C.byref(out), ro, stream))
        return DeviceBatch(self.ctx, out), list(ro)

    def partition_exchange(self, b: DeviceBatch, pred, exprs, keys: Sequence[int], semi: "Bloom" = None,
                           stream=None) -> DeviceBatch:
        """Fused hash-partition + shuffle over NVLink peer memory
        (tq_pipeline_partition_exchange): the rows every rank sends to this one,
        in unspecified order.  Collective."""
        pp, _k1 = _pred(pred)
        arr, n, _k2 = _exprs(exprs)
        out = TqBatchC()
        Context._check(lib().tq_pipeline_partition_exchange(self.handle, C.byref(b.c), pp, arr, n, _u32(keys),
                                                            len(keys), semi.handle if semi else None,
                                                            C.byref(out), stream))
        return DeviceBatch(self.ctx, out)

    def broadcast(self, b: DeviceBatch, pred, exprs, stream=None) -> DeviceBatch:
        """Fused filter/project + broadcast over NVLink peer memory
        (tq_pipeline_broadcast): every rank's passing rows, unspecified order.  Collective."""
        pp, _k1 = _pred(pred)
        arr, n, _k2 = _exprs(exprs)
        out = TqBatchC()
        Context._check(lib().tq_pipeline_broadcast(self.handle, C.byref(b.c), pp, arr, n, C.byref(out), stream))
        return DeviceBatch(self.ctx, out)

    def allgather(self, b: DeviceBatch, stream=None) -> Tuple[DeviceBatch, List[int]]:
        ro = (C.c_uint64 * (self.n + 1))()
        out = TqBatchC()
        Context._check(lib().tq_comm_allgather(self.handle, C.byref(b.c), C.byref(out), ro, stream))
        return DeviceBatch(self.ctx, out), list(ro)

    def bloom_union(self, bloom: "Bloom", stream=None):
        Context._check(lib().tq_comm_bloom_union(self.handle, bloom.handle, stream))

    def gather_table_blooms(self, table: JoinTable, stream=None) -> "Bloom":
        """Partitioned LIP filter: part d = rank d's join-table Bloom filter
        (tq_comm_gather_table_blooms).  Collective."""
        h = C.c_void_p()
        Context._check(lib().tq_comm_gather_table_blooms(self.handle, table.handle, C.byref(h), stream))
        return Bloom(self.ctx, h)

    def last_exchange_capacity(self) -> int:
        """Most rows any rank received in the last partition_exchange (same on every rank)."""
        return lib().tq_comm_last_exchange_capacity(self.handle)

    def bytes_sent(self) -> int:
        return lib().tq_comm_bytes_sent(self.handle)

    def close(self):
        if self.handle:
            lib().tq_comm_destroy(self.handle)
            self.handle = None


class Pool:
    """Pinned FixedBufferPool (reference pool.hpp:29-56) — the Host tier."""

    def __init__(self, buffer_size: int, capacity: int):
        h = C.c_void_p()
        Context._check(lib().tq_pool_create(buffer_size, capacity, C.byref(h)))
        self.handle = h

    def free_count(self) -> int:
        return lib().tq_pool_free_count(self.handle)

    def acquire(self, n: int) -> List[int]:
        ids = (C.c_uint32 * max(1, n))()
        Context._check(lib().tq_pool_acquire(self.handle, n, ids))
        return list(ids)[:n]

    def release(self, ids: Sequence[int]):
        arr = (C.c_uint32 * max(1, len(ids)))(*ids)
        Context._check(lib().tq_pool_release(self.handle, arr, len(ids)))

    def encode(self, hb: HostBatch) -> "Chunked":
        hc = hb.to_c()
        h = C.c_void_p()
        Context._check(lib().tq_chunked_encode(self.handle, C.byref(hc), C.byref(h)))
        return Chunked(h)

    def spill(self, ctx: Context, db: DeviceBatch, stream=None) -> "Chunked":
        h = C.c_void_p()
        Context._check(lib().tq_spill(ctx.handle, self.handle, C.byref(db.c), C.byref(h), stream))
        ctx.sync(stream)
        return Chunked(h)

    def close(self):
        if self.handle:
            lib().tq_pool_destroy(self.handle)
            self.handle = None


class Chunked:
    """ChunkedBatch (reference chunked.hpp:22-53) in a Pool."""

    def __init__(self, h):
        self.handle = h

    def layout(self):
        nbuf, tail, total = C.c_uint64(), C.c_uint64(), C.c_uint64()
        n = lib().tq_chunked_layout(self.handle, C.byref(nbuf), C.byref(tail), C.byref(total), None, 0)
        segs = (C.c_uint32 * (3 * max(1, n)))()
        lib().tq_chunked_layout(self.handle, None, None, None, segs, n)
        return nbuf.value, tail.value, total.value, [tuple(segs[3 * i:3 * i + 3]) for i in range(n)]

    def decode(self) -> HostBatch:
        out = TqBatchC()
        Context._check(lib().tq_chunked_decode(self.handle, C.byref(out)))
        try:
            return HostBatch.from_c(out)
        finally:
            lib().tq_host_batch_free(C.byref(out))

    def load(self, ctx: Context, stream=None) -> DeviceBatch:
        out = TqBatchC()
        Context._check(lib().tq_load(ctx.handle, self.handle, C.byref(out), stream))
        ctx.sync(stream)
        return DeviceBatch(ctx, out)

    def release(self):
        if self.handle:
            lib().tq_chunked_release(self.handle)
            self.handle = None


def estimate_reservation(samples, ema_peak, ema_ratio, input_bytes, multiplier, safety=1.25) -> int:
    return lib().tq_estimate_reservation(samples, ema_peak, ema_ratio, input_bytes, multiplier, safety)


OOM_ACTIONS = ("retry", "split", "abort")


def on_oom_decide(estimate: int, capacity: int, splittable: bool) -> Tuple[str, int]:
    """SPEC.md:390-398 on_oom rule -> (action, new estimate)."""
    e = C.c_uint64()
    a = lib().tq_on_oom_decide(estimate, capacity, 1 if splittable else 0, C.byref(e))
    return OOM_ACTIONS[a], e.value


def engine_run_query(ctx: Context, query: int, tables: dict, comm: "Comm" = None, **opts):
    """Run a benchmark query DAG on the C++ worker runtime (include/tq_engine.h).
    tables: {table_id: DeviceBatch or HostBatch}.  Returns (HostBatch, metrics)."""
    import json
    arr = (TqBatchC * 8)()
    keep = []
    for t, b in tables.items():
        if isinstance(b, DeviceBatch):
            arr[t] = b.c
        else:
            c = b.to_c()
            keep.append(c)
            arr[t] = c
    o = TqEngineOptsC()
    for k, v in opts.items():
        setattr(o, k, v.encode() if isinstance(v, str) else v)
    out = TqBatchC()
    buf = C.create_string_buffer(1 << 16)
    Context._check(lib().tq_engine_run_query(ctx.handle, comm.handle if comm else None, query, arr, C.byref(o),
                                             C.byref(out), buf, len(buf)))
    try:
        res = HostBatch.from_c(out)
    finally:
        lib().tq_host_batch_free(C.byref(out))
    return res, json.loads(buf.value.decode() or "{}")


class Tcf:
    """A TCF file (include/tq_storage.h): footer read on open
    (exactly two reads), per-row-group byte-range fetch into the pinned Host
    pool (a Chunked batch: .decode() on the host, .load(ctx) to the device)."""

    @staticmethod
    def write(path: str, table: HostBatch, row_group_bytes: int, names: Sequence[str] = None):
        hc = table.to_c()
        nm = None
        if names:
            nm = (C.c_char_p * len(names))(*[n.encode() for n in names])
        Context._check(lib().tq_tcf_write(path.encode(), C.byref(hc), nm, row_group_bytes))

    def __init__(self, path: str):
        h = C.c_void_p()
        Context._check(lib().tq_tcf_open(path.encode(), C.byref(h)))
        self.handle = h

    @property
    def row_groups(self) -> int:
        return lib().tq_tcf_row_groups(self.handle)

    @property
    def ncols(self) -> int:
        return lib().tq_tcf_ncols(self.handle)

    def rows(self, rg: int) -> int:
        return lib().tq_tcf_rows(self.handle, rg)

    def reads(self) -> int:
        return lib().tq_tcf_reads(self.handle)

    def column(self, c: int):
        col = TqColumnC()
        name = lib().tq_tcf_column(self.handle, c, C.byref(col))
        return (name.decode() if name else None), col.kind, col.precision, col.scale

    def plan_ranges(self, cols: Sequence[int], row_groups: Sequence[int]) -> List[Tuple[int, int]]:
        n = C.c_uint64()
        cap = max(1, len(cols) * len(row_groups))
        out = (C.c_uint64 * (2 * cap))()
        Context._check(lib().tq_tcf_plan_ranges(self.handle, _u32(cols), len(cols), _u32(row_groups), len(row_groups),
                                                out, cap, C.byref(n)))
        return [(out[2 * i], out[2 * i + 1]) for i in range(n.value)]

    def fetch(self, pool: "Pool", rg: int, cols: Sequence[int], max_connections: int = 4) -> "Chunked":
        h = C.c_void_p()
        Context._check(lib().tq_tcf_fetch(self.handle, pool.handle, rg, _u32(cols), len(cols), max_connections,
                                          C.byref(h)))
        return Chunked(h)

    def close(self):
        if self.handle:
            lib().tq_tcf_close(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def coalesce_ranges(ranges: Sequence[Tuple[int, int]], max_gap: int, max_merged: int) -> List[Tuple[int, int]]:
    """SPEC.md coalesce_ranges (tq_coalesce_ranges)."""
    n = len(ranges)
    flat = (C.c_uint64 * max(2, 2 * n))(*[v for r in ranges for v in r])
    out = (C.c_uint64 * max(2, 2 * n))()
    k = lib().tq_coalesce_ranges(flat, n, max_gap, max_merged, out)
    return [(out[2 * i], out[2 * i + 1]) for i in range(k)]


def engine_run_query_tcf(ctx: Context, query: int, paths: dict, comm: "Comm" = None, **opts):
    """Run a query DAG on the C++ worker runtime over TCF files (paths:
    {table_id: path}); every row group is a Storage-tier batch the executors
    fetch into the pinned pool and move to the device.  Returns (HostBatch, metrics)."""
    import json
    arr = (C.c_char_p * 8)(*[paths[t].encode() if t in paths else None for t in range(8)])
    o = TqEngineOptsC()
    for k, v in opts.items():
        setattr(o, k, v.encode() if isinstance(v, str) else v)
    out = TqBatchC()
    buf = C.create_string_buffer(1 << 16)
    Context._check(lib().tq_engine_run_query_tcf(ctx.handle, comm.handle if comm else None, query, arr, C.byref(o),
                                                 C.byref(out), buf, len(buf)))
    try:
        res = HostBatch.from_c(out)
    finally:
        lib().tq_host_batch_free(C.byref(out))
    return res, json.loads(buf.value.decode() or "{}")
