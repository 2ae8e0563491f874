"""Host-side columnar batches (numpy) and the ctypes mirror of include/tq_types.h.

`HostBatch` is the Python view of the reference's ColumnBatch
(reference proj/include/tierq/columnar/types.hpp:104-143): per column a values
byte section, an optional LSB-first validity bitmap and, for Utf8, int32
offsets.  It is plumbing for tests and the bench: the operators themselves run
in libtq_gpu.so (CUDA) behind the C-ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

INT64, FLOAT64, BOOL, UTF8, DECIMAL = 0, 1, 2, 3, 4
KIND_NAMES = {INT64: "int64", FLOAT64: "float64", BOOL: "bool", UTF8: "utf8", DECIMAL: "decimal"}
WIDTH = {INT64: 8, FLOAT64: 8, BOOL: 1, DECIMAL: 16, UTF8: 0}
MEM_HOST, MEM_DEVICE = 0, 1

# Errc ordinals + 1 (reference proj/include/tierq/common.hpp:34-53)
ERRC = [
    "PoolExhausted", "CorruptLayout", "MalformedBatch", "SchemaMismatch", "NotTcf",
    "CorruptFooter", "UnknownColumn", "CorruptRowGroup", "IoError", "ReservationImpossible",
    "ReservationExceeded", "NoEligibleVictims", "OutOfMemoryUnsplittable", "CorruptFrame",
    "PeerDisconnected", "InvalidPlan", "WorkerFailure", "Internal",
]


class TqError(RuntimeError):
    """Mirror of tierq::Error (common.hpp:57-66): carries the Errc name."""

    def __init__(self, status: int, msg: str = ""):
        self.status = status
        self.errc = ERRC[status - 1] if 1 <= status <= len(ERRC) else f"status{status}"
        super().__init__(f"{self.errc}: {msg}")


class TqColumnC(C.Structure):
    _fields_ = [
        ("kind", C.c_uint8), ("precision", C.c_uint8), ("scale", C.c_uint8), ("_pad", C.c_uint8 * 5),
        ("values", C.c_void_p), ("values_bytes", C.c_uint64),
        ("validity", C.c_void_p), ("offsets", C.c_void_p),
    ]


class TqBatchC(C.Structure):
    _fields_ = [
        ("rows", C.c_uint64), ("ncols", C.c_uint32), ("mem", C.c_uint32),
        ("cols", C.POINTER(TqColumnC)), ("owner", C.c_void_p),
    ]


class TqExprNodeC(C.Structure):
    _fields_ = [
        ("tag", C.c_uint8), ("op", C.c_uint8), ("kind", C.c_uint8), ("scale", C.c_uint8),
        ("is_null", C.c_uint8), ("_pad", C.c_uint8 * 3), ("column", C.c_uint32), ("_pad2", C.c_uint32),
        ("lo", C.c_uint64), ("hi", C.c_uint64),
    ]


class TqExprC(C.Structure):
    _fields_ = [("nodes", C.POINTER(TqExprNodeC)), ("len", C.c_uint32), ("_pad", C.c_uint32)]


class TqAggC(C.Structure):
    _fields_ = [("fn", C.c_uint32), ("column", C.c_uint32)]


assert C.sizeof(TqColumnC) == 40 and C.sizeof(TqBatchC) == 32 and C.sizeof(TqExprNodeC) == 32


def bitmap_bytes(rows: int) -> int:
    return (rows + 7) // 8


def pack_validity(valid: np.ndarray) -> np.ndarray:
    """bool[rows] -> LSB-first bitmap (types.hpp:91-100), padding bits zero."""
    return np.packbits(np.asarray(valid, dtype=bool), bitorder="little")


def unpack_validity(bm: Optional[np.ndarray], rows: int) -> np.ndarray:
    if bm is None:
        return np.ones(rows, dtype=bool)
    return np.unpackbits(np.asarray(bm, dtype=np.uint8), bitorder="little", count=rows).astype(bool)


@dataclass
class HostColumn:
    kind: int
    values: np.ndarray  # uint8 raw LE bytes
    validity: Optional[np.ndarray] = None  # uint8 bitmap
    offsets: Optional[np.ndarray] = None  # int32 (Utf8)
    precision: int = 0
    scale: int = 0

    # ---- typed views -------------------------------------------------------
    def i64(self) -> np.ndarray:
        return self.values.view(np.int64)

    def f64(self) -> np.ndarray:
        return self.values.view(np.float64)

    def dec_words(self) -> np.ndarray:
        """(rows, 2) int64: [:,0] low word (as int64 bits), [:,1] high word."""
        return self.values.view(np.int64).reshape(-1, 2)

    def dec_ints(self) -> List[int]:
        w = self.values.view(np.uint64).reshape(-1, 2)
        out = []
        for lo, hi in w.tolist():
            v = (hi << 64) | lo
            if v >= 1 << 127:
                v -= 1 << 128
            out.append(v)
        return out


@dataclass
class HostBatch:
    rows: int
    cols: List[HostColumn] = field(default_factory=list)
    _keep: list = field(default_factory=list, repr=False)

    # ---- constructors ------------------------------------------------------
    @staticmethod
    def col_i64(vals, valid=None) -> HostColumn:
        a = np.ascontiguousarray(np.asarray(vals, dtype=np.int64))
        return HostColumn(INT64, a.view(np.uint8).copy(), None if valid is None else pack_validity(valid))

    @staticmethod
    def col_f64(vals, valid=None) -> HostColumn:
        a = np.ascontiguousarray(np.asarray(vals, dtype=np.float64))
        return HostColumn(FLOAT64, a.view(np.uint8).copy(), None if valid is None else pack_validity(valid))

    @staticmethod
    def col_bool(vals, valid=None) -> HostColumn:
        a = np.asarray(vals, dtype=bool).astype(np.uint8)
        return HostColumn(BOOL, a.copy(), None if valid is None else pack_validity(valid))

    @staticmethod
    def col_dec(vals, precision=11, scale=2, valid=None) -> HostColumn:
        """vals: python ints (any int128) or an int64 numpy array (sign-extended)."""
        if isinstance(vals, np.ndarray) and vals.dtype == np.int64:
            w = np.empty((len(vals), 2), dtype=np.int64)
            w[:, 0] = vals
            w[:, 1] = np.where(vals < 0, -1, 0)
        else:
            vals = list(vals)
            w = np.empty((len(vals), 2), dtype=np.uint64)
            for i, v in enumerate(vals):
                v &= (1 << 128) - 1
                w[i, 0] = v & 0xFFFFFFFFFFFFFFFF
                w[i, 1] = v >> 64
        return HostColumn(DECIMAL, w.view(np.uint8).reshape(-1).copy(),
                          None if valid is None else pack_validity(valid), None, precision, scale)

    @staticmethod
    def col_utf8(strs: Sequence[str], valid=None) -> HostColumn:
        bs = [s.encode() for s in strs]
        off = np.zeros(len(bs) + 1, dtype=np.int32)
        off[1:] = np.cumsum([len(b) for b in bs]) if bs else []
        vals = np.frombuffer(b"".join(bs), dtype=np.uint8).copy()
        return HostColumn(UTF8, vals, None if valid is None else pack_validity(valid), off)

    def validity_of(self, c: int) -> np.ndarray:
        return unpack_validity(self.cols[c].validity, self.rows)

    # ---- ctypes ------------------------------------------------------------
    def to_c(self) -> TqBatchC:
        n = len(self.cols)
        arr = (TqColumnC * max(n, 1))()
        keep = [arr]
        for i, c in enumerate(self.cols):
            vals = np.ascontiguousarray(c.values, dtype=np.uint8)
            if vals.size == 0:
                vals = np.zeros(1, dtype=np.uint8)
                nbytes = 0
            else:
                nbytes = vals.size
            keep.append(vals)
            arr[i].kind, arr[i].precision, arr[i].scale = c.kind, c.precision, c.scale
            arr[i].values = vals.ctypes.data
            arr[i].values_bytes = nbytes
            if c.validity is not None:
                v = np.ascontiguousarray(c.validity, dtype=np.uint8)
                if v.size == 0:
                    v = np.zeros(1, dtype=np.uint8)
                keep.append(v)
                arr[i].validity = v.ctypes.data
            if c.offsets is not None:
                o = np.ascontiguousarray(c.offsets, dtype=np.int32)
                keep.append(o)
                arr[i].offsets = o.ctypes.data
        b = TqBatchC(self.rows, n, MEM_HOST, C.cast(arr, C.POINTER(TqColumnC)), None)
        b._keep = keep  # type: ignore[attr-defined]
        return b

    @staticmethod
    def from_c(b: TqBatchC) -> "HostBatch":
        """Copy a HOST tq_batch into numpy (caller frees the C batch)."""
        assert b.mem == MEM_HOST
        out = HostBatch(int(b.rows))
        for i in range(b.ncols):
            c = b.cols[i]
            nb = int(c.values_bytes)
            vals = np.ctypeslib.as_array(C.cast(c.values, C.POINTER(C.c_uint8)), (nb,)).copy() if nb else \
                np.zeros(0, dtype=np.uint8)
            val = None
            if c.validity:
                m = bitmap_bytes(out.rows)
                val = np.ctypeslib.as_array(C.cast(c.validity, C.POINTER(C.c_uint8)), (m,)).copy() if m else \
                    np.zeros(0, dtype=np.uint8)
            off = None
            if c.kind == UTF8:
                off = np.ctypeslib.as_array(C.cast(c.offsets, C.POINTER(C.c_int32)), (out.rows + 1,)).copy()
            out.cols.append(HostColumn(int(c.kind), vals, val, off, int(c.precision), int(c.scale)))
        return out

    def nbytes(self) -> int:
        """batch_size_bytes (types.cpp:166-170)."""
        t = 0
        for c in self.cols:
            t += c.values.size
            t += 0 if c.validity is None else c.validity.size
            t += 0 if c.offsets is None else c.offsets.size * 4
        return t

    # ---- logical rows (for tests) -----------------------------------------
    def column_py(self, c: int) -> list:
        col = self.cols[c]
        valid = self.validity_of(c)
        if col.kind == INT64:
            vals = col.i64().tolist()
        elif col.kind == FLOAT64:
            vals = col.f64().tolist()
        elif col.kind == BOOL:
            vals = [bool(x) for x in col.values.tolist()]
        elif col.kind == DECIMAL:
            vals = col.dec_ints()
        else:
            o = col.offsets
            raw = col.values.tobytes()
            vals = [raw[o[i]:o[i + 1]].decode() for i in range(self.rows)]
        return [v if ok else None for v, ok in zip(vals, valid.tolist())]

    def to_rows(self) -> list:
        cols = [self.column_py(c) for c in range(len(self.cols))]
        return list(zip(*cols)) if cols else [()] * self.rows


def _sort_keys(b: HostBatch, exact_only: bool):
    keys = []
    for c, col in enumerate(b.cols):
        valid = b.validity_of(c)
        if col.kind == INT64:
            keys.append(np.where(valid, col.i64(), 0))
        elif col.kind == DECIMAL:
            w = col.dec_words()
            keys.append(np.where(valid, w[:, 0].view(np.uint64), 0))
            keys.append(np.where(valid, w[:, 1], 0))
        elif col.kind == BOOL:
            keys.append(np.where(valid, col.values, 0))
        elif col.kind == FLOAT64:
            if exact_only:
                continue
            keys.append(np.where(valid, col.f64(), 0.0))
        else:
            o = col.offsets
            raw = col.values.tobytes()
            s = np.array([raw[o[i]:o[i + 1]] for i in range(b.rows)], dtype=object)
            _, inv = np.unique(s, return_inverse=True) if b.rows else (None, np.zeros(0, np.int64))
            keys.append(np.where(valid, inv, -1))
        keys.append(~valid)
    return keys


def canonical_order(b: HostBatch) -> np.ndarray:
    if b.rows == 0:
        return np.zeros(0, dtype=np.int64)
    keys = _sort_keys(b, exact_only=True) + _sort_keys(b, exact_only=False)
    return np.lexsort(keys[::-1])


def assert_batches_equal(got: HostBatch, want: HostBatch, rtol: float = 1e-9, ordered: bool = False):
    """Canonical-sort comparison: integers/decimals/bools/strings and
    validity bit-exact, Float64 within `rtol` relative (north star: 1e-9)."""
    assert got.rows == want.rows, f"row count {got.rows} != {want.rows}"
    assert len(got.cols) == len(want.cols), f"ncols {len(got.cols)} != {len(want.cols)}"
    for c, (g, w) in enumerate(zip(got.cols, want.cols)):
        assert g.kind == w.kind, f"col {c}: kind {g.kind} != {w.kind}"
        if g.kind == DECIMAL:
            assert g.scale == w.scale, f"col {c}: scale {g.scale} != {w.scale}"
    if got.rows == 0:
        return
    og = np.arange(got.rows) if ordered else canonical_order(got)
    ow = np.arange(want.rows) if ordered else canonical_order(want)
    for c, (g, w) in enumerate(zip(got.cols, want.cols)):
        vg, vw = got.validity_of(c)[og], want.validity_of(c)[ow]
        assert np.array_equal(vg, vw), f"col {c}: validity differs at rows {np.nonzero(vg != vw)[0][:10]}"
        if g.kind == UTF8:
            cg, cw = got.column_py(c), want.column_py(c)
            pg = [cg[i] for i in og]
            pw = [cw[i] for i in ow]
            assert pg == pw, f"col {c}: utf8 values differ"
            continue
        if g.kind == FLOAT64:
            a, b = g.f64()[og][vg], w.f64()[ow][vw]
            ok = np.isclose(a, b, rtol=rtol, atol=0.0) | (a == b)
            assert ok.all(), f"col {c}: float mismatch e.g. {a[~ok][:5]} vs {b[~ok][:5]}"
            continue
        width = WIDTH[g.kind]
        a = g.values.reshape(-1, width)[og][vg]
        b = w.values.reshape(-1, width)[ow][vw]
        if not np.array_equal(a, b):
            bad = np.nonzero((a != b).any(axis=1))[0][:5]
            raise AssertionError(f"col {c} ({KIND_NAMES[g.kind]}): values differ at sorted rows {bad}")
