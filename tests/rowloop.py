"""Pure-Python row-loop micro-oracles (test infrastructure).

SPEC.md:713 ("filter/project also carry independent row-loop micro-oracles")
and SPEC.md:699 (nested-loop join).  These are deliberately naive and share
no code with oracle/tq_oracle.cpp or the CUDA path: they evaluate the Expr
tree per row with Python integers (int128 / int64 wrap emulated explicitly).
Typing rules: DESIGN.md §3.
"""
from __future__ import annotations

from paper_2508_05029_b200.columnar import BOOL, DECIMAL, FLOAT64, INT64, UTF8, HostBatch
from paper_2508_05029_b200.expr import (ADD, EQ, EX_AND, EX_ARITH, EX_CMP, EX_COL, EX_LIT, EX_NOT, EX_OR, GE,
                                        GT, LE, LT, MUL, NE, SUB, Expr)

M128 = (1 << 128) - 1
M64 = (1 << 64) - 1


def wrap128(v: int) -> int:
    v &= M128
    return v - (1 << 128) if v >> 127 else v


def wrap64(v: int) -> int:
    v &= M64
    return v - (1 << 64) if v >> 63 else v


def typeof(e: Expr, b: HostBatch):
    """-> (cls, scale) with cls in 'I','D','F','B','S'."""
    if e.tag == EX_COL:
        c = b.cols[e.column]
        return {INT64: ("I", 0), DECIMAL: ("D", c.scale), FLOAT64: ("F", 0), BOOL: ("B", 0), UTF8: ("S", 0)}[c.kind]
    if e.tag == EX_LIT:
        return {INT64: ("I", 0), DECIMAL: ("D", e.scale), FLOAT64: ("F", 0), BOOL: ("B", 0)}[e.kind]
    if e.tag == EX_ARITH:
        ta, tb = typeof(e.children[0], b), typeof(e.children[1], b)
        if "F" in (ta[0], tb[0]):
            return ("F", 0)
        if "D" in (ta[0], tb[0]):
            return ("D", ta[1] + tb[1] if e.op == MUL else max(ta[1], tb[1]))
        return ("I", 0)
    return ("B", 0)


def to_float(v, t):
    if t[0] == "F":
        return v
    if t[0] == "I":
        return float(v)
    return float(v) / (10.0 ** t[1])


def eval_row(e: Expr, b: HostBatch, cols, r: int):
    """-> python value or None (null)."""
    if e.tag == EX_COL:
        return cols[e.column][r]
    if e.tag == EX_LIT:
        if e.is_null:
            return None
        return bool(e.value) if e.kind == BOOL else e.value
    if e.tag == EX_NOT:
        a = eval_row(e.children[0], b, cols, r)
        return None if a is None else (not a)
    a = eval_row(e.children[0], b, cols, r)
    c = eval_row(e.children[1], b, cols, r)
    if a is None or c is None:
        return None
    if e.tag == EX_AND:
        return bool(a and c)
    if e.tag == EX_OR:
        return bool(a or c)
    ta, tb = typeof(e.children[0], b), typeof(e.children[1], b)
    if e.tag == EX_ARITH:
        t = typeof(e, b)
        if t[0] == "F":
            x, y = to_float(a, ta), to_float(c, tb)
            return x + y if e.op == ADD else x - y if e.op == SUB else x * y
        x, y = int(a), int(c)
        if t[0] == "D" and e.op != MUL:
            x = wrap128(x * 10 ** (t[1] - ta[1]))
            y = wrap128(y * 10 ** (t[1] - tb[1]))
        r_ = x + y if e.op == ADD else x - y if e.op == SUB else x * y
        return wrap64(r_) if t[0] == "I" else wrap128(r_)
    # compare
    if ta[0] == "S":
        x, y = a.encode(), c.encode()
    elif "F" in (ta[0], tb[0]):
        x, y = to_float(a, ta), to_float(c, tb)
    elif ta[0] == "B":
        x, y = int(a), int(c)
    else:
        s = max(ta[1], tb[1])
        x, y = wrap128(int(a) * 10 ** (s - ta[1])), wrap128(int(c) * 10 ** (s - tb[1]))
    return {LT: x < y, LE: x <= y, EQ: x == y, NE: x != y, GE: x >= y, GT: x > y}[e.op]


def filter_rows(b: HostBatch, pred: Expr):
    cols = [b.column_py(c) for c in range(len(b.cols))]
    return [r for r in range(b.rows) if eval_row(pred, b, cols, r) is True]


def project_values(b: HostBatch, e: Expr):
    cols = [b.column_py(c) for c in range(len(b.cols))]
    return [eval_row(e, b, cols, r) for r in range(b.rows)]
