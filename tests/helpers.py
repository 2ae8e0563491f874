"""Seeded random batches / expressions for parity tests (test infrastructure)."""
from __future__ import annotations

import random

import numpy as np

from paper_2508_05029_b200.columnar import BOOL, DECIMAL, FLOAT64, INT64, UTF8, HostBatch
from paper_2508_05029_b200.expr import (ADD, MUL, SUB, And, Arith, Cmp, Col, Dec, Lit, Not, Null, Or)


def rand_valid(rng: np.random.Generator, n: int, null_frac: float):
    if null_frac <= 0:
        return None
    return rng.random(n) >= null_frac


def rand_batch(seed: int, rows: int, kinds=(INT64, DECIMAL, FLOAT64, BOOL, INT64), null_frac=0.1,
               small=True, utf8=False) -> HostBatch:
    """Columns in `kinds` order; values small so comparisons/keys collide."""
    rng = np.random.default_rng(seed)
    b = HostBatch(rows)
    for k in kinds:
        valid = rand_valid(rng, rows, null_frac)
        if k == INT64:
            v = rng.integers(-20, 20, rows) if small else rng.integers(-(1 << 62), 1 << 62, rows)
            b.cols.append(HostBatch.col_i64(v, valid))
        elif k == DECIMAL:
            v = rng.integers(-5000, 5000, rows) if small else rng.integers(-(1 << 62), 1 << 62, rows)
            b.cols.append(HostBatch.col_dec(v.astype(np.int64), 11, 2, valid))
        elif k == FLOAT64:
            b.cols.append(HostBatch.col_f64(np.round(rng.normal(0, 10, rows), 3), valid))
        elif k == BOOL:
            b.cols.append(HostBatch.col_bool(rng.random(rows) < 0.5, valid))
    if utf8:
        words = ["", "a", "bb", "ccc", "hello", "wörld"]
        b.cols.append(HostBatch.col_utf8([words[i] for i in rng.integers(0, len(words), rows)],
                                         rand_valid(rng, rows, null_frac)))
    return b


def rand_numeric_expr(r: random.Random, kinds, depth: int):
    """Random numeric expression over columns of `kinds` (no bool/utf8)."""
    num_cols = [i for i, k in enumerate(kinds) if k in (INT64, DECIMAL, FLOAT64)]
    if depth <= 0 or r.random() < 0.3:
        x = r.random()
        if x < 0.6:
            return Col(r.choice(num_cols))
        if x < 0.75:
            return Lit(r.randint(-10, 10))
        if x < 0.9:
            return Dec(r.randint(-500, 500), r.choice([0, 1, 2, 3]))
        if x < 0.95:
            return Lit(float(r.randint(-4, 4)) / 2.0, FLOAT64)
        return Null(r.choice([INT64, DECIMAL]), 2)
    op = r.choice([ADD, SUB, MUL])
    return Arith(op, rand_numeric_expr(r, kinds, depth - 1), rand_numeric_expr(r, kinds, depth - 1))


def rand_pred(r: random.Random, kinds, depth: int):
    bool_cols = [i for i, k in enumerate(kinds) if k == BOOL]
    if depth <= 0 or r.random() < 0.35:
        if bool_cols and r.random() < 0.2:
            return Col(r.choice(bool_cols))
        op = r.choice(["<", "<=", "=", "!=", ">=", ">"])
        return Cmp(op, rand_numeric_expr(r, kinds, 1), rand_numeric_expr(r, kinds, 1))
    x = r.random()
    if x < 0.4:
        return And(rand_pred(r, kinds, depth - 1), rand_pred(r, kinds, depth - 1))
    if x < 0.75:
        return Or(rand_pred(r, kinds, depth - 1), rand_pred(r, kinds, depth - 1))
    return Not(rand_pred(r, kinds, depth - 1))
