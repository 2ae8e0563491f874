"""Expr trees and their prefix serialization (tq_expr_node[]).

    Expr := ColumnRef(index) | Literal(value) | Compare(op, a, b)
          | Arith(op, a, b) | And(a, b) | Or(a, b) | Not(a)

Null rule: any null operand -> null; a null predicate filters the row out.
Typing/promotion rules are recorded in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from typing import Optional, Tuple

from .columnar import BOOL, DECIMAL, FLOAT64, INT64, TqExprC, TqExprNodeC

EX_COL, EX_LIT, EX_CMP, EX_ARITH, EX_AND, EX_OR, EX_NOT = range(7)
LT, LE, EQ, NE, GE, GT = range(6)
ADD, SUB, MUL = range(3)
CMP_NAMES = {"<": LT, "<=": LE, "=": EQ, "==": EQ, "!=": NE, ">=": GE, ">": GT}
ARITH_NAMES = {"+": ADD, "-": SUB, "*": MUL}


@dataclass(frozen=True)
class Expr:
    tag: int
    op: int = 0
    children: Tuple["Expr", ...] = ()
    column: int = 0
    kind: int = INT64
    scale: int = 0
    is_null: bool = False
    value: object = 0  # int / float / bool

    # operator sugar
    def __lt__(self, o): return Cmp("<", self, _lift(o))
    def __le__(self, o): return Cmp("<=", self, _lift(o))
    def __gt__(self, o): return Cmp(">", self, _lift(o))
    def __ge__(self, o): return Cmp(">=", self, _lift(o))
    def eq(self, o): return Cmp("=", self, _lift(o))
    def ne(self, o): return Cmp("!=", self, _lift(o))
    def __add__(self, o): return Arith("+", self, _lift(o))
    def __sub__(self, o): return Arith("-", self, _lift(o))
    def __mul__(self, o): return Arith("*", self, _lift(o))
    def __and__(self, o): return And(self, o)
    def __or__(self, o): return Or(self, o)
    def __invert__(self): return Not(self)

    def nodes(self):
        yield self
        for c in self.children:
            yield from c.nodes()

    def serialize(self) -> "SerializedExpr":
        ns = list(self.nodes())
        arr = (TqExprNodeC * len(ns))()
        for i, n in enumerate(ns):
            a = arr[i]
            a.tag, a.op, a.kind, a.scale, a.is_null, a.column = n.tag, n.op, n.kind, n.scale, int(n.is_null), n.column
            if n.tag == EX_LIT and not n.is_null:
                if n.kind == FLOAT64:
                    a.lo = struct.unpack("<Q", struct.pack("<d", float(n.value)))[0]
                elif n.kind == BOOL:
                    a.lo = 1 if n.value else 0
                else:
                    v = int(n.value) & ((1 << 128) - 1)
                    a.lo = v & 0xFFFFFFFFFFFFFFFF
                    a.hi = v >> 64 if n.kind == DECIMAL else 0
        return SerializedExpr(arr, len(ns))


class SerializedExpr:
    def __init__(self, arr, n):
        self.arr = arr
        self.n = n

    def c(self) -> TqExprC:
        return TqExprC(C.cast(self.arr, C.POINTER(TqExprNodeC)), self.n, 0)


def _lift(o) -> Expr:
    if isinstance(o, Expr):
        return o
    if isinstance(o, bool):
        return Lit(o, BOOL)
    if isinstance(o, int):
        return Lit(o, INT64)
    if isinstance(o, float):
        return Lit(o, FLOAT64)
    raise TypeError(o)


def Col(i: int) -> Expr:
    return Expr(EX_COL, column=i)


def Lit(v, kind: int = INT64, scale: int = 0) -> Expr:
    return Expr(EX_LIT, kind=kind, scale=scale, value=v)


def Dec(v: int, scale: int = 2) -> Expr:
    """Decimal literal given as the scaled integer (Dec(100, 2) == 1.00)."""
    return Expr(EX_LIT, kind=DECIMAL, scale=scale, value=v)


def Null(kind: int = INT64, scale: int = 0) -> Expr:
    return Expr(EX_LIT, kind=kind, scale=scale, is_null=True)


def Cmp(op, a: Expr, b: Expr) -> Expr:
    return Expr(EX_CMP, op=CMP_NAMES[op] if isinstance(op, str) else op, children=(a, b))


def Arith(op, a: Expr, b: Expr) -> Expr:
    return Expr(EX_ARITH, op=ARITH_NAMES[op] if isinstance(op, str) else op, children=(a, b))


def And(a: Expr, b: Expr) -> Expr:
    return Expr(EX_AND, children=(a, b))


def Or(a: Expr, b: Expr) -> Expr:
    return Expr(EX_OR, children=(a, b))


def Not(a: Expr) -> Expr:
    return Expr(EX_NOT, children=(a,))


def all_of(*es: Expr) -> Optional[Expr]:
    out = None
    for e in es:
        out = e if out is None else And(out, e)
    return out
