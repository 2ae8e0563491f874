"""The benchmark query DAGs expressed over the fused
pipeline entry points of the C-ABI.  Plans match oracle/tq_oracle.cpp's
query() operator for operator; decimal literals are scaled integers at
scale 2 (Dec(100) == 1.00)."""
from __future__ import annotations

from .expr import Col, Dec, Lit, all_of

# lineitem columns
L_ORDERKEY, L_PARTKEY, L_SUPPKEY, L_QUANTITY, L_EXTPRICE, L_DISCOUNT, L_TAX, L_RETURNFLAG, L_LINESTATUS, \
    L_SHIPDATE = range(10)
O_ORDERKEY, O_CUSTKEY, O_ORDERDATE, O_SHIPPRIORITY, O_YEAR = range(5)
AGG_SUM, AGG_COUNT, AGG_COUNT_STAR, AGG_MIN, AGG_MAX, AGG_AVG = range(6)

# Q6: sum(ep * disc) where 1994-01-01 <= shipdate < 1995-01-01, disc in [.05,.07], qty < 24
Q6_PRED = (((Col(L_SHIPDATE) >= 8766) & (Col(L_SHIPDATE) < 9131)) &
           (((Col(L_DISCOUNT) >= Dec(5)) & (Col(L_DISCOUNT) <= Dec(7))) & (Col(L_QUANTITY) < Dec(2400))))
Q6_EXPRS = [Col(L_EXTPRICE) * Col(L_DISCOUNT)]
Q6_AGGS = [(AGG_SUM, 0)]

# Q1: group by returnflag, linestatus where shipdate <= 1998-09-02
Q1_PRED = Col(L_SHIPDATE) <= 10471
_DP = Col(L_EXTPRICE) * (Dec(100) - Col(L_DISCOUNT))
Q1_EXPRS = [Col(L_RETURNFLAG), Col(L_LINESTATUS), Col(L_QUANTITY), Col(L_EXTPRICE), Col(L_DISCOUNT), _DP,
            _DP * (Dec(100) + Col(L_TAX))]
Q1_KEYS = [0, 1]
Q1_AGGS = [(AGG_SUM, 2), (AGG_SUM, 3), (AGG_SUM, 5), (AGG_SUM, 6), (AGG_AVG, 2), (AGG_AVG, 3), (AGG_AVG, 4),
           (AGG_COUNT_STAR, 0)]

# bytes of lineitem each query's scan reads (columns referenced x width)
Q1_SCAN_BYTES_PER_ROW = 8 + 8 + 16 + 16 + 16 + 16 + 8   # rf, ls, qty, ep, disc, tax, shipdate
Q6_SCAN_BYTES_PER_ROW = 8 + 16 + 16 + 16                # shipdate, qty, ep, disc


def q6(ctx, lineitem, stream=None):
    return ctx.pipeline_aggregate(lineitem, Q6_PRED, Q6_EXPRS, [], Q6_AGGS, stream)


def q1(ctx, lineitem, stream=None):
    return ctx.pipeline_aggregate(lineitem, Q1_PRED, Q1_EXPRS, Q1_KEYS, Q1_AGGS, stream)


# Scan projection pushdown: the columns of lineitem each query reads, and the
# same plans re-indexed over that narrower batch (what a columnar scan loads).
Q1_SCAN = [L_RETURNFLAG, L_LINESTATUS, L_QUANTITY, L_EXTPRICE, L_DISCOUNT, L_TAX, L_SHIPDATE]
Q6_SCAN = [L_SHIPDATE, L_QUANTITY, L_EXTPRICE, L_DISCOUNT]


def remap(e, cols):
    """Rewrite ColumnRef(i) -> ColumnRef(cols.index(i))."""
    from dataclasses import replace
    from .expr import EX_COL
    if e.tag == EX_COL:
        return replace(e, column=cols.index(e.column))
    return replace(e, children=tuple(remap(c, cols) for c in e.children))


def q1_scan(ctx, scan, stream=None, partial=False):
    """Q1 over the pushed-down 7-column scan batch.  partial=True returns the
    mergeable per-worker state (sums + counts) used for multi-GPU Q1."""
    aggs = Q1_AGGS if not partial else [(AGG_SUM, 2), (AGG_SUM, 3), (AGG_SUM, 5), (AGG_SUM, 6), (AGG_SUM, 4),
                                         (AGG_COUNT_STAR, 0)]
    return ctx.pipeline_aggregate(scan, remap(Q1_PRED, Q1_SCAN), [remap(e, Q1_SCAN) for e in Q1_EXPRS], Q1_KEYS,
                                  aggs, stream)


def q6_scan(ctx, scan, stream=None):
    return ctx.pipeline_aggregate(scan, remap(Q6_PRED, Q6_SCAN), [remap(e, Q6_SCAN) for e in Q6_EXPRS], [], Q6_AGGS,
                                  stream)
