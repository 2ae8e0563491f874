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


_Q1_SCAN_PRED = remap(Q1_PRED, Q1_SCAN)
_Q1_SCAN_EXPRS = [remap(e, Q1_SCAN) for e in Q1_EXPRS]
_Q1_PARTIAL_AGGS = [(AGG_SUM, 2), (AGG_SUM, 3), (AGG_SUM, 5), (AGG_SUM, 6), (AGG_SUM, 4), (AGG_COUNT_STAR, 0)]
_Q6_SCAN_PRED = remap(Q6_PRED, Q6_SCAN)
_Q6_SCAN_EXPRS = [remap(e, Q6_SCAN) for e in Q6_EXPRS]


def q1_scan(ctx, scan, stream=None, partial=False):
    """Q1 over the pushed-down 7-column scan batch.  partial=True returns the
    mergeable per-worker state (sums + counts) used for multi-GPU Q1."""
    return ctx.pipeline_aggregate(scan, _Q1_SCAN_PRED, _Q1_SCAN_EXPRS, Q1_KEYS,
                                  _Q1_PARTIAL_AGGS if partial else Q1_AGGS, stream)


def q6_scan(ctx, scan, stream=None):
    return ctx.pipeline_aggregate(scan, _Q6_SCAN_PRED, _Q6_SCAN_EXPRS, [], Q6_AGGS, stream)


# ---------------------------------------------------------------- join queries
C_CUSTKEY, C_NATIONKEY, C_MKTSEGMENT = range(3)
S_SUPPKEY, S_NATIONKEY = range(2)
P_PARTKEY, P_COLOR = range(2)
PS_PARTKEY, PS_SUPPKEY, PS_SUPPLYCOST = range(3)
N_NATIONKEY, N_REGIONKEY = range(2)
R_REGIONKEY, R_NAME = range(2)
REV = Col(L_EXTPRICE) * (Dec(100) - Col(L_DISCOUNT))


def q3(ctx, customer, orders, lineitem):
    """Q3-style: customer(BUILDING) >< orders(< 1995-03-15) >< lineitem(> 1995-03-15), group by
    (l_orderkey, o_orderdate, o_shippriority) sum(revenue)."""
    # customer contributes no columns: the build side of a semi-join
    ct = ctx.pipeline_build(customer, Col(C_MKTSEGMENT).eq(1), [C_CUSTKEY], semi=True)
    of = ctx.pipeline_probe(ct, orders, Col(O_ORDERDATE) < 9204,
                            [Col(O_ORDERKEY), Col(O_ORDERDATE), Col(O_SHIPPRIORITY), Col(O_CUSTKEY)], [3], [])
    ot = ctx.join_build(of, [0])
    j = ctx.pipeline_probe(ot, lineitem, Col(L_SHIPDATE) > 9204, [Col(L_ORDERKEY), REV], [0], [1, 2])
    # j: [o_orderdate, o_shippriority, l_orderkey, rev]
    out = ctx.aggregate_execute(j, [2, 0, 1], [(AGG_SUM, 3)])
    for t in (ct, ot):
        t.free()
    return out


def q5(ctx, region, nation, customer, orders, lineitem, supplier):
    """Q5-style: ASIA nations, local supplier revenue per nation (1994)."""
    rt = ctx.pipeline_build(region, Col(R_NAME).eq(2), [R_REGIONKEY], semi=True)  # semi-joins: no build columns
    nf = ctx.pipeline_probe(rt, nation, None, [Col(N_NATIONKEY), Col(N_REGIONKEY)], [1], [])
    nt = ctx.join_build(nf, [0], semi=True)
    cf = ctx.pipeline_probe(nt, customer, None, [Col(C_CUSTKEY), Col(C_NATIONKEY)], [1], [])
    ct = ctx.join_build(cf, [0])
    of = ctx.pipeline_probe(ct, orders, (Col(O_ORDERDATE) >= 8766) & (Col(O_ORDERDATE) < 9131),
                            [Col(O_ORDERKEY), Col(O_CUSTKEY)], [1], [1])  # [c_nationkey, o_orderkey, o_custkey]
    ot = ctx.join_build(of, [1])
    lj = ctx.pipeline_probe(ot, lineitem, None, [Col(L_ORDERKEY), Col(L_SUPPKEY), REV], [0], [0])
    # lj: [c_nationkey, l_orderkey, l_suppkey, rev]
    st = ctx.join_build(supplier, [S_SUPPKEY, S_NATIONKEY])
    sj = ctx.pipeline_probe(st, lj, None, None, [2, 0], [S_NATIONKEY])
    # sj: [s_nationkey, c_nationkey, l_orderkey, l_suppkey, rev]
    out = ctx.aggregate_execute(sj, [0], [(AGG_SUM, 4)])
    for t in (rt, nt, ct, ot, st):
        t.free()
    return out


def q9(ctx, part, partsupp, lineitem, supplier, orders):
    """Q9-style: profit of 'green' parts per (nation, year)."""
    pt = ctx.pipeline_build(part, Col(P_COLOR) < 54, [P_PARTKEY], semi=True)  # semi-join: no part columns
    psf = ctx.pipeline_probe(pt, partsupp, None, None, [PS_PARTKEY], [])
    pst = ctx.join_build(psf, [PS_PARTKEY, PS_SUPPKEY])
    lj = ctx.pipeline_probe(pst, lineitem, None,
                            [Col(L_ORDERKEY), Col(L_PARTKEY), Col(L_SUPPKEY), Col(L_QUANTITY), Col(L_EXTPRICE),
                             Col(L_DISCOUNT)], [1, 2], [PS_SUPPLYCOST])
    # lj: [ps_supplycost, l_orderkey, l_partkey, l_suppkey, qty, ep, disc]
    st = ctx.join_build(supplier, [S_SUPPKEY])
    sj = ctx.pipeline_probe(st, lj, None, None, [3], [S_NATIONKEY])
    # sj: [s_nationkey, ps_supplycost, l_orderkey, l_partkey, l_suppkey, qty, ep, disc]
    ot = ctx.join_build(orders, [O_ORDERKEY])
    amt = Col(6) * (Dec(100) - Col(7)) - Col(1) * Col(5)
    oj = ctx.pipeline_probe(ot, sj, None, [Col(0), amt, Col(2)], [2], [O_YEAR])
    # oj: [o_year, s_nationkey, amt, l_orderkey]
    out = ctx.aggregate_execute(oj, [1, 0], [(AGG_SUM, 2)])
    for t in (pt, pst, st, ot):
        t.free()
    return out


QUERY_TABLES = {3: ["customer", "orders", "lineitem"],
                5: ["region", "nation", "customer", "orders", "lineitem", "supplier"],
                9: ["part", "partsupp", "lineitem", "supplier", "orders"]}
TABLE_IDS = {"orders": 0, "lineitem": 1, "customer": 2, "supplier": 3, "part": 4, "partsupp": 5, "nation": 6,
             "region": 7}


def run_join_query(ctx, q: int, tables: dict):
    args = [tables[n] for n in QUERY_TABLES[q]]
    return {3: q3, 5: q5, 9: q9}[q](ctx, *args)


# ---------------------------------------------------------------- distributed (one rank per GPU)
def q3_distributed(ctx, comm, customer, orders, lineitem, stats=None, lip=True, fused=False):
    """Config 4: Q3-style shuffle join over each rank's row-group subset.
    customer_f is broadcast (exchange_decide: 24 MB <= 16 MiB x N at SF100),
    orders_f and lineitem_f are hash-partitioned on orderkey (fnv1a64 mod N)
    and exchanged all-to-all over NVLink; the build/probe/aggregate that
    follows is co-partitioned, so each rank's groups are final.
    lip=True adds Lookahead Information Passing: a Bloom filter
    of the orders_f keys drops lineitem rows that cannot join before they are
    partitioned and shipped (same result).  Unfused: one filter of each rank's
    local orders_f, OR-ed across ranks.  Fused: the all-gathered Bloom filters
    of the ranks' (already shuffled) orders_f join tables, one part per rank.
    fused=True replaces each partition + all-to-all pair with the fused
    partition/scatter over NVLink peer memory (tq_pipeline_partition_exchange):
    rows are written once, straight into their destination rank's window."""
    n = comm.n
    if fused:  # filter + broadcast in one kernel over NVLink peer memory
        cf = cb = comm.broadcast(customer, Col(C_MKTSEGMENT).eq(1), [Col(C_CUSTKEY)])
    else:
        cf = ctx.pipeline_materialize(customer, Col(C_MKTSEGMENT).eq(1), [Col(C_CUSTKEY)])
        cb, _ = comm.allgather(cf)
    ct = ctx.join_build(cb, [0], semi=True)  # customer contributes no columns: a semi-join build
    of = ctx.pipeline_probe(ct, orders, Col(O_ORDERDATE) < 9204,
                            [Col(O_ORDERKEY), Col(O_ORDERDATE), Col(O_SHIPPRIORITY), Col(O_CUSTKEY)], [3], [])
    bloom = None
    ot = None
    if fused:
        # orders_f is shuffled first; each rank's orders_f table carries a Bloom
        # filter of its partition (sized from the window capacity every rank
        # agrees on), and the all-gathered filters are the LIP filter of the
        # lineitem shuffle: a row is checked against its destination's part
        orx = comm.partition_exchange(of, None, None, [0])
        ot = ctx.join_build(orx, [0], bloom_keys=comm.last_exchange_capacity())
        if lip:
            bloom = comm.gather_table_blooms(ot)
        lrx = comm.partition_exchange(lineitem, Col(L_SHIPDATE) > 9204, [Col(L_ORDERKEY), REV], [0], bloom)
        lp = lrx
    else:
        if lip:
            bloom = ctx.bloom_build(of, [0], expected_keys=of.rows * n)
            comm.bloom_union(bloom)
        op, ooff = ctx.hash_partition(of, [0], n)
        orx, _ = comm.exchange(op, ooff)
        if lip:
            lp, loff = ctx.pipeline_partition_semi(lineitem, Col(L_SHIPDATE) > 9204, [Col(L_ORDERKEY), REV], [0], n,
                                                   bloom)
        else:
            lp, loff = ctx.pipeline_partition(lineitem, Col(L_SHIPDATE) > 9204, [Col(L_ORDERKEY), REV], [0], n)
        lrx, _ = comm.exchange(lp, loff)
        ot = ctx.join_build(orx, [0])
    j = ctx.pipeline_probe(ot, lrx, None, None, [0], [1, 2])
    out = ctx.aggregate_execute(j, [2, 0, 1], [(AGG_SUM, 3)])
    if stats is not None:
        stats.update({"orders_f_rows": of.rows, "lineitem_shipped_rows": None if fused else lp.rows,
                      "recv_orders": orx.rows, "recv_lineitem": lrx.rows, "lip": lip, "fused": fused})
    for t in (ct, ot):
        t.free()
    if bloom is not None:
        bloom.free()
    return out
