"""GPU parity: every operator through the C-ABI (libtq_gpu.so, sm_100a) vs the
CPU oracle on the same seeded inputs.  Integer / decimal / bool / row-set
results bit-exact after canonical sort; Float64 within 1e-9 relative."""
import random

import numpy as np
import pytest

import oracle as O
import rowloop
from helpers import rand_batch, rand_numeric_expr, rand_pred
from paper_2508_05029_b200.columnar import (BOOL, DECIMAL, FLOAT64, INT64, HostBatch, assert_batches_equal)
from paper_2508_05029_b200.expr import Col, Dec, Lit, Null, all_of

pytestmark = pytest.mark.gpu
AGG_SUM, AGG_COUNT, AGG_COUNT_STAR, AGG_MIN, AGG_MAX, AGG_AVG = range(6)


@pytest.fixture(scope="module", params=["jit", "interp"])
def ctx(request):
    """Every parity test runs twice: NVRTC-specialised kernels and the AOT
    interpreter kernels (the same skeleton, two program policies)."""
    from paper_2508_05029_b200.ops import Context
    c = Context(0)
    c.set_jit(request.param == "jit")
    yield c
    if request.param == "jit":
        rep = c.jit_report()
        assert int(rep["failed"]) == 0, rep
        assert int(rep["jit_launches"]) > 0, rep
    c.close()


def test_roundtrip(ctx):
    b = rand_batch(1, 1000, null_frac=0.2)
    got = ctx.upload(b).to_host()
    assert_batches_equal(got, b, ordered=True)


@pytest.mark.parametrize("t", range(8))
def test_datagen_bit_identical(ctx, t):
    sf = 0.01
    g = ctx.datagen(t, sf).to_host()
    want = O.datagen(t, sf)
    assert_batches_equal(g, want, ordered=True)


def test_spec_examples(ctx):
    b = ctx.upload(HostBatch(4, [HostBatch.col_i64([1, 7, 3, 0], [True, True, True, False])]))
    assert ctx.filter_execute(b, Col(0) < 5).to_host().column_py(0) == [1, 3]
    assert ctx.filter_execute(b, Lit(True, BOOL)).to_host().column_py(0) == [1, 7, 3, None]
    a = ctx.upload(HostBatch(4, [HostBatch.col_i64([9, 9, 9, 1]), HostBatch.col_i64([1, 2, 3, 4])]))
    p = ctx.upload(HostBatch(3, [HostBatch.col_i64([9, 2, 9])]))
    assert ctx.join_execute(a, p, [0], [0]).rows == 6
    one = ctx.upload(HostBatch(5, [HostBatch.col_i64([3] * 5)]))
    assert ctx.aggregate_execute(one, [0], [(AGG_COUNT_STAR, 0)]).to_host().to_rows() == [(3, 5)]
    empty = ctx.upload(HostBatch(0, [HostBatch.col_i64([])]))
    assert ctx.aggregate_execute(empty, [0], [(AGG_COUNT_STAR, 0)]).rows == 0
    same = ctx.upload(HostBatch(50, [HostBatch.col_i64([7] * 50), HostBatch.col_i64(list(range(50)))]))
    _, offs = ctx.hash_partition(same, [0], 8)
    sizes = np.diff(offs)
    assert (sizes > 0).sum() == 1 and sizes.sum() == 50


@pytest.mark.parametrize("seed", range(24))
def test_filter_parity(ctx, seed):
    kinds = (INT64, DECIMAL, FLOAT64, BOOL, INT64)
    rows = [0, 1, 31, 513, 4000, 20000][seed % 6]
    b = rand_batch(seed, rows, kinds, null_frac=0.1 if seed % 3 else 0.0)
    pred = rand_pred(random.Random(seed), kinds, 3)
    got = ctx.filter_execute(ctx.upload(b), pred).to_host()
    want = O.filter_execute(b, pred)
    assert_batches_equal(got, want, ordered=True)
    if rows <= 600:
        assert_batches_equal(got, O.take(b, rowloop.filter_rows(b, pred)), ordered=True)


@pytest.mark.parametrize("seed", range(24))
def test_project_parity(ctx, seed):
    kinds = (INT64, DECIMAL, FLOAT64, BOOL, DECIMAL)
    rows = [1, 100, 512, 3333][seed % 4]
    b = rand_batch(seed, rows, kinds, null_frac=0.1, small=seed % 3 != 0)
    r = random.Random(seed)
    exprs = [rand_numeric_expr(r, kinds, 3) for _ in range(3)] + [rand_pred(r, kinds, 2), Col(1), Col(3)]
    got = ctx.project_execute(ctx.upload(b), exprs).to_host()
    want = O.project_execute(b, exprs)
    assert_batches_equal(got, want, ordered=True)


@pytest.mark.parametrize("seed", range(8))
def test_partition_parity(ctx, seed):
    b = rand_batch(seed, [10, 700, 5000, 70000][seed % 4], (INT64, DECIMAL, BOOL, FLOAT64), null_frac=0.05)
    keys = [[0], [1], [0, 1], [2]][seed % 4]
    n = [1, 2, 4, 8, 3, 16, 64, 7][seed]
    d, offs = ctx.hash_partition(ctx.upload(b), keys, n)
    got = d.to_host()
    want = O.hash_partition(b, keys, n)
    assert offs[-1] == b.rows
    for p in range(n):
        part = O.slice_(got, offs[p], offs[p + 1] - offs[p])
        assert_batches_equal(part, want[p], ordered=True)  # stable within a part


@pytest.mark.parametrize("seed", range(10))
def test_join_parity(ctx, seed):
    a = rand_batch(seed, [5, 300, 2000, 20000, 100][seed % 5], (INT64, DECIMAL, BOOL), null_frac=0.05)
    b = rand_batch(seed + 99, [7, 500, 3000, 30000, 0][seed % 5], (INT64, DECIMAL, FLOAT64), null_frac=0.05)
    rng = np.random.default_rng(seed)
    for x in (a, b):
        x.cols[1] = HostBatch.col_dec(rng.integers(0, 3, x.rows), 11, 2, x.validity_of(1))
    keys = ([0], [0]) if seed % 2 else ([0, 1], [0, 1])
    got = ctx.join_execute(ctx.upload(a), ctx.upload(b), *keys).to_host()
    want = O.join_execute(a, b, *keys)
    assert_batches_equal(got, want)


@pytest.mark.parametrize("dups_probed", [False, True])
def test_probe_unique_then_duplicate_keys(ctx, dups_probed):
    """A probe assumes unique build keys and runs single-pass; a probe key with
    a second build match makes it discard that pass and re-run two-pass (and
    the table remembers it).  Duplicates no probe key reaches keep one pass."""
    rng = np.random.default_rng(7)
    nb = 50000
    bkeys = rng.permutation(np.arange(1, 4 * nb, 4))[:nb].astype(np.int64)  # unique
    bkeys[:20] = bkeys[20:40] if dups_probed else -bkeys[:20]              # 20 duplicated keys / unreachable negatives
    if not dups_probed:
        bkeys[20:40] = bkeys[:20]                                          # duplicates among the negatives
    build = HostBatch(nb, [HostBatch.col_i64(bkeys), HostBatch.col_i64(rng.integers(0, 100, nb))])
    npr = 200000
    probe = HostBatch(npr, [HostBatch.col_i64(rng.integers(0, 4 * nb, npr)), HostBatch.col_dec(rng.integers(0, 999, npr))])
    want = O.join_execute(build, probe, [0], [0])
    t = ctx.join_build(ctx.upload(build), [0])
    dp = ctx.upload(probe)
    for _ in range(2):  # the second probe reuses the table (and its uniqueness hint)
        assert_batches_equal(ctx.join_probe(t, dp, [0]).to_host(), want)
    t.free()


@pytest.mark.parametrize("out_of_range", [False, True])
def test_probe_exact_bitmap_semi_join(ctx, out_of_range):
    """Dense one-word build keys get an exact membership bitmap (no Bloom false
    positives); a semi-join probe (no build columns) over proven-unique keys
    then never reads the table.  A key outside [0, 32 x words) disables it."""
    from paper_2508_05029_b200.expr import Col
    rng = np.random.default_rng(11)
    nb = 30000
    bkeys = rng.permutation(np.arange(0, 4 * nb))[:nb].astype(np.int64)
    if out_of_range:
        bkeys[7] = -5
        bkeys[9] = 1 << 40
    build = HostBatch(nb, [HostBatch.col_i64(bkeys), HostBatch.col_i64(rng.integers(0, 100, nb))])
    npr = 100000
    pk = rng.integers(-100, 4 * nb + 100, npr).astype(np.int64)
    pk[:3] = [-5, 1 << 40, 4 * nb]
    probe = HostBatch(npr, [HostBatch.col_i64(pk), HostBatch.col_i64(rng.integers(0, 50, npr))])
    t = ctx.join_build(ctx.upload(build), [0])
    dp = ctx.upload(probe)
    semi = ctx.pipeline_probe(t, dp, Col(1) < 40, [Col(0), Col(1)], [0], []).to_host()
    keys = set(bkeys.tolist())
    want = [(int(k), int(v)) for k, v in zip(pk, probe.cols[1].values.view(np.int64)) if v < 40 and int(k) in keys]
    assert sorted(semi.to_rows()) == sorted(want)
    full = ctx.join_probe(t, dp, [0]).to_host()  # with build columns: the table is read
    assert_batches_equal(full, O.join_execute(build, probe, [0], [0]))
    t.free()


@pytest.mark.parametrize("case", ["unique", "duplicates", "out_of_range"])
def test_semi_join_build(ctx, case):
    """tq_join_build_semi: dense unique keys -> bitmap only (no hash table);
    duplicate or out-of-range keys -> falls back to a real table.  Either way
    the (inner-join) result equals the oracle's."""
    from paper_2508_05029_b200.columnar import TqError
    from paper_2508_05029_b200.expr import Col
    rng = np.random.default_rng(3)
    nb = 20000
    bkeys = rng.permutation(np.arange(1, 3 * nb))[:nb].astype(np.int64)
    if case == "duplicates":
        bkeys[100:110] = bkeys[200:210]
    if case == "out_of_range":
        bkeys[5] = -3
    build = HostBatch(nb, [HostBatch.col_i64(bkeys)])
    npr = 80000
    probe = HostBatch(npr, [HostBatch.col_i64(rng.integers(-10, 3 * nb + 10, npr)),
                            HostBatch.col_dec(rng.integers(0, 999, npr))])
    t = ctx.join_build(ctx.upload(build), [0], semi=True)
    got = ctx.pipeline_probe(t, ctx.upload(probe), None, [Col(0), Col(1)], [0], []).to_host()
    want = O.join_execute(build, probe, [0], [0])  # build key column first, then probe columns
    want = HostBatch(want.rows, want.cols[1:])
    assert_batches_equal(got, want)
    if case == "unique":  # a semi-only table cannot hand out build columns
        with pytest.raises(TqError):
            ctx.pipeline_probe(t, ctx.upload(probe), None, [Col(0)], [0], [0])
    t.free()


@pytest.mark.parametrize("seed", range(12))
def test_aggregate_parity(ctx, seed):
    kinds = (INT64, DECIMAL, FLOAT64, BOOL, INT64)
    rows = [0, 10, 1000, 20000, 100000, 777][seed % 6]
    b = rand_batch(seed, rows, kinds, null_frac=0.1 if seed % 2 else 0.0, small=seed % 5 != 4)
    keys = [[0], [3], [0, 3], [], [1, 4], [0, 1, 3]][seed % 6]
    aggs = [(AGG_SUM, 1), (AGG_SUM, 0), (AGG_SUM, 2), (AGG_COUNT, 1), (AGG_COUNT_STAR, 0), (AGG_MIN, 1),
            (AGG_MAX, 2), (AGG_AVG, 1), (AGG_AVG, 0), (AGG_MIN, 3), (AGG_MAX, 0), (AGG_AVG, 2)]
    got = ctx.aggregate_execute(ctx.upload(b), keys, aggs).to_host()
    want = O.aggregate_execute(b, keys, aggs)
    assert_batches_equal(got, want)


def test_aggregate_many_groups(ctx):
    """More groups than the per-CTA table: exercises the global table + regrowth."""
    rng = np.random.default_rng(5)
    n = 400000
    b = HostBatch(n, [HostBatch.col_i64(rng.integers(0, 150000, n)), HostBatch.col_dec(rng.integers(0, 10**9, n))])
    aggs = [(AGG_SUM, 1), (AGG_COUNT_STAR, 0), (AGG_MAX, 1)]
    got = ctx.aggregate_execute(ctx.upload(b), [0], aggs).to_host()
    want = O.aggregate_execute(b, [0], aggs)
    assert_batches_equal(got, want)


@pytest.mark.parametrize("seed", range(3))
def test_aggregate_mixed_magnitudes(ctx, seed):
    """Mostly small sums with rare values beyond 2^46 in the same groups: the
    per-lane 64-bit planes take the small ones, the large ones go to the
    global int128 table; sums must still be exact (and wrap like the oracle)."""
    rng = np.random.default_rng(100 + seed)
    n = 300000
    big = rng.random(n) < 0.01
    iv = np.where(big, rng.integers(-(1 << 62), 1 << 62, n), rng.integers(-1000, 1000, n))
    dv = np.where(big, rng.integers(-(1 << 62), 1 << 62, n), rng.integers(-10**6, 10**6, n))
    b = HostBatch(n, [HostBatch.col_i64(rng.integers(0, 6, n)), HostBatch.col_i64(iv),
                      HostBatch.col_dec(dv.astype(np.int64), 11, 2)])
    aggs = [(AGG_SUM, 1), (AGG_SUM, 2), (AGG_COUNT_STAR, 0), (AGG_AVG, 2), (AGG_MIN, 2), (AGG_MAX, 1)]
    got = ctx.aggregate_execute(ctx.upload(b), [0], aggs).to_host()
    want = O.aggregate_execute(b, [0], aggs)
    assert_batches_equal(got, want)


@pytest.mark.parametrize("seed", range(6))
def test_take_concat_slice_parity(ctx, seed):
    rng = np.random.default_rng(seed)
    b = rand_batch(seed, int(rng.integers(1, 3000)), (INT64, DECIMAL, BOOL, FLOAT64),
                   null_frac=0.2 if seed % 2 else 0.0, utf8=True)
    d = ctx.upload(b)
    ids = rng.integers(0, b.rows, int(rng.integers(0, 5000))).tolist()
    assert_batches_equal(ctx.take(d, ids).to_host(), O.take(b, ids), ordered=True)
    b2 = rand_batch(seed + 7, int(rng.integers(0, 100)), (INT64, DECIMAL, BOOL, FLOAT64), null_frac=0.0, utf8=True)
    d2 = ctx.upload(b2)
    got = ctx.concat([d, d2, d]).to_host()
    want = O.concat([b, b2, b])
    assert_batches_equal(got, want, ordered=True)
    assert [c.validity is not None for c in got.cols] == [c.validity is not None for c in want.cols]
    s = int(rng.integers(0, b.rows))
    n = int(rng.integers(0, b.rows - s + 1))
    assert_batches_equal(ctx.slice(d, s, n).to_host(), O.slice_(b, s, n), ordered=True)


def test_invalid_plan_errors(ctx):
    from paper_2508_05029_b200.columnar import TqError
    b = ctx.upload(HostBatch(3, [HostBatch.col_i64([1, 2, 3])]))
    with pytest.raises(TqError) as e:
        ctx.filter_execute(b, Col(5) < 1)
    assert e.value.errc == "InvalidPlan"
    with pytest.raises(TqError) as e:
        ctx.filter_execute(b, Col(0) + 1)  # non-bool predicate
    assert e.value.errc == "InvalidPlan"


@pytest.mark.parametrize("q", ["q1", "q6"])
def test_query_pipelines(ctx, q):
    """Fused Filter->Project->Aggregate pipelines vs the
    oracle's operator-by-operator DAG, full-width and scan-pushed-down."""
    from paper_2508_05029_b200 import queries
    sf = 0.05
    li = ctx.datagen(O.T_LINEITEM, sf)
    want = O.query(int(q[1]), {O.T_LINEITEM: O.datagen(O.T_LINEITEM, sf)}, 4)
    full = getattr(queries, q)(ctx, li).to_host()
    assert_batches_equal(full, want)
    scan = li.select(queries.Q1_SCAN if q == "q1" else queries.Q6_SCAN)
    pushed = getattr(queries, q + "_scan")(ctx, scan).to_host()
    assert_batches_equal(pushed, want)


@pytest.mark.parametrize("q", [3, 5, 9])
def test_join_queries(ctx, q):
    """Multi-join DAGs (build/probe pipelines + aggregate) vs the oracle."""
    from paper_2508_05029_b200 import queries
    sf = 0.05
    names = queries.QUERY_TABLES[q]
    dev = {n: ctx.datagen(queries.TABLE_IDS[n], sf) for n in names}
    got = queries.run_join_query(ctx, q, dev).to_host()
    host = {queries.TABLE_IDS[n]: O.datagen(queries.TABLE_IDS[n], sf) for n in names}
    want = O.query(q, host, 4)
    assert want.rows > 0
    assert_batches_equal(got, want)


@pytest.mark.parametrize("seed", range(6))
def test_streaming_aggregate_state(ctx, seed):
    """tq_agg_update over row-group slices + tq_agg_finalize == one aggregate."""
    kinds = (INT64, DECIMAL, FLOAT64, BOOL, INT64)
    b = rand_batch(seed, 20000, kinds, null_frac=0.1 if seed % 2 else 0.0)
    keys = [[0], [3], [0, 3], [], [1, 4], [0, 1, 3]][seed]
    aggs = [(AGG_SUM, 1), (AGG_SUM, 0), (AGG_SUM, 2), (AGG_COUNT, 1), (AGG_COUNT_STAR, 0), (AGG_MIN, 1),
            (AGG_MAX, 2), (AGG_AVG, 1), (AGG_AVG, 0), (AGG_MIN, 3), (AGG_MAX, 0), (AGG_AVG, 2)]
    d = ctx.upload(b)
    parts = [ctx.slice(d, s, min(3000, b.rows - s)) for s in range(0, b.rows, 3000)]
    got = ctx.agg_stream(parts, None, None, keys, aggs).to_host()
    assert_batches_equal(got, O.aggregate_execute(b, keys, aggs))


@pytest.mark.parametrize("seed", range(3))
def test_partition_semi_bloom(ctx, seed):
    """LIP: partition with a build-side Bloom filter keeps every row whose key
    is in the build set (no false negatives), drops most others, and the join
    result is unchanged."""
    rng = np.random.default_rng(seed)
    build = HostBatch(2000, [HostBatch.col_i64(rng.integers(0, 100000, 2000))])
    probe = HostBatch(50000, [HostBatch.col_i64(rng.integers(0, 100000, 50000)),
                              HostBatch.col_dec(rng.integers(0, 10**6, 50000))])
    db, dp = ctx.upload(build), ctx.upload(probe)
    bloom = ctx.bloom_build(db, [0])
    part, offs = ctx.pipeline_partition_semi(dp, None, None, [0], 4, bloom)
    got = part.to_host()
    keys = set(build.cols[0].i64().tolist())
    kept = got.cols[0].i64().tolist()
    must = [k for k in probe.cols[0].i64().tolist() if k in keys]
    assert set(must) <= set(kept) and len([k for k in kept if k in keys]) == len(must)
    assert len(kept) < 0.2 * probe.rows            # most non-joining rows dropped
    j1 = O.join_execute(build, got, [0], [0])
    assert_batches_equal(j1, O.join_execute(build, probe, [0], [0]))


@pytest.mark.parametrize("distinct", [40, 200000])
def test_aggregate_publication_stress(ctx, distinct):
    """Many lanes insert the same NEW keys at once (every key's first
    occurrences are spread over the whole grid): a reader that observed a
    published slot must compare the keys written before the publication, or
    the same key lands in two slots (duplicate groups).  40 keys stress the
    per-CTA shared-memory table, 200K the global table.  50 repetitions."""
    rng = np.random.default_rng(1234 + distinct)
    n = 2_000_000
    k = rng.integers(0, distinct, n).astype(np.int64) * 7919 + 3
    b = HostBatch(n, [HostBatch.col_i64(k), HostBatch.col_dec(rng.integers(-10**6, 10**6, n))])
    aggs = [(AGG_SUM, 1), (AGG_COUNT_STAR, 0)]
    want = O.aggregate_execute(b, [0], aggs)
    d = ctx.upload(b)
    for _ in range(50):
        got = ctx.aggregate_execute(d, [0], aggs)
        assert got.rows == want.rows  # no key was inserted twice
        got.free()
    assert_batches_equal(ctx.aggregate_execute(d, [0], aggs).to_host(), want)


@pytest.mark.parametrize("t", [0, 1, 2, 5])
def test_datagen_shard_bit_identical(ctx, t):
    """GPU row-group subsets (tq_datagen_shard) == the oracle's shards."""
    sf = 0.02
    for s in (0, 3):
        g = ctx.datagen(t, sf, shard=s, nshards=4).to_host()
        assert_batches_equal(g, O.datagen(t, sf, 4, s, 4), ordered=True)


@pytest.mark.parametrize("case", ["clustered", "shuffled", "nulls", "sparse", "huge"])
def test_aggregate_direct_dense_key(ctx, case):
    """One integer group key over >= 4M rows: a range pass sizes a DIRECT
    table (slot = key - min) when the keys are dense — clustered keys (like
    lineitem by orderkey) are reduced per warp run before one atomic per run;
    a null key gets its own slot; a sparse key range falls back to the hash
    table.  Every path equals the oracle."""
    rng = np.random.default_rng({"clustered": 1, "shuffled": 2, "nulls": 3, "sparse": 4, "huge": 5}[case])
    n = 4_500_000
    if case == "sparse":
        k = rng.integers(0, 1 << 40, n // 8).repeat(8)[:n]
    else:
        k = np.sort(rng.integers(-1000, n // 4, n))
        if case == "shuffled":
            k = rng.permutation(k)
    valid = rng.random(n) >= 0.01 if case == "nulls" else None
    # "huge": runs whose integer sums pass int64 (the direct table's limb
    # form cannot hold them: the aggregate re-runs exactly on the hash table)
    v = rng.integers(1 << 61, 1 << 62, n) if case == "huge" else rng.integers(-10**9, 10**9, n)
    f = rng.integers(-400, 400, n) * 0.25  # exact in binary: float sums do not depend on the order
    b = HostBatch(n, [HostBatch.col_i64(k.astype(np.int64), valid), HostBatch.col_dec(v.astype(np.int64)),
                      HostBatch.col_f64(f, rng.random(n) >= 0.05)])
    aggs = [(AGG_SUM, 1), (AGG_COUNT_STAR, 0), (AGG_MIN, 1), (AGG_MAX, 2), (AGG_AVG, 1), (AGG_SUM, 2),
            (AGG_COUNT, 2), (AGG_MIN, 2)]
    got = ctx.aggregate_execute(ctx.upload(b), [0], aggs).to_host()
    assert_batches_equal(got, O.aggregate_execute(b, [0], aggs))


@pytest.mark.parametrize("case", ["fixed", "utf8", "small", "many_inputs"])
def test_rebatch_matches_reference(ctx, case):
    """tq_rebatch == the reference's rebatch (transform.cpp:122-154): the same
    cut points (row counts from the reference library itself) and the same rows."""
    seed = {"fixed": 1, "utf8": 2, "small": 3, "many_inputs": 4}[case]
    rows = {"fixed": 50000, "utf8": 30000, "small": 100, "many_inputs": 20000}[case]
    b = rand_batch(seed, rows, (INT64, DECIMAL, BOOL), null_frac=0.1, utf8=case == "utf8")
    target = {"fixed": 64 << 10, "utf8": 40 << 10, "small": 1 << 20, "many_inputs": 50 << 10}[case]
    d = ctx.upload(b)
    ins = [ctx.slice(d, s, min(3000, b.rows - s)) for s in range(0, b.rows, 3000)] if case == "many_inputs" else [d]
    parts = ctx.rebatch(ins, target)
    want_rows = O.ref_rebatch_rows(b, target)
    assert [p.rows for p in parts] == want_rows
    at = 0
    for p in parts:
        assert_batches_equal(p.to_host(), O.slice_(b, at, p.rows), ordered=True)
        at += p.rows
    if len(want_rows) > 1:  # every output but the last in [target / 2, 2 * target] bytes
        sizes = [O.ref_batch_size_bytes(O.slice_(b, int(s), n)) for s, n in zip(np.cumsum([0] + want_rows[:-1]), want_rows)]
        assert all(target // 2 <= x <= 2 * target for x in sizes[:-1])


@pytest.mark.parametrize("seed", range(6))
def test_utf8_payload_and_partition_keys(ctx, seed):
    """Utf8 columns through filter / project / partition (carried as row ids
    through the kernel, gathered after with the reference take semantics) and
    Utf8 partition keys (fnv1a64 over the string bytes, chained with the other
    keys; a null string adds no bytes) — equal to the oracle."""
    kinds = (INT64, DECIMAL, BOOL)
    rows = [0, 1, 700, 5000, 40000, 3][seed]
    b = rand_batch(seed, rows, kinds, null_frac=0.1 if seed % 2 else 0.0, utf8=True)
    u = len(kinds)  # the Utf8 column
    d = ctx.upload(b)
    pred = rand_pred(random.Random(seed), kinds, 2)
    assert_batches_equal(ctx.filter_execute(d, pred).to_host(), O.filter_execute(b, pred), ordered=True)
    exprs = [Col(u), Col(0) + 1, Col(u), Col(1)]
    assert_batches_equal(ctx.project_execute(d, exprs).to_host(), O.project_execute(b, exprs), ordered=True)
    for keys, n in (([u], 4), ([0, u], 3), ([1], 8)):
        part, offs = ctx.hash_partition(d, keys, n)
        got = part.to_host()
        want = O.hash_partition(b, keys, n)
        assert offs[-1] == b.rows
        for p in range(n):
            assert_batches_equal(O.slice_(got, offs[p], offs[p + 1] - offs[p]), want[p], ordered=True)


def _utf8_group_batch(seed, rows, null_frac):
    rng = np.random.default_rng(seed)
    words = ["", "a", "ab", "abc", "b", "ba", "ASIA", "EUROPE", "ünï", "a" * 40] + [f"w{i}" for i in range(50)]
    names = [words[i] for i in rng.integers(0, len(words), rows)]
    b = HostBatch(rows)
    b.cols.append(HostBatch.col_utf8(names, (rng.random(rows) >= null_frac) if null_frac else None))
    b.cols.append(HostBatch.col_i64(rng.integers(0, 3, rows)))
    b.cols.append(HostBatch.col_dec(rng.integers(-5000, 5000, rows).astype(np.int64), 11, 2))
    b.cols.append(HostBatch.col_utf8([words[i] for i in rng.integers(0, 4, rows)]))  # a second Utf8 column
    return b


@pytest.mark.parametrize("seed,rows,null_frac", [(0, 0, 0.0), (1, 1, 0.0), (2, 700, 0.0), (3, 5000, 0.2),
                                                 (4, 40000, 0.1)])
def test_utf8_group_keys(ctx, seed, rows, null_frac):
    """aggregate_execute with Utf8 group keys (alone, with an Int64 key, two Utf8
    keys): the GPU groups by the strings' fnv1a64 after checking every row's
    string against its hash's representative row, and gathers each group's
    string back — equal to the oracle's byte-exact interning."""
    b = _utf8_group_batch(seed, rows, null_frac)
    d = ctx.upload(b)
    aggs = [(0, 2), (2, 0), (3, 1), (5, 2)]  # SUM(dec), COUNT(*), MIN(k), AVG(dec)
    for keys in ([0], [1, 0], [0, 3], [3, 0, 1]):
        got = ctx.aggregate_execute(d, keys, aggs).to_host()
        assert_batches_equal(got, O.aggregate_execute(b, keys, aggs), ordered=False)


def test_utf8_group_key_errors(ctx):
    b = _utf8_group_batch(9, 100, 0.0)
    d = ctx.upload(b)
    with pytest.raises(Exception, match="InvalidPlan"):
        ctx.aggregate_execute(d, [0], [(3, 3)])  # MIN over a Utf8 column


@pytest.mark.parametrize("seed,nb,np_,null_frac", [(0, 0, 50, 0.0), (1, 60, 0, 0.0), (2, 120, 1500, 0.0),
                                                  (3, 200, 4000, 0.15)])
def test_utf8_join_keys_and_payloads(ctx, seed, nb, np_, null_frac):
    """join_execute with Utf8 keys (alone / with an Int64 key) and Utf8 payloads
    on both sides: candidate pairs from the fnv1a64 of the bytes, pairs whose
    strings differ dropped, strings gathered by row id — equal to the oracle's
    byte-exact dictionary join.  Also Int64 keys with Utf8 payloads only."""
    b = _utf8_group_batch(seed, nb, null_frac)
    p = _utf8_group_batch(seed + 50, np_, null_frac)
    db, dp = ctx.upload(b), ctx.upload(p)
    # ([1], [1]): an Int64 key with 3 values — Utf8 payloads only (the output is ~nb x np / 3 rows)
    for bk, pk in (([0], [0]), ([1, 0], [1, 0]), ([3], [0])) + ((([1], [1]),) if nb * np_ <= 200000 else ()):
        got = ctx.join_execute(db, dp, bk, pk).to_host()
        assert_batches_equal(got, O.join_execute(b, p, bk, pk), ordered=False)


def test_utf8_join_key_type_mismatch(ctx):
    b = _utf8_group_batch(7, 50, 0.0)
    db = ctx.upload(b)
    with pytest.raises(Exception, match="InvalidPlan"):
        ctx.join_execute(db, db, [0], [1])  # Utf8 build key vs Int64 probe key


@pytest.mark.parametrize("seed", range(4))
def test_async_filter_and_partition(ctx, seed):
    """tq_filter_async / tq_hash_partition_async: no host sync; the
    output carries the input's row count as capacity, the count / part starts
    arrive in a pinned slot after the stream event, and the trimmed batch equals
    the synchronous operator's (stable order, same part offsets)."""
    from paper_2508_05029_b200.ops import PinnedU64
    rows = [0, 1, 3000, 70000][seed]
    b = rand_batch(seed, rows, (INT64, DECIMAL, BOOL, INT64), null_frac=0.1 if seed % 2 else 0.0)
    d = ctx.upload(b)
    pred = rand_pred(random.Random(seed), (INT64, DECIMAL, BOOL, INT64), 2)
    slot = PinnedU64(2)
    try:
        got = ctx.filter_async(d, pred, slot)
        assert got.rows == rows  # capacity until trimmed
        ctx.sync()
        assert slot[0] == 0
        got.set_rows(slot[1])
        assert_batches_equal(got.to_host(), ctx.filter_execute(d, pred).to_host(), ordered=True)
    finally:
        slot.free()
    for nparts in (1, 7):
        slot = PinnedU64(nparts + 1)
        try:
            got = ctx.hash_partition_async(d, [0, 3], nparts, slot)
            ctx.sync()
            want, offs = ctx.hash_partition(d, [0, 3], nparts)
            assert slot.values() == offs
            got.set_rows(slot[nparts])
            assert_batches_equal(got.to_host(), want.to_host(), ordered=True)
        finally:
            slot.free()
