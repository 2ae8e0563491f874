"""CPU tests of the ORACLE itself: golden vectors, SPEC inline examples,
reference-substrate parity (oracle/_ref), naive-vs-hash cross checks.
No GPU needed."""
import json
import os
import random
import struct

import numpy as np
import pytest

import oracle as O
import rowloop
from helpers import rand_batch, rand_numeric_expr, rand_pred
from paper_2508_05029_b200.columnar import (BOOL, DECIMAL, FLOAT64, INT64, UTF8, HostBatch,
                                            assert_batches_equal)
from paper_2508_05029_b200.expr import Col, Dec, Lit, Null, all_of

GOLD = os.path.join(os.path.dirname(__file__), "golden")
AGG_SUM, AGG_COUNT, AGG_COUNT_STAR, AGG_MIN, AGG_MAX, AGG_AVG = range(6)


def load_golden(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- Appendix B vectors
def test_fnv_golden():
    assert O.fnv1a64(b"") == 0xCBF29CE484222325
    assert O.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert O.fnv1a64(b"foobar") == 0x85944171F73967E8
    table = {0: (0xA8C7F832281A39C5, 1, 1, 5), 1: (0x89CD31291D2AEFA4, 0, 0, 4), 42: (0xFF3ADD6B3789DAEF, 1, 3, 7),
             -1: (0x8CF51A8BFCA3883D, 1, 1, 5), 6000000: (0xE356695487F57C65, 1, 1, 5)}
    for k, (h, m2, m4, m8) in table.items():
        got = O.fnv1a64(struct.pack("<q", k))
        assert got == h, (k, hex(got))
        assert (got % 2, got % 4, got % 8) == (m2, m4, m8)
    chained = O.fnv1a64(struct.pack("<q", 11), O.fnv1a64(struct.pack("<q", 7)))
    assert chained == 0x74014FA0744B2289


def test_splitmix_golden():
    assert [O.splitmix_nth(42, k) for k in range(1, 5)] == [
        0xBDD732262FEB6E95, 0x28EFE333B266F103, 0x47526757130F9F52, 0x581CE1FF0E4AE394]
    assert [O.splitmix_nth(0, k) for k in range(1, 4)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                          0x06C45D188009454F]


def test_golden_fixture_vectors():
    g = load_golden("hash_rng.json")
    for item in g["fnv"]:
        assert O.fnv1a64(bytes.fromhex(item["bytes"]), int(item["seed"])) == int(item["hash"])
    for item in g["splitmix"]:
        seed = int(item["seed"])
        assert [O.splitmix_nth(seed, k + 1) for k in range(len(item["out"]))] == [int(x) for x in item["out"]]


def test_against_reference_hash_rng():
    L = O.ref()
    if L is None:
        pytest.skip("oracle/_ref not built")
    import ctypes as C
    rng = random.Random(3)
    for _ in range(200):
        data = bytes(rng.randrange(256) for _ in range(rng.randrange(40)))
        seed = rng.getrandbits(64)
        assert L.tqr_fnv1a64(data, len(data), seed) == O.fnv1a64(data, seed)
    out = (C.c_uint64 * 1000)()
    L.tqr_splitmix(12345, 1000, out)
    assert list(out) == [O.splitmix_nth(12345, k) for k in range(1, 1001)]


# ---------------------------------------------------------------- substrate vs reference
def _utf8_batch(seed, rows, nulls=0.2):
    return rand_batch(seed, rows, kinds=(INT64, DECIMAL, BOOL, FLOAT64), null_frac=nulls, utf8=True)


@pytest.mark.parametrize("seed", range(6))
def test_take_concat_slice_match_reference(seed):
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(seed)
    b = _utf8_batch(seed, int(rng.integers(0, 50)), nulls=0.2 if seed % 2 else 0.0)
    ids = rng.integers(0, max(b.rows, 1), int(rng.integers(0, 60))).tolist() if b.rows else []
    assert_batches_equal(O.take(b, ids), O.ref_take(b, ids), ordered=True)
    b2 = _utf8_batch(seed + 100, int(rng.integers(0, 30)), nulls=0.0)
    assert_batches_equal(O.concat([b, b2, b]), O.ref_concat([b, b2, b]), ordered=True)
    if b.rows:
        s = int(rng.integers(0, b.rows))
        n = int(rng.integers(0, b.rows - s + 1))
        assert_batches_equal(O.slice_(b, s, n), O.ref_slice(b, s, n), ordered=True)


def test_take_concat_golden_fixture():
    """Fixture produced by the reference's own take/concat (tests/golden/make_golden.py)."""
    g = load_golden("substrate.json")
    for case in g["take"]:
        b = HostBatch(case["rows"], [HostBatch.col_i64(case["x"], case["valid"])])
        out = O.take(b, case["ids"])
        assert out.column_py(0) == [None if v is None else v for v in case["want"]]
        assert (out.cols[0].validity is not None) == case["want_bitmap"]
    for case in g["concat"]:
        parts = [HostBatch(len(p["x"]), [HostBatch.col_i64(p["x"], p["valid"])]) for p in case["parts"]]
        out = O.concat(parts)
        assert out.column_py(0) == case["want"]
        assert (out.cols[0].validity is not None) == case["want_bitmap"]


# ---------------------------------------------------------------- SPEC inline examples
def test_spec_filter_example():
    # SPEC.md:565  x < 5 on [1,7,3,null] -> [1,3]
    b = HostBatch(4, [HostBatch.col_i64([1, 7, 3, 0], [True, True, True, False])])
    out = O.filter_execute(b, Col(0) < 5)
    assert out.column_py(0) == [1, 3]
    # Literal(true) -> identity
    out = O.filter_execute(b, Lit(True, BOOL))
    assert out.column_py(0) == [1, 7, 3, None]


def test_spec_project_example():
    b = HostBatch(3, [HostBatch.col_i64([1, 2, 3]), HostBatch.col_i64([10, 20, 30])])
    out = O.project_execute(b, [Col(0), Col(1), Col(0) + Col(1)])
    assert out.column_py(2) == [11, 22, 33]
    assert_batches_equal(O.project_execute(b, [Col(0), Col(1)]), b, ordered=True)


def test_spec_partition_examples():
    b = rand_batch(1, 100)
    parts = O.hash_partition(b, [0], 1)
    assert_batches_equal(parts[0], b, ordered=True)
    same = HostBatch(50, [HostBatch.col_i64([7] * 50), HostBatch.col_i64(list(range(50)))])
    parts = O.hash_partition(same, [0], 8)
    assert sum(p.rows > 0 for p in parts) == 1
    # union of parts == input multiset
    parts = O.hash_partition(b, [0, 1], 4)
    assert_batches_equal(O.concat(parts), b)
    # Appendix B: pid of int64 key 42 mod 8 == 7
    k = HostBatch(1, [HostBatch.col_i64([42])])
    assert O.partition_ids(k, [0], 8).tolist() == [7]


def test_spec_join_examples():
    a = HostBatch(3, [HostBatch.col_i64([1, 2, 3])])
    b = HostBatch(3, [HostBatch.col_i64([4, 5, 6])])
    assert O.join_execute(a, b, [0], [0]).rows == 0
    # key present k=3 times build, m=2 times probe -> 6
    a = HostBatch(4, [HostBatch.col_i64([9, 9, 9, 1]), HostBatch.col_i64([1, 2, 3, 4])])
    b = HostBatch(3, [HostBatch.col_i64([9, 2, 9])])
    assert O.join_execute(a, b, [0], [0]).rows == 6
    # null keys never match
    a = HostBatch(2, [HostBatch.col_i64([0, 0], [False, True])])
    b = HostBatch(2, [HostBatch.col_i64([0, 0], [False, True])])
    assert O.join_execute(a, b, [0], [0]).rows == 1


def test_spec_aggregate_examples():
    b = HostBatch(5, [HostBatch.col_i64([3] * 5)])
    out = O.aggregate_execute(b, [0], [(AGG_COUNT_STAR, 0)])
    assert out.to_rows() == [(3, 5)]
    empty = HostBatch(0, [HostBatch.col_i64([])])
    assert O.aggregate_execute(empty, [0], [(AGG_COUNT_STAR, 0)]).rows == 0
    # nulls skipped except count(*); avg = sum / count
    b = HostBatch(4, [HostBatch.col_i64([1, 1, 1, 1]), HostBatch.col_dec(np.array([100, 300, 0, 0]), 11, 2,
                                                                        [True, True, False, False])])
    out = O.aggregate_execute(b, [0], [(AGG_SUM, 1), (AGG_COUNT, 1), (AGG_COUNT_STAR, 1), (AGG_AVG, 1),
                                       (AGG_MIN, 1), (AGG_MAX, 1)])
    assert out.to_rows() == [(1, 400, 2, 4, 2.0, 100, 300)]


# ---------------------------------------------------------------- randomized cross checks
@pytest.mark.parametrize("seed", range(30))
def test_filter_vs_rowloop(seed):
    kinds = (INT64, DECIMAL, FLOAT64, BOOL, INT64)
    b = rand_batch(seed, 200, kinds, null_frac=0.1)
    pred = rand_pred(random.Random(seed), kinds, 3)
    got = O.filter_execute(b, pred)
    want = O.take(b, rowloop.filter_rows(b, pred))
    assert_batches_equal(got, want, ordered=True)


@pytest.mark.parametrize("seed", range(30))
def test_project_vs_rowloop(seed):
    kinds = (INT64, DECIMAL, FLOAT64, BOOL, DECIMAL)
    b = rand_batch(seed, 150, kinds, null_frac=0.1, small=seed % 3 != 0)
    e = rand_numeric_expr(random.Random(seed), kinds, 3)
    got = O.project_execute(b, [e]).column_py(0)
    want = rowloop.project_values(b, e)
    for g, w in zip(got, want):
        if isinstance(w, float) or isinstance(g, float):
            assert (g is None) == (w is None)
            if w is not None:
                assert g == pytest.approx(w, rel=1e-9, abs=0) or g == w
        else:
            assert g == w


@pytest.mark.parametrize("seed", range(12))
def test_join_hash_vs_naive(seed):
    a = rand_batch(seed, 120, (INT64, DECIMAL, BOOL), null_frac=0.05)
    b = rand_batch(seed + 1000, 150, (INT64, DECIMAL, FLOAT64), null_frac=0.05)
    rng = np.random.default_rng(seed)
    for x in (a, b):  # few distinct decimal keys so composite keys collide
        x.cols[1] = HostBatch.col_dec(rng.integers(0, 3, x.rows), 11, 2, x.validity_of(1))
    keys_b, keys_p = ([0], [0]) if seed % 2 else ([0, 1], [0, 1])
    h = O.join_execute(a, b, keys_b, keys_p, naive=False)
    n = O.join_execute(a, b, keys_b, keys_p, naive=True)
    assert h.rows > 0
    assert_batches_equal(h, n)


@pytest.mark.parametrize("seed", range(12))
def test_aggregate_hash_vs_naive(seed):
    kinds = (INT64, DECIMAL, FLOAT64, BOOL, INT64)
    b = rand_batch(seed, 300, kinds, null_frac=0.1)
    keys = [[0], [3], [0, 3], []][seed % 4]
    aggs = [(AGG_SUM, 1), (AGG_SUM, 0), (AGG_SUM, 2), (AGG_COUNT, 1), (AGG_COUNT_STAR, 0), (AGG_MIN, 1),
            (AGG_MAX, 2), (AGG_AVG, 1), (AGG_AVG, 0), (AGG_MIN, 3)]
    h = O.aggregate_execute(b, keys, aggs)
    n = O.aggregate_execute(b, keys, aggs, naive=True)
    assert_batches_equal(h, n)


# ---------------------------------------------------------------- datagen / queries
def test_datagen_shapes():
    sf = 0.01
    li = O.datagen(O.T_LINEITEM, sf)
    od = O.datagen(O.T_ORDERS, sf)
    assert od.rows == 15000
    assert li.rows == O.table_rows(O.T_LINEITEM, sf)
    assert 3.5 * od.rows < li.rows < 4.5 * od.rows
    ok = li.cols[0].i64()
    assert ok.min() == 1 and ok.max() == od.rows and np.all(np.diff(ok) >= 0)
    ship = li.cols[9].i64()
    assert 8036 <= ship.min() and ship.max() <= 10440 + 121
    # counter-based generator == reference SplitMix64(seed).next_below sequence
    L = O.ref()
    if L is not None:
        import ctypes as C
        seed = O.fnv1a64(b"customer.c_nationkey", 42)
        n = 500
        out = (C.c_uint64 * n)()
        L.tqr_splitmix_below(seed, 25, n, out)
        cu = O.datagen(O.T_CUSTOMER, sf)
        assert cu.cols[1].i64()[:n].tolist() == list(out)


@pytest.mark.parametrize("q", [1, 3, 5, 6, 9])
def test_queries_threads_agree(q):
    sf = 0.01
    tabs = {t: O.datagen(t, sf) for t in O.QUERY_TABLES[q]}
    one = O.query(q, tabs, nthreads=1)
    many = O.query(q, tabs, nthreads=4)
    assert one.rows > 0
    assert_batches_equal(many, one)


def test_q6_selectivity():
    li = O.datagen(O.T_LINEITEM, 0.01)
    shipdate, disc, qty = li.cols[9].i64(), li.cols[5].dec_words()[:, 0], li.cols[3].dec_words()[:, 0]
    m = (shipdate >= 8766) & (shipdate < 9131) & (disc >= 5) & (disc <= 7) & (qty < 2400)
    assert 0.01 < m.mean() < 0.03
    out = O.query(6, {O.T_LINEITEM: li})
    ep = li.cols[4].dec_words()[:, 0]
    assert out.column_py(0)[0] == int((ep[m].astype(object) * disc[m].astype(object)).sum())


@pytest.mark.parametrize("t", range(8))
def test_datagen_shards_concat_to_full_table(t):
    """A worker's row-group subset (tqo_datagen_shard) is a contiguous slice of
    the full table: the shards concatenate back to it, value for value."""
    sf = 0.02
    full = O.datagen(t, sf, 4)
    parts = [O.datagen(t, sf, 4, s, 5) for s in range(5)]
    cat = O.concat(parts)
    assert cat.rows == full.rows
    for a, b in zip(cat.cols, full.cols):
        assert (a.values == b.values).all()


# ---------------------------------------------------------------- Utf8 group keys
def _utf8_key_batch(seed, rows, null_frac):
    """(Utf8 name, Int64 k, Int64 v): few distinct strings, incl. the empty one
    and strings that share prefixes, so byte equality (not a prefix) decides."""
    rng = np.random.default_rng(seed)
    words = ["", "a", "ab", "abc", "b", "ba", "ASIA", "EUROPE", "ünï", "a" * 40]
    names = [words[i] for i in rng.integers(0, len(words), rows)]
    nv = rng.random(rows) >= null_frac
    b = HostBatch(rows)
    b.cols.append(HostBatch.col_utf8(names, nv if null_frac else None))
    b.cols.append(HostBatch.col_i64(rng.integers(0, 3, rows)))
    b.cols.append(HostBatch.col_i64(rng.integers(-100, 100, rows)))
    return b, names, nv


def _py_group(names, nv, ks, vs, use_k):
    out = {}
    for i in range(len(names)):
        key = (names[i] if nv[i] else None,) + ((int(ks[i]),) if use_k else ())
        s, n, mn = out.get(key, (0, 0, None))
        v = int(vs[i])
        out[key] = (s + v, n + 1, v if mn is None else min(mn, v))
    return out


@pytest.mark.parametrize("seed,rows,null_frac", [(0, 0, 0.0), (1, 1, 0.0), (2, 500, 0.0), (3, 3000, 0.2)])
@pytest.mark.parametrize("naive", [False, True])
def test_oracle_utf8_group_keys(seed, rows, null_frac, naive):
    """aggregate_execute over a Utf8 key (alone and with an Int64 key): one group
    per distinct string by its bytes, a null string its own group — against a
    Python dict; the output key column is Utf8 (bitmap iff the input had one)."""
    b, names, nv = _utf8_key_batch(seed, rows, null_frac)
    ks, vs = b.cols[1].i64(), b.cols[2].i64()
    for keys, use_k in (([0], False), ([1, 0], True)):
        got = O.aggregate_execute(b, keys, [(AGG_SUM, 2), (AGG_COUNT_STAR, 0), (AGG_MIN, 2)], naive=naive)
        want = _py_group(names, nv, ks, vs, use_k)
        ucol = keys.index(0)
        assert got.cols[ucol].kind == UTF8
        assert (got.cols[ucol].validity is not None) == (null_frac > 0 and rows > 0)
        rows_got = {}
        strs = got.column_py(ucol)
        kcol = got.column_py(1 - ucol) if use_k else None
        sums, cnts, mins = got.column_py(len(keys)), got.column_py(len(keys) + 1), got.column_py(len(keys) + 2)
        for g in range(got.rows):
            key = (strs[g],) + ((kcol[g],) if use_k else ())
            rows_got[key] = (sums[g], cnts[g], mins[g])
        assert rows_got == want


def test_oracle_utf8_aggregate_input_rejected():
    b, _, _ = _utf8_key_batch(5, 10, 0.0)
    with pytest.raises(Exception, match="InvalidPlan"):
        O.aggregate_execute(b, [1], [(AGG_MIN, 0)])


@pytest.mark.parametrize("seed,nb,np_,null_frac", [(0, 0, 5, 0.0), (1, 7, 0, 0.0), (2, 60, 300, 0.0),
                                                  (3, 200, 900, 0.2)])
@pytest.mark.parametrize("naive", [False, True])
def test_oracle_utf8_join_keys(seed, nb, np_, null_frac, naive):
    """join_execute on (Utf8) and (Int64, Utf8) keys: rows match iff the strings'
    bytes are equal (a null string never matches), duplicates on both sides give
    every pair — against a Python nested loop over the row tuples."""
    bb, bnames, bnv = _utf8_key_batch(seed, nb, null_frac)
    pb, pnames, pnv = _utf8_key_batch(seed + 100, np_, null_frac)
    for bk, pk in (([0], [0]), ([1, 0], [1, 0])):
        got = O.join_execute(bb, pb, bk, pk, naive=naive)
        want = []
        for p in range(np_):
            for b in range(nb):
                if not (bnv[b] and pnv[p]) or bnames[b] != pnames[p]:
                    continue
                if len(bk) == 2 and bb.cols[1].i64()[b] != pb.cols[1].i64()[p]:
                    continue
                want.append((bnames[b], int(bb.cols[1].i64()[b]), int(bb.cols[2].i64()[b]),
                             pnames[p], int(pb.cols[1].i64()[p]), int(pb.cols[2].i64()[p])))
        assert got.cols[0].kind == UTF8 and got.cols[3].kind == UTF8
        rows = list(zip(*[got.column_py(c) for c in range(6)])) if got.rows else []
        assert sorted(rows) == sorted(want)
