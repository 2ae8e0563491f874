"""The scan side: TCF files (SPEC.md:128-229 storage module) and
the byte-range preload of a row group's needed columns into the pinned Host
pool as a chunked batch — the object tq_load moves to the device.  CPU tests
(the pool falls back to plain host memory without a driver) + one GPU test."""
import os

import numpy as np
import pytest

import oracle as O
from helpers import rand_batch
from paper_2508_05029_b200.columnar import BOOL, DECIMAL, FLOAT64, INT64, HostBatch, TqError, assert_batches_equal
from paper_2508_05029_b200.ops import Pool, Tcf, coalesce_ranges


def _write(tmp_path, b, target, names=None):
    path = str(tmp_path / "t.tcf")
    Tcf.write(path, b, target, names)
    return path


def test_write_read_footer_two_reads(tmp_path):
    """1M Int64 rows at a 1 MiB target -> ~8 row groups (SPEC example); the
    footer read issues exactly two datasource reads."""
    b = HostBatch(1_000_000, [HostBatch.col_i64(np.arange(1_000_000))])
    f = Tcf(_write(tmp_path, b, 1 << 20, ["x"]))
    assert f.reads() == 2
    assert 7 <= f.row_groups <= 9
    assert sum(f.rows(g) for g in range(f.row_groups)) == b.rows
    assert f.column(0)[:2] == ("x", INT64)
    f.close()


@pytest.mark.parametrize("seed", range(4))
def test_full_scan_equivalence(tmp_path, seed):
    """Every row group fetched into the pool (all columns) and decoded,
    concatenated == the written table (validity, Decimal, Bool, Utf8)."""
    b = rand_batch(seed, [0, 1, 5000, 33333][seed], (INT64, DECIMAL, BOOL, FLOAT64), null_frac=0.1 * (seed % 2),
                   utf8=True)
    f = Tcf(_write(tmp_path, b, 4096))
    pool = Pool(1 << 12, 4096)
    parts = []
    for g in range(f.row_groups):
        cb = f.fetch(pool, g, list(range(f.ncols)), max_connections=3)
        parts.append(cb.decode())
        cb.release()
    assert pool.free_count() == 4096
    got = O.concat(parts) if parts else None
    if b.rows:
        assert_batches_equal(got, b, ordered=True)
    else:
        assert f.row_groups == 0
    f.close()
    pool.close()


def test_column_subset_and_ranges(tmp_path):
    """plan_ranges: 2 row groups x 3 of 5 columns -> 6 ranges sorted by offset;
    a subset fetch equals the projection of those row groups."""
    b = rand_batch(9, 20000, (INT64, DECIMAL, BOOL, FLOAT64, INT64), null_frac=0.05)
    f = Tcf(_write(tmp_path, b, 64 << 10))
    assert f.row_groups >= 2
    rs = f.plan_ranges([0, 2, 4], [0, 1])
    assert len(rs) == 6 and rs == sorted(rs)
    pool = Pool(1 << 16, 256)
    cb = f.fetch(pool, 1, [4, 1])
    start = f.rows(0)
    want = O.slice_(HostBatch(b.rows, [b.cols[4], b.cols[1]]), start, f.rows(1))
    assert_batches_equal(cb.decode(), want, ordered=True)
    cb.release()
    f.close()
    pool.close()


def test_coalesce_examples():
    assert coalesce_ranges([], 64, 1 << 20) == []                                   # SPEC: [] -> []
    assert coalesce_ranges([(0, 100), (150, 100)], 64, 1 << 20) == [(0, 250)]       # gap 50 <= 64
    assert coalesce_ranges([(0, 100), (200, 100)], 64, 1 << 20) == [(0, 100), (200, 100)]  # gap 100 > 64
    assert coalesce_ranges([(0, 100), (100, 100)], 0, 150) == [(0, 100), (100, 100)]  # max_merged bound


def test_errors(tmp_path):
    p = str(tmp_path / "short.tcf")
    open(p, "wb").write(b"TCF1")
    with pytest.raises(TqError) as e:
        Tcf(p)
    assert e.value.errc == "NotTcf"
    b = HostBatch(10, [HostBatch.col_i64(np.arange(10))])
    f = Tcf(_write(tmp_path, b, 1024))
    with pytest.raises(TqError) as e:
        f.plan_ranges([3], [0])
    assert e.value.errc == "UnknownColumn"
    f.close()


@pytest.mark.gpu
def test_tcf_row_group_to_device(tmp_path):
    """Byte-range preload into the pinned pool, then load_to_device (one
    cudaMemcpyAsync per segment): the device batch equals the row group."""
    from paper_2508_05029_b200.ops import Context
    ctx = Context(0)
    b = rand_batch(3, 50000, (INT64, DECIMAL, BOOL), null_frac=0.1, utf8=True)
    f = Tcf(_write(tmp_path, b, 256 << 10))
    pool = Pool(1 << 20, 64)
    at = 0
    for g in range(f.row_groups):
        cb = f.fetch(pool, g, [0, 1, 2, 3])
        d = cb.load(ctx)
        assert_batches_equal(d.to_host(), O.slice_(b, at, f.rows(g)), ordered=True)
        at += f.rows(g)
        cb.release()
        d.free()
    f.close()
    pool.close()
    ctx.close()
