"""GPU: Device<->Host tier moves and the C++ worker runtime (BatchHolders,
Memory / Pre-loading / Compute executors, run_task lifecycle) running the
benchmark query DAGs vs the oracle — with resident tables, with Host-tier
tables under a Device budget (spill / load_to_device / preload), and through
the on_oom retry path."""
import os

import numpy as np
import pytest

import oracle as O
from helpers import rand_batch
from paper_2508_05029_b200.columnar import BOOL, DECIMAL, FLOAT64, INT64, assert_batches_equal
from paper_2508_05029_b200.ops import Context, Pool, engine_run_query

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("seed", range(4))
def test_spill_load_roundtrip(ctx, seed):
    b = rand_batch(seed, [0, 7, 5000, 123457][seed], (INT64, DECIMAL, BOOL, FLOAT64), null_frac=0.1 * (seed % 2))
    p = Pool([64, 4096, 1 << 20, 1 << 16][seed], 4096)
    d = ctx.upload(b)
    cb = p.spill(ctx, d)                       # one cudaMemcpyAsync per segment, D2H
    assert_batches_equal(cb.decode(), b, ordered=True)
    back = cb.load(ctx)                        # load_to_device, H2D
    assert_batches_equal(back.to_host(), b, ordered=True)
    cb.release()
    p.close()


@pytest.mark.parametrize("q", [1, 3, 5, 6, 9])
def test_engine_queries_resident(ctx, q):
    sf = 0.05
    tabs = {t: ctx.datagen(t, sf) for t in O.QUERY_TABLES[q]}
    got, m = engine_run_query(ctx, q, tabs, compute_threads=4, batch_rows=64 * 1024)
    want = O.query(q, {t: O.datagen(t, sf) for t in O.QUERY_TABLES[q]}, 8)
    assert_batches_equal(got, want)
    assert m["tasks"] > 0


@pytest.mark.parametrize("q", [3, 9])
def test_engine_host_tables_under_budget(ctx, q):
    """Config-5 path: tables start in the pinned Host tier, a Device budget
    forces spills; results stay identical."""
    sf = 0.05
    host = {t: O.datagen(t, sf) for t in O.QUERY_TABLES[q]}
    total = sum(b.nbytes() for b in host.values())
    got, m = engine_run_query(ctx, q, host, compute_threads=4, batch_rows=32 * 1024, preload=1,
                              device_budget=max(total // 3, 48 << 20))
    want = O.query(q, host, 8)
    assert_batches_equal(got, want)
    assert m["loads"] + m["preloads"] > 0, m


@pytest.mark.parametrize("case", ["retry", "split", "unsplittable"])
def test_engine_on_oom_paths(ctx, case):
    """run_task's on_oom forced in a real query by injecting
    ReservationExceeded into the lineitem probe tasks (filter + project + probe): the doubled
    estimate is retried; a multi-batch task whose doubled estimate exceeds
    the Device capacity is split in two; a single-batch one aborts the query
    with OutOfMemoryUnsplittable.  Results stay identical to the oracle."""
    from paper_2508_05029_b200.columnar import TqError
    sf = 0.05
    tabs = {t: ctx.datagen(t, sf) for t in O.QUERY_TABLES[3]}
    want = O.query(3, {t: O.datagen(t, sf) for t in O.QUERY_TABLES[3]}, 8)
    opts = dict(compute_threads=2, batch_rows=32 * 1024, device_budget=4 << 30, inject_oom_op="lineitem_probe")
    if case == "retry":
        got, m = engine_run_query(ctx, 3, tabs, inject_oom_mode=1, inject_oom_count=2, **opts)
        assert (m["oom_retries"], m["splits"]) == (2, 0), m
        assert_batches_equal(got, want)
    elif case == "split":
        got, m = engine_run_query(ctx, 3, tabs, task_batches=4, inject_oom_mode=2, inject_oom_count=1, **opts)
        assert m["splits"] == 1 and m["oom_retries"] == 0, m
        assert_batches_equal(got, want)
    else:
        with pytest.raises(TqError) as e:
            engine_run_query(ctx, 3, tabs, task_batches=1, inject_oom_mode=2, inject_oom_count=1, **opts)
        assert e.value.errc == "OutOfMemoryUnsplittable"


@pytest.mark.parametrize("q", [3, 9])
def test_engine_over_tcf_files(ctx, q, tmp_path):
    """The scan side end to end: the query's tables written as TCF files, every
    row group a Storage-tier batch that the executors fetch into the pinned
    pool (byte ranges) and move to the device; with a Device budget and the
    Pre-loading executor.  Result == the oracle."""
    from paper_2508_05029_b200.ops import Tcf, engine_run_query_tcf
    sf = 0.05
    host = {t: O.datagen(t, sf) for t in O.QUERY_TABLES[q]}
    paths = {}
    for t, b in host.items():
        paths[t] = str(tmp_path / f"t{t}.tcf")
        Tcf.write(paths[t], b, 256 << 10)
    got, m = engine_run_query_tcf(ctx, q, paths, compute_threads=4, preload=1,
                                  device_budget=max(sum(b.nbytes() for b in host.values()) // 3, 48 << 20))
    assert_batches_equal(got, O.query(q, host, 8))
    assert m["storage_reads"] >= sum(Tcf(p).row_groups for p in paths.values()), m


@pytest.mark.parametrize("q", [5, 9])
def test_engine_host_tier_spill_stress(ctx, q):
    """The config-5 shape at SF1 (Host-tier tables, a Device budget below the
    data, several batches per table) repeated: spills run on the Memory executor
    concurrently with the compute threads, so every handle a kernel reads must be
    pinned first (a concatenated build batch once was not — wrong Q9 groups in
    about half of the runs).  Every repetition equals the oracle."""
    sf = 1.0
    host = {t: O.datagen(t, sf) for t in O.QUERY_TABLES[q]}
    total = sum(b.nbytes() for b in host.values())
    want = O.query(q, host, 8)
    spills = 0
    for _ in range(4):
        got, m = engine_run_query(ctx, q, host, compute_threads=4, batch_rows=256 * 1024, preload=1,
                                  device_budget=max(int(total / 1.5), 64 << 20))
        assert_batches_equal(got, want)
        spills += m["spills"]
    assert spills > 0


@pytest.mark.timeout(300)
def test_engine_abort_does_not_hang():
    """Q9 under a Device budget tight enough that a probe task may not fit
    (OutOfMemoryUnsplittable) while other tasks wait for memory
    and spills are queued: whichever way each run goes (an exact result or the
    abort), the query returns — the tear-down releases waiting tasks (one once
    kept the executor threads from joining: a hang).  Run in a subprocess with a
    deadline, 4 times."""
    import subprocess
    import sys
    code = r"""
import os, sys
sys.path[:0] = [%r, %r]
import oracle as O
from paper_2508_05029_b200.ops import Context, engine_run_query
from paper_2508_05029_b200.columnar import TqError, assert_batches_equal
ctx = Context(0)
host = {t: O.datagen(t, 1.0) for t in O.QUERY_TABLES[9]}
total = sum(b.nbytes() for b in host.values())
want = O.query(9, host, 8)
for _ in range(4):
    try:
        got, m = engine_run_query(ctx, 9, host, compute_threads=4, batch_rows=512 * 1024, preload=1,
                                  device_budget=int(total / 2.5))
        assert_batches_equal(got, want)
        print("exact", flush=True)
    except TqError as e:
        assert "OutOfMemoryUnsplittable" in str(e), e
        print("aborted", flush=True)
""" % (ROOT, os.path.join(ROOT, "oracle"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    assert len(r.stdout.split()) == 4, r.stdout
