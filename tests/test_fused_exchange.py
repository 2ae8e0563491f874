"""Fused partition + scatter into peer receive windows
(tq_pipeline_partition_exchange) on one GPU (a world-1 communicator: every row
goes to this rank's own window) vs the oracle's filter + project.  The output
order is unspecified, so batches are compared after canonical sort.  The
multi-rank path (real NVLink peer windows) is tests/test_multigpu.py
(modes fused / fused_nolip)."""
import random

import pytest

import oracle as O
from helpers import rand_batch, rand_numeric_expr, rand_pred
from paper_2508_05029_b200.columnar import BOOL, DECIMAL, FLOAT64, INT64, assert_batches_equal
from paper_2508_05029_b200.expr import Col

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["jit", "interp"])
def env(request):
    from paper_2508_05029_b200.ops import Comm, Context
    c = Context(0)
    c.set_jit(request.param == "jit")
    comm = Comm(c, 0, 1, Comm.unique_id())
    yield c, comm
    comm.close()
    c.close()


@pytest.mark.parametrize("seed", range(10))
def test_fused_partition_exchange_world1(env, seed):
    ctx, comm = env
    kinds = (INT64, DECIMAL, FLOAT64, BOOL, INT64)
    rows = [0, 1, 513, 20000, 250000][seed % 5]
    b = rand_batch(seed, rows, kinds, null_frac=0.1 if seed % 2 else 0.0, small=seed % 3 != 0)
    r = random.Random(seed)
    # seed % 4 == 0: no predicate -> every row is shipped (first window guess
    # overflows for the large cases and the call re-runs with a grown window)
    pred = None if seed % 4 == 0 else rand_pred(r, kinds, 2)
    exprs = [Col(0), Col(1), rand_numeric_expr(r, kinds, 2), Col(3), Col(2)]
    keys = [[0], [1], [0, 3]][seed % 3]
    got = comm.partition_exchange(ctx.upload(b), pred, exprs, keys).to_host()
    filtered = O.filter_execute(b, pred) if pred is not None else b
    want = O.project_execute(filtered, exprs)
    assert_batches_equal(got, want)


def test_fused_exchange_repeated_calls_reuse_window(env):
    """Back-to-back calls of different widths share (and grow) one window."""
    ctx, comm = env
    for i, rows in enumerate([1000, 300000, 5000, 300000]):
        b = rand_batch(40 + i, rows, (INT64, DECIMAL, INT64), null_frac=0.05)
        exprs = [Col(0), Col(1)] if i % 2 else [Col(0), Col(1), Col(2), Col(1)]
        got = comm.partition_exchange(ctx.upload(b), None, exprs, [0]).to_host()
        assert_batches_equal(got, O.project_execute(b, exprs))
