"""CPU (gloo, world_size 2) tests of the multi-worker host logic: the
distributed Q3 plan — broadcast of customer_f, fnv1a64-mod-N hash partition,
all-to-all exchange, co-partitioned join + aggregate — executed with the
oracle's operators over each worker's row-group subset must equal the
single-node result; plus exchange_phase1 / exchange_decide / assign_files
(SPEC.md:571-588, 661-667)."""
import os
import pickle
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from paper_2508_05029_b200.exchange import (BROADCAST, HASH_PARTITION, assign_files, exchange_decide,  # noqa: E402
                                            exchange_phase1, shard_range)


def test_exchange_phase1_examples():
    assert exchange_phase1(10 << 20, 0.25) == 40 << 20
    assert exchange_phase1(0, 1.0) == 0
    assert exchange_phase1(123, 0.01) is None                 # below sample fraction
    assert exchange_phase1(5 << 20, 1.0) == 5 << 20           # scan complete: exact bytes


def test_exchange_decide_examples():
    d = exchange_decide([1 << 20], [1 << 30], 1, 10 << 20)
    assert d.strategy == BROADCAST and d.broadcast_side == 0
    d = exchange_decide([1 << 30], [1 << 30], 4)
    assert d.strategy == HASH_PARTITION
    # identical on every worker for identical inputs
    assert exchange_decide([5, 6], [7, 8], 2) == exchange_decide([5, 6], [7, 8], 2)
    # the smaller side is broadcast, whichever it is; ties -> side 0
    assert exchange_decide([1 << 30], [1 << 20], 1).broadcast_side == 1
    assert exchange_decide([7], [7], 1).broadcast_side == 0
    # config 4 at SF100: customer_f 24 MB broadcast for N >= 2, orders/lineitem partitioned
    assert exchange_decide([24_000_000], [10 ** 10], 2).strategy == BROADCAST
    assert exchange_decide([24_000_000], [10 ** 10], 1).strategy == HASH_PARTITION


def test_assign_files_examples():
    assert sorted(map(len, assign_files([1, 1, 1, 1], 4))) == [1, 1, 1, 1]
    sizes = [5, 1, 9, 3, 3, 7, 2, 8, 4, 6, 1, 2]
    out = assign_files(sizes, 3)
    assert sorted(i for w in out for i in w) == list(range(len(sizes)))
    loads = [sum(sizes[i] for i in w) for w in out]
    assert max(loads) / min(loads) <= 1.5
    lo, hi = shard_range(10, 1, 3)
    assert (lo, hi) == (3, 6)


def _worker(rank, world, port, sf, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import numpy as np
    import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = {t: O.datagen(t, sf) for t in (O.T_CUSTOMER, O.T_ORDERS, O.T_LINEITEM)}
        # row-group subsets (tq_datagen_shard semantics): orders by range, lineitem = lines of those orders
        olo, ohi = shard_range(full[O.T_ORDERS].rows, rank, world)
        okeys = full[O.T_LINEITEM].cols[0].i64()
        lsel = np.nonzero((okeys > olo) & (okeys <= ohi))[0].tolist()
        clo, chi = shard_range(full[O.T_CUSTOMER].rows, rank, world)
        cust = O.slice_(full[O.T_CUSTOMER], clo, chi - clo)
        orders = O.slice_(full[O.T_ORDERS], olo, ohi - olo)
        line = O.take(full[O.T_LINEITEM], lsel)
        from paper_2508_05029_b200.expr import Col, Dec
        from paper_2508_05029_b200 import queries as Q
        # broadcast customer_f
        cf = O.project_execute(O.filter_execute(cust, Col(2).eq(1)), [Col(0)])
        allc = [None] * world
        dist.all_gather_object(allc, pickle.dumps(cf))
        cb = O.concat([pickle.loads(x) for x in allc])
        oj = O.join_execute(cb, O.filter_execute(orders, Col(2) < 9204), [0], [1])
        of = O.project_execute(oj, [Col(1), Col(3), Col(4)])
        lf = O.project_execute(O.filter_execute(line, Col(9) > 9204), [Col(0), Q.REV])

        def shuffle(b):
            parts = O.hash_partition(b, [0], world)
            got = [None] * world
            for dst in range(world):  # all-to-all as world gathers
                recv = [None] * world
                dist.all_gather_object(recv, pickle.dumps(parts[dst]))
                if dst == rank:
                    got = [pickle.loads(x) for x in recv]
            return O.concat(got)

        orx, lrx = shuffle(of), shuffle(lf)
        j = O.join_execute(orx, lrx, [0], [0])
        agg = O.aggregate_execute(j, [3, 1, 2], [(0, 4)])
        res = [None] * world
        dist.all_gather_object(res, pickle.dumps(agg))
        if rank == 0:
            got = O.concat([pickle.loads(x) for x in res])
            want = O.query(3, full, 4)
            from paper_2508_05029_b200.columnar import assert_batches_equal
            assert_batches_equal(got, want)
            # groups are disjoint across workers (co-partitioned on orderkey)
            keys = [set(pickle.loads(x).cols[0].i64().tolist()) for x in res]
            assert not (keys[0] & keys[1])
            q.put("ok")
    except Exception as e:  # pragma: no cover
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


def test_distributed_q3_plan_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29650
    ps = [ctx.Process(target=_worker, args=(r, 2, port, 0.02, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    assert all(p.exitcode == 0 for p in ps)
    assert q.get(timeout=5) == "ok"
