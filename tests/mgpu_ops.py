"""torchrun helper (one process per GPU) for multi-rank operator checks that
are not whole queries.  Run by tests/test_multigpu.py; exits non-zero on a
mismatch.  Modes (TQ_MODE):
  validity  the fused partition exchange / broadcast when ranks DISAGREE on
            which columns can be null (rank 0 has nulls, rank 1 has no
            bitmaps, rank 2 an empty input): every rank must lay out its
            window identically and the output must carry the nulls.
  utf8      Utf8 payload / key columns through the NCCL exchange.
  engine    the C++ worker runtime's distributed plans (tq_engine_run_query
            with a communicator) for Q1 / Q3 / Q5 / Q6 / Q9: exchange_decide
            (adaptive), forced Broadcast and forced HashPartition (SPEC.md:613
            strategy equivalence), fused NVLink and NCCL exchanges; the union
            of the workers' results must equal the oracle every time."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def validity(ctx, comm, rank, world):
    import oracle as O
    from helpers import rand_batch
    from paper_2508_05029_b200.columnar import DECIMAL, INT64
    from paper_2508_05029_b200.expr import Col
    rows = 0 if rank == 2 else 20000 + 3000 * rank
    b = rand_batch(50 + rank, rows, (INT64, DECIMAL, INT64), null_frac=0.1 if rank == 0 else 0.0)
    d = ctx.upload(b)
    exprs = [Col(0), Col(1), Col(2) + 1]
    px = comm.partition_exchange(d, None, exprs, [0]).to_host()
    bc = comm.broadcast(d, Col(2) < 5, [Col(1), Col(0)]).to_host()
    ins = [None] * world
    outs = [None] * world
    dist.all_gather_object(ins, b)
    dist.all_gather_object(outs, (px, bc))
    if rank != 0:
        return True
    from paper_2508_05029_b200.columnar import assert_batches_equal
    allin = O.concat(ins)
    assert_batches_equal(O.concat([o[0] for o in outs]), O.project_execute(allin, exprs))
    want_bc = O.project_execute(O.filter_execute(allin, Col(2) < 5), [Col(1), Col(0)])
    for o in outs:  # every rank receives every broadcast row
        assert_batches_equal(o[1], want_bc)
    return True


def utf8(ctx, comm, rank, world):
    """Utf8 columns through the NCCL exchange (tq_comm_exchange): each rank
    hash-partitions a batch with Utf8 payload and key columns (nulls on rank 0,
    an empty input on rank 2) and exchanges it; rank r must receive, in sender
    order, every sender's part r — strings, offsets and bitmaps exactly."""
    import numpy as np
    import oracle as O
    from paper_2508_05029_b200.columnar import HostBatch, assert_batches_equal
    rng = np.random.default_rng(70 + rank)
    rows = 0 if rank == 2 else 3000 + 500 * rank
    words = ["", "a", "bc", "def", "ASIA", "ünï", "x" * 50] + [f"w{i}" for i in range(40)]
    b = HostBatch(rows)
    b.cols.append(HostBatch.col_utf8([words[i] for i in rng.integers(0, len(words), rows)],
                                     (rng.random(rows) > 0.1) if rank == 0 else None))
    b.cols.append(HostBatch.col_i64(rng.integers(0, 100, rows)))
    b.cols.append(HostBatch.col_utf8([words[i] for i in rng.integers(0, len(words), rows)]))
    d = ctx.upload(b)
    parts, offs = ctx.hash_partition(d, [0, 1], world)
    got, _ = comm.exchange(parts, offs)
    got = got.to_host()
    # the fused API with Utf8 columns (routed through the NCCL exchange / all-gather)
    px = comm.partition_exchange(d, None, None, [0, 1]).to_host()
    bc = comm.broadcast(d, None, None).to_host()
    ins = [None] * world
    outs = [None] * world
    dist.all_gather_object(ins, b)
    dist.all_gather_object(outs, (got, px, bc))
    if rank != 0:
        return True
    for r in range(world):
        want = O.concat([O.hash_partition(ins[s], [0, 1], world)[r] for s in range(world)])
        assert_batches_equal(outs[r][0], want, ordered=True)
        assert_batches_equal(outs[r][1], want, ordered=True)
        assert_batches_equal(outs[r][2], O.concat(ins), ordered=True)
    return True


def engine(ctx, comm, rank, world):
    import oracle as O
    from paper_2508_05029_b200.columnar import assert_batches_equal
    from paper_2508_05029_b200.ops import engine_run_query
    sf = float(os.environ.get("TQ_SF", "0.1"))
    queries = [int(q) for q in os.environ.get("TQ_QUERIES", "1,3,5,6,9").split(",")]
    cases = [("adaptive", 0, 0), ("broadcast", 1, 0), ("hash", 2, 0), ("hash_nccl", 2, 1)]
    ok = True
    for q in queries:
        tabs = {t: ctx.datagen(t, sf, shard=rank, nshards=world) for t in O.QUERY_TABLES[q]}
        want = O.query(q, {t: O.datagen(t, sf) for t in O.QUERY_TABLES[q]}, 8) if rank == 0 else None
        for name, force, impl in cases:
            out, m = engine_run_query(ctx, q, tabs, comm=comm, compute_threads=4, batch_rows=64 * 1024,
                                      force_exchange=force, exchange_impl=impl)
            parts = [None] * world
            dist.all_gather_object(parts, out)
            if rank == 0:
                try:
                    assert_batches_equal(O.concat(parts), want)
                    print(f"  q{q} {name}: ok rows={want.rows} decisions="
                          f"{[(d['pair'], d['strategy']) for d in m['exchange_decisions']]}")
                except AssertionError as e:
                    print(f"  q{q} {name}: MISMATCH {e}")
                    ok = False
        for v in tabs.values():
            v.free()
    flag = [ok]
    dist.broadcast_object_list(flag, src=0)
    assert flag[0]


def main():
    if os.environ.get("TQ_MGPU_TRACE"):
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ["TQ_MGPU_TRACE"]), exit=True)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    from paper_2508_05029_b200.ops import Comm, Context
    ctx = Context(local)
    uid = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = Comm(ctx, rank, world, uid[0])
    mode = os.environ.get("TQ_MODE", "validity")
    rc = 0
    try:
        {"validity": validity, "engine": engine, "utf8": utf8}[mode](ctx, comm, rank, world)
    except AssertionError as e:
        print("MISMATCH", mode, str(e)[:2000], flush=True)
        rc = 1
    # every rank reaches the same barrier whether its check passed or not
    flags = [None] * world
    dist.all_gather_object(flags, rc)
    rc = max(flags)
    if rank == 0 and rc == 0:
        print(f"mgpu ops ok: mode={mode} world={world}")
    comm.close()
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(rc)


if __name__ == "__main__":
    main()
