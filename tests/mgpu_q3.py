"""torchrun helper (one process per GPU): distributed Q3 through NCCL vs the
oracle.  Run by tests/test_multigpu.py; exits non-zero on mismatch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    from paper_2508_05029_b200 import queries
    from paper_2508_05029_b200.ops import Comm, Context
    ctx = Context(local)
    uid = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = Comm(ctx, rank, world, uid[0])
    sf = float(os.environ.get("TQ_SF", "0.1"))
    t = {name: ctx.datagen(queries.TABLE_IDS[name], sf, shard=rank, nshards=world)
         for name in ("customer", "orders", "lineitem")}
    if os.environ.get("TQ_ENGINE") == "1":
        # the C++ worker runtime with ExchangeOps (broadcast customer_f, hash orders_f / lineitem_f)
        from paper_2508_05029_b200.ops import engine_run_query
        out, m = engine_run_query(ctx, 3, {queries.TABLE_IDS[k]: v for k, v in t.items()}, comm=comm,
                                  compute_threads=4, batch_rows=256 * 1024)
    else:
        out = queries.q3_distributed(ctx, comm, t["customer"], t["orders"], t["lineitem"],
                                     lip=os.environ.get("TQ_LIP", "1") == "1",
                                     fused=os.environ.get("TQ_FUSED", "0") == "1").to_host()
    parts = [None] * world
    dist.all_gather_object(parts, out)
    rc = 0
    if rank == 0:
        import oracle as O
        from paper_2508_05029_b200.columnar import assert_batches_equal
        got = O.concat(parts)
        want = O.query(3, {tt: O.datagen(tt, sf) for tt in O.QUERY_TABLES[3]}, 8)
        try:
            assert_batches_equal(got, want)
            print(f"mgpu q3 ok: world={world} rows={got.rows} nvlink_bytes_sent={comm.bytes_sent()}")
        except AssertionError as e:
            print("MISMATCH", e)
            rc = 1
    comm.close()
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(rc)


if __name__ == "__main__":
    main()
