"""Stage-by-stage device timing of the config-4 Q3 shuffle plan on N ranks
(one process per GPU).  Prints, per stage, rank 0's time and the max over
ranks (CUDA events on each rank's stream, barrier before each repetition).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tools/profile_q3_dist.py --sf 100
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2508_05029_b200 import queries as Q  # noqa: E402
from paper_2508_05029_b200.expr import Col  # noqa: E402
from paper_2508_05029_b200.ops import Comm, Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=float, default=100)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nolip", action="store_true")
    ap.add_argument("--fused", action="store_true", help="fused partition + NVLink scatter")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    free, _ = torch.cuda.mem_get_info(local)
    ctx = Context(local, pool_reserve_bytes=int(free * 0.7))
    uid = [Comm.unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    comm = Comm(ctx, rank, world, uid[0])
    st = torch.cuda.ExternalStream(ctx.stream())
    t = {n: ctx.datagen(Q.TABLE_IDS[n], a.sf, shard=rank, nshards=world) for n in ("customer", "orders", "lineitem")}
    ctx.sync()
    lip = not a.nolip
    n = world
    for rep in range(a.reps):
        if world > 1:
            dist.barrier()
        marks = []
        ctx.profile(rep == a.reps - 1)
        if rep == a.reps - 1 and os.environ.get("TQ_HOST_TIMING") == "1":
            import ctypes as C
            from paper_2508_05029_b200.ops import lib
            lib().tq_host_timing_report(C.create_string_buffer(1 << 16), 1 << 16)  # only the last rep

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            marks.append((name, e))
        mark("start")
        if a.fused:
            cf = cb = comm.broadcast(t["customer"], Col(Q.C_MKTSEGMENT).eq(1), [Col(Q.C_CUSTKEY)])
            mark("customer filter+broadcast")
        else:
            cf = ctx.pipeline_materialize(t["customer"], Col(Q.C_MKTSEGMENT).eq(1), [Col(Q.C_CUSTKEY)])
            mark("customer filter")
            cb, _ = comm.allgather(cf)
            mark("customer allgather")
        ct = ctx.join_build(cb, [0], semi=True)
        mark("customer build")
        of = ctx.pipeline_probe(ct, t["orders"], Col(Q.O_ORDERDATE) < 9204,
                                [Col(Q.O_ORDERKEY), Col(Q.O_ORDERDATE), Col(Q.O_SHIPPRIORITY), Col(Q.O_CUSTKEY)],
                                [3], [])
        mark("orders filter+probe")
        bloom = None
        if a.fused:
            orx = comm.partition_exchange(of, None, None, [0])
            op = orx
            mark("orders fused partition+scatter")
            ot = ctx.join_build(orx, [0], bloom_keys=comm.last_exchange_capacity())
            mark("orders_f build")
            if lip:
                bloom = comm.gather_table_blooms(ot)
                mark("LIP gather table blooms")
            lrx = comm.partition_exchange(t["lineitem"], Col(Q.L_SHIPDATE) > 9204, [Col(Q.L_ORDERKEY), Q.REV], [0],
                                          bloom)
            lp = lrx
            mark("lineitem fused filter+semi+partition+scatter")
        else:
            if lip:
                bloom = ctx.bloom_build(of, [0], expected_keys=of.rows * n)
                mark("LIP bloom build")
                comm.bloom_union(bloom)
                mark("LIP bloom union")
            op, ooff = ctx.hash_partition(of, [0], n)
            mark("orders partition")
            orx, _ = comm.exchange(op, ooff)
            mark("orders exchange")
            if lip:
                lp, loff = ctx.pipeline_partition_semi(t["lineitem"], Col(Q.L_SHIPDATE) > 9204,
                                                       [Col(Q.L_ORDERKEY), Q.REV], [0], n, bloom)
            else:
                lp, loff = ctx.pipeline_partition(t["lineitem"], Col(Q.L_SHIPDATE) > 9204, [Col(Q.L_ORDERKEY), Q.REV],
                                                  [0], n)
            mark("lineitem filter+partition")
            lrx, _ = comm.exchange(lp, loff)
            mark("lineitem exchange")
            ot = ctx.join_build(orx, [0])
            mark("orders_f build")
        j = ctx.pipeline_probe(ot, lrx, None, None, [0], [1, 2])
        mark("lineitem probe")
        out = ctx.aggregate_execute(j, [2, 0, 1], [(Q.AGG_SUM, 3)])
        mark("aggregate")
        torch.cuda.synchronize()
        ctx.sync()
        times = [(n1, e0.elapsed_time(e1)) for (_, e0), (n1, e1) in zip(marks, marks[1:])]
        if world > 1:
            allt = [None] * world
            dist.all_gather_object(allt, times)
        else:
            allt = [times]
        if rank == 0 and rep == a.reps - 1:
            print(f"world={world} sf={a.sf:g} lip={lip} fused={a.fused}")
            for i, (name, ms) in enumerate(times):
                mx = max(r[i][1] for r in allt)
                print(f"  {name:28s} rank0 {ms:8.3f} ms   max {mx:8.3f} ms", flush=True)
            tot = [sum(x[1] for x in r) for r in allt]
            print(f"  total rank0 {tot[0]:.3f} ms  max {max(tot):.3f} ms", flush=True)
            if os.environ.get("TQ_HOST_TIMING") == "1":
                import ctypes as C
                from paper_2508_05029_b200.ops import lib
                buf = C.create_string_buffer(1 << 16)
                lib().tq_host_timing_report(buf, len(buf))
                print(buf.value.decode())
            prof = ctx.profile_report()
            print("  kernels (rank0): " + ", ".join(f"{k} {v[0]}x {v[1]:.3f} ms" for k, v in sorted(prof.items())))
        for x in {id(x): x for x in (cf, cb, of, op, orx, lp, lrx, j, out)}.values():
            x.free()
        for x in (ct, ot):
            x.free()
        if bloom is not None:
            bloom.free()
    comm.close()
    ctx.close()


if __name__ == "__main__":
    main()
