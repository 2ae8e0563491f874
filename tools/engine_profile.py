"""Distributed engine profile (torchrun, one process per GPU): runs
tq_engine_run_query for a query over each rank's row-group subset several
times and prints rank 0's executor metrics (per-operator tasks / ms, exchange
decisions, run_ms) next to the Python fused plan's time.

    torchrun --nproc-per-node 2 tools/engine_profile.py [--q 3] [--sf 100]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]


def main():
    import torch
    import torch.distributed as dist
    ap = argparse.ArgumentParser()
    ap.add_argument("--q", type=int, default=3)
    ap.add_argument("--sf", type=float, default=100)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--threads", type=int, default=4)
    ap.add_argument("--pre-python", type=int, default=0, help="run the Python Q3 plans first (as bench.py)")
    ap.add_argument("--pre5", type=int, default=0, help="run config 5 (Host-tier Q5/Q9) first (as bench.py)")
    ap.add_argument("--keep", type=int, default=1)
    ap.add_argument("--kprof", type=int, default=0, help="per-kernel CUDA-event profile of the last rep")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    from paper_2508_05029_b200 import queries
    from paper_2508_05029_b200.ops import Comm, Context, engine_run_query
    ctx = Context(local, pool_reserve_bytes=int(float(os.environ.get("TQ_POOL_RESERVE_GB", "0")) * 1e9))
    uid = [Comm.unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    comm = Comm(ctx, rank, world, uid[0])
    names = queries.QUERY_TABLES[a.q]
    if a.pre5:
        # what bench.py runs before config 4: config 5 (Host-tier tables, Device budget)
        for q in (5, 9):
            host = {}
            for n in queries.QUERY_TABLES[q]:
                d = ctx.datagen(queries.TABLE_IDS[n], 12.5)
                host[queries.TABLE_IDS[n]] = d.to_host()
                d.free()
            data_bytes = sum(b.nbytes() for b in host.values())
            for _ in range(2):
                engine_run_query(ctx, q, host, compute_threads=4, preload=1, batch_rows=4 << 20,
                                 device_budget=max(int(data_bytes / 2.5), 1 << 30))
            del host
        if rank == 0:
            print("pre5 done", flush=True)
    t = {queries.TABLE_IDS[n]: ctx.datagen(queries.TABLE_IDS[n], a.sf, shard=rank, nshards=world) for n in names}
    if a.pre_python and a.q == 3:
        # what bench.py runs before the engine line: the Python fused plan (results kept)
        kept = []
        for fused in ((True, False, True) if a.pre_python == 1 else (True,)):
            if world > 1:
                dist.barrier()
            kept.append(queries.q3_distributed(ctx, comm, t[queries.TABLE_IDS["customer"]],
                                               t[queries.TABLE_IDS["orders"]], t[queries.TABLE_IDS["lineitem"]],
                                               {}, fused=fused, lip=a.pre_python != 2))
        ctx.sync()
        if not a.keep:
            for k in kept:
                k.free()
            kept = []
    for i in range(a.reps + 1):
        if world > 1:
            dist.barrier()
        if a.kprof and i == a.reps:
            ctx.profile(True)
        if i == a.reps and os.environ.get("TQ_HOST_TIMING") == "1":  # host phases of the last rep only
            import ctypes as C
            from paper_2508_05029_b200.ops import lib
            lib().tq_host_timing_report(C.create_string_buffer(1 << 16), 1 << 16)
        import ctypes as _C
        from paper_2508_05029_b200.ops import lib as _lib
        _lib().tq_device_bytes_reserved.restype = _C.c_uint64
        _lib().tq_device_bytes_reserved.argtypes = [_C.c_void_p]
        res0 = _lib().tq_device_bytes_reserved(ctx.handle)
        t0 = time.perf_counter()
        _, m = engine_run_query(ctx, a.q, t, comm=comm if world > 1 else None, compute_threads=a.threads,
                                batch_rows=1 << 40)
        wall = (time.perf_counter() - t0) * 1e3
        if rank == 0 and i:
            from paper_2508_05029_b200.ops import lib
            lib().tq_device_bytes_reserved.restype = __import__("ctypes").c_uint64
            lib().tq_device_bytes_reserved.argtypes = [__import__("ctypes").c_void_p]
            print("pool reserved GB before / after", res0 / 1e9, lib().tq_device_bytes_reserved(ctx.handle) / 1e9,
                  "in use GB", ctx.bytes_in_use() / 1e9, flush=True)
            ops = sorted(m["ops"].items(), key=lambda kv: -kv[1]["ms"])
            print(json.dumps({"rep": i, "wall_ms": round(wall, 3), "run_ms": round(m["run_ms"], 3),
                              "setup_ms": round(m["setup_ms"], 3), "tasks": m["tasks"],
                              "ops": {k: (v["tasks"], round(v["ms"], 3), round(v["gpu_ms"], 3), round(v["call_ms"], 3))
                                      for k, v in ops}}), flush=True)
            print("timeline", json.dumps([(n, k, round(a, 3), round(b, 3)) for n, k, a, b in m["timeline"]]),
                  flush=True)
    if rank == 0:
        print("jit", ctx.jit_report(), flush=True)
        if a.kprof:
            print("kernels", json.dumps({k: (v[0], round(v[1], 3)) for k, v in ctx.profile_report().items()}), flush=True)
    if rank == 0 and os.environ.get("TQ_HOST_TIMING") == "1":
        import ctypes as C
        from paper_2508_05029_b200.ops import lib
        buf = C.create_string_buffer(1 << 16)
        lib().tq_host_timing_report(buf, len(buf))
        print(buf.value.decode(), flush=True)
    comm.close()
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
