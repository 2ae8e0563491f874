#!/usr/bin/env python
"""bench.py — TPC-H Q1-style group-by over synthetic lineitem SF10 per GPU
(BASELINE.json configs[1]) through libtq_gpu.so, plus the reference arm.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tq|reference]

Prints ONE JSON line (rank 0).  Timing: CUDA events on the stream the
pipeline kernels run on, W untimed warm-up steps, K timed steps bracketed by a
barrier + device synchronize, max over ranks.  Inputs (5.3 GB of scanned
columns per GPU) are larger than the 126 MB L2, so no flush is needed.
N > 1: one process per GPU (torchrun); each rank generates and scans its own
row-group subset of an SF(10*N) lineitem (weak scaling); the per-rank partial
aggregates (4 groups) are merged on rank 0 after timing.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep stdout to the one JSON line

METRIC = "query latency (ms) and input rows/sec per TPC-H-style query at 1/2/4/8 B200"
SF_PER_GPU = float(os.environ.get("TQ_BENCH_SF", "10"))  # override: quick test runs only
Q1_BYTES_PER_ROW = 88  # rf 8 + ls 8 + qty 16 + ep 16 + disc 16 + tax 16 + shipdate 8


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return None


def ncu_traffic(kernel: str):
    """dram bytes/launch of `kernel` from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line). Each rank polls NVML for its OWN GPU
    from a background thread that runs from just before the opening event to
    just after the closing synchronize (ctypes NVML calls release the GIL, so
    the launching thread is not held up); rank 0 merges every rank's samples. (An nvidia-smi -lms subprocess block-buffers its
    output and produced no samples inside a ~10 ms timed region.)"""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.h = None
        self.sm, self.mx, self.bits = [], None, 0
        if os.environ.get("TQ_BENCH_CLOCKS", "1") == "0":
            return
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(device).uuid))
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.h = None

    def sample(self):
        if self.h is None:
            return
        try:
            self.sm.append(float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)))
            self.bits |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        except Exception:
            pass

    def start(self, period_s: float = 0.001):
        """Background sampler thread for the timed region (NVML calls release the GIL)."""
        import threading
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                self.sample()
                time.sleep(period_s)
        self._thr = threading.Thread(target=run, daemon=True)
        self._thr.start()

    def stop(self):
        if getattr(self, "_thr", None):
            self._stop.set()
            self._thr.join()
            self._thr = None

    def report(self, world: int):
        mine = {"sm": self.sm, "mx": self.mx, "bits": self.bits}
        alls = [mine]
        if world > 1:
            import torch.distributed as dist
            alls = [None] * world
            dist.all_gather_object(alls, mine)
        sm = [x for a in alls for x in a["sm"]]
        if not sm:
            return None
        bits = 0
        for a in alls:
            bits |= a["bits"]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(a["mx"] or 0 for a in alls),
                "reasons": sorted(n for n, b in self.REASONS.items() if bits & b), "samples": len(sm),
                "samples_by_rank": [len(a["sm"]) for a in alls],
                "source": "NVML clocks/event reasons polled by every rank for its own GPU inside the timed region"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, x: float) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_ranks(world, x: float) -> list:
    if world == 1:
        return [x]
    import torch
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, x)
    return out


def sum_over_ranks(world, x: float) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def host_info(nthreads: int) -> dict:
    """What bounds the CPU baseline on this box: core count,
    cgroup CPU quota, CPU model and host memory read bandwidth."""
    info = {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    for path in ("/sys/fs/cgroup/cpu.max", "/sys/fs/cgroup/cpu/cpu.cfs_quota_us"):
        try:
            with open(path) as f:
                info["cgroup_cpu_max"] = f.read().strip()
                break
        except OSError:
            continue
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        info["read_bw_gbs_1thread"] = round(O.host_read_bw(1 << 30, 1, 3), 2)
        info["read_bw_gbs_all"] = round(O.host_read_bw(1 << 30, nthreads, 3), 2)
    except Exception as e:  # the reference build (oracle/_ref) is missing
        info["read_bw_error"] = str(e)[:120]
    return info


def cpu_q1_fused_ref(li_host, nthreads: int, reps: int):
    """Q1 as one fused pass over the REFERENCE's own ColumnBatch accessors
    (oracle/_ref, compiled from the reference sources): rows/s list + result."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    r = O.RefResident(li_host)
    try:
        res, _ = r.q1_fused(nthreads)  # warm
        rates = []
        for _ in range(reps):
            res, sec = r.q1_fused(nthreads)
            rates.append(li_host.rows / sec)
    finally:
        r.close()
    return rates, res


def cpu_q1_sample(sf: float, nthreads: int, reps: int):
    """Oracle (CPU port) Q1 on a bounded lineitem sample; returns rows/s list."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    li = O.datagen(O.T_LINEITEM, sf, nthreads)
    tabs = {O.T_LINEITEM: li}
    O.query(1, tabs, nthreads)  # warm
    rates = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.query(1, tabs, nthreads)
        rates.append(li.rows / (time.perf_counter() - t0))
    return rates, li.rows


def run_reference(args, world, rank):
    """--impl reference: the reference path's CPU implementation on this box's
    host cores, on the SAME workload as the GPU arm (Q1 over lineitem SF10):
    one fused pass per step over the reference's own ColumnBatch / Column
    accessors (oracle/_ref, built from the reference sources; the reference
    ships no operator code), all host threads, the batch resident
    in host memory (as the GPU arm's tables are in HBM)."""
    if rank != 0:
        return
    nthreads = len(os.sched_getaffinity(0)) or os.cpu_count() or 1
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    li = O.datagen(O.T_LINEITEM, SF_PER_GPU, nthreads)
    r = O.RefResident(li)
    try:
        for _ in range(args.warmup):
            r.q1_fused(nthreads)
        ts = []
        for _ in range(args.steps):
            _, sec = r.q1_fused(nthreads)
            ts.append(sec)
    finally:
        r.close()
    sec = sum(ts) / len(ts)
    value = li.rows / sec
    sample = (f"full lineitem SF{SF_PER_GPU:g} ({li.rows} rows, same workload as the GPU arm); fused Q1 over the "
              f"reference's Column::i64_at / dec_at, {nthreads} threads")
    line = {
        "metric": METRIC, "value": value, "unit": "rows/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int128", "data": "synthetic",
        "config": {"workload": f"TPC-H Q1-style filter+project+group-by over lineitem SF{SF_PER_GPU:g} per GPU",
                   "query": "q1", "sf_per_gpu": SF_PER_GPU, "rows_per_gpu": li.rows, "same_config": True},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": nthreads, "kind": "reference", "sample": sample,
                         "host": host_info(nthreads)},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def timed(ctx, fn, reps, world, stream, keep=False):
    """median device ms of fn() over reps (after one warm-up), max over ranks;
    keep=True also returns the last output (host copy) for the parity check."""
    import torch
    fn().free()
    ctx.sync()
    ms = []
    last = None
    for i in range(reps):
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ctx.sync()
        ms.append(e0.elapsed_time(e1))
        if keep and i == reps - 1:
            last = out.to_host()
        out.free()
    if os.environ.get("TQ_BENCH_VERBOSE"):
        print(f"[timed rank{os.environ.get('RANK', '0')}] {[round(x, 3) for x in ms]}", file=sys.stderr, flush=True)
    m = max_over_ranks(world, statistics.median(ms))
    return (m, last) if keep else m


class OracleTables:
    """The CPU oracle's copy of the synthetic tables (test infrastructure: the
    parity checker of the timed results, never the thing measured)."""

    def __init__(self, nthreads):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        self.O = O
        self.nthreads = nthreads
        self.cache = {}

    def get(self, t, sf):
        if (t, sf) not in self.cache:
            self.cache[(t, sf)] = self.O.datagen(t, sf, self.nthreads)
        return self.cache[(t, sf)]

    def query(self, q, sf):
        return self.O.query(q, {t: self.get(t, sf) for t in self.O.QUERY_TABLES[q]}, self.nthreads)

    def drop(self):
        self.cache.clear()


def local_device() -> int:
    return int(os.environ.get("LOCAL_RANK", "0"))


def pinned_h2d_gbs(device: int, stream, nbytes: int = 1 << 30, reps: int = 5) -> float:
    """Pinned host -> device copy bandwidth on this box, measured in the same run
    (the denominator of the config-5 Host-tier runs' H2D GB/s): best of `reps`
    1-GiB cudaMemcpyAsync copies, CUDA events on the bench stream."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
    best = 0.0
    with torch.cuda.stream(stream):
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dst.copy_(src, non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del src, dst
    return best


def check(got, want) -> str:
    """'exact' (integers / decimals / keys bit-exact after canonical sort,
    Float64 within 1e-9 relative) or the mismatch."""
    from paper_2508_05029_b200.columnar import assert_batches_equal
    try:
        assert_batches_equal(got, want)
        return "exact"
    except AssertionError as e:
        return f"MISMATCH: {str(e)[:200]}"


def q3_sharded_parity(got, sf, nthreads, shards=(0, 57), nshards=100) -> str:
    """Config-4 result (Q3 at SF100) vs the oracle, exact on sampled orderkey
    shards: the group-by key l_orderkey is co-partitioned with the orders
    row-group subsets, so the result's groups whose orderkey lies in orders
    shard s are exactly the oracle's Q3 over (all customers, orders shard s,
    lineitem shard s = the lines of those orders)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle as O
    no = O.table_rows(O.T_ORDERS, sf)
    cust = O.datagen(O.T_CUSTOMER, sf, nthreads)
    keys = got.cols[0].i64()
    groups = 0
    for s in shards:
        lo, hi = no * s // nshards, no * (s + 1) // nshards  # orderkeys lo+1 .. hi
        tabs = {O.T_CUSTOMER: cust, O.T_ORDERS: O.datagen(O.T_ORDERS, sf, nthreads, s, nshards),
                O.T_LINEITEM: O.datagen(O.T_LINEITEM, sf, nthreads, s, nshards)}
        want = O.query(3, tabs, nthreads)
        sel = O.take(got, np.nonzero((keys > lo) & (keys <= hi))[0].tolist())
        r = check(sel, want)
        if r != "exact":
            return f"shard {s}: {r}"
        groups += want.rows
    return f"exact on orderkey shards {list(shards)} of {nshards} ({groups} groups)"


def run_suite(args, ctx, world, rank, stream, oracle, parity):
    """The other BASELINE.json configs: Q6/Q3/Q5/Q9 at SF10 on one GPU, and the
    config-4 Q3 shuffle join (broadcast + NCCL all-to-all over NVLink) at
    SF{shuffle_sf} total, strong scaling over the N GPUs.  Every timed result
    is checked against the CPU oracle (`parity`, filled in place)."""
    import torch.distributed as dist
    from paper_2508_05029_b200 import queries
    from paper_2508_05029_b200.ops import Comm
    suite = {}
    do_parity = os.environ.get("TQ_BENCH_PARITY", "1") == "1"
    if world == 1:
        sf = SF_PER_GPU
        names = ["customer", "orders", "lineitem", "supplier", "part", "partsupp", "nation", "region"]
        t = {n: ctx.datagen(queries.TABLE_IDS[n], sf) for n in names}
        li6 = t["lineitem"].select(queries.Q6_SCAN)
        ms, out = timed(ctx, lambda: queries.q6_scan(ctx, li6), 5, world, stream, keep=True)
        key = f"q6_sf{sf:g}"
        suite[key] = {"ms": ms, "rows_per_s": t["lineitem"].rows / (ms * 1e-3),
                      "hbm_gbs": t["lineitem"].rows * queries.Q6_SCAN_BYTES_PER_ROW / (ms * 1e-3) / 1e9}
        if do_parity:
            parity[key] = suite[key]["parity"] = check(out, oracle.query(6, sf))
        for q in (3, 5, 9):
            rows = sum(t[n].rows for n in queries.QUERY_TABLES[q])
            ms, out = timed(ctx, lambda: queries.run_join_query(ctx, q, t), 3, world, stream, keep=True)
            key = f"q{q}_sf{sf:g}"
            suite[key] = {"ms": ms, "rows_per_s": rows / (ms * 1e-3)}
            if do_parity:
                parity[key] = suite[key]["parity"] = check(out, oracle.query(q, sf))
        for v in t.values():
            v.free()
        oracle.drop()
        # per-operator HBM roofline (each SPEC operator alone, SF10, kernel
        # time vs algorithmic bytes; tools/op_roofline.py)
        if os.environ.get("TQ_BENCH_OPS", "1") == "1":
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import op_roofline
            peaks = measured_peaks()
            suite["operators_sf10"] = op_roofline.measure(ctx, sf, stream, peaks["hbm_gbs"] if peaks else 6538.6)
        # config 5 (one worker's share: SF100 / 8 GPUs): Q5 / Q9 on the C++ worker
        # runtime with the tables in the pinned Host tier and a Device budget of a
        # quarter of the data, so scans go through load_to_device / preload and
        # holders spill (PCIe-bound by design)
        from paper_2508_05029_b200.ops import engine_run_query
        sf5 = args.spill_sf
        h2d_peak = pinned_h2d_gbs(local_device(), stream)
        for q in (5, 9):
            names = queries.QUERY_TABLES[q]
            host = {}
            for n in names:
                d = ctx.datagen(queries.TABLE_IDS[n], sf5)
                host[queries.TABLE_IDS[n]] = d.to_host()
                d.free()
            data_bytes = sum(b.nbytes() for b in host.values())
            rows = sum(b.rows for b in host.values())
            runs = []
            for _ in range(2):
                res, m = engine_run_query(ctx, q, host, compute_threads=4, preload=1, batch_rows=4 << 20,
                                          device_budget=max(int(data_bytes / 2.5), 1 << 30))
                runs.append(m)
            m = runs[-1]
            key = f"q{q}_engine_hosttier_sf{sf5:g}"
            suite[key] = {
                "ms": m["run_ms"], "rows_per_s": rows / (m["run_ms"] * 1e-3), "host_tier_bytes": data_bytes,
                "device_budget": m["device_capacity"], "loads": m["loads"], "preloads": m["preloads"],
                "spills": m["spills"], "spill_bytes": m["spill_bytes"], "h2d_bytes": m["load_bytes"],
                "h2d_gbs": m["load_bytes"] / (m["run_ms"] * 1e-3) / 1e9, "pinned_h2d_probe_gbs": h2d_peak,
                "h2d_frac_of_probe": m["load_bytes"] / (m["run_ms"] * 1e-3) / 1e9 / h2d_peak if h2d_peak else None,
                "oom_retries": m["oom_retries"],
                "tasks": m["tasks"], "timing": "host wall clock of tq_engine_run_query's run phase"}
            if do_parity:
                parity[key] = suite[key]["parity"] = check(res, oracle.O.query(q, host, oracle.nthreads))
            del host
    # config 4: distributed shuffle join
    uid = [Comm.unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    comm = Comm(ctx, rank, world, uid[0])
    sf = args.shuffle_sf
    t = {n: ctx.datagen(queries.TABLE_IDS[n], sf, shard=rank, nshards=world) for n in ("customer", "orders", "lineitem")}
    rows = sum_over_ranks(world, float(sum(v.rows for v in t.values())))
    results = {}
    for fused in (True, False):
        b0 = comm.bytes_sent()
        stats = {}
        ms, out = timed(ctx, lambda: queries.q3_distributed(ctx, comm, t["customer"], t["orders"], t["lineitem"], stats,
                                                            fused=fused), 3, world, stream, keep=True)
        sent = (comm.bytes_sent() - b0) / 4.0  # 1 warm-up + 3 timed runs
        key = f"q3_shuffle_sf{sf:g}" if fused else f"q3_shuffle_nccl_sf{sf:g}"
        results[key] = out
        suite[key] = {
            "ms": ms, "rows_per_s": rows / (ms * 1e-3), "scaling": "strong", "n_gpus": world,
            "nvlink_bytes_sent_per_gpu": sent, "nvlink_gbs_per_gpu": sent / (ms * 1e-3) / 1e9,
            "nvlink_frac_of_770": sent / (ms * 1e-3) / 770e9,
            "exchange": ("customer_f broadcast (allgather); orders_f, lineitem_f: fused partition + scatter into "
                         "the destination rank's CUDA-IPC window over NVLink (fnv1a64 mod N)") if fused else
                        ("customer_f broadcast (allgather); orders_f, lineitem_f hash-partitioned (fnv1a64 mod N) "
                         "then NCCL grouped send/recv"),
            "recv_rows_rank0": {k: v for k, v in stats.items()},
        }
    if world > 1:
        # LIP off: the lineitem shuffle ships every filtered row; the scatter
        # kernels' NVLink throughput = bytes stored into other ranks' windows /
        # the scatter kernels' time (CUDA events around each launch)
        queries.q3_distributed(ctx, comm, t["customer"], t["orders"], t["lineitem"], fused=True, lip=False).free()
        ctx.sync()
        barrier(world)
        b0 = comm.bytes_sent()
        ctx.profile(True)
        queries.q3_distributed(ctx, comm, t["customer"], t["orders"], t["lineitem"], fused=True, lip=False).free()
        ctx.sync()
        prof = ctx.profile_report()
        ctx.profile(False)
        sent = comm.bytes_sent() - b0
        n_sc, sc_ms = prof.get("pipe_scatter", (0, 0.0))
        n_bc, bc_ms = prof.get("pipe_broadcast", (0, 0.0))
        gbs = sent / ((sc_ms + bc_ms) * 1e-3) / 1e9 if sc_ms else None
        gbs = max_over_ranks(world, gbs or 0.0)
        suite[f"q3_shuffle_nolip_sf{sf:g}_scatter"] = {
            "nvlink_bytes_sent_per_gpu": sent, "scatter_kernels_ms": sc_ms + bc_ms, "launches": n_sc + n_bc,
            "nvlink_gbs_per_gpu": gbs, "nvlink_frac_of_770": gbs / 770.0 if gbs else None,
            "what": "fused partition + scatter / broadcast kernels of config 4 without LIP: remote bytes stored "
                    "over NVLink per GPU / those kernels' CUDA-event time (max over ranks)"}
    # the same query through the C++ worker runtime (tq_engine_run_query): its
    # distributed Q3 plan decides the exchanges itself (exchange_decide) and
    # runs them over the same fused NVLink kernels; one batch per table shard
    from paper_2508_05029_b200.ops import engine_run_query
    tabs = {queries.TABLE_IDS[n]: v for n, v in t.items()}
    runs = []
    for i in range(4):
        barrier(world)
        if i == 3:
            ctx.profile(True)
        res, m = engine_run_query(ctx, 3, tabs, comm=comm if world > 1 else None, compute_threads=4,
                                  batch_rows=1 << 40)
        if i:
            runs.append(m["run_ms"])
    eprof = ctx.profile_report()
    ctx.profile(False)
    key = f"q3_shuffle_engine_sf{sf:g}"
    ms = max_over_ranks(world, statistics.median(runs))
    results[key] = res
    suite[key] = {"ms": ms, "rows_per_s": rows / (ms * 1e-3), "scaling": "strong", "n_gpus": world,
                  "timing": "host wall clock of tq_engine_run_query's run phase (median of 3), max over ranks",
                  "exchange_decisions": m.get("exchange_decisions"), "tasks": m.get("tasks"),
                  "runs_ms_rank0": [round(r, 3) for r in runs], "spills": m.get("spills"),
                  "ops_ms_last_run": {k: [round(v["ms"], 3), round(v.get("gpu_ms", 0.0), 3)] for k, v in
                                      sorted(m.get("ops", {}).items(), key=lambda kv: -kv[1]["ms"])[:6]},
                  "kernels_last_run": {k: (v[0], round(v[1], 3)) for k, v in eprof.items()},
                  "timeline_last_run": [(n, k, round(a, 3), round(b, 3)) for n, k, a, b in m.get("timeline", [])]}
    for v in t.values():
        v.free()
    comm.close()
    if do_parity:
        # the ranks' results concatenated (co-partitioned groups: disjoint)
        import torch.distributed as dist
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        full = {}
        for key, out in results.items():
            parts = [out]
            if world > 1:
                parts = [None] * world
                dist.all_gather_object(parts, out)
            full[key] = O.concat(parts)
        if rank == 0:
            k_f, k_n = f"q3_shuffle_sf{sf:g}", f"q3_shuffle_nccl_sf{sf:g}"
            r = q3_sharded_parity(full[k_f], sf, oracle.nthreads)
            parity[k_f] = suite[k_f]["parity"] = r
            # the unfused (NCCL) plan: the whole result equals the fused plan's
            # (two GPU code paths), and the same oracle shards
            same = check(full[k_n], full[k_f])
            parity[k_n] = suite[k_n]["parity"] = (
                q3_sharded_parity(full[k_n], sf, oracle.nthreads) + f"; full result vs fused plan: {same}")
            k_e = f"q3_shuffle_engine_sf{sf:g}"
            parity[k_e] = suite[k_e]["parity"] = (
                q3_sharded_parity(full[k_e], sf, oracle.nthreads) + f"; full result vs fused plan: "
                f"{check(full[k_e], full[k_f])}")
    return suite


def run_tq(args, world, rank, local):
    import ctypes as C

    import numpy as np
    import torch

    from paper_2508_05029_b200 import queries
    from paper_2508_05029_b200.columnar import HostBatch, TqBatchC
    from paper_2508_05029_b200.ops import Context, DeviceBatch, lib

    torch.cuda.set_device(local)
    # map most of the GPU's memory into the context's pool once: the suite's
    # SF100 tables and the queries' temporaries then never map memory mid-query
    free, _ = torch.cuda.mem_get_info(local)
    ctx = Context(local, pool_reserve_bytes=int(free * 0.7))
    sf_total = SF_PER_GPU * world
    li = ctx.datagen(1, sf_total, shard=rank, nshards=world)
    scan = li.select(queries.Q1_SCAN)
    rows = scan.rows
    stream = torch.cuda.ExternalStream(ctx.stream())
    partial = world > 1

    def step():
        out = queries.q1_scan(ctx, scan, partial=partial)
        return out

    for _ in range(args.warmup):
        step().free()
    ctx.sync()
    barrier(world)
    clocks = Clocks(local)
    clocks.start()
    ctx.profile(True)
    l0 = ctx.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    outs = []
    for _ in range(args.steps):
        outs.append(step())
    e1.record(stream)
    torch.cuda.synchronize()
    ctx.sync()
    clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    launches = ctx.kernel_launches() - l0
    prof = ctx.profile_report()
    ctx.profile(False)
    ck = clocks.report(world)
    barrier(world)
    ms_max = max_over_ranks(world, ms)
    ms_ranks = gather_ranks(world, round(ms, 4))
    total_rows = sum_over_ranks(world, float(rows))
    result = outs[-1].to_host()
    for o in outs:
        o.free()

    # ---- end to end through the public API: pinned host columns -> H2D ->
    # Q1 -> D2H of the result, every step
    host = ctx.download(scan)
    pinned = []
    hb = HostBatch(host.rows)
    for c in host.cols:
        p = C.c_void_p()
        Context._check(lib().tq_pinned_alloc(max(1, c.values.size), C.byref(p)))
        arr = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)), (max(1, c.values.size),))
        arr[:c.values.size] = c.values
        pinned.append(p)
        hb.cols.append(type(c)(c.kind, arr[:c.values.size], None, None, c.precision, c.scale))
    del host
    hc = hb.to_c()
    h2d = sum(c.values.size for c in hb.cols)

    def e2e_step():
        out = TqBatchC()
        Context._check(lib().tq_batch_upload(ctx.handle, C.byref(hc), C.byref(out), None))
        d = DeviceBatch(ctx, out)
        r = queries.q1_scan(ctx, d, partial=partial)
        res = r.to_host()
        r.free()
        d.free()
        return res

    for _ in range(max(1, min(args.warmup, 2))):
        e2e_step()
    ctx.sync()
    barrier(world)
    ee = max(2, min(args.steps, 5))
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(ee):
        res = e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3) / ee
    e2e_ms = max_over_ranks(world, e2e_ms)
    d2h = res.nbytes()
    for p in pinned:
        lib().tq_pinned_free(p)

    # ---- correctness of what was timed vs the CPU oracle
    nthreads = os.cpu_count() or 1
    oracle = OracleTables(nthreads)
    parity = {}
    q1_want = None
    if os.environ.get("TQ_BENCH_PARITY", "1") == "1":
        key = f"q1_sf{SF_PER_GPU:g}_per_gpu"
        if world == 1:
            q1_want = oracle.query(1, sf_total)
            parity[key] = check(result, q1_want)
        elif rank == 0:
            # each rank returns its shard's partial aggregates (merged after
            # timing): rank 0's partial vs the oracle's operators on that shard
            O = oracle.O
            shard = O.datagen(O.T_LINEITEM, sf_total, nthreads, 0, world)
            proj = O.project_execute(O.filter_execute(shard, queries.Q1_PRED), queries.Q1_EXPRS)
            parity[key] = "rank-0 shard partial: " + check(result, O.aggregate_execute(proj, queries.Q1_KEYS,
                                                                                        queries._Q1_PARTIAL_AGGS))
            del shard, proj

    cpu = None
    if rank == 0 and world == 1:
        # two CPU implementations on this box's cores, the faster is the baseline:
        # the materialising oracle port (SF1 sample) and one fused pass over the
        # reference's own accessors (full SF10, the GPU arm's workload)
        nthreads = len(os.sched_getaffinity(0)) or os.cpu_count() or 1
        rates, srows = cpu_q1_sample(1.0, nthreads, 3)
        port = {"value": statistics.median(rates), "unit": "rows/s", "cores": nthreads, "kind": "port",
                "sample": f"oracle Q1 on lineitem SF1 ({srows} rows), median of 3, {nthreads} threads"}
        fused = None
        try:
            li_host = oracle.get(oracle.O.T_LINEITEM, sf_total)
            frates, fres = cpu_q1_fused_ref(li_host, nthreads, 3)
            fused = {"value": statistics.median(frates), "unit": "rows/s", "cores": nthreads, "kind": "reference",
                     "sample": f"fused Q1 over the reference's Column accessors, full lineitem SF{sf_total:g} "
                               f"({li_host.rows} rows), median of 3, {nthreads} threads",
                     "parity": check(fres, q1_want if q1_want is not None else oracle.query(1, sf_total))}
        except Exception as e:
            fused = {"error": str(e)[:200]}
        best = fused if fused and fused.get("value", 0) > port["value"] else port
        cpu = dict(best)
        cpu["alternatives"] = {"port": port, "reference_fused": fused}
        cpu["host"] = host_info(nthreads)
    oracle.drop()

    del li, scan
    suite = run_suite(args, ctx, world, rank, stream, oracle, parity) if args.suite else None
    if rank != 0:
        ctx.close()
        return
    peaks = measured_peaks()
    peak = peaks["hbm_gbs"] if peaks else 6650.0
    n_agg, agg_ms = prof.get("pipe_agg", (0, 0.0))
    kern_ms = agg_ms / max(1, n_agg)
    achieved = Q1_BYTES_PER_ROW * rows / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else None
    value = total_rows / (ms_max * 1e-3)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "rows/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_max,
        "ms_per_step_by_rank": ms_ranks,
        "parity": parity,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int128",
        "data": "synthetic (counter-based SplitMix64 TPC-H-style tables, DESIGN.md §4)",
        "config": {
            "workload": f"TPC-H Q1-style filter+project+group-by over lineitem SF{SF_PER_GPU:g} per GPU",
            "query": "q1", "sf_per_gpu": SF_PER_GPU, "rows_per_gpu": rows, "scan_bytes_per_row": Q1_BYTES_PER_ROW,
            "l2": "scanned columns (%.1f GB/GPU) > 126 MB L2; no flush needed" % (rows * Q1_BYTES_PER_ROW / 1e9),
            "parallelism": f"dp{world} (row-group subsets, partial aggregates merged)",
        },
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": ncu_traffic("pipe_agg"),
            "traffic_unit": "bytes/launch (dram read+write, ncu)",
            "kernel": "tq_jit_main = pipe_body<SINK_AGG> (NVRTC-specialised)", "kernel_ms": kern_ms,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "B200_PROFILING.md fallback",
            "algorithmic_bytes_per_row": Q1_BYTES_PER_ROW,
        },
        "cpu_baseline": cpu,
        "e2e": {"value": total_rows / (e2e_ms * 1e-3), "unit": "rows/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": launches,
        "kernels_ms": {k: v[1] / max(1, v[0]) for k, v in prof.items()},
        "clocks": ck,
        "jit": ctx.jit_report(),
        "suite": suite,
    }
    print(json.dumps(line), flush=True)
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tq", choices=["tq", "reference"])
    ap.add_argument("--suite", type=int, default=1, help="also time the other BASELINE configs")
    ap.add_argument("--shuffle-sf", type=float, default=100.0, help="total SF of the config-4 shuffle join")
    ap.add_argument("--spill-sf", type=float, default=12.5, help="SF of the config-5 Host-tier engine runs")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_tq(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
