"""Per-operator HBM roofline: every SPEC operator of the hot path run alone on
synthetic lineitem / orders (SF10, inputs far larger than the 126 MB L2),
timed with CUDA events on the context stream, against its ALGORITHMIC bytes
(each referenced input column read once + each materialised output written
once + one table entry per build row / probed row).

    python tools/op_roofline.py [--sf 10]       (bench.py embeds measure())

`op_ms` brackets the whole operator call (its kernels, scans, fix-ups and the
host sync that returns the row count); `kernel_ms` is the sum of the
operator's pipeline-kernel launches (CUDA events around each launch).
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def measure(ctx, sf: float, stream, peak_gbs: float, reps: int = 5) -> dict:
    import torch

    from paper_2508_05029_b200 import queries as Q
    from paper_2508_05029_b200.expr import Col

    li = ctx.datagen(Q.TABLE_IDS["lineitem"], sf)
    od = ctx.datagen(Q.TABLE_IDS["orders"], sf)
    L = li.select([Q.L_ORDERKEY, Q.L_EXTPRICE, Q.L_DISCOUNT, Q.L_SHIPDATE])  # 8 + 16 + 16 + 8 = 48 B/row
    n = L.rows
    rev = Col(1) * (Q.Dec(100) - Col(2))
    proj = ctx.project_execute(L, [Col(0), rev])  # orderkey, rev: 24 B/row (input of the partition op)
    ot = ctx.join_build(od.select([Q.O_ORDERKEY, Q.O_ORDERDATE]), [0])  # every lineitem row matches once
    res = {}

    only = os.environ.get("TQ_OPS")

    def run(name, fn, algo_bytes, note, rows_in):
        if only and name not in only.split(","):
            return
        fn().free()
        ctx.sync()
        op, kern = [], []
        out_rows = 0
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ctx.profile(True)
            e0.record(stream)
            out = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ctx.sync()
            prof = ctx.profile_report()
            ctx.profile(False)
            op.append(e0.elapsed_time(e1))
            kern.append(sum(v[1] for v in prof.values()))
            by_kernel = {k: round(v[1], 4) for k, v in prof.items()}
            out_rows = out.rows if hasattr(out, "rows") else 0
            out.free()
        op_ms, k_ms = statistics.median(op), statistics.median(kern)
        b = algo_bytes(out_rows)
        res[name] = {"rows_in": rows_in, "rows_out": out_rows, "algorithmic_bytes": b,
                     "op_ms": round(op_ms, 4), "kernel_ms": round(k_ms, 4),
                     "kernel_gbs": round(b / (k_ms * 1e-3) / 1e9, 1) if k_ms else None,
                     "kernel_frac_of_hbm": round(b / (k_ms * 1e-3) / 1e9 / peak_gbs, 3) if k_ms else None,
                     "op_gbs": round(b / (op_ms * 1e-3) / 1e9, 1), "kernels_ms": by_kernel, "note": note}

    run("filter_execute", lambda: ctx.filter_execute(L, Col(3) > 9204),
        lambda m: n * 48 + m * 48, "4 lineitem cols, shipdate > 1995-03-15 (54%); COUNT pass + stable EMIT pass", n)
    run("project_execute", lambda: ctx.project_execute(L, [Col(0), rev]),
        lambda m: n * 40 + m * 24, "orderkey, ep*(100-disc): dense single pass", n)
    run("hash_partition", lambda: _Part(ctx.hash_partition(proj, [0], 8)),
        lambda m: n * 24 + m * 24, "fnv1a64(orderkey) mod 8, stable per part; COUNT + EMIT", n)
    run("join_build", lambda: _Tab(ctx.join_build(od.select([Q.O_ORDERKEY, Q.O_ORDERDATE]), [0]), od.rows),
        lambda m: od.rows * (8 + 16 + 4), "orders.orderkey: 16-B {row, key} entry (128-bit CAS) + Bloom word", od.rows)
    run("join_probe_pkfk", lambda: ctx.join_probe(ot, L, [0]),
        lambda m: n * 48 + n * 16 + m * (16 + 48),
        "every lineitem row matches one order: table (512 MB) entry per row, output = build cols + probe cols", n)
    run("pipeline_probe_filtered", lambda: ctx.pipeline_probe(ot, li, Col(Q.L_SHIPDATE) > 9204, [Col(Q.L_ORDERKEY), Q.REV],
                                                         [0], [1]),
        lambda m: n * 48 + m * (16 + 32), "lineitem filter (54%) + project + probe of all orders (every passing row matches)", n)
    run("aggregate_q1", lambda: Q.q1_scan(ctx, li.select(Q.Q1_SCAN)),
        lambda m: n * Q.Q1_SCAN_BYTES_PER_ROW, "Q1 filter+project+group-by (4 groups, 8 aggregates)", n)
    run("aggregate_high_card", lambda: ctx.aggregate_execute(proj, [0], [(Q.AGG_SUM, 1)]),
        lambda m: n * 24 + m * 24, "group by orderkey (15M groups per SF10), Sum(rev)", n)
    ot.free()
    proj.free()
    li.free()
    od.free()
    return res


class _Part:
    """(batch, offsets) -> freeable with a row count."""
    def __init__(self, r):
        self.b = r[0]
        self.rows = self.b.rows

    def free(self):
        self.b.free()


class _Tab:
    def __init__(self, t, rows):
        self.t = t
        self.rows = rows

    def free(self):
        self.t.free()


def main():
    import json

    import torch

    from paper_2508_05029_b200.ops import Context
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=float, default=10)
    a = ap.parse_args()
    ctx = Context(0)
    st = torch.cuda.ExternalStream(ctx.stream())
    peak = 6538.6
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = json.load(f)["hbm_gbs"]
    except Exception:
        pass
    r = measure(ctx, a.sf, st, peak)
    if os.environ.get("TQ_HOST_TIMING") == "1":
        import ctypes as C
        from paper_2508_05029_b200.ops import lib
        buf = C.create_string_buffer(1 << 16)
        lib().tq_host_timing_report(buf, len(buf))
        print(buf.value.decode())
    for k, v in r.items():
        print(f"{k:22s} op {v['op_ms']:7.3f} ms  kernels {v['kernel_ms']:7.3f} ms  {v['kernel_gbs']} GB/s "
              f"({v['kernel_frac_of_hbm']})  rows {v['rows_in']} -> {v['rows_out']}")
    print(json.dumps(r))
    ctx.close()


if __name__ == "__main__":
    main()
