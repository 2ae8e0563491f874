"""Config-5 parity check outside the bench: Q5 / Q9 on the C++ engine with the
tables in the pinned Host tier and a Device budget (as bench.py), against the
oracle, a few repetitions.

    python tools/engine_hosttier_check.py [--sf 12.5] [--reps 3] [--q 9]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=float, default=12.5)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--q", type=int, default=9)
    a = ap.parse_args()
    import oracle as O
    from paper_2508_05029_b200 import queries
    from paper_2508_05029_b200.columnar import assert_batches_equal
    from paper_2508_05029_b200.ops import Context, engine_run_query
    ctx = Context(0)
    host = {}
    for n in queries.QUERY_TABLES[a.q]:
        d = ctx.datagen(queries.TABLE_IDS[n], a.sf)
        host[queries.TABLE_IDS[n]] = d.to_host()
        d.free()
    data_bytes = sum(b.nbytes() for b in host.values())
    want = O.query(a.q, host, os.cpu_count() or 1)
    for i in range(a.reps):
        res, m = engine_run_query(ctx, a.q, host, compute_threads=4, preload=1, batch_rows=4 << 20,
                                  device_budget=max(int(data_bytes / 2.5), 1 << 30))
        try:
            assert_batches_equal(res, want, ordered=False)
            ok = "exact"
        except AssertionError as e:
            ok = "MISMATCH " + str(e)[:200]
        print(f"rep {i}: {ok} rows {res.rows} vs {want.rows} spills {m['spills']} retries {m['oom_retries']} "
              f"splits {m.get('splits')} tasks {m['tasks']}", flush=True)


if __name__ == "__main__":
    main()
