import sys, time
sys.path[:0] = ['/root/repo', '/root/repo/oracle']
from paper_2508_05029_b200.ops import Context, engine_run_query
from paper_2508_05029_b200 import queries
ctx = Context(0)
sf5 = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
for q in (5, 9):
    t0 = time.time()
    names = queries.QUERY_TABLES[q]
    host = {}
    for n in names:
        d = ctx.datagen(queries.TABLE_IDS[n], sf5)
        host[queries.TABLE_IDS[n]] = d.to_host()
        d.free()
    data_bytes = sum(b.nbytes() for b in host.values())
    print(q, "datagen+download", time.time() - t0, "s", data_bytes / 1e9, "GB", flush=True)
    for budget_div in (0, 4):
        t0 = time.time()
        kw = dict(compute_threads=4, preload=1, batch_rows=4 << 20)
        if budget_div:
            kw["device_budget"] = max(int(data_bytes / 2.5), 1 << 30)
        _, m = engine_run_query(ctx, q, host, **kw)
        print(q, "budget_div", budget_div, "wall", time.time() - t0, {k: v for k, v in m.items() if k != 'ops'}, flush=True)
        print("   ops", {k: (v['tasks'], round(v['ms'], 1)) for k, v in m['ops'].items()}, flush=True)
