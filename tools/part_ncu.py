"""One hash_partition of the op_roofline workload (SF10 lineitem orderkey +
revenue, 8 parts) for an ncu capture of its kernels:

    ncu --set full --import-source on -k regex:tq_jit_main -o gpurun_out/part python tools/part_ncu.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]


def main():
    from paper_2508_05029_b200 import queries as Q
    from paper_2508_05029_b200.expr import Col
    from paper_2508_05029_b200.ops import Context
    ctx = Context(0)
    li = ctx.datagen(Q.TABLE_IDS["lineitem"], float(os.environ.get("SF", "10")))
    L = li.select([Q.L_ORDERKEY, Q.L_EXTPRICE, Q.L_DISCOUNT, Q.L_SHIPDATE])
    proj = ctx.project_execute(L, [Col(0), Col(1) * (Q.Dec(100) - Col(2))])
    for _ in range(2):
        out, _ = ctx.hash_partition(proj, [0], 8)
        ctx.sync()
        out.free()
    print("ok")


if __name__ == "__main__":
    main()
