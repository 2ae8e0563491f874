"""Print an ncu --csv launch list (gpu__time_duration + dram bytes) one launch per line.
    python tools/launches.py gpurun_out/x.csv"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = OrderedDict()
for r in rows[1:]:
    d.setdefault(r[ii], {"k": r[ki][:50]})[r[mi]] = r[vi]
for k, v in d.items():
    print(k, v["k"], v.get("gpu__time_duration.sum"), v.get("dram__bytes_read.sum"), v.get("dram__bytes_write.sum"))
