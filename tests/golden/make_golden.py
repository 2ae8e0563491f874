"""Regenerate tests/golden/*.json from the REFERENCE's own code.

Runs only in the build container where /root/reference exists: it loads
oracle/_ref/libtierq_ref.so (built from /root/reference/proj sources by
oracle/build_ref.sh) and records its fnv1a64 / SplitMix64 outputs and its
take / concat results (reference transform.cpp:49-120) on seeded inputs.
The committed JSON is what the CPU and GPU tests check against, so they run
on boxes without /root/reference.

    python tests/golden/make_golden.py
"""
import ctypes as C
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import oracle as O  # noqa: E402
from paper_2508_05029_b200.columnar import HostBatch  # noqa: E402


def main():
    L = O.ref()
    assert L is not None, "build oracle/_ref first (make -C oracle)"
    rng = random.Random(2508_05029)
    fnv = []
    for n in [0, 1, 3, 8, 16, 31]:
        data = bytes(rng.randrange(256) for _ in range(n))
        for seed in (0xCBF29CE484222325, rng.getrandbits(64)):
            fnv.append({"bytes": data.hex(), "seed": str(seed), "hash": str(L.tqr_fnv1a64(data, n, seed))})
    for k in [0, 1, 42, -1, 6000000, 2**62, -(2**63)]:
        data = (k & (2**64 - 1)).to_bytes(8, "little")
        fnv.append({"bytes": data.hex(), "seed": str(0xCBF29CE484222325),
                    "hash": str(L.tqr_fnv1a64(data, 8, 0xCBF29CE484222325))})
    sm = []
    for seed in [0, 42, 7, 2**64 - 1, O.fnv1a64(b"lineitem.l_shipdate", 42)]:
        out = (C.c_uint64 * 16)()
        L.tqr_splitmix(seed, 16, out)
        sm.append({"seed": str(seed), "out": [str(x) for x in out]})
    with open(os.path.join(HERE, "hash_rng.json"), "w") as f:
        json.dump({"source": "reference proj/include/tierq/common.hpp:128-158 via oracle/_ref", "fnv": fnv,
                   "splitmix": sm}, f, indent=1)

    takes, concats = [], []
    for case in range(12):
        rows = rng.randrange(0, 20)
        x = [rng.randrange(-100, 100) for _ in range(rows)]
        valid = None if case % 3 == 0 else [rng.random() > 0.3 for _ in range(rows)]
        b = HostBatch(rows, [HostBatch.col_i64(x, valid)])
        ids = [rng.randrange(rows) for _ in range(rng.randrange(0, 25))] if rows else []
        out = O.ref_take(b, ids)
        takes.append({"rows": rows, "x": x, "valid": valid, "ids": ids, "want": out.column_py(0),
                      "want_bitmap": out.cols[0].validity is not None})
    for case in range(8):
        parts = []
        for _ in range(rng.randrange(1, 4)):
            rows = rng.randrange(0, 10)
            x = [rng.randrange(-100, 100) for _ in range(rows)]
            valid = None if rng.random() < 0.5 else [rng.random() > 0.3 for _ in range(rows)]
            parts.append({"x": x, "valid": valid})
        out = O.ref_concat([HostBatch(len(p["x"]), [HostBatch.col_i64(p["x"], p["valid"])]) for p in parts])
        concats.append({"parts": parts, "want": out.column_py(0), "want_bitmap": out.cols[0].validity is not None})
    with open(os.path.join(HERE, "substrate.json"), "w") as f:
        json.dump({"source": "reference proj/src/columnar/transform.cpp:49-120 via oracle/_ref", "take": takes,
                   "concat": concats}, f, indent=1)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
