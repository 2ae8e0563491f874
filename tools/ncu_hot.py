"""Summarise an ncu report's SASS source page: top basic blocks by executed
instructions and by stall samples (needs --set full --import-source on).

    python tools/ncu_hot.py gpurun_out/prof.ncu-rep [kernel-regex]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    iS, iW, iI = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    tot = sum(int(r[iI] or 0) for r in data)
    totw = sum(int(r[iW] or 0) for r in data)
    print(f"warp instructions {tot}  stall samples {totw}  sass lines {len(data)}")
    blocks, cur = [], None
    for i, r in enumerate(data):
        n, w = int(r[iI] or 0), int(r[iW] or 0)
        if cur and cur["n"] == n:
            cur["end"] = i
            cur["w"] += w
        else:
            cur = {"start": i, "end": i, "n": n, "w": w}
            blocks.append(cur)
    for key, label in (("inst", "by instructions"), ("w", "by stall samples")):
        print("--", label)
        f = (lambda b: b["n"] * (b["end"] - b["start"] + 1)) if key == "inst" else (lambda b: b["w"])
        for b in sorted(blocks, key=lambda b: -f(b))[:12]:
            ln = b["end"] - b["start"] + 1
            print(f"  [{b['start']:5d}-{b['end']:5d}] exec {b['n']:>10d} x {ln:3d} = {b['n'] * ln:>11d}  "
                  f"samples {b['w']:6d} ({100 * b['w'] / max(1, totw):4.1f}%)  {data[b['start']][iS].strip()[:48]}")
    hot = sorted(range(len(data)), key=lambda i: -int(data[i][iW] or 0))[:15]
    print("-- hottest instructions by samples")
    for i in hot:
        print(f"  {i:5d} samples {data[i][iW]:>6} exec {data[i][iI]:>10}  {data[i][iS].strip()[:70]}")


if __name__ == "__main__":
    main()
