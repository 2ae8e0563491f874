"""Summarise ncu reports (.ncu-rep) into profiles/: one JSON record per kernel
launch with duration, DRAM bytes, throughput and top stall reasons.

    python tools/ncu_summary.py gpurun_out/prof_q1.ncu-rep --label q1_agg --out profiles/r01_ncu_q1.json
"""
import argparse
import csv
import io
import json
import subprocess

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--label", default="")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    recs = []
    for v in rows[2:]:
        d = dict(zip(hdr, v))
        rec = {"kernel": d.get("Kernel Name", ""), "label": a.label}
        for k in KEEP:
            if k in d:
                u = units[hdr.index(k)]
                rec[k] = d[k] + (f" {u}" if u else "")
        stalls = []
        for k, x in d.items():
            if "issue_stalled" in k and k.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(x), k.split("stalled_")[1].split("_per")[0]))
                except ValueError:
                    pass
        rec["top_stalls"] = [f"{n}={s:.2f}" for s, n in sorted(stalls, reverse=True)[:5]]
        # bytes per launch in bytes for roofline.traffic
        def to_bytes(s):
            num, _, unit = s.partition(" ")
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
            return float(num.replace(",", "")) * mult
        try:
            rec["dram_bytes_per_launch"] = to_bytes(rec["dram__bytes_read.sum"]) + to_bytes(rec["dram__bytes_write.sum"])
        except KeyError:
            pass
        recs.append(rec)
    with open(a.out, "w") as f:
        json.dump(recs, f, indent=1)
    print(json.dumps(recs, indent=1)[:3000])


if __name__ == "__main__":
    main()
