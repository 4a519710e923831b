#!/usr/bin/env python
"""Summarise an ncu report (run here, no GPU needed) and optionally record its DRAM
traffic for bench.py's roofline.traffic.

    python tools/ncu_summary.py gpurun_out/r2e/c5.ncu-rep [--csv profiles/x.csv]
        [--traffic-key n400_w8_C32_s256_g1]

--traffic-key writes {dram_bytes, dram_read, dram_write, capture, source_hash} into
profiles/ncu_traffic.json; source_hash is the hash of the SpMMV kernel sources at
the time of the call (bench.py reports the traffic only while they are unchanged),
so run it on the tree the capture was taken from.
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        kernels.append((d, u))
    return kernels


def value(d, u, key):
    v = d.get(key)
    if v in (None, ""):
        return None
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * SCALE.get(u.get(key, ""), 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--csv")
    ap.add_argument("--traffic-key")
    a = ap.parse_args()
    ks = load(a.rep)
    lines = []
    for d, u in ks:
        rec = {"kernel": d.get("Kernel Name"), "id": d.get("ID")}
        for m in METRICS:
            rec[m] = value(d, u, m)
        lines.append(rec)
        print(json.dumps(rec))
    if a.csv:
        with open(a.csv, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=list(lines[0].keys()))
            w.writeheader()
            w.writerows(lines)
    if a.traffic_key:
        from bench import kernel_source_hash
        rec = lines[-1]
        rd, wr = rec["dram__bytes_read.sum"], rec["dram__bytes_write.sum"]
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        tr = json.load(open(path)) if os.path.exists(path) else {}
        tr[a.traffic_key] = {"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
                             "capture": os.path.relpath(a.csv or a.rep, ROOT), "kernel": rec["kernel"],
                             "duration_s": rec["gpu__time_duration.sum"], "source_hash": kernel_source_hash()}
        with open(path, "w") as f:
            json.dump(tr, f, indent=1)
        print("recorded", a.traffic_key, tr[a.traffic_key])


if __name__ == "__main__":
    main()
