#!/usr/bin/env python
"""Summarise an ncu report (--set full) into the numbers DESIGN.md / profiles/ cite.

Usage: python benchmarks/ncu_summary.py report.ncu-rep [--bytes ALGORITHMIC_BYTES]
Prints one JSON object per profiled kernel: duration, DRAM bytes read/written,
DRAM throughput, occupancy, registers, issue activity, top stall reasons and,
with --bytes, the achieved algorithmic bandwidth.
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__cluster_dim_x": "cluster_x",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--bytes", type=float, default=None)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for v in rows[2:]:
        out = {"kernel": v[hdr.index("Kernel Name")]}
        for i, h in enumerate(hdr):
            if h in KEYS:
                try:
                    val = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                out[KEYS[h]] = val * SCALE.get(units[i], 1.0)
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    out.setdefault("stalls", {})[h.split("stalled_")[1].split("_per_issue")[0]] = float(v[i])
                except ValueError:
                    pass
        if "stalls" in out:
            out["stalls"] = dict(sorted(out["stalls"].items(), key=lambda kv: -kv[1])[:6])
        if "dram_read" in out and "dram_write" in out:
            out["dram_bytes"] = out["dram_read"] + out["dram_write"]
        if a.bytes and "duration" in out:
            out["algorithmic_GBps"] = a.bytes / out["duration"] / 1e9
        print(json.dumps(out))


if __name__ == "__main__":
    main()
