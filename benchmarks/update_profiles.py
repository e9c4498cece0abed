#!/usr/bin/env python
"""Copy the judged evidence of a capture run (benchmarks/capture_profiles.sh,
under gpurun_out/) into profiles/ with a round tag: ncu summaries (JSON), raw
ncu pages (CSV) of the top kernels, the launch list, the bench line and the
per-config lines.

Usage: python benchmarks/update_profiles.py TAG   (e.g. r01c)
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
W = "gaussian_problem(20000,20000,0) quadratic alpha=5e-3*(m+n)=200, fp32 C/X storage"


def summ(rep):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "benchmarks", "ncu_summary.py"), rep],
                         capture_output=True, text=True, check=True).stdout.strip().splitlines()
    return json.loads(out[0])


def raw(rep, dst):
    with open(dst, "w") as f:
        subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], stdout=f, check=True)


def l2_compression(rep):
    """L2 generic-compression figures of the memory-workload section."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    got = {}
    for ln in out.splitlines():
        if "L2 Compression" in ln:
            parts = ln.split()
            try:
                got[" ".join(parts[:-2]) if parts[-2] in ("%", "sector") else " ".join(parts[:-1])] = float(parts[-1].replace(",", ""))
            except ValueError:
                pass
    return got


def sass_tma(kernel):
    """Counts of Blackwell async-copy SASS (UTMALDG = 2-D TMA loads, UBLKCP =
    1-D bulk copies) and of LDGSTS (per-thread cp.async) in the kernel's code."""
    so = os.path.join(ROOT, "paper_2305_18483_b200", "libotdr_dev.so")
    try:
        out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    except Exception:
        return None
    name = kernel.split("<")[0].split("(")[0].split()[-1]
    counts, cur = {}, None
    for ln in out.splitlines():
        if "Function :" in ln:
            cur = ln
        elif cur and name in cur:
            for op in ("UTMALDG", "UBLKCP", "LDGSTS", "SYNCS"):
                if op in ln:
                    counts[op] = counts.get(op, 0) + 1
    return counts


def main():
    tag = sys.argv[1]
    if os.path.exists(os.path.join(OUT, "stream.ncu-rep")):
        s = summ(os.path.join(OUT, "stream.ncu-rep"))
        it = 20  # capture_profiles.sh: the timed launch of bench.py --steps 20 --warmup 5
        raw(os.path.join(OUT, "stream.ncu-rep"), os.path.join(PROF, f"{tag}_stream_20000_f32_raw.csv"))
        json.dump({"workload": W, "kernel": s["kernel"],
                   "source": f"profiles/{tag}_stream_20000_f32_raw.csv (ncu --set full --clock-control none; "
                             "the timed launch of bench.py --steps 20 --warmup 5 = ONE launch running "
                             "iterations 6..25)",
                   "iterations_in_launch": it, "dram_bytes_read": s["dram_read"],
                   "dram_bytes_write": s["dram_write"], "dram_bytes_per_launch": s["dram_bytes"],
                   "dram_bytes_per_iteration": s["dram_bytes"] / it,
                   "algorithmic_bytes_per_iteration": 12 * 20000 * 20000,
                   "duration_us_ncu": s["duration"] * 1e6, "duration_per_iteration_us_ncu": s["duration"] * 1e6 / it,
                   "dram_throughput_pct_of_ncu_peak": s["dram_throughput_pct"], "registers": s["registers"],
                   "grid": s["grid"], "stalls": s.get("stalls"), "issue_active_pct": s.get("issue_active_pct"),
                   "x_allocation": "generic-compressible HBM (first 3.2 GB of X; OTDR_COMPRESS)",
                   "sass_tma": sass_tma(s["kernel"]),
                   "l2_compression": l2_compression(os.path.join(OUT, "stream.ncu-rep"))},
                  open(os.path.join(PROF, "ncu_stream_summary.json"), "w"), indent=1)
    if os.path.exists(os.path.join(OUT, "sweep.ncu-rep")):
        s = summ(os.path.join(OUT, "sweep.ncu-rep"))
        json.dump({"workload": W, "kernel": s["kernel"],
                   "source": "ncu --set full, one launch of the graph-path sweep kernel (bench.py --steps 2)",
                   "dram_bytes_read": s["dram_read"], "dram_bytes_write": s["dram_write"],
                   "dram_bytes_per_launch": s["dram_bytes"], "dram_bytes_per_iteration": s["dram_bytes"],
                   "algorithmic_bytes_per_launch": 12 * 20000 * 20000, "duration_us_ncu": s["duration"] * 1e6,
                   "dram_throughput_pct": s["dram_throughput_pct"], "registers": s["registers"], "grid": s["grid"]},
                  open(os.path.join(PROF, "ncu_sweep_summary.json"), "w"), indent=1)
    if os.path.exists(os.path.join(OUT, "gl.ncu-rep")):
        s = summ(os.path.join(OUT, "gl.ncu-rep"))
        s["workload"] = "adaptation_problem(10000,10000,10 classes,0), GroupLasso lambda=1e-3, fp32 (cfg3)"
        s["algorithmic_bytes_per_launch"] = 12 * 10000 * 10000
        s["algorithmic_GBps"] = 12 * 10000 * 10000 / s["duration"] / 1e9
        raw(os.path.join(OUT, "gl.ncu-rep"), os.path.join(PROF, f"{tag}_gl_pipe_cfg3_raw.csv"))
        json.dump(s, open(os.path.join(PROF, f"{tag}_gl_pipe_cfg3_summary.json"), "w"), indent=1)
    if os.path.exists(os.path.join(OUT, "glstream.ncu-rep")):
        s = summ(os.path.join(OUT, "glstream.ncu-rep"))
        s["workload"] = "cfg3 (10000^2, 10 classes, lambda 1e-3, fp32): ONE gl_stream_kernel launch of 2 DR iterations"
        s["iterations_in_launch"] = 2
        s["algorithmic_bytes_per_iteration"] = 12 * 10000 * 10000
        s["dram_bytes_per_iteration"] = s["dram_bytes"] / 2
        s["algorithmic_GBps"] = 2 * 12 * 10000 * 10000 / s["duration"] / 1e9
        json.dump(s, open(os.path.join(PROF, f"{tag}_gl_stream_cfg3_summary.json"), "w"), indent=1)
    for src, dst in (("launches.csv", f"{tag}_launches_20000_f32.csv"), ("configs.log", f"{tag}_configs.jsonl")):
        if os.path.exists(os.path.join(OUT, src)):
            shutil.copy(os.path.join(OUT, src), os.path.join(PROF, dst))
    if os.path.exists(os.path.join(OUT, "bench.log")):
        lines = [ln for ln in open(os.path.join(OUT, "bench.log")) if ln.startswith("{")]
        if lines:
            open(os.path.join(PROF, f"{tag}_bench.jsonl"), "w").write(lines[-1])


if __name__ == "__main__":
    main()
