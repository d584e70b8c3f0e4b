#!/usr/bin/env python3
"""Measure the DRAM traffic of one fused step launch per (config, batch
width) with ncu and write it keyed by the step kernel's source hash
(bench.kernel_hash) -- the `roofline.traffic` that bench.py reports.

    python tools/r2/traffic.py c5:128 c5:64 c5:32 c3:128 [--out gpurun_out/traffic.json]

One ncu pass per case (application replay: the whole process re-runs, so no
kernel-replay save/restore of the 69 GB blocks), after the same command ran
without ncu.  The launch measured is the 3rd step launch (steady state)."""

import argparse
import csv
import io
import json
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import bench  # noqa: E402

METRICS = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct"


def measure(cfg, p):
    cmd = [sys.executable, os.path.join(REPO, "tools", "prof_step.py"), "--config", cfg,
           "--probes", str(p), "--steps", "4"]
    subprocess.run(cmd, check=True, capture_output=True)  # must exit 0 without ncu first
    out = subprocess.run(["ncu", "--replay-mode", "application", "--metrics", METRICS,
                          "--clock-control", "none", "-k", "regex:kpm_step", "-s", "2", "-c", "1",
                          "--csv"] + cmd, check=True, capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 14 and r[0].isdigit()]
    vals = {r[12]: float(r[14].replace(",", "")) for r in rows}
    kern = rows[0][4] if rows else "?"
    return {"dram_bytes": int(vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]),
            "dram_read": int(vals["dram__bytes_read.sum"]),
            "dram_write": int(vals["dram__bytes_write.sum"]),
            "ncu_ms": vals["gpu__time_duration.sum"] / 1e6,
            "l2_hit_pct": vals.get("lts__t_sector_hit_rate.pct"), "kernel": kern,
            "kernel_sha": bench.kernel_hash(),
            "source": f"ncu --replay-mode application --metrics dram__bytes_read.sum,"
                      f"dram__bytes_write.sum -s 2 -c 1 tools/prof_step.py --config {cfg} "
                      f"--probes {p} ({time.strftime('%Y-%m-%d')})"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="+")
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "traffic.json"))
    a = ap.parse_args()
    rec = {"note": "DRAM bytes of one fused step launch, keyed config/P; valid while "
                   "kernel_sha == bench.kernel_hash() (tests/test_bench_contract.py checks it)",
           "entries": {}}
    if os.path.exists(a.out):
        with open(a.out) as f:
            rec = json.load(f)
    for case in a.cases:
        cfg, p = case.split(":")
        rec["entries"][f"{cfg}/P{p}"] = measure(cfg, int(p))
        print(case, rec["entries"][f"{cfg}/P{p}"], flush=True)
        with open(a.out, "w") as f:
            json.dump(rec, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
