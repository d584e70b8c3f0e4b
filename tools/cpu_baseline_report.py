#!/usr/bin/env python3
"""SURVEY §8(d) CPU baseline, run on the GPU box's own host cores: the
reference's CPU path -- its compiled Cython csr_matvec (oracle/_ref) inside the
recurrence glue restated with the identical numpy calls (kpm.py:73-152) --
timed with threads=1 and threads=<all cores> on the same probe matrix, per
config.  C1, C2 (LDOS), C4: full M where it fits the per-run budget, else the
first K moments; C3, C5: the first moments over a probe-column sample (the
paper's Table 1 method).  Every line states what was measured and what is an
extrapolation (seconds per moment x M, x P / sampled probes: the SpMM and the
einsums are linear in the probe count).

Test infrastructure (it executes oracle/): not part of the product path.

    python tools/cpu_baseline_report.py [--configs c1,c2,c3,c4,c5] [--budget 90]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402
from oracle import netdos_oracle as orc  # noqa: E402

# (probe columns sampled at all threads, at 1 thread, moment cap) per config
PLAN = {"c1": (20, 20, None), "c2": (64, 64, None), "c3": (8, 2, 10),
        "c4": (64, 64, None), "c5": (4, 1, 4)}


def _mem_free_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 1e9
    except Exception:
        return float("inf")


def run_cfg(cfg, budget):
    kind, prm, P, M = bench.CONFIGS[cfg]
    ldos = cfg == "c2"
    t0 = time.perf_counter()
    rp, ci, data, _ = bench._oracle_graph(cfg)
    t_graph = time.perf_counter() - t0
    n, nnz = rp.shape[0] - 1, ci.shape[0]
    engine = "ref" if orc.ref_spmv() is not None else "c"
    op = orc.CSROp(rp, ci, data, engine=engine)
    del rp, ci, data
    ps_all, ps_one, mcap = PLAN[cfg]
    z_all = orc.make_probes(n, ps_all, "rademacher", seed=prm.get("seed", 0))
    fn = orc.ldos_num if ldos else orc.dos_contrib
    out = []
    for threads, ps in ((orc.cpu_threads(), ps_all), (1, ps_one)):
        z = np.ascontiguousarray(z_all[:, :ps])
        # one step (T_0, T_1 = H z, two collects) sizes the run to the budget
        fn(op, z, 1, threads=threads)  # warm-up (OpenMP team, page faults)
        t1 = time.perf_counter()
        fn(op, z, 1, threads=threads)
        t_one = time.perf_counter() - t1
        k = M if mcap is None else min(M, mcap)
        k = int(max(2, min(k, budget / max(t_one, 1e-9))))
        t1 = time.perf_counter()
        res = fn(op, z, k, threads=threads)
        dt = time.perf_counter() - t1
        assert np.isfinite(res).all()
        s_per_moment = dt / k
        full = s_per_moment * M * (P / ps)
        units = nnz * ps * k
        out.append({
            "config": cfg, "mode": "ldos" if ldos else "dos", "threads": threads,
            "n": n, "nnz": nnz, "probes_sampled": ps, "probes_config": P,
            "moments_measured": k, "moments_config": M, "seconds": round(dt, 3),
            "s_per_moment": round(s_per_moment, 4),
            "G_units_per_s": round(units / dt / 1e9, 4),
            "full_run_s": round(full, 2),
            "full_run_kind": ("measured" if (k == M and ps == P) else
                              "extrapolated (s/moment x M x P/probes_sampled)"),
            "kind": "reference" if engine == "ref" else "port",
            "graph_prep_s": round(t_graph, 2)})
        print(json.dumps(out[-1]), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--budget", type=float, default=90.0,
                    help="seconds per (config, thread count) run")
    a = ap.parse_args()
    print(json.dumps({"host_cores": os.cpu_count(), "affinity": orc.cpu_threads(),
                      "mem_free_gb": round(_mem_free_gb(), 1)}), flush=True)
    for cfg in a.configs.split(","):
        if cfg == "c5" and _mem_free_gb() < 120:
            print(json.dumps({"config": cfg, "skipped": "host memory < 120 GB free"}), flush=True)
            continue
        run_cfg(cfg, a.budget)


if __name__ == "__main__":
    main()
