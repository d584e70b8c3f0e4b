#!/usr/bin/env python3
"""Time-to-solution of every BASELINE config through the public API on one
B200 (graph generation / upload, probes, motif filtering and the full moment
run), next to the recurrence-only time.  Prints one JSON line per config.

    python tools/config_report.py [--configs c1,c2,c3,c4,c5]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1905_09758_b200 as kp  # noqa: E402
from paper_1905_09758_b200 import _lib  # noqa: E402


def _sync():
    _lib.Context.get().synchronize()


def run(cfg):
    rec = {"config": cfg}
    t0 = time.perf_counter()
    if cfg == "c1":
        g = kp.erdos_renyi(10_000, 1e-3, seed=0)
        rec["graph_s"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        res = kp.kpm_dos(g, m_max=200, nz=20, probe_kind="rademacher", seed=0, bins=100)
        rec["solve_s"] = time.perf_counter() - t1
        rec["nnz"], rec["units"] = g.nnz, g.nnz * 20 * 200
    elif cfg == "c2":
        g = kp.preferential_attachment(1_000_000, 5, seed=1)
        rec["graph_s"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        mom, _ = kp.kpm_pdos(g, m_max=100, nz=64, probe_kind="rademacher", seed=1)
        rec["solve_s"] = time.perf_counter() - t1
        rec["nnz"], rec["units"] = g.nnz, g.nnz * 64 * 100
    elif cfg in ("c3", "c5"):
        scale, seed, P, M = (24, 2, 128, 500) if cfg == "c3" else (26, 4, 256, 1000)
        dev = kp.DeviceGraph.rmat(scale, 16, seed)
        _sync()
        rec["graph_s"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        sop = kp.rescale_operator(kp.NormalizedAdjacencyOperator(dev), (-1.0, 1.0))
        mom = kp.dos_moments(sop, kp.make_probes(dev.n, P, "rademacher", seed=seed), M)
        kp.histogram_from_moments(mom, bins=50)
        rec["solve_s"] = time.perf_counter() - t1
        rec["nnz"], rec["units"] = dev.nnz, dev.nnz * P * M
    elif cfg == "c4":
        g = kp.testkit.motif_heavy()
        rec["graph_s"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        insts = kp.detect_motifs(g, seed=3)
        rec["detect_s"] = time.perf_counter() - t1
        t2 = time.perf_counter()
        res = kp.kpm_dos(g, m_max=300, nz=64, probe_kind="rademacher", seed=3, bins=50,
                         custom_instances=insts)
        rec["filter_and_solve_s"] = time.perf_counter() - t2
        rec["solve_s"] = time.perf_counter() - t1
        rec["removed"] = res.adjustment.deflated_dim
        rec["nnz"], rec["units"] = g.nnz, g.nnz * 64 * 300
    rec["G_units_per_s_solve"] = round(rec["units"] / rec["solve_s"] / 1e9, 2)
    for k in list(rec):
        if isinstance(rec[k], float):
            rec[k] = round(rec[k], 4)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    a = ap.parse_args()
    # warm the CUDA context and kernel modules first (a one-time process
    # cost of ~1.4 s that would otherwise land on the first config)
    t0 = time.perf_counter()
    tiny = kp.build_csr([(0, 1), (1, 2), (2, 0)])
    kp.kpm_dos(tiny, m_max=4, nz=2, probe_kind="rademacher")
    kp.kpm_pdos(tiny, m_max=4, nz=2, probe_kind="rademacher")
    print(json.dumps({"warmup_s": round(time.perf_counter() - t0, 3)}), flush=True)
    for cfg in a.configs.split(","):
        print(json.dumps(run(cfg)), flush=True)


if __name__ == "__main__":
    main()
