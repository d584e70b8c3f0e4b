#!/usr/bin/env python3
"""Device Lanczos vs the reference algorithm on one B200.

Laplacian of R-MAT(scale, 16): estimate_spectral_range (100 steps, one start
vector) and gql_dos (20 probes x 50 steps, one lockstep block) on the device;
the reference's lanczos_factorize (restated in oracle/, over the reference's
own compiled SpMV on all host cores) for a bounded number of steps.

    python tools/lanczos_bench.py [--scale 20] [--ref-steps 20]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1905_09758_b200 as kp  # noqa: E402
from oracle import netdos_oracle as orc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ref-steps", type=int, default=20)
    a = ap.parse_args()
    g = kp.DeviceGraph.rmat(a.scale, 16, seed=2).to_host()
    op = kp.build_operator(g, "laplacian")
    rec = {"graph": f"R-MAT {a.scale} ef16 Laplacian", "n": g.n, "nnz": int(op.indices.shape[0])}
    z = np.random.default_rng(0).standard_normal(g.n)
    kp.lanczos_factorize(op, z, 3)   # warm: upload + modules
    for steps in (20, 100):
        t0 = time.perf_counter()
        f = kp.lanczos_factorize(op, z, steps)
        rec[f"device_factorize_{steps}_s"] = round(time.perf_counter() - t0, 4)
    t0 = time.perf_counter()
    rng_ = kp.estimate_spectral_range(op, steps=100)
    rec["device_range_100_s"] = round(time.perf_counter() - t0, 4)
    rec["range"] = [round(x, 6) for x in rng_]
    probes = kp.make_probes(g.n, 20, "rademacher", seed=1)
    _ = probes.columns
    t0 = time.perf_counter()
    kp.gql_dos(op, probes, 50, bins=50)
    rec["device_gql_20x50_s"] = round(time.perf_counter() - t0, 4)
    ip, ix, dd = op.csr_arrays()
    threads = orc.cpu_threads()
    t0 = time.perf_counter()
    ra, rb, _, _ = orc.lanczos_factorize(
        lambda x: orc.csr_matvec(ip, ix, dd, x, threads=threads, engine="ref"), z, a.ref_steps)
    rec[f"reference_factorize_{a.ref_steps}_s"] = round(time.perf_counter() - t0, 3)
    rec["reference_threads"] = threads
    f = kp.lanczos_factorize(op, z, a.ref_steps)
    rec["alphas_max_rel_diff"] = float(np.abs(f.alphas - ra).max() / np.abs(ra).max())
    rec["betas_max_rel_diff"] = float(np.abs(f.betas - rb).max() / np.abs(rb).max())
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
