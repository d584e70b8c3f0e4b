#!/usr/bin/env python3
"""Experiment: implicit h_ij = dinv_i*dinv_j (random dinv gathers) versus
stored h values (coalesced stream) on an R-MAT config."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1905_09758_b200 as kp
from paper_1905_09758_b200 import _lib
from paper_1905_09758_b200.kpm import Run

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--probes", type=int, default=128)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
ctx = _lib.Context.get(0)
dev = kp.DeviceGraph.rmat(a.scale, 16, 2)
rp, ci, dinv = dev.export()
ci = ci.astype(np.int64)
rows = np.repeat(np.arange(dev.n, dtype=np.int64), np.diff(rp))
vals = (1.0 * dinv[rows]) * dinv[ci]
del rows
exp = kp.DeviceGraph.from_csr(dev.n, rp, ci, vals)
del vals
for name, g in (("implicit", dev), ("explicit", exp)):
    run = Run(g, a.probes, _lib.MODE_DOS_DOUBLING, 2 * a.steps + 8)
    run.set_probes(kp.make_probes(g.n, a.probes, "rademacher", seed=2))
    run.advance(2)
    run.set_timing(True)
    run.advance(a.steps)
    ms, n = run.kernel_time()
    run.free()
    print(json.dumps({"exp": name, "scale": a.scale, "P": a.probes, "ms_per_step": round(ms / n, 3)}))
