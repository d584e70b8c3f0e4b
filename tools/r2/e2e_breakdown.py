#!/usr/bin/env python3
"""Where the end-to-end call spends its time beside the recurrence steps
(C5 by default): host CSR upload + graph build, twin build, run allocation,
probe generation, steps, result, frees."""
import argparse
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1905_09758_b200 as kp  # noqa: E402
from paper_1905_09758_b200 import _lib  # noqa: E402
from paper_1905_09758_b200.kpm import Run  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--moments", type=int, default=100)
a = ap.parse_args()
ctx = _lib.Context.get(0)
kind, prm, P, M = bench.CONFIGS[a.config]
dev = bench.build_graph(a.config, ctx)
rp, ci, _ = dev.export()
n, nnz = dev.n, dev.nnz
dev.free()
_t1, hrp = bench._pinned(rp)
_t2, hci = bench._pinned(ci)
del rp, ci


def lap(label, t0):
    ctx.synchronize()
    t = time.perf_counter()
    print(f"{label:28s} {t - t0:8.3f} s", flush=True)
    return t


t = time.perf_counter()
t_all = t
g = kp.DeviceGraph.from_csr(n, hrp, hci, ctx=ctx)
t = lap("from_csr (H2D + schedule)", t)
twin = g.prepare(128)
t = lap(f"prepare (twin={twin})", t)
fam = kp.make_probes(n, P, "rademacher", seed=prm["seed"])
for b0 in range(0, P, 128):
    b1 = min(P, b0 + 128)
    run = Run(g, b1 - b0, _lib.MODE_DOS_DOUBLING, a.moments)
    t = lap("run create", t)
    run.set_probes(fam.column_slice(b0, b1))
    t = lap("set_probes (+ init step)", t)
    run.advance()
    t = lap(f"advance {run.total_steps} steps", t)
    out = np.empty((a.moments + 1, b1 - b0))
    run.result(out)
    t = lap("result", t)
    run.free()
    t = lap("run free", t)
g.free()
t = lap("graph free", t)
print(f"{'total':28s} {t - t_all:8.3f} s")
