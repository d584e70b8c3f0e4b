#!/usr/bin/env python3
"""Minimal driver for ncu: build a config graph on the device and run a few
fused KPM steps (no timing, no CPU work)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_1905_09758_b200 as kp  # noqa: E402
from paper_1905_09758_b200 import _lib  # noqa: E402
from paper_1905_09758_b200.kpm import Run  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--mode", type=int, default=_lib.MODE_DOS_DOUBLING)
ap.add_argument("--probes", type=int, default=0)
a = ap.parse_args()
ctx = _lib.Context.get(0)
dev = bench.build_graph(a.config, ctx)
kind, prm, P, M = bench.CONFIGS[a.config]
P = a.probes or P
run = Run(dev, P, a.mode, max(M, 2 * a.steps + 2))
run.set_probes(kp.make_probes(dev.n, P, "rademacher", seed=prm.get("seed", 0)))
run.advance(a.steps)
ctx.synchronize()
print("ok", dev.n, dev.nnz, dev.max_degree)
