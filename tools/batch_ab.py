#!/usr/bin/env python3
"""A/B of probe-column batching on one box: dos_contrib over the same probes
with batch=P (one wide run) vs batch=64 (compact 64-column runs), and the
step kernel of one wide run with and without 64-column tiles; interleaved."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1905_09758_b200 as kp  # noqa: E402
from paper_1905_09758_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--probes", type=int, default=128)
ap.add_argument("--moments", type=int, default=100)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
ctx = _lib.Context.get(0)
dev = bench.build_graph(a.config, ctx)
kind, prm, _, _ = bench.CONFIGS[a.config]
probes = kp.make_probes(dev.n, a.probes, "rademacher", seed=prm.get("seed", 0))
sop = kp.rescale_operator(kp.NormalizedAdjacencyOperator(dev), (-1.0, 1.0))
ref = None
for rep in range(a.reps):
    for tag, batch, tile in (("wide-tiles", a.probes, "1"), ("wide-bulk", a.probes, "0"),
                             ("batch64", 64, "1"), ("batch32", 32, "1")):
        os.environ["KPM_TILE"] = tile
        ctx.synchronize()
        t0 = time.perf_counter()
        c = kp.dos_contrib(sop, probes, a.moments, batch=batch)
        ctx.synchronize()
        dt = time.perf_counter() - t0
        same = None if ref is None else bool(np.array_equal(c, ref))
        ref = c if ref is None else ref
        units = dev.nnz * a.probes * a.moments
        print(json.dumps({"rep": rep, "tag": tag, "s": round(dt, 4),
                          "G_units_s": round(units / dt / 1e9, 1), "bitwise_same": same}),
              flush=True)
