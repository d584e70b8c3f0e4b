#!/usr/bin/env python3
"""Time fused KPM steps (CUDA events on the library stream) for one config;
used to compare kernel variants (KPM_LIB=<path to a libkpm build>)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_1905_09758_b200 as kp  # noqa: E402
from paper_1905_09758_b200 import _lib  # noqa: E402
from paper_1905_09758_b200.kpm import Run  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--mode", type=int, default=_lib.MODE_DOS_DOUBLING)
ap.add_argument("--probes", type=int, default=0)
ap.add_argument("--tag", default="")
a = ap.parse_args()
ctx = _lib.Context.get(0)
dev = bench.build_graph(a.config, ctx)
kind, prm, P, M = bench.CONFIGS[a.config]
P = a.probes or P
run = Run(dev, P, a.mode, max(M, 2 * (a.steps + a.warmup) + 2))
run.set_probes(kp.make_probes(dev.n, P, "rademacher", seed=prm.get("seed", 0)))
run.advance(a.warmup)
ctx.synchronize()
run.set_timing(True)
run.advance(a.steps)
ms, n = run.kernel_time()
ldos = a.mode == _lib.MODE_LDOS
per = ms / n
model = bench._bytes_per_step(dev.n, dev.nnz, P, ldos)
units = dev.nnz * P * (2 if a.mode == _lib.MODE_DOS_DOUBLING else 1)
print(json.dumps({"tag": a.tag or os.environ.get("KPM_LIB", "default"), "config": a.config,
                  "P": P, "mode": a.mode, "ms_per_step": round(per, 3),
                  "G_units_s": round(units / per / 1e6, 1),
                  "model_GBs": round(model / per / 1e6, 1), "n_heavy": None}))
