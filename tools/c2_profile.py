#!/usr/bin/env python3
"""Time the pieces of C2's end-to-end kpm_pdos (BA 1M, 64 probes, LDOS, 100
moments): operator, graph upload, probe generation, recurrence, result D2H."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1905_09758_b200 as kp  # noqa: E402
from paper_1905_09758_b200 import _lib  # noqa: E402
from paper_1905_09758_b200.kpm import Run  # noqa: E402

ctx = _lib.Context.get(0)
g = kp.preferential_attachment(1_000_000, 5, seed=1)
for rep in range(3):
    rec = {}
    t = time.perf_counter()
    res, _ = kp.kpm_pdos(g, m_max=100, nz=64, probe_kind="rademacher", seed=1)
    rec["kpm_pdos_s"] = time.perf_counter() - t
    t = time.perf_counter()
    sop = kp.scaled_operator_for(g, "normalized-adjacency")
    dev = sop.device_graph()
    ctx.synchronize()
    rec["operator_and_device_graph_s"] = time.perf_counter() - t
    probes = kp.make_probes(g.n, 64, "rademacher", seed=1)
    t = time.perf_counter()
    run = Run(dev, 64, _lib.MODE_LDOS, 100)
    run.set_probes(probes)
    ctx.synchronize()
    rec["run_create_probes_s"] = time.perf_counter() - t
    t = time.perf_counter()
    run.advance()
    ctx.synchronize()
    rec["advance_s"] = time.perf_counter() - t
    t = time.perf_counter()
    out = np.empty((g.n, 101))
    run.result(out, probes.trace_scale)
    rec["result_d2h_fresh_s"] = time.perf_counter() - t
    run.free()
    # the same D2H into memory that is already paged in
    run = Run(dev, 64, _lib.MODE_LDOS, 100)
    run.set_probes(probes)
    run.advance()
    ctx.synchronize()
    t = time.perf_counter()
    run.result(out, probes.trace_scale)
    rec["result_d2h_touched_s"] = time.perf_counter() - t
    run.free()
    print(json.dumps({k: round(v, 4) for k, v in rec.items()}), flush=True)
