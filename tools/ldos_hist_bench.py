#!/usr/bin/env python3
"""Per-node histograms at C2 scale on one B200.

BA(1e6, 5, seed 1), 64 Rademacher probes, 100 moments, 50 bins:
  * pdos_moments (808 MB of moments D2H) + the reference's host product
    `(values * jackson) @ table` (density.py:83-91, numpy/BLAS on all cores)
  * pdos_moments + histogram_from_moments (moments H2D again, device kernel)
  * pdos_histogram (moments stay in HBM; only the (n, 50) masses come back)
  * the binning kernel alone on HBM-resident moments (CUDA events)
Checks that all three histograms agree (per-row L1 <= 1e-9).

    python tools/ldos_hist_bench.py
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_09758_b200 as kp  # noqa: E402
from paper_1905_09758_b200 import _lib  # noqa: E402


def best(fn, reps=3):
    out, t = None, 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        t = min(t, time.perf_counter() - t0)
    return out, t


def main():
    g = kp.preferential_attachment(1_000_000, 5, seed=1)
    sop = kp.rescale_operator(kp.NormalizedAdjacencyOperator(g), (-1.0, 1.0))
    z = kp.make_probes(g.n, 64, "rademacher", seed=1)
    M, B = 100, 50
    kp.pdos_histogram(sop, z, M, bins=B, negativity_tol=10.0)   # warm
    rec = {"config": "C2 BA 1e6 m5, P=64, M=100, bins=50", "n": g.n, "nnz": g.nnz}

    mom, t_mom = best(lambda: kp.pdos_moments(sop, z, M))
    rec["pdos_moments_s"] = round(t_mom, 4)
    edges = sop.scale_map.from_scaled(np.linspace(-1.0, 1.0, B + 1))
    table = kp.cheb_bin_masses(M, sop.scale_map.to_scaled(edges))
    jack = kp.jackson_coefficients(M)
    host, t_host = best(lambda: (mom.values * jack) @ table)
    rec["reference_host_product_s"] = round(t_host, 4)
    rec["host_threads"] = torch.get_num_threads()
    h1, t_h1 = best(lambda: kp.histogram_from_moments(mom, bins=B, negativity_tol=10.0))
    rec["device_hist_from_host_moments_s"] = round(t_h1, 4)
    h2, t_h2 = best(lambda: kp.pdos_histogram(sop, z, M, bins=B, negativity_tol=10.0))
    rec["pdos_histogram_s"] = round(t_h2, 4)
    rec["moments_then_reference_product_s"] = round(t_mom + t_host, 4)
    assert np.abs(h1.masses - host).sum(axis=1).max() <= 1e-9
    assert np.abs(h2.masses - host).sum(axis=1).max() <= 1e-9

    # kernel alone on HBM-resident moments, events on the library stream
    ctx = _lib.Context.get()
    lib = _lib.load()
    dv, dm = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(lib.kpm_device_alloc(ctx.handle, mom.values.nbytes, ctypes.byref(dv)))
    _lib.check(lib.kpm_device_alloc(ctx.handle, 8 * g.n * B, ctypes.byref(dm)))
    _lib.check(lib.kpm_memcpy(ctx.handle, dv, _lib.ptr(mom.values), mom.values.nbytes, 0))
    ctx.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream)
    mn = ctypes.c_double()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(lib.kpm_ldos_histogram(ctx.handle, dv, g.n, M + 1, M, _lib.ptr(jack),
                                          _lib.ptr(table), B, dm, None, ctypes.byref(mn)))
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    lib.kpm_device_free(ctx.handle, dv)
    lib.kpm_device_free(ctx.handle, dm)
    kt = min(ts) / 1e3
    rec["binning_call_device_s"] = round(kt, 5)
    moved = 8 * g.n * (M + 1) + 8 * g.n * B
    rec["binning_GB_per_s"] = round(moved / kt / 1e9, 1)
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
