#!/usr/bin/env python3
"""Per-node histogram fixtures written BY THE
REFERENCE: pdos_moments + histogram_from_moments (kpm.py:120-152,
density.py:63-108) on small seeded graphs.  Build container only; writes
tests/golden/density.npz.

    python tests/golden/make_density_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import netdos_oracle as orc  # noqa: E402

assert orc.ref_spmv() is not None, "run `make -C oracle` first"
sys.path.insert(0, "/root/reference/pkg/src")
import netdos  # noqa: E402
from netdos import histogram_from_moments, make_probes, pdos_moments  # noqa: E402
from netdos.pipeline import scaled_operator_for  # noqa: E402
from netdos.testkit import erdos_renyi, preferential_attachment  # noqa: E402

assert netdos.KERNEL_BACKEND == "cython"


def main():
    out = {}
    graphs = {"ba": preferential_attachment(400, 3, seed=7),
              "er": erdos_renyi(300, 0.02, seed=8)}
    for name, g in graphs.items():
        out[f"{name}_row_ptr"] = g.row_ptr
        out[f"{name}_col_idx"] = g.col_idx
        sop = scaled_operator_for(g, "normalized-adjacency", range_=(-1.0, 1.0))
        for kind, nz, m in ((("rademacher", 24, 60),) if name == "ba"
                            else (("gaussian", 10, 33),)):
            tag = f"{name}_{kind}"
            z = make_probes(g.n, nz, kind=kind, seed=5)
            mom = pdos_moments(sop, z, m)
            out[f"{tag}_values"] = mom.values
            edges = np.array([-1.0, -0.7, -0.1, 0.0, 0.25, 0.9, 1.0])
            mom_raw = pdos_moments(sop, z, m, normalized=False)
            out[f"{tag}_raw_values"] = mom_raw.values
            calls = {
                "h50": (mom, dict(bins=50, negativity_tol=1.0)),
                "h50tol": (mom, dict(bins=50)),
                "h7raw": (mom, dict(bins=7, damping=False)),
                "hedges": (mom, dict(edges=edges, negativity_tol=1.0)),
                "neg": (mom, dict(bins=80, damping=False, negativity_tol=1e-9)),
                "rawh20": (mom_raw, dict(bins=20, negativity_tol=10.0)),
            }
            for key, (mm, kw) in calls.items():
                try:
                    h = histogram_from_moments(mm, **kw)
                except ValueError as exc:
                    out[f"{tag}_{key}_error"] = np.array(str(exc))
                else:
                    out[f"{tag}_{key}_masses"] = h.masses
                    out[f"{tag}_{key}_norm"] = h.normalization
                    out[f"{tag}_{key}_edges"] = h.edges
    np.savez_compressed(os.path.join(HERE, "density.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
