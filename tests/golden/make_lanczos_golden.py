#!/usr/bin/env python3
"""Lanczos / GQL fixtures written BY THE REFERENCE:
lanczos_factorize, lanczos_quadrature, estimate_spectral_range, gql_dos,
gql_pdos and gql_dos_pipeline on small seeded graphs for every operator kind.
Build container only; writes tests/golden/lanczos.npz.

    python tests/golden/make_lanczos_golden.py
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
from netdos import (build_csr, build_operator, estimate_spectral_range, gql_dos,  # noqa: E402
                    gql_pdos, lanczos_factorize, lanczos_quadrature, make_probes)
from netdos.pipeline import gql_dos_pipeline, scaled_operator_for  # noqa: E402
from netdos.testkit import erdos_renyi, preferential_attachment  # noqa: E402

assert netdos.KERNEL_BACKEND == "cython"
KINDS = ("adjacency", "laplacian", "normalized-adjacency", "normalized-laplacian")


def main():
    out = {}
    graphs = {"er": erdos_renyi(200, 0.04, seed=14), "ba": preferential_attachment(300, 2, seed=4)}
    for gname, g in graphs.items():
        out[f"{gname}/row_ptr"] = g.row_ptr
        out[f"{gname}/col_idx"] = g.col_idx
        z = np.random.default_rng(3).standard_normal(g.n)
        out[f"{gname}/z"] = z
        for kind in KINDS:
            op = build_operator(g, kind)
            tag = f"{gname}/{kind}"
            f = lanczos_factorize(op, z, 40)
            out[f"{tag}/alphas"] = f.alphas
            out[f"{tag}/betas"] = f.betas
            out[f"{tag}/exhausted"] = np.array(f.exhausted)
            out[f"{tag}/range"] = np.array(estimate_spectral_range(op, probe_seed=2, steps=60))
            q = lanczos_quadrature(op, z, 12)
            out[f"{tag}/q_nodes"] = q.nodes
            out[f"{tag}/q_weights"] = q.weights
            probes = make_probes(g.n, 8, kind="rademacher", seed=3)
            h = gql_dos(op, probes, 30, bins=40)
            out[f"{tag}/gql_edges"] = h.edges
            out[f"{tag}/gql_masses"] = h.masses
            out[f"{tag}/gql_norm"] = np.array(h.normalization)
            q = gql_pdos(op, 7, 10)
            out[f"{tag}/pdos_nodes"] = q.nodes
            out[f"{tag}/pdos_weights"] = q.weights
        h = gql_dos_pipeline(g, "laplacian", steps=25, nz=6, probe_kind="gaussian", seed=5,
                             bins=30)
        out[f"{gname}/pipeline_edges"] = h.edges
        out[f"{gname}/pipeline_masses"] = h.masses
        sop = scaled_operator_for(g, "normalized-laplacian", seed=1)
        q = lanczos_quadrature(sop, z, 15)
        out[f"{gname}/scaled_nodes"] = q.nodes
        out[f"{gname}/scaled_weights"] = q.weights
    # exhausted Krylov spaces
    tri = build_csr([(0, 1), (1, 2), (0, 2)])
    q = lanczos_quadrature(build_operator(tri, "adjacency"), np.ones(3), 5)
    out["tri/nodes"], out["tri/exhausted"] = q.nodes, np.array(q.exhausted)
    loop = build_csr([(0, 1), (2, 2, 3.0)], allow_self_loops=True)
    q = gql_pdos(build_operator(loop, "adjacency"), 2, 4)
    out["loop/nodes"], out["loop/weights"] = q.nodes, q.weights
    out["loop/exhausted"] = np.array(q.exhausted)
    np.savez_compressed(os.path.join(HERE, "lanczos.npz"), **out)
    print(len(out), "arrays")


if __name__ == "__main__":
    main()
