#!/usr/bin/env python3
"""Write the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Runs only in the build container, where /root/reference exists: it imports the
unmodified reference package (netdos 0.1.0) from /root/reference/pkg/src with
its own compiled Cython kernel (built unchanged from _spmv.c by
oracle/build_ref.sh into oracle/_ref/, so KERNEL_BACKEND == "cython"), runs
the hot-path functions on small seeded inputs and the C1 config, and stores
inputs, outputs and SHA-256 digests.  The GPU box never runs this script; the
tests read the committed .npz/.json files.

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import netdos_oracle as orc  # noqa: E402

assert orc.ref_spmv() is not None, "run `make -C oracle` first"
sys.path.insert(0, "/root/reference/pkg/src")
import netdos  # noqa: E402
from netdos import (MotifKind, OperatorKind, ProbeKind, build_csr,  # noqa: E402
                    build_operator, detect_motifs, dos_moments, filter_probes,
                    histogram_from_moments, make_probes, pdos_moments)
from netdos.graph import _csr_from_canonical  # noqa: E402
from netdos.pipeline import kpm_dos, scaled_operator_for  # noqa: E402
from netdos.testkit import erdos_renyi, preferential_attachment  # noqa: E402

assert netdos.KERNEL_BACKEND == "cython", netdos.KERNEL_BACKEND


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def t_block(sop, z, steps):
    """T_steps block via the reference's own recurrence driver."""
    from netdos.kpm import _recurrence
    box = {}

    def collect(m, t):
        if m == steps:
            box["t"] = t.copy()

    _recurrence(sop, z, steps, collect, 1)
    return box["t"]


def graph_case(name, g, nz, seed, m_dos, m_pdos, store_blocks, out):
    sop = scaled_operator_for(g, OperatorKind.NORMALIZED_ADJACENCY)
    p = make_probes(g.n, nz, ProbeKind.RADEMACHER, seed=seed)
    d = dos_moments(sop, p, m_dos)
    contrib = np.empty((m_dos + 1, nz))
    from netdos.kpm import _recurrence

    def col(m, t):
        contrib[m] = np.einsum("ij,ij->j", p.columns, t)

    _recurrence(sop, p.columns, m_dos, col, 1)
    pd = pdos_moments(sop, p, m_pdos)
    h = histogram_from_moments(d, bins=50)
    rec = {
        f"{name}/n": np.int64(g.n),
        f"{name}/row_ptr": g.row_ptr, f"{name}/col_idx": g.col_idx,
        f"{name}/degrees": g.degrees(), f"{name}/op_data": sop.base.data,
        f"{name}/op_indptr": sop.base.indptr, f"{name}/op_indices": sop.base.indices,
        f"{name}/probes": p.columns, f"{name}/dos_values": d.values,
        f"{name}/dos_contrib": contrib, f"{name}/pdos_values": pd.values,
        f"{name}/hist_masses": h.masses, f"{name}/hist_edges": h.edges,
        f"{name}/meta": np.array([nz, seed, m_dos, m_pdos], dtype=np.int64),
    }
    for s in store_blocks:
        rec[f"{name}/T{s}"] = t_block(sop, p.columns, s)
    out.update(rec)


def main():
    out = {}
    summary = {"reference": "netdos 0.1.0 (/root/reference/pkg), KERNEL_BACKEND=cython",
               "numpy": np.__version__}

    # --- tiny closed-form graphs + small random graphs (full arrays) -------
    tri = build_csr([(0, 1), (0, 2), (1, 2)])
    p3 = build_csr([(0, 1), (1, 2)])
    star = build_csr([(0, 1), (0, 2), (0, 3)])
    edges = []
    for i in range(4):
        for j in range(5):
            if j + 1 < 5:
                edges.append((i * 5 + j, i * 5 + j + 1))
            if i + 1 < 4:
                edges.append((i * 5 + j, (i + 1) * 5 + j))
    grid = build_csr(edges)
    # isolated trailing nodes exercise the d^-1/2 = 0 convention
    iso = build_csr([(0, 1), (1, 2), (2, 3), (0, 3), (4, 5)], n=9)
    for name, g in [("triangle", tri), ("path3", p3), ("star4", star), ("grid4x5", grid),
                    ("isolated9", iso)]:
        graph_case(name, g, 3, 1, 12, 8, (1, 2, 5), out)
    graph_case("er200", erdos_renyi(200, 0.05, seed=3), 7, 11, 40, 20, (1, 2, 3, 10), out)
    graph_case("ba300", preferential_attachment(300, 3, seed=4), 20, 5, 60, 30,
               (1, 2, 3, 10), out)
    graph_case("ba_p64", preferential_attachment(500, 2, seed=9), 64, 2, 30, 30, (1, 7), out)

    # --- explicit-values mode: Laplacian with a shifted/scaled range -------
    g = erdos_renyi(60, 0.1, seed=21)
    sop = scaled_operator_for(g, OperatorKind.LAPLACIAN, seed=0)
    p = make_probes(g.n, 5, ProbeKind.GAUSSIAN, seed=8)
    d = dos_moments(sop, p, 30)
    out.update({"lap60/indptr": sop.base.indptr, "lap60/indices": sop.base.indices,
                "lap60/data": sop.base.data,
                "lap60/shift_scale": np.array([sop.shift, sop.scale]),
                "lap60/probes": p.columns, "lap60/dos_values": d.values,
                "lap60/T3": t_block(sop, p.columns, 3),
                "lap60/pdos_values": pdos_moments(sop, p, 15).values})

    # --- probe generators ---------------------------------------------------
    for kind in ("rademacher", "gaussian", "hadamard"):
        out[f"probes/{kind}"] = make_probes(1000, 8, kind, seed=17).columns
    out["probes/std_basis"] = make_probes(6, 4, "standard-basis", seed=0).columns

    # --- _csr_from_canonical on raw pairs after canonicalise + unique ------
    rng = np.random.default_rng(5)
    u = rng.integers(0, 700, size=4000)
    v = rng.integers(0, 700, size=4000)
    a, b = np.minimum(u, v), np.maximum(u, v)
    keep = a != b
    key = np.unique(a[keep] * 700 + b[keep])
    gc = _csr_from_canonical(700, key // 700, key % 700, np.ones(key.size), False)
    out.update({"canon/u": u, "canon/v": v, "canon/row_ptr": gc.row_ptr,
                "canon/col_idx": gc.col_idx})

    # --- motif detection + probe filtering (C4 semantics, small) ----------
    base = preferential_attachment(400, 2, seed=7)
    bu, bv, _ = base.edge_list()
    rng = np.random.default_rng(3)
    us, vs = list(bu.tolist()), list(bv.tolist())
    nxt = base.n
    for _ in range(40):  # pendant-twin pairs on random hubs
        hub = int(rng.integers(0, base.n))
        us += [hub, hub]
        vs += [nxt, nxt + 1]
        nxt += 2
    for _ in range(10):  # 4-node stars attached by their centre
        att = int(rng.integers(0, base.n))
        c = nxt
        us += [att, c, c, c]
        vs += [c, c + 1, c + 2, c + 3]
        nxt += 4
    for _ in range(6):  # dangling two-chains (two per hub -> +-1/sqrt 2)
        hub = int(rng.integers(0, base.n))
        us += [hub, nxt, hub, nxt + 2]
        vs += [nxt, nxt + 1, nxt + 2, nxt + 3]
        nxt += 4
    a, b = np.minimum(us, vs), np.maximum(us, vs)
    key = np.unique(np.asarray(a, dtype=np.int64) * nxt + np.asarray(b, dtype=np.int64))
    gm = _csr_from_canonical(nxt, key // nxt, key % nxt, np.ones(key.size), False)
    insts = detect_motifs(gm, seed=3)
    pm = make_probes(gm.n, 16, ProbeKind.RADEMACHER, seed=3)
    filt, adj = filter_probes(pm, insts)
    sopm = scaled_operator_for(gm, OperatorKind.NORMALIZED_ADJACENCY)
    dm = dos_moments(sopm, filt, 80, effective_dim=gm.n - adj.deflated_dim)
    hm = histogram_from_moments(dm, bins=40, filter_adjustment=adj)
    res = kpm_dos(gm, m_max=80, nz=16, probe_kind=ProbeKind.RADEMACHER, seed=3, bins=40,
                  filter_kinds=("open-twin", "closed-twin", "dangling-two-chain"))
    assert np.array_equal(res.moments.values, dm.values)
    out.update({"motif/u": key // nxt, "motif/v": key % nxt, "motif/n": np.int64(nxt),
                "motif/row_ptr": gm.row_ptr, "motif/col_idx": gm.col_idx,
                "motif/probes": pm.columns, "motif/filtered": filt.columns,
                "motif/dos_values": dm.values, "motif/hist_masses": hm.masses})
    summary["motif"] = {
        "removed": {repr(k): v for k, v in adj.removed.items()},
        "total_dim": adj.total_dim,
        "instances": [[i.kind.value, list(i.nodes), i.eigenvalue, i.multiplicity,
                       [[[int(k), float(v)] for k, v in vec.items()] for vec in i.eigvecs],
                       {k: (list(map(list, v)) if k == "chains" else v)
                        for k, v in i.detail.items()}]
                      for i in insts],
    }

    # --- generators + the C1 config (digests; C1 moments in full) ---------
    gens = {}
    for (n, p_, s) in [(10000, 1e-3, 0), (500, 0.02, 1), (3000, 0.004, 9)]:
        g = erdos_renyi(n, p_, seed=s)
        gens[f"er_{n}_{p_}_{s}"] = {"nnz": g.nnz, "row_ptr": sha(g.row_ptr),
                                    "col_idx": sha(g.col_idx)}
    for (n, m, s) in [(300, 3, 4), (5000, 5, 1), (20000, 5, 1)]:
        g = preferential_attachment(n, m, seed=s)
        gens[f"ba_{n}_{m}_{s}"] = {"nnz": g.nnz, "row_ptr": sha(g.row_ptr),
                                   "col_idx": sha(g.col_idx)}
    if os.environ.get("GOLDEN_FULL_BA", "1") == "1":
        for (n, m, s) in [(1_000_000, 5, 1), (2_000_000, 4, 3)]:
            t0 = time.time()
            g = preferential_attachment(n, m, seed=s)
            gens[f"ba_{n}_{m}_{s}"] = {"nnz": g.nnz, "row_ptr": sha(g.row_ptr),
                                       "col_idx": sha(g.col_idx),
                                       "ref_seconds": time.time() - t0}
    summary["generators"] = gens

    g = erdos_renyi(10000, 1e-3, seed=0)
    sop = scaled_operator_for(g, OperatorKind.NORMALIZED_ADJACENCY)
    p = make_probes(g.n, 20, ProbeKind.RADEMACHER, seed=0)
    t0 = time.perf_counter()
    d = dos_moments(sop, p, 200)
    t_ref = time.perf_counter() - t0
    h = histogram_from_moments(d, bins=100)
    c1 = {"nnz": g.nnz, "row_ptr": sha(g.row_ptr), "col_idx": sha(g.col_idx),
          "dinv_data": sha(sop.base.data), "probes": sha(p.columns),
          "T1": sha(t_block(sop, p.columns, 1)), "T2": sha(t_block(sop, p.columns, 2)),
          "T7": sha(t_block(sop, p.columns, 7)), "dos_seconds_1thread": t_ref}
    summary["c1"] = c1
    out["c1/dos_values"] = d.values
    out["c1/hist_masses"] = h.masses

    # C2-shaped, reduced n (the full 1e6-node LDOS oracle run is ~2 min at 8
    # threads; tests run the oracle at full size on the GPU box instead)
    g = preferential_attachment(20000, 5, seed=1)
    sop = scaled_operator_for(g, OperatorKind.NORMALIZED_ADJACENCY)
    p = make_probes(g.n, 64, ProbeKind.RADEMACHER, seed=1)
    pd = pdos_moments(sop, p, 100)
    rows = np.random.default_rng(0).choice(g.n, 64, replace=False)
    rows.sort()
    out["c2s/rows"] = rows
    out["c2s/pdos_rows"] = pd.values[rows]
    out["c2s/global_values"] = pd.global_values
    summary["c2s"] = {"pdos_values": sha(pd.values), "probes": sha(p.columns)}

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
