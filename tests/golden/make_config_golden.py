#!/usr/bin/env python3
"""Config-scale fixtures (BASELINE.json C2-C5) written by the REFERENCE's code.

SURVEY.md §8c subset parity, committed so the ``-m gpu`` suite checks the full
lengths in seconds (tests/test_gpu_configs.py):

* ``c3``: R-MAT scale 24 / ef 16 / seed 2 (harness generator, C restatement
  pinned bit-exact against the device one), probe columns 0-3 of
  ``make_probes(n, 128, RADEMACHER, seed=2)``, all 500 moments: the per-probe
  contribution matrix ``contrib[m, j] = z_j^T T_m z_j`` (kpm.py:104-108).
* ``c5``: R-MAT scale 26 / ef 16 / seed 4, columns 0-1 of the 256-probe
  family, the first 100 moments.
* ``c4``: the reference's OWN ``kpm_dos`` pipeline (pipeline.py:62-91) on the
  motif-heavy graph, full config: detect_motifs + filter_probes + 64 probes x
  300 moments + the 50-bin histogram; plus the per-probe contributions of the
  first 4 filtered columns.
* ``c2``: the reference's OWN ``kpm_pdos`` (pipeline.py:94-100) on BA(1e6, 5,
  seed 1), 64 probes x 100 moments: global values, the per-node rows of a
  seeded node sample (+ the 32 highest-degree nodes) and their histograms.

Engines: in this container (``/root/reference`` present) the recurrence is the
reference's own ``netdos.kpm._recurrence`` over a reference
``SymmetricCSROperator`` and the reference's compiled Cython kernel
(``KERNEL_BACKEND == "cython"``).  C5 needs ~60 GB of host memory for the
reference's int64/fp64 operator arrays, so it is generated on the GPU box's
host (196 GB) where ``/root/reference`` is absent: there the recurrence is the
oracle's restated glue (oracle/netdos_oracle.py ``recurrence``, pinned to the
reference by tests/test_oracle.py) around the same compiled Cython kernel
(oracle/_ref, built unchanged from the reference's _spmv.c).  The CSR comes from
the oracle's C restatement of ``_csr_from_canonical`` (bit-exact vs the device
loader, tests/test_gpu_configs.py) and the operator values from
``operators.py:108-110`` (bit-identical to ``build_operator``).

    python tests/golden/make_config_golden.py c3 c4 c2     # here
    python tests/golden/make_config_golden.py c5 --out gpurun_out   # GPU box host
"""

from __future__ import annotations

import argparse
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

REF_SRC = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(REF_SRC)
if HAVE_REF:
    # register the reference's compiled kernel (oracle/_ref) as
    # netdos._kernels._spmv before netdos is imported -> KERNEL_BACKEND "cython"
    assert orc.ref_spmv() is not None, "run `make -C oracle` first"
    sys.path.insert(0, REF_SRC)

THREADS = orc.cpu_threads()


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def _rmat_csr(scale, seed):
    u, v = orc.rmat_edges(scale, 16 << scale, seed)
    rp, ci = orc.csr_from_edges(1 << scale, u, v)
    del u, v
    return rp, ci


def _columns(n, seed, cols):
    """Columns j of make_probes(n, P, RADEMACHER, seed): SeedSequence(seed,
    spawn_key=(j,)) is SeedSequence(seed).spawn(P)[j] (pinned by
    tests/test_oracle.py)."""
    return np.ascontiguousarray(np.stack([orc.rademacher_column(n, seed, j) for j in cols], 1))


def _contrib(rp, ci, data, z, m_max):
    """Per-probe contributions through the reference's recurrence driver."""
    n = rp.shape[0] - 1
    contrib = np.empty((m_max + 1, z.shape[1]))

    def collect(m, t):
        contrib[m] = np.einsum("ij,ij->j", z, t)

    if HAVE_REF:
        import netdos
        from netdos.kpm import _recurrence
        from netdos.operators import OperatorKind, SymmetricCSROperator, rescale_operator

        assert netdos.KERNEL_BACKEND == "cython", netdos.KERNEL_BACKEND
        op = SymmetricCSROperator(n, rp, ci, data, OperatorKind.NORMALIZED_ADJACENCY)
        sop = rescale_operator(op, (-1.0, 1.0))
        _recurrence(sop, z, m_max, collect, THREADS)
        engine = "reference netdos.kpm._recurrence + compiled Cython csr_matvec"
    else:
        assert orc.ref_spmv() is not None, "oracle/_ref not built"
        op = orc.CSROp(rp, ci, data, engine="ref")
        orc.recurrence(op, z, m_max, collect, THREADS)
        engine = "oracle recurrence (restated kpm.py:73-89) + reference's compiled Cython csr_matvec"
    return contrib, engine


def rmat_subset(name, scale, seed, family, cols, m_max, out):
    t0 = time.time()
    rp, ci = _rmat_csr(scale, seed)
    n, nnz = rp.shape[0] - 1, ci.shape[0]
    log(name, "csr", n, nnz, f"{time.time() - t0:.1f}s")
    dinv = orc.dinv_of(rp)
    data = orc.normadj_values(rp, ci, dinv)
    z = _columns(n, seed, cols)
    t0 = time.time()
    contrib, engine = _contrib(rp, ci, data, z, m_max)
    log(name, "recurrence", f"{time.time() - t0:.1f}s")
    out[f"{name}/contrib"] = contrib
    out[f"{name}/cols"] = np.asarray(cols, dtype=np.int64)
    meta = {"n": int(n), "nnz": int(nnz), "m_max": m_max, "family": family, "seed": seed,
            "row_ptr_sha": sha(rp), "probe_sha": sha(z), "engine": engine,
            "threads": THREADS, "seconds": round(time.time() - t0, 1)}
    return meta


def c2(out):
    import netdos
    from netdos import ProbeKind, histogram_from_moments
    from netdos.pipeline import kpm_pdos
    from netdos.testkit import preferential_attachment

    assert netdos.KERNEL_BACKEND == "cython"
    t0 = time.time()
    g = preferential_attachment(1_000_000, 5, seed=1)
    log("c2 graph", f"{time.time() - t0:.1f}s")
    t0 = time.time()
    mom, sop = kpm_pdos(g, m_max=100, nz=64, probe_kind=ProbeKind.RADEMACHER, seed=1,
                        threads=THREADS)
    log("c2 kpm_pdos", f"{time.time() - t0:.1f}s")
    deg = np.diff(g.row_ptr)
    rng = np.random.default_rng(20261021)
    sample = np.unique(np.concatenate([rng.choice(g.n, 2000, replace=False),
                                       np.argsort(-deg, kind="stable")[:32]]))
    rows = mom.values[sample]
    out["c2/nodes"] = sample.astype(np.int64)
    out["c2/rows"] = rows
    out["c2/global_values"] = mom.global_values
    out["c2/row_sum"] = mom.values.sum(axis=0)
    # per-node histograms of the sample (density.py:63-108 on per-node moments)
    from netdos.kpm import ChebMoments
    sub = ChebMoments(mode=mom.mode, values=rows, scale_map=mom.scale_map,
                      probe_meta=mom.probe_meta)
    # per-node series of 64 probes dip below the default 1e-3 negativity
    # guard (density.py:102-107): the masses are what is pinned here
    h = histogram_from_moments(sub, bins=50, negativity_tol=np.inf)
    out["c2/hist_rows"] = h.masses
    out["c2/hist_edges"] = h.edges
    hg = histogram_from_moments(ChebMoments(mode="global", values=mom.global_values,
                                            scale_map=mom.scale_map,
                                            probe_meta=mom.probe_meta), bins=50)
    out["c2/hist_global"] = hg.masses
    return {"n": int(g.n), "nnz": int(g.row_ptr[-1]), "m_max": 100, "nz": 64, "seed": 1,
            "engine": "reference netdos.pipeline.kpm_pdos (Cython kernel)",
            "threads": THREADS, "sample": int(sample.shape[0]),
            "row_ptr_sha": sha(g.row_ptr), "seconds": round(time.time() - t0, 1)}


def c4(out):
    import netdos
    from netdos import ProbeKind
    from netdos.graph import _csr_from_canonical
    from netdos.kpm import _recurrence
    from netdos.pipeline import kpm_dos
    from netdos.testkit import preferential_attachment

    assert netdos.KERNEL_BACKEND == "cython"
    # the C4 harness rule (paper_1905_09758_b200/testkit.py motif_heavy_edges,
    # DESIGN.md §8), written out here over the reference's own generator
    n_ba, m, seed, twin_pairs, stars = 2_000_000, 4, 3, 500_000, 100_000
    t0 = time.time()
    gba = preferential_attachment(n_ba, m, seed=seed)
    rows = np.repeat(np.arange(n_ba, dtype=np.int64), np.diff(gba.row_ptr))
    keep = rows < gba.col_idx
    bu, bv = rows[keep], gba.col_idx[keep]
    rng = np.random.default_rng([seed, 0xC4])
    hubs = rng.integers(0, n_ba, size=twin_pairs)
    att = rng.integers(0, n_ba, size=stars)
    leaf = n_ba + 2 * np.arange(twin_pairs, dtype=np.int64)
    c = n_ba + 2 * twin_pairs + 4 * np.arange(stars, dtype=np.int64)
    u = np.concatenate([bu, hubs, hubs, att, c, c, c]).astype(np.int64)
    v = np.concatenate([bv, leaf, leaf + 1, c, c + 1, c + 2, c + 3]).astype(np.int64)
    n = n_ba + 2 * twin_pairs + 4 * stars
    g = _csr_from_canonical(n, np.minimum(u, v), np.maximum(u, v), np.ones(u.shape[0]), False)
    log("c4 graph", n, g.row_ptr[-1], f"{time.time() - t0:.1f}s")
    t0 = time.time()
    res = kpm_dos(g, m_max=300, nz=64, probe_kind=ProbeKind.RADEMACHER, seed=3, bins=50,
                  filter_kinds=("open-twin", "closed-twin", "dangling-two-chain"),
                  threads=THREADS)
    log("c4 kpm_dos", f"{time.time() - t0:.1f}s")
    adj = res.adjustment
    out["c4/values"] = res.moments.values
    out["c4/hist_masses"] = res.histogram.masses
    out["c4/hist_edges"] = res.histogram.edges
    # per-probe contributions of the first 4 filtered columns
    z = np.ascontiguousarray(adj.probes.columns[:, :4]) if hasattr(adj, "probes") else None
    if z is None:
        from netdos import filter_probes, make_probes
        p = make_probes(n, 64, ProbeKind.RADEMACHER, seed=3)
        fp, _ = filter_probes(p, res.instances)
        z = np.ascontiguousarray(fp.columns[:, :4])
    contrib = np.empty((301, 4))

    def collect(mm, t):
        contrib[mm] = np.einsum("ij,ij->j", z, t)

    _recurrence(res.scaled_op, z, 300, collect, THREADS)
    out["c4/contrib4"] = contrib
    out["c4/filtered4_sum"] = z.sum(axis=0)
    return {"n": int(n), "nnz": int(g.row_ptr[-1]), "m_max": 300, "nz": 64, "seed": 3,
            "deflated_dim": int(adj.deflated_dim),
            "removed": {str(k): int(c_) for k, c_ in sorted(adj.removed.items())},
            "instances": len(res.instances), "row_ptr_sha": sha(g.row_ptr),
            "col_idx_sha": sha(g.col_idx),
            "engine": "reference netdos.pipeline.kpm_dos (Cython kernel)", "threads": THREADS,
            "seconds": round(time.time() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--out", default=HERE)
    args = ap.parse_args()
    for cfg in args.configs:
        out = {}
        if cfg == "c3":
            meta = rmat_subset("c3", 24, 2, 128, [0, 1, 2, 3], 500, out)
        elif cfg == "c5":
            meta = rmat_subset("c5", 26, 4, 256, [0, 1], 100, out)
        elif cfg == "c4":
            meta = c4(out)
        else:
            meta = c2(out)
        os.makedirs(args.out, exist_ok=True)
        np.savez_compressed(os.path.join(args.out, f"config_{cfg}.npz"), **out)
        with open(os.path.join(args.out, f"config_{cfg}.json"), "w") as f:
            json.dump(meta, f, indent=1, sort_keys=True)
        log(cfg, "written", meta)


if __name__ == "__main__":
    main()
