"""Config-scale parity on the B200 (BASELINE.json configs C1-C5).

At full size the CPU oracle cannot run every moment of every probe (SURVEY §8c:
~9 h for C3), so each config is checked (a) bit-exactly where the path is
integer/deterministic (CSR, degrees, d^-1/2, T_m blocks), (b) against the
oracle on probe subsets / moment prefixes, and (c) through size-independent
properties (d_0 = 1, |d_m| <= 1 + 5/sqrt(nz), doubling == direct, per-node rows
averaging to the global moments, batch invariance).
"""

import os

import numpy as np
import pytest

import paper_1905_09758_b200 as kp
from paper_1905_09758_b200 import _lib
from paper_1905_09758_b200.kpm import Run

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _normwise(got, want):
    return np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300)


def _d2h(ptr, shape, ctx):
    out = np.empty(shape)
    _lib.check(_lib.load().kpm_memcpy(ctx.handle, _lib.ptr(out), ptr, out.nbytes, 1))
    ctx.synchronize()
    return out


def _sop(dev):
    return kp.rescale_operator(kp.NormalizedAdjacencyOperator(dev), (-1.0, 1.0))


_THREADS = len(os.sched_getaffinity(0))
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _fixture(cfg):
    """tests/golden/config_<cfg>.npz/.json: written by the reference's code
    (tests/golden/make_config_golden.py)."""
    with np.load(os.path.join(GOLDEN, f"config_{cfg}.npz")) as f:
        arrs = {k: f[k] for k in f.files}
    with open(os.path.join(GOLDEN, f"config_{cfg}.json")) as f:
        import json
        return arrs, json.load(f)


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _global_hist(values, bins=50):
    """histogram_from_moments on a global moment vector of the normalized
    adjacency (scale map identity)."""
    mom = kp.ChebMoments(mode="global", values=values, scale_map=kp.ScaleMap(0.0, 1.0),
                         probe_meta={})
    return kp.histogram_from_moments(mom, bins=bins).masses


def _subset_vs_fixture(cfg, scale, seed, family):
    """SURVEY §8c subset parity at the FULL moment length: the device CSR
    (row_ptr SHA) and the per-probe contributions of the fixture's probe
    columns (production doubling path and the direct estimator) against the
    reference's recurrence; the subset's finished moments and their damped
    histogram (L1 <= 1e-6)."""
    ref, meta = _fixture(cfg)
    dev = kp.DeviceGraph.rmat(scale, 16, seed)
    assert (dev.n, dev.nnz) == (meta["n"], meta["nnz"])
    rp, _, _ = dev.export()
    assert _sha(rp) == meta["row_ptr_sha"]
    cols = ref[f"{cfg}/cols"]
    want = ref[f"{cfg}/contrib"]
    m_max = want.shape[0] - 1
    probes = kp.make_probes(dev.n, family, "rademacher", seed=seed).column_slice(
        int(cols[0]), int(cols[-1]) + 1)
    sop = _sop(dev)
    got = kp.dos_contrib(sop, probes, m_max)
    got_direct = kp.dos_contrib(sop, probes, m_max, doubling=False)
    for j in range(want.shape[1]):
        assert _normwise(got[:, j], want[:, j]) <= 1e-9, j
        assert _normwise(got_direct[:, j], want[:, j]) <= 1e-12, j
    d_got = got.sum(axis=1) / (probes.nz * dev.n)   # kpm.py:115
    d_want = want.sum(axis=1) / (probes.nz * dev.n)
    assert _normwise(d_got, d_want) <= 1e-9
    l1 = np.abs(_global_hist(d_got) - _global_hist(d_want)).sum()
    assert l1 <= 1e-6
    print(cfg, "subset", want.shape, "normwise", _normwise(got, want), "direct",
          _normwise(got_direct, want), "hist L1", l1)
    dev.free()


@pytest.mark.parametrize("order", ["reference", "twin"])
def test_c3_probe_subset_full_length_vs_reference(kpm_ctx, monkeypatch, order):
    """C3: columns 0-3 of the 128-probe family x all 500 moments -- in the
    reference's neighbour order (what 4 columns run by default) and on the
    gather-ordered twin (what the 128-probe batches of the bench run)."""
    monkeypatch.setenv("KPM_REORDER", "1" if order == "twin" else "0")
    _subset_vs_fixture("c3", 24, 2, 128)


@pytest.mark.parametrize("order", ["reference", "twin"])
def test_c5_probe_subset_full_length_vs_reference(kpm_ctx, monkeypatch, order):
    """C5: columns 0-1 of the 256-probe family x the first 100 moments."""
    monkeypatch.setenv("KPM_REORDER", "1" if order == "twin" else "0")
    _subset_vs_fixture("c5", 26, 4, 256)


def test_c3_rmat24_csr_bitexact_and_probe_subset(oracle, kpm_ctx):
    """C3: R-MAT scale 24 built on the device == oracle CSR (C restatement of
    _csr_from_canonical on the same draws), bit for bit; T_2 of two probe
    columns bit-exact; 10 moments of 2 probes vs the oracle recurrence."""
    scale, ef, seed = 24, 16, 2
    dev = kp.DeviceGraph.rmat(scale, ef, seed)
    rp, ci, dinv = dev.export()
    u, v = oracle.rmat_edges(scale, ef << scale, seed)
    orp, oci = oracle.csr_from_edges(1 << scale, u, v)
    del u, v
    assert np.array_equal(rp, orp)
    assert np.array_equal(ci, oci.astype(np.int32))
    assert np.array_equal(dinv, oracle.dinv_of(orp))
    del orp
    data = oracle.normadj_values(rp, oci, dinv)
    probes = kp.make_probes(dev.n, 128, "rademacher", seed=seed).column_slice(5, 7)
    z = probes.columns
    run = Run(dev, 2, _lib.MODE_DOS_DIRECT, 12)
    run.set_probes(probes)
    run.advance(2)
    ptr, ld, _ = run.block()
    t2 = _d2h(ptr, (dev.n, ld), kpm_ctx)[:, :2]
    run.free()
    assert np.array_equal(t2, oracle.c_recurrence_block(rp, oci, data, z, 2, threads=16))
    want = oracle.c_dos_contrib(rp, oci, data, z, 10, threads=16)
    got = kp.dos_contrib(_sop(dev), probes, 10, doubling=False)
    assert _normwise(got, want) <= 1e-12
    got_d = kp.dos_contrib(_sop(dev), probes, 10, doubling=True)
    assert _normwise(got_d, want) <= 1e-9


def test_c3_full_probe_block_properties(kpm_ctx):
    """C3 with all 128 probes, 500 moments: d_0 = 1, statistical bound, the
    doubling and direct estimators agree, batch (= GPU-shard) invariance."""
    dev = kp.DeviceGraph.rmat(24, 16, 2)
    sop = _sop(dev)
    probes = kp.make_probes(dev.n, 128, "rademacher", seed=2)
    mom = kp.dos_moments(sop, probes, 500)
    assert mom.values[0] == pytest.approx(1.0, abs=1e-14)
    assert np.all(np.isfinite(mom.values))
    assert np.abs(mom.values).max() <= 1.0 + 5.0 / np.sqrt(128)
    direct = kp.dos_moments(sop, probes, 40, doubling=False)
    assert _normwise(mom.values[:41], direct.values) <= 1e-9
    c_full = kp.dos_contrib(sop, probes, 20)
    c_half = kp.dos_contrib(sop, probes, 20, batch=64)
    assert np.array_equal(c_full, c_half)
    h = kp.histogram_from_moments(mom, bins=50)
    assert h.masses.sum() == pytest.approx(1.0, abs=1e-12)


def test_c2_ba1m_ldos_full_vs_oracle_and_reference(oracle, kpm_ctx):
    """C2 in full: BA(1e6, 5, seed 1), LDOS with 64 Rademacher probes x 100
    moments -- all 1e6 nodes x 101 moments against the oracle's per-node sums
    (C restatement of kpm.py:133-148, all host threads), the reference's own
    kpm_pdos on a 2,032-node sample (tests/golden/config_c2.npz), and the
    per-node damped histograms of that sample (density.py:63-108, L1 <= 1e-6
    per node) and of the global values."""
    g = kp.preferential_attachment(1_000_000, 5, seed=1)
    ref, meta = _fixture("c2")
    assert _sha(g.row_ptr) == meta["row_ptr_sha"]
    mom, sop = kp.kpm_pdos(g, m_max=100, nz=64, probe_kind="rademacher", seed=1)
    assert mom.values.shape == (g.n, 101)
    nodes = ref["c2/nodes"]
    assert np.max(np.abs(mom.values[nodes] - ref["c2/rows"])) <= 1e-12
    assert _normwise(mom.global_values, ref["c2/global_values"]) <= 1e-12
    hist = kp.pdos_histogram(sop, kp.make_probes(g.n, 64, "rademacher", seed=1), 100,
                             bins=50, negativity_tol=np.inf)
    l1 = np.abs(hist.masses[nodes] - ref["c2/hist_rows"]).sum(axis=1)
    assert l1.max() <= 1e-6, l1.max()
    lg = np.abs(_global_hist(mom.global_values) - ref["c2/hist_global"]).sum()
    assert lg <= 1e-6
    # every node, every moment, against the oracle
    z = kp.make_probes(g.n, 64, "rademacher", seed=1).columns
    data = oracle.normadj_values_c(g.row_ptr, g.col_idx, oracle.dinv_of(g.row_ptr))
    num = oracle.c_ldos_num(g.row_ptr, g.col_idx, data, z, 100, threads=_THREADS)
    want = (num / num[0]).T
    err = np.max(np.abs(mom.values - want))
    assert err <= 1e-12, err
    glob = kp.dos_moments(sop, kp.make_probes(g.n, 64, "rademacher", seed=1), 100,
                          doubling=False)
    assert _normwise(mom.global_values, glob.values) <= 1e-9
    assert np.abs(mom.values[:, 0] - 1.0).max() == 0.0
    print("c2 full: max |err| vs oracle", err, "sample hist L1 max", l1.max(), "global L1", lg)


def test_c4_full_config_vs_reference_pipeline(oracle, kpm_ctx):
    """C4 in full against the reference's OWN kpm_dos (tests/golden/config_c4):
    BA(2e6, 4, 3) + 500k pendant-twin pairs + 100k stars; detection, device
    deflation of all 64 probes, 300 filtered moments, the spike re-inserted
    50-bin histogram (L1 <= 1e-6); plus the per-probe contributions of the
    first 4 filtered columns over all 300 moments."""
    from paper_1905_09758_b200 import motifs as M

    ref, meta = _fixture("c4")
    g = kp.testkit.motif_heavy()
    assert g.n == meta["n"] and _sha(g.row_ptr) == meta["row_ptr_sha"]
    assert _sha(g.col_idx) == meta["col_idx_sha"]
    res = kp.kpm_dos(g, m_max=300, nz=64, probe_kind="rademacher", seed=3, bins=50,
                     filter_kinds=("open-twin", "closed-twin", "dangling-two-chain"))
    adj = res.adjustment
    assert adj.deflated_dim == meta["deflated_dim"]
    assert {str(k): int(c) for k, c in sorted(adj.removed.items())} == meta["removed"]
    assert len(res.instances) == meta["instances"]
    assert _normwise(res.moments.values, ref["c4/values"]) <= 1e-9
    l1 = np.abs(res.histogram.masses - ref["c4/hist_masses"]).sum()
    assert l1 <= 1e-6, l1
    # the first 4 filtered columns, all 300 moments
    arrays, _ = M.deflation_vectors(res.instances, g.n)
    filt = M.project_probes(kp.make_probes(g.n, 64, "rademacher", seed=3).columns[:, :4].copy(),
                            arrays)
    assert np.max(np.abs(filt.sum(axis=0) - ref["c4/filtered4_sum"])) <= 1e-9
    sop = kp.scaled_operator_for(g, "normalized-adjacency")
    got = kp.dos_contrib(sop, kp.ProbeMatrix(g.n, 4, "rademacher", 3, columns=filt), 300)
    for j in range(4):
        assert _normwise(got[:, j], ref["c4/contrib4"][:, j]) <= 1e-9, j
    print("c4 full: moments normwise", _normwise(res.moments.values, ref["c4/values"]),
          "hist L1", l1)


def test_c5_rmat26_one_gpu_batch(kpm_ctx):
    """C5: R-MAT scale 26 (~1e9 edges) fits one B200 with a 128-probe batch;
    int32 column limit, degrees, and a short run's invariants."""
    dev = kp.DeviceGraph.rmat(26, 16, 4)
    assert dev.n == 1 << 26
    assert 1.8e9 < dev.nnz < (1 << 31) - 1
    sop = _sop(dev)
    probes = kp.make_probes(dev.n, 256, "rademacher", seed=4).column_slice(0, 8)
    d = kp.dos_moments(sop, probes, 20)
    dd = kp.dos_moments(sop, probes, 20, doubling=False)
    assert d.values[0] == pytest.approx(1.0, abs=1e-14)
    assert _normwise(d.values, dd.values) <= 1e-9


def test_c5_rmat26_csr_rowranges_bitexact(oracle, kpm_ctx):
    """SURVEY §8c, CSR bit-exactness at C5 by row ranges: the oracle restates
    _csr_from_canonical on every draw touching rows [a, b) (the generator run
    in 2^27-draw chunks), and rows [a, b) of the device CSR (row_ptr offsets,
    int32 col_idx, d^-1/2) must equal it bit for bit.  Ranges: the highest-
    degree ids [0, 4096), a middle window and the sparse tail."""
    scale, ef, seed = 26, 16, 4
    n = 1 << scale
    dev = kp.DeviceGraph.rmat(scale, ef, seed)
    rp, ci, dinv = dev.export()
    ranges = [(0, 4096), ((1 << 25), (1 << 25) + (1 << 18)), (n - (1 << 18), n)]
    n_draws = ef << scale
    chunk = 1 << 27
    sel = [([], []) for _ in ranges]
    for e0 in range(0, n_draws, chunk):
        u, v = oracle.rmat_edges(scale, n_draws, seed, e0=e0, count=min(chunk, n_draws - e0))
        for (a, b), (su, sv) in zip(ranges, sel):
            m = ((u >= a) & (u < b)) | ((v >= a) & (v < b))
            su.append(u[m])
            sv.append(v[m])
        del u, v
    for (a, b), (su, sv) in zip(ranges, sel):
        orp, oci = oracle.csr_from_edges(n, np.concatenate(su), np.concatenate(sv))
        want_rp = orp[a:b + 1] - orp[a]
        got_rp = rp[a:b + 1] - rp[a]
        assert np.array_equal(got_rp, want_rp), (a, b)
        assert np.array_equal(ci[rp[a]:rp[b]], oci[orp[a]:orp[b]].astype(np.int32)), (a, b)
        assert np.array_equal(dinv[a:b], oracle.dinv_of(orp[a:b + 1] - orp[a])), (a, b)
        print("c5 rows", a, b, "nnz", int(rp[b] - rp[a]))
