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


# SURVEY §8c subset parity: C3 4 probes x all 500 moments, C5 2 probes x the
# first 100 moments against the oracle recurrence.  The oracle needs ~15 min
# (C3) / ~6 min (C5) on 16 host cores, so the default suite runs the same
# comparison over a moment prefix; KPM_FULL_SUBSET=1 runs the full lengths
# (profiles/r01_subset_parity.log).
_FULL = os.environ.get("KPM_FULL_SUBSET") == "1"
_THREADS = len(os.sched_getaffinity(0))


def _host_ram_gb():
    return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30


def _subset_parity(oracle, dev, probes, m_max):
    """GPU per-probe contributions (production doubling path, and direct)
    vs the oracle's sequential recurrence on the same CSR and probe columns."""
    rp, ci, dinv = dev.export()
    ci = ci.astype(np.int64)
    data = oracle.normadj_values(rp, ci, dinv)
    want = oracle.c_dos_contrib(rp, ci, data, probes.columns, m_max, threads=_THREADS)
    del ci, data
    sop = _sop(dev)
    got = kp.dos_contrib(sop, probes, m_max)
    got_direct = kp.dos_contrib(sop, probes, m_max, doubling=False)
    for j in range(want.shape[1]):
        assert _normwise(got[:, j], want[:, j]) <= 1e-9, j
        assert _normwise(got_direct[:, j], want[:, j]) <= 1e-12, j
    # the finished moments (kpm.py:115) of the subset
    d_got = got.sum(axis=1) / (probes.nz * dev.n)
    d_want = want.sum(axis=1) / (probes.nz * dev.n)
    assert _normwise(d_got, d_want) <= 1e-9
    return _normwise(got, want)


def test_c3_probe_subset_vs_oracle(oracle, kpm_ctx):
    """C3: columns 0-3 of the 128-probe family, all 500 moments with
    KPM_FULL_SUBSET=1 (else the first 30)."""
    dev = kp.DeviceGraph.rmat(24, 16, 2)
    probes = kp.make_probes(dev.n, 128, "rademacher", seed=2).column_slice(0, 4)
    err = _subset_parity(oracle, dev, probes, 500 if _FULL else 30)
    print("c3 subset normwise", err, "full" if _FULL else "prefix")


def test_c5_probe_subset_vs_oracle(oracle, kpm_ctx):
    """C5: columns 0-1 of the 256-probe family, the first 100 moments with
    KPM_FULL_SUBSET=1 (else the first 6); the oracle holds int64 indices and
    fp64 values for 2.1e9 nonzeros (~34 GB of host memory)."""
    if _host_ram_gb() < 96:
        pytest.skip("needs ~96 GB of host memory for the C5 oracle operator")
    dev = kp.DeviceGraph.rmat(26, 16, 4)
    probes = kp.make_probes(dev.n, 256, "rademacher", seed=4).column_slice(0, 2)
    err = _subset_parity(oracle, dev, probes, 100 if _FULL else 6)
    print("c5 subset normwise", err, "full" if _FULL else "prefix")


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


def test_c2_ba1m_ldos_vs_oracle(oracle, kpm_ctx):
    """C2: BA(1e6, 5, seed 1) (the reference's generator, SHA-pinned), LDOS
    with 64 Rademacher probes, 100 moments; the oracle per-node sums over the
    first 12 moments for all 1e6 nodes; global consistency over all 100."""
    g = kp.preferential_attachment(1_000_000, 5, seed=1)
    mom, sop = kp.kpm_pdos(g, m_max=100, nz=64, probe_kind="rademacher", seed=1)
    assert mom.values.shape == (g.n, 101)
    z = kp.make_probes(g.n, 64, "rademacher", seed=1).columns
    data = oracle.normadj_values(g.row_ptr, g.col_idx)
    num = oracle.c_ldos_num(g.row_ptr, g.col_idx, data, z, 12, threads=16)
    want = (num / num[0]).T
    assert np.max(np.abs(mom.values[:, :13] - want)) <= 1e-12
    glob = kp.dos_moments(sop, kp.make_probes(g.n, 64, "rademacher", seed=1), 100,
                          doubling=False)
    assert _normwise(mom.global_values, glob.values) <= 1e-9
    assert np.abs(mom.values[:, 0] - 1.0).max() == 0.0


def test_c4_motif_pipeline_vs_oracle(oracle, kpm_ctx):
    """C4: BA(2e6, 4, 3) + 500k pendant-twin pairs + 100k stars; detection,
    device deflation of 64 probes, filtered DOS with 300 moments.  The
    deflation of 4 probe columns is re-done by the oracle's sequential loop
    (motifs.py:400-403) and their first 20 moments by the oracle recurrence."""
    from paper_1905_09758_b200 import motifs as M

    g = kp.testkit.motif_heavy()
    assert g.n == 3_400_000
    res = kp.kpm_dos(g, m_max=300, nz=64, probe_kind="rademacher", seed=3, bins=50,
                     filter_kinds=("open-twin", "closed-twin", "dangling-two-chain"))
    r = res.adjustment.deflated_dim
    assert r > 600_000
    # the bin masses telescope to d_0 (n-r)/n + r/n (re-inserted spikes)
    d0 = res.moments.values[0]
    assert abs(res.histogram.masses.sum() - (d0 * (g.n - r) / g.n + r / g.n)) < 1e-9
    arrays, removed = M.deflation_vectors(res.instances, g.n)
    assert removed == res.adjustment.removed
    z = kp.make_probes(g.n, 64, "rademacher", seed=3).columns[:, :4]
    zf = oracle.project_out(z, arrays)
    filt = M.project_probes(kp.make_probes(g.n, 64, "rademacher", seed=3).columns, arrays)
    assert np.max(np.abs(filt[:, :4] - zf)) <= 1e-12
    data = oracle.normadj_values(g.row_ptr, g.col_idx)
    want = oracle.c_dos_contrib(g.row_ptr, g.col_idx, data, zf, 20, threads=16)
    sop = kp.scaled_operator_for(g, "normalized-adjacency")
    got = kp.dos_contrib(sop, kp.ProbeMatrix(g.n, 4, "rademacher", 3, columns=filt[:, :4]),
                         20)
    assert _normwise(got, want) <= 1e-9


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
