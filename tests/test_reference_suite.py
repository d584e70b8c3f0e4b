"""The reference's own tests for the hot path (pkg/tests/test_kpm.py,
test_motifs.py, test_operators.py, test_density.py, test_acceptance.py
criteria 1-3 and 9), re-run against this package.  Same graphs, seeds,
probes and tolerances; every moment here is computed by the B200 kernels
(GPU-marked) -- the closed forms and the dense eigen-oracle are the checks."""

import time

import numpy as np
import pytest

import paper_1905_09758_b200 as kp
from paper_1905_09758_b200 import testkit
from paper_1905_09758_b200.kpm import chebyshev_values
from paper_1905_09758_b200.pipeline import scaled_operator_for

gpu = pytest.mark.gpu


@pytest.fixture
def triangle():
    return kp.build_csr([(0, 1), (0, 2), (1, 2)])


@pytest.fixture
def path3():
    return kp.build_csr([(0, 1), (1, 2)])


@pytest.fixture
def star4():
    return kp.build_csr([(0, 1), (0, 2), (0, 3)])


def _scaled(g, kind="normalized-adjacency", seed=0):
    return scaled_operator_for(g, kind, seed=seed)


def _dense_from_graph(g, kind):
    """Independent dense construction of each operator family (conftest.py:34-51)."""
    a = np.zeros((g.n, g.n))
    for i in range(g.n):
        sl = g.neighbor_slice(i)
        for j, w in zip(g.col_idx[sl].tolist(), g.weights[sl].tolist()):
            a[i, j] = w
    deg = a.sum(axis=1)
    if kind == "adjacency":
        return a
    if kind == "laplacian":
        return np.diag(deg) - a
    with np.errstate(divide="ignore"):
        dinv = np.where(deg > 0, 1.0 / np.sqrt(np.where(deg > 0, deg, 1.0)), 0.0)
    na = dinv[:, None] * a * dinv[None, :]
    return na if kind == "normalized-adjacency" else np.eye(g.n) - na


# ----------------------------------------------------------- test_kpm.py
@gpu
def test_dos_moment_zero_is_one(star4):
    mom = kp.dos_moments(_scaled(star4), kp.make_probes(4, 3, "rademacher", seed=1), 0)
    assert mom.values.shape == (1,)
    assert mom.values[0] == pytest.approx(1.0, abs=1e-14)


@gpu
@pytest.mark.parametrize("doubling", [True, False])
def test_k3_first_two_moments_vanish(triangle, doubling):
    p = kp.make_probes(3, 3, "standard-basis", seed=0)
    mom = kp.dos_moments(_scaled(triangle), p, 2, doubling=doubling)
    assert mom.values[1] == pytest.approx(0.0, abs=1e-14)
    assert mom.values[2] == pytest.approx(0.0, abs=1e-14)


@gpu
@pytest.mark.parametrize("doubling", [True, False])
def test_p3_moments_match_closed_form(path3, doubling):
    p = kp.make_probes(3, 3, "standard-basis", seed=0)
    mom = kp.dos_moments(_scaled(path3), p, 4, doubling=doubling)
    want = chebyshev_values(4, np.array([-1.0, 0.0, 1.0])).mean(axis=1)
    assert np.abs(mom.values - want).max() < 1e-13


@gpu
@pytest.mark.parametrize("doubling", [True, False])
def test_moment_exactness_against_eigenvalue_oracle(doubling):
    rng = np.random.default_rng(100)
    for kind in ("normalized-adjacency", "laplacian"):
        n = int(rng.integers(40, 120))
        g = kp.erdos_renyi(n, 0.08, seed=int(rng.integers(1 << 30)))
        sop = _scaled(g, kind)
        p = kp.make_probes(n, n, "standard-basis", seed=0)
        mom = kp.dos_moments(sop, p, 50, doubling=doubling)
        ev = testkit.exact_spectrum(sop.base).eigenvalues
        want = testkit.oracle_moments(sop.scale_map.to_scaled(ev), 50)
        assert np.abs(mom.values - want).max() < 1e-10


@gpu
def test_pdos_zero_degree_moment_is_one(star4):
    sop = _scaled(star4)
    for kind in ("rademacher", "gaussian", "hadamard"):
        mom = kp.pdos_moments(sop, kp.make_probes(4, 3, kind, seed=2), 3)
        assert np.abs(mom.values[:, 0] - 1.0).max() < 1e-12


@gpu
def test_p3_center_second_moment(path3):
    mom = kp.pdos_moments(_scaled(path3), kp.make_probes(3, 3, "standard-basis"), 2)
    assert mom.values[1, 2] == pytest.approx(1.0, abs=1e-13)


@gpu
def test_star_leaf_first_moment_zero(star4):
    mom = kp.pdos_moments(_scaled(star4), kp.make_probes(4, 4, "standard-basis"), 1)
    assert np.abs(mom.values[1:, 1]).max() < 1e-14


@gpu
def test_pdos_rows_average_to_global_moments():
    g = kp.erdos_renyi(80, 0.06, seed=6)
    sop = _scaled(g)
    for kind in ("rademacher", "hadamard", "standard-basis"):
        nz = g.n if kind == "standard-basis" else 12
        p = kp.make_probes(g.n, nz, kind, seed=5)
        per_node = kp.pdos_moments(sop, p, 25)
        glob = kp.dos_moments(sop, p, 25)
        assert np.abs(per_node.values.mean(axis=0) - glob.values).max() < 1e-10


@gpu
def test_pdos_exact_probes_match_node_oracle():
    g = kp.erdos_renyi(70, 0.08, seed=8)
    sop = _scaled(g, "normalized-laplacian")
    mom = kp.pdos_moments(sop, kp.make_probes(g.n, g.n, "standard-basis"), 30)
    spec = testkit.exact_spectrum(sop.base, want_vectors=True)
    t = chebyshev_values(30, sop.scale_map.to_scaled(spec.eigenvalues))
    assert np.abs(mom.values - (spec.eigenvectors ** 2) @ t.T).max() < 1e-10


@gpu
def test_polynomial_integration_exactness():
    g = kp.erdos_renyi(50, 0.1, seed=12)
    sop = _scaled(g)
    mom = kp.dos_moments(sop, kp.make_probes(g.n, g.n, "standard-basis"), 24)
    coef = np.random.default_rng(3).standard_normal(25)
    ev = sop.scale_map.to_scaled(testkit.exact_spectrum(sop.base).eigenvalues)
    assert coef @ mom.values == pytest.approx((coef @ chebyshev_values(24, ev)).mean(),
                                              abs=1e-8)


@gpu
def test_statistical_moment_bound():
    g = kp.erdos_renyi(300, 0.03, seed=2)
    sop = _scaled(g)
    for kind in ("rademacher", "hadamard", "gaussian"):
        mom = kp.dos_moments(sop, kp.make_probes(g.n, 16, kind, seed=3), 200)
        assert np.abs(mom.values).max() <= 1.0 + 5.0 / np.sqrt(16)


@gpu
def test_recurrence_blowup_detected(path3):
    bad = kp.rescale_operator(kp.build_operator(path3, "laplacian"), (0.0, 1.5))
    with pytest.raises(kp.RecurrenceBlowupError, match="margin"):
        kp.dos_moments(bad, kp.make_probes(3, 2, "rademacher", seed=0), 600)


@gpu
def test_hadamard_not_worse_than_rademacher_for_trace_noise():
    g = kp.erdos_renyi(256, 0.05, seed=4)
    sop = _scaled(g)
    exact = kp.dos_moments(sop, kp.make_probes(g.n, g.n, "standard-basis"), 60)
    errs = {}
    for kind in ("hadamard", "rademacher"):
        errs[kind] = np.mean([np.abs(kp.dos_moments(sop, kp.make_probes(g.n, 8, kind, s),
                                                    60).values - exact.values).max()
                              for s in range(8)])
    assert errs["hadamard"] < 2.0 * errs["rademacher"]


@gpu
def test_per_node_statistical_moment_bound():
    g = kp.erdos_renyi(150, 0.05, seed=8)
    mom = kp.pdos_moments(_scaled(g), kp.make_probes(g.n, 16, "hadamard", seed=4), 120)
    assert np.abs(mom.values).max() <= 1.0 + 5.0 / np.sqrt(16)


# ------------------------------------------------------ test_motifs.py
@gpu
def test_star_filtered_moments_identity(star4):
    insts = kp.detect_motifs(star4, kinds={kp.MotifKind.OPEN_TWIN})
    sop = _scaled(star4)
    probes = kp.make_probes(4, 4, "standard-basis")
    filtered, adj = kp.filter_probes(probes, insts)
    m_unf = kp.dos_moments(sop, probes, 30)
    m_fil = kp.dos_moments(sop, filtered, 30, effective_dim=4 - adj.deflated_dim)
    t0 = chebyshev_values(30, np.array([0.0]))[:, 0]
    assert np.abs(m_fil.values - (4 * m_unf.values - 2 * t0) / 2).max() < 1e-12


@gpu
def test_filter_probes_annihilates_difference(star4):
    insts = kp.detect_motifs(star4, kinds={kp.MotifKind.OPEN_TWIN})
    filtered, adj = kp.filter_probes(kp.make_probes(4, 6, "gaussian", seed=3), insts)
    z = filtered.columns
    assert np.abs(z[1] - z[2]).max() < 1e-12 and np.abs(z[2] - z[3]).max() < 1e-12
    assert adj.deflated_dim == 2 and adj.removed == {0.0: 2}


@gpu
def test_trace_decomposition_on_planted_graphs():
    rng = np.random.default_rng(5)
    for _ in range(6):
        g = kp.preferential_attachment(int(rng.integers(80, 300)), 1,
                                       seed=int(rng.integers(1 << 30)))
        insts = kp.detect_motifs(g)
        if not insts:
            continue
        sop = _scaled(g)
        probes = kp.make_probes(g.n, g.n, "standard-basis")
        filtered, adj = kp.filter_probes(probes, insts)
        r = adj.deflated_dim
        m_unf = kp.dos_moments(sop, probes, 50)
        m_fil = kp.dos_moments(sop, filtered, 50, effective_dim=g.n - r)
        removed = np.zeros(51)
        for lam, cnt in adj.removed.items():
            removed += cnt * chebyshev_values(50, np.array([lam]))[:, 0]
        assert np.abs(g.n * m_unf.values - ((g.n - r) * m_fil.values + removed)).max() < 1e-8


@gpu
def test_custom_instance_deflation():
    g = kp.build_csr([(0, 1), (1, 2)])
    inst = kp.MotifInstance(kind=kp.MotifKind.CUSTOM, nodes=(0, 2), eigenvalue=0.0,
                            eigvecs=({0: 1 / np.sqrt(2), 2: -1 / np.sqrt(2)},))
    filtered, adj = kp.filter_probes(kp.make_probes(3, 3, "standard-basis"), [inst])
    m_fil = kp.dos_moments(_scaled(g), filtered, 8, effective_dim=2)
    want = chebyshev_values(8, np.array([-1.0, 1.0])).mean(axis=1)
    assert np.abs(m_fil.values - want).max() < 1e-12


# --------------------------------------------------- test_operators.py
@gpu
def test_operator_matches_dense_definition_entrywise():
    rng = np.random.default_rng(3)
    for trial in range(6):
        n = int(rng.integers(5, 40))
        edges = set()
        target = min(int(rng.integers(n, 3 * n)), n * (n - 1) // 2)
        while len(edges) < target:
            u, v = rng.integers(0, n, size=2)
            if u != v:
                edges.add((min(u, v), max(u, v)))
        w = trial % 2
        g = kp.build_csr([(int(u), int(v), 1.0 + w * float((u * v) % 4)) for u, v in edges],
                         n=n)
        for kind in kp.OperatorKind:
            op = kp.build_operator(g, kind)
            assert np.allclose(testkit.dense_matrix(op), _dense_from_graph(g, kind.value),
                               atol=1e-14)


@gpu
def test_isolated_node_conventions():
    g = kp.build_csr([(0, 1)], n=3)
    na = testkit.dense_matrix(kp.build_operator(g, "normalized-adjacency"))
    nl = testkit.dense_matrix(kp.build_operator(g, "normalized-laplacian"))
    assert np.array_equal(na[2], np.zeros(3))
    assert np.array_equal(nl[2], np.array([0, 0, 1.0]))


@gpu
def test_small_spectra(triangle, path3, star4):
    sp = testkit.exact_spectrum(kp.build_operator(triangle, "normalized-adjacency"))
    assert np.allclose(sp.eigenvalues, [-0.5, -0.5, 1.0], atol=1e-12)
    sp = testkit.exact_spectrum(kp.build_operator(path3, "normalized-adjacency"))
    assert np.allclose(sp.eigenvalues, [-1.0, 0.0, 1.0], atol=1e-12)
    sp = testkit.exact_spectrum(kp.build_operator(star4, "laplacian"))
    assert np.allclose(sp.eigenvalues, [0.0, 1.0, 1.0, 4.0], atol=1e-12)


@gpu
def test_apply_is_linear():
    g = kp.erdos_renyi(60, 0.1, seed=2)
    rng = np.random.default_rng(4)
    for kind in kp.OperatorKind:
        op = kp.build_operator(g, kind)
        x, y = rng.standard_normal((2, g.n))
        lhs = op.apply(0.7 * x - 1.3 * y)
        rhs = 0.7 * op.apply(x) - 1.3 * op.apply(y)
        assert np.abs(lhs - rhs).max() <= 1e-12 * max(np.abs(rhs).max(), 1.0)


@gpu
def test_k3_adjacency_exact_krylov_range(triangle):
    op = kp.build_operator(triangle, "adjacency")
    lo, hi = kp.estimate_spectral_range(op, probe_seed=1, steps=3, margin=0.0)
    assert abs(lo + 1.0) < 1e-9 and abs(hi - 2.0) < 1e-9


@gpu
def test_entrywise_equality_at_500_nodes():
    g = kp.erdos_renyi(500, 0.02, seed=9)
    for kind in ("normalized-adjacency", "laplacian"):
        assert np.allclose(testkit.dense_matrix(kp.build_operator(g, kind)),
                           _dense_from_graph(g, kind), atol=1e-14)


# ------------------------------------------------------- test_density.py
def test_single_bin_carries_all_mass():
    m = kp.ChebMoments("global", np.array([1.0, 0.3, -0.2]), kp.ScaleMap(0.0, 1.0), {})
    h = kp.histogram_from_moments(m, bins=1, damping=False)
    assert h.masses[0] == pytest.approx(1.0, abs=1e-14)


def test_bin_table_telescopes_to_unit_mass():
    table = kp.cheb_bin_masses(40, np.linspace(-1, 1, 33))
    assert table[0].sum() == pytest.approx(1.0, abs=1e-14)
    assert np.abs(table[1:].sum(axis=1)).max() < 1e-13


def test_spike_reinsertion_bookkeeping():
    m = kp.ChebMoments("global", np.array([1.0, 0.0, 0.0]), kp.ScaleMap(0.0, 1.0), {})
    adj = kp.FilterAdjustment(removed={0.0: 2, 0.5: 1}, total_dim=10)
    h = kp.histogram_from_moments(m, bins=4, damping=False, filter_adjustment=adj)
    assert h.masses.sum() == pytest.approx(1.0, abs=1e-14)


def test_bins_must_be_positive():
    m = kp.ChebMoments("global", np.array([1.0]), kp.ScaleMap(0.0, 1.0), {})
    with pytest.raises(ValueError, match="bins"):
        kp.histogram_from_moments(m, bins=0)


@gpu
def test_p3_exact_moments_recover_thirds(path3):
    mom = kp.dos_moments(_scaled(path3), kp.make_probes(3, 3, "standard-basis"), 400)
    h = kp.histogram_from_moments(mom, bins=3)
    assert np.allclose(h.masses, [1 / 3] * 3, atol=0.02)


# ------------------------------------------------- test_acceptance.py
@gpu
def test_criterion_01_kpm_histogram_matches_oracle():
    g = testkit.erdos_renyi(2000, 0.01, seed=1)
    t0 = time.perf_counter()
    res = kp.kpm_dos(g, operator="normalized-adjacency", m_max=500, nz=20,
                     probe_kind="hadamard", seed=7, bins=50, damping=True)
    elapsed = time.perf_counter() - t0
    ev = testkit.exact_spectrum(kp.build_operator(g, "normalized-adjacency")).eigenvalues
    oracle = testkit.oracle_histogram(ev, res.histogram.edges)
    assert float(np.abs(res.histogram.masses - oracle).sum()) < 0.05
    assert elapsed < 60.0


@gpu
def test_criterion_02_motif_filtering_improves_and_trace_identity():
    g = testkit.preferential_attachment(3000, 1, seed=0)
    kinds = ("open-twin", "closed-twin", "dangling-two-chain")
    ev = testkit.exact_spectrum(kp.build_operator(g, "normalized-adjacency")).eigenvalues
    unf = kp.kpm_dos(g, m_max=100, nz=20, seed=11, bins=50)
    fil = kp.kpm_dos(g, m_max=100, nz=20, seed=11, bins=50, filter_kinds=kinds)
    oracle = testkit.oracle_histogram(ev, unf.histogram.edges)
    assert np.abs(fil.histogram.masses - oracle).sum() < np.abs(unf.histogram.masses -
                                                                oracle).sum()
    sop = scaled_operator_for(g, "normalized-adjacency")
    probes = kp.make_probes(g.n, g.n, "standard-basis")
    filtered, adj = kp.filter_probes(probes, kp.detect_motifs(g, seed=11))
    r = adj.deflated_dim
    m_unf = kp.dos_moments(sop, probes, 100)
    m_fil = kp.dos_moments(sop, filtered, 100, effective_dim=g.n - r)
    removed = np.zeros(101)
    for lam, cnt in adj.removed.items():
        removed += cnt * chebyshev_values(100, np.array([lam]))[:, 0]
    assert np.abs(g.n * m_unf.values - ((g.n - r) * m_fil.values + removed)).max() < 1e-8


@gpu
def test_criterion_03_moment_exactness_suite():
    rng = np.random.default_rng(2024)
    kinds = ["normalized-adjacency", "adjacency", "laplacian", "normalized-laplacian"]
    worst = 0.0
    for trial in range(25):
        n = int(rng.integers(40, 301))
        g = testkit.erdos_renyi(n, float(rng.uniform(0.02, 0.1)),
                                seed=int(rng.integers(1 << 30)))
        sop = scaled_operator_for(g, kinds[trial % 4], seed=trial)
        ev = sop.scale_map.to_scaled(testkit.exact_spectrum(sop.base).eigenvalues)
        mom = kp.dos_moments(sop, kp.make_probes(n, n, "standard-basis"), 50)
        worst = max(worst, float(np.abs(mom.values - testkit.oracle_moments(ev, 50)).max()))
    assert worst < 1e-10


@gpu
def test_criterion_09_scaling():
    def per_moment_seconds(g):
        sop = scaled_operator_for(g, "normalized-adjacency")
        probes = kp.make_probes(g.n, 20, "hadamard", seed=1)
        best = np.inf
        for _ in range(3):
            t0 = time.perf_counter()
            kp.dos_moments(sop, probes, 10)
            best = min(best, (time.perf_counter() - t0) / 10)
        return best

    g_small = testkit.erdos_renyi(20_000, 1e5 / (20_000 * 19_999 / 2), seed=1)
    g_big = testkit.erdos_renyi(200_000, 1e6 / (200_000 * 199_999 / 2), seed=1)
    assert per_moment_seconds(g_big) / per_moment_seconds(g_small) <= 30.0
